# racecheck over the restructured k-means (warp-0 Lloyd, collectives) and K1t K-slices
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_quantize.py::test_quantize_any_matches_oracle[True-case3]" \
  "tests/test_gpu_quantize.py::test_lossless_rows_and_constant_rows" \
  "tests/test_gpu_quantize.py::test_near_duplicate_centroids_take_the_cta_kernel" \
  "tests/test_gpu_gemv_tc.py::test_k_slices[16-4096-256]" > gpurun_out/racecheck_r2b.log 2>&1
echo "racecheck exit $?" >> gpurun_out/racecheck_r2b.log
grep -E "RACECHECK SUMMARY|passed|exit" gpurun_out/racecheck_r2b.log
grep "Race reported" gpurun_out/racecheck_r2b.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head
