# compute-sanitizer memcheck + synccheck over this session's kernel changes: k-means
# (warp-0 Lloyd, chunk-sum M-step, repairs, bail path), K1t K-slices, K2 two-chunk step
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q \
    "tests/test_gpu_quantize.py::test_quantize_any_matches_oracle[True-case3]" \
    "tests/test_gpu_quantize.py::test_lossless_rows_and_constant_rows" \
    "tests/test_gpu_quantize.py::test_near_duplicate_centroids_take_the_cta_kernel" \
    "tests/test_gpu_gemv_tc.py::test_k_slices[16-4096-256]" \
    "tests/test_gpu_gemv_tc.py::test_k_slices[3-14336-128]" \
    "tests/test_gpu_k2.py::test_k2_formats[any4]" "tests/test_gpu_k2.py::test_k2_m_sweep[300]" \
    > gpurun_out/sanitizer_r2b_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_r2b_$tool.log
done
for f in gpurun_out/sanitizer_r2b_*.log; do tail -n 4 "$f"; done
