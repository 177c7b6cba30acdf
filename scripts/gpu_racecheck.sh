# compute-sanitizer racecheck (shared-memory hazards) over the hand-written kernels:
# K1a single + dependent chain, K1t, K2, the bit-exact gemm_fused and the k-means
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 30 python -m pytest -x -q \
  "tests/test_gpu_gemm.py::test_tc_gemm_matches_reference[1-any4-gemv]" \
  "tests/test_gpu_gemm.py::test_tc_gemm_matches_reference[2-any3-gemv]" \
  "tests/test_gpu_gemm.py::test_gemm_chain_matches_single_launches" \
  "tests/test_gpu_gemv_tc.py::test_formats_and_m[1-any4]" \
  "tests/test_gpu_k2.py::test_k2_formats[any4]" \
  "tests/test_gpu_gemm.py::test_fused_bit_exact_vs_reference[5-any4]" \
  "tests/test_gpu_quantize.py::test_quantize_any_matches_oracle[True-case1]" "tests/test_gpu_quantize.py::test_lossless_rows_and_constant_rows" > gpurun_out/racecheck_r2.log 2>&1
echo "racecheck exit $?" >> gpurun_out/racecheck_r2.log
tail -n 30 gpurun_out/racecheck_r2.log
