# compute-sanitizer memcheck + synccheck over the K1a changes of this round (builder warp, x loaded
# from L2, two half rings) and K1t's slot changes: single GEMVs, ragged K, the dependent chains
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q \
    "tests/test_gpu_gemm.py::test_tc_gemm_matches_reference[1-any4-gemv]" \
    "tests/test_gpu_gemm.py::test_tc_gemm_matches_reference[2-any3-gemv]" \
    "tests/test_gpu_gemm.py::test_gemv_ragged_k[300-1000-2]" \
    "tests/test_gpu_gemm.py::test_gemm_chain_matches_single_launches" \
    "tests/test_gpu_gemm.py::test_gemm_chain_edge_cases" \
    "tests/test_gpu_gemv_tc.py::test_formats_and_m[4-any4]" \
    "tests/test_gpu_gemv_tc.py::test_chain_decoder_pattern[2]" \
    > gpurun_out/sanitizer_r2c_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_r2c_$tool.log
done
for f in gpurun_out/sanitizer_r2c_*.log; do tail -n 4 "$f"; done
