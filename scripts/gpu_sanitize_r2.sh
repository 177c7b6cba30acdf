# compute-sanitizer memcheck + synccheck over the round-2 kernels (K1t, K2, exact gemm_fused,
# prepack^-1, fused TP gather): small parity tests, log tails under gpurun_out/
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -x -q \
    "tests/test_gpu_gemv_tc.py::test_formats_and_m[1-any4]" "tests/test_gpu_gemv_tc.py::test_chain_decoder_pattern[2]" \
    "tests/test_gpu_k2.py::test_k2_formats[any4]" "tests/test_gpu_k2.py::test_k2_m_sweep[200]" \
    "tests/test_gpu_gemm.py::test_fused_bit_exact_vs_reference[5-any4]" "tests/test_gpu_pack.py::test_prepack_inverse_round_trip[shape0-3-128-any4]" \
    "tests/test_gpu_tp.py::test_fused_allgather_equals_unsharded[2-2]" > gpurun_out/sanitizer_r2_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_r2_$tool.log
done
for f in gpurun_out/sanitizer_r2_*.log; do tail -n 4 "$f"; done
