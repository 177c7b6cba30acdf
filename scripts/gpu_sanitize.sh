# compute-sanitizer (memcheck + racecheck + synccheck) over small GEMV-chain and k-means runs
mkdir -p gpurun_out
: > gpurun_out/sanitizer.txt
for tool in memcheck racecheck synccheck; do
  echo "=== $tool gemm" >> gpurun_out/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -k "test_tc_gemm_shapes and gemv and 1024" >> gpurun_out/sanitizer.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer.txt
  echo "=== $tool kmeans" >> gpurun_out/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_quantize.py -x -q -k "not config1 and not slow" >> gpurun_out/sanitizer.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer.txt
done
echo "=== memcheck chain" >> gpurun_out/sanitizer.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -k "chain" >> gpurun_out/sanitizer.txt 2>&1
echo "exit $?" >> gpurun_out/sanitizer.txt
