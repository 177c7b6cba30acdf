# compute-sanitizer memcheck + synccheck over the rows around the path (stats, eval
# metrics, file -> device load) and the 3-row GEMV
mkdir -p gpurun_out
: > gpurun_out/sanitizer_aux.txt
for tool in memcheck synccheck racecheck; do
  echo "=== $tool stats/eval/file" >> gpurun_out/sanitizer_aux.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_stats.py tests/test_file_io.py -x -q -m gpu -k "not 4096 and not 4097" >> gpurun_out/sanitizer_aux.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_aux.txt
done
echo "=== memcheck gemv m=3" >> gpurun_out/sanitizer_aux.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -k "ragged and 3-" >> gpurun_out/sanitizer_aux.txt 2>&1
echo "exit $?" >> gpurun_out/sanitizer_aux.txt
echo done
