# k-means experiment builds: golden / fingerprint / oracle tests and rows/s per variant
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/build/exp/$v/libanyq_b200.so; fi
  echo "== $v" >> gpurun_out/km_var.txt
  ANYQ_LIB=$lib timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_quantize.py tests/test_gpu_headline.py -q -k "not chain and not single_gemm and not wide" 2>&1 | grep -E "passed|failed|FAILED" >> gpurun_out/km_var.txt
  ANYQ_LIB=$lib ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096 4096x14336 2>&1 | grep -v "^\[kmeans" >> gpurun_out/km_var.txt
done
cat gpurun_out/km_var.txt
