# k-means: parity tests, then the phase breakdown and rows/s (config 1 and a K=14336 row set)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_quantize.py tests/test_gpu_learner.py tests/test_gpu_golden.py tests/test_gpu_headline.py -x -q -k "not chain and not single_gemm and not wide" > gpurun_out/km_tests.txt 2>&1
tail -n 3 gpurun_out/km_tests.txt
ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096 4096x14336 > gpurun_out/km_prof.txt 2>&1
grep -v "^\[kmeans" gpurun_out/km_prof.txt; grep "^\[kmeans" gpurun_out/km_prof.txt | tail -n 1
