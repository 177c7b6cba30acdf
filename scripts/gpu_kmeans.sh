# k-means iteration on a B200: parity tests of the quantizer, then the timing probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantize.py tests/test_gpu_golden.py tests/test_reference_suite.py tests/test_dist.py -x -q > gpurun_out/pytest_km.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_km.log
timeout 300 python scripts/prof_kmeans.py 148 1024 4096 4096 16384 > gpurun_out/prof_kmeans.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kmeans_launches.csv python scripts/prof_kmeans.py 4096 > /dev/null 2>&1
echo done
