mkdir -p gpurun_out
ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096 > gpurun_out/prof_kmeans_dbg.txt 2>&1
echo done
