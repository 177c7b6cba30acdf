mkdir -p gpurun_out
: > gpurun_out/prof_kmeans_dbg.txt
timeout 300 python scripts/prof_kmeans.py 4096 4096x14336 1024x4096 4096x1024 >> gpurun_out/prof_kmeans_dbg.txt 2>&1
echo done
