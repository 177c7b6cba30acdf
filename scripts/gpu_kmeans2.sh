mkdir -p gpurun_out
: > gpurun_out/prof_kmeans_dbg.txt
for G in 1 2 4; do echo "G=$G" >> gpurun_out/prof_kmeans_dbg.txt; ANYQ_KM_G=$G ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096 >> gpurun_out/prof_kmeans_dbg.txt 2>&1; done
echo "G=auto" >> gpurun_out/prof_kmeans_dbg.txt
ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096x14336 16384 >> gpurun_out/prof_kmeans_dbg.txt 2>&1
echo done
