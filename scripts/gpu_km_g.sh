# k-means row-group size sweep (ANYQ_KM_G) on the current library
mkdir -p gpurun_out
for G in 1 2 4 8; do
  echo "== G=$G" >> gpurun_out/km_g.txt
  ANYQ_KM_G=$G ANYQ_KM_DEBUG=1 timeout 300 python scripts/prof_kmeans.py 4096 4096x14336 >> gpurun_out/km_g.txt 2>&1
done
grep -v "^\[kmeans" gpurun_out/km_g.txt
