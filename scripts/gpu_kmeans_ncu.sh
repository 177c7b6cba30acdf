mkdir -p gpurun_out
ANYQ_KM_G=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_kmeans_warp -c 1 -o gpurun_out/km_warp python scripts/prof_kmeans.py 4096 > gpurun_out/km_ncu.log 2>&1
echo done
