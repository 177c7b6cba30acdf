mkdir -p gpurun_out
cd scripts && ./ubench_mma_issue > ../gpurun_out/ubench_mma.txt 2>&1; ./ubench_tcgen05 > ../gpurun_out/ubench_tc.txt 2>&1; cd ..
timeout 300 python scripts/gemv_probe.py --paths 1,2 --ms 1,2,4 > gpurun_out/probe.txt 2>&1
echo done
