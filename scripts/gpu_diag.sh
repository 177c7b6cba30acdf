mkdir -p gpurun_out
timeout 120 python scripts/trace_gemm.py 1024 4096 1 > gpurun_out/trace_kv.txt 2>&1
timeout 120 python scripts/trace_gemm.py 4096 4096 1 > gpurun_out/trace_q.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_q.csv python scripts/prof_one.py 4096 4096 1 5 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_lutgemm -s 2 -c 1 -o gpurun_out/lutgemm_q python scripts/prof_one.py 4096 4096 1 4 > gpurun_out/ncu_full.log 2>&1
echo done
