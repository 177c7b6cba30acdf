# Round-2 profiles: bench launch list + one ncu --set full capture per hot kernel.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 8 --warmup 3 --quick --no-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lutgemv -s 2 -c 1 -o gpurun_out/r2_chain python scripts/prof_chain.py > gpurun_out/ncu_r2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lutgemv_tc -s 1 -c 1 -o gpurun_out/r2_k1t_gate_m4 python scripts/prof_gemv.py gate 4 5 3 >> gpurun_out/ncu_r2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lutgemm_k2 -s 1 -c 1 -o gpurun_out/r2_k2_gate_m64 python scripts/prof_gemv.py gate 64 6 3 >> gpurun_out/ncu_r2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_exact_fast -c 1 -o gpurun_out/r2_exact python scripts/prof_exact.py >> gpurun_out/ncu_r2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kmeans_warp -c 1 -o gpurun_out/r2_kmeans python scripts/prof_kmeans.py 4096 >> gpurun_out/ncu_r2.log 2>&1

echo done
# summaries on the box (the reports themselves exceed the copy-back limit)
python scripts/ncu_summarize.py gpurun_out/r2_chain.ncu-rep gpurun_out/r2_ncu_chain.json "k_lutgemv<1> chain: one Llama-3-8B decoder layer (q,k,v,o,gate,up,down), M=1" 117383168
python scripts/ncu_summarize.py gpurun_out/r2_k1t_gate_m4.ncu-rep gpurun_out/r2_ncu_k1t_gate_m4.json "k_lutgemv_tc<4> (K1t): gate 14336x4096 at M=4" 31690752
python scripts/ncu_summarize.py gpurun_out/r2_k2_gate_m64.ncu-rep gpurun_out/r2_ncu_k2_gate_m64.json "k_lutgemm_k2<64> (K2): gate 14336x4096 at M=64" 33259520
python scripts/ncu_summarize.py gpurun_out/r2_exact.ncu-rep gpurun_out/r2_ncu_exact.json "k_gemm_exact_fast<1>: bit-exact gemm_fused, 4096x4096 any4 at M=1"
python scripts/ncu_summarize.py gpurun_out/r2_kmeans.ncu-rep gpurun_out/r2_ncu_kmeans.json "k_kmeans_warp: 4096x4096 any4 g128 (config 1)"
mkdir -p gpurun_out/keep; cp gpurun_out/r2_chain.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/r2_*.ncu-rep
