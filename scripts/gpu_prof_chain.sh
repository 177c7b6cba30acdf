# ncu --set full (source-attributed) of the 8B-layer chain and of gate at M=1.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lutgemv -s 2 -c 1 -o gpurun_out/${OUT:-chain_full} python scripts/prof_chain.py > gpurun_out/ncu_chain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lutgemv -s 2 -c 1 -o gpurun_out/${OUT:-chain_full}_gate python scripts/prof_gemv.py gate 1 1 4 >> gpurun_out/ncu_chain.log 2>&1
echo done
