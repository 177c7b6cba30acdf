mkdir -p gpurun_out
timeout 120 python scripts/trace_chain.py 1 > gpurun_out/trace_chain.txt 2>&1
timeout 300 python scripts/gemv_probe.py --paths 1 --ms 1 --shapes q,gate --chain > gpurun_out/probe.txt 2>&1
ANYQ_GV_XTMA=1 timeout 300 python scripts/gemv_probe.py --paths 1 --ms 1 --shapes q,gate --chain > gpurun_out/probe_xtma.txt 2>&1
echo done
