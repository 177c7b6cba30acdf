mkdir -p gpurun_out
timeout 120 python scripts/trace_gemv.py gate 1 > gpurun_out/trace_gemv_gate.txt 2>&1
timeout 300 python scripts/gemv_probe.py --paths ${PATHS:-1} --ms ${MS:-1} --shapes ${SHAPES:-q,k,gate,down} > gpurun_out/probe.txt 2>&1
echo done
