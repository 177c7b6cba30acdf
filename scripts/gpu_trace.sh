mkdir -p gpurun_out
timeout 120 python scripts/trace_gemv.py q 1 > gpurun_out/trace_gemv_q.txt 2>&1
timeout 120 python scripts/trace_gemv.py k 1 > gpurun_out/trace_gemv_k.txt 2>&1
timeout 120 python scripts/trace_gemv.py gate 1 > gpurun_out/trace_gemv_gate.txt 2>&1
echo done
