mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gemm.log
timeout 120 python scripts/trace_gemv.py gate 1 > gpurun_out/trace_gemv_gate.txt 2>&1
timeout 300 python scripts/gemv_probe.py --paths ${PATHS:-1} --ms ${MS:-1} --shapes ${SHAPES-q,k,gate,down} --chain > gpurun_out/probe.txt 2>&1
echo done
