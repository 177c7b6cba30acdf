# One iteration of the GEMV kernel loop on a B200: parity tests, chain trace, probe.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_gemm.py tests/test_dist.py -x -q > gpurun_out/pytest_gemm.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gemm.log
timeout 120 python scripts/trace_chain.py ${MS:-1} > gpurun_out/trace_chain.txt 2>&1
timeout 300 python scripts/gemv_probe.py --paths 1 --ms ${MS:-1,2} --shapes ${SHAPES-q,k,gate,down} --chain > gpurun_out/probe.txt 2>&1
echo done
