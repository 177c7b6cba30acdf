# K1t iteration: parity tests, then timing vs K1a.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv_tc.py -x -q ${TARGS} > gpurun_out/pytest_k1t.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k1t.log
timeout 300 python scripts/gemv_probe.py --paths ${PATHS:-1,5} --ms ${MS:-1,2,4,8,16} --shapes ${SHAPES-q,k,gate,down} --chain --chain-paths 1,5 > gpurun_out/probe_k1t.txt 2>&1
echo done
