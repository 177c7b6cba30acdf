# K1e (tensor-core GEMV) iteration: parity tests of the GEMV paths, then the
# probe with the MMA compute warps and with the FHFMA ones for comparison.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -k "gemv or chain or tc_gemm" > gpurun_out/pytest_k1e.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_k1e.log
ANYQ_GV_MMA=1 timeout 300 python scripts/gemv_probe.py --paths 1 --ms ${MS:-1,2,3,4} --shapes ${SHAPES-q,k,gate,down,gate70} --chain > gpurun_out/probe_mma.txt 2>&1
ANYQ_GV_MMA=0 timeout 300 python scripts/gemv_probe.py --paths 1 --ms ${MS:-1,2,3,4} --shapes ${SHAPES-q,k,gate,down,gate70} --chain > gpurun_out/probe_fma.txt 2>&1
echo done
