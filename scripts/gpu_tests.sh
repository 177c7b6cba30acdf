# Full GPU test suite (+ the given extra pytest args), log under gpurun_out/.
mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest tests -m gpu -x -q -rs ${ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
echo done
