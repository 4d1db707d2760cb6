set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -rf ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_pytest_gpu.log 2>&1
tail -30 gpurun_out/t_pytest_gpu.log
