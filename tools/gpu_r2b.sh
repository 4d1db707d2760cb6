mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_api_surface.py tests/test_gpu_sharded.py -m gpu -q -rf > gpurun_out/b_pytest_new.log 2>&1; tail -30 gpurun_out/b_pytest_new.log
timeout 2400 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_multiprocess.py --deselect tests/test_gpu_api_surface.py --deselect tests/test_gpu_sharded.py > gpurun_out/b_pytest_rest.log 2>&1; tail -8 gpurun_out/b_pytest_rest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/b_bench.log 2>&1; tail -1 gpurun_out/b_bench.log | cut -c1-400
