set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
for c in ts1 wl1 sl1 wl2; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/r1_bench_$c.log 2>&1; done
timeout 600 python bench.py --config wl3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r1_bench_wl3.log 2>&1
tail -3 gpurun_out/*.log
