# round 2, first pass: GPU tests (all), smoke, default bench + reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
nproc > gpurun_out/a_nproc.txt; lscpu | head -20 >> gpurun_out/a_nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -x -p no:randomly --durations=30 > gpurun_out/a_pytest.log 2>&1; tail -40 gpurun_out/a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; tail -2 gpurun_out/a_smoke.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/a_ref.log 2>&1; tail -1 gpurun_out/a_ref.log | cut -c1-1500
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench.log 2>&1; tail -1 gpurun_out/a_bench.log | cut -c1-3000
