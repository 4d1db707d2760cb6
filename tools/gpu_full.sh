# full GPU check: tests, smoke, bench lines for every BASELINE config
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/f_pytest.log 2>&1; tail -8 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -2 gpurun_out/f_smoke.log
for c in ${BENCH_CONFIGS:-ts1 wl1 sl1 wl2}; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f_bench_$c.log 2>&1; tail -1 gpurun_out/f_bench_$c.log | cut -c1-400; done
