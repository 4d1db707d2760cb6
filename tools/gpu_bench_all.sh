# bench lines of every BASELINE config + the reference arm + GPU tests + smoke (no ncu)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/v_pytest.log 2>&1; tail -2 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -1 gpurun_out/v_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/v_bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_bench_ref.log 2>&1
