# round-2 evidence, part A: GPU tests, smoke, every bench line + the reference arm (logs only)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/v2_pytest.log 2>&1; tail -3 gpurun_out/v2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1; tail -1 gpurun_out/v2_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/v2_bench_$c.log 2>&1; tail -1 gpurun_out/v2_bench_$c.log | cut -c1-120
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/v2_ref_$c.log 2>&1; tail -1 gpurun_out/v2_ref_$c.log | cut -c1-120
done
