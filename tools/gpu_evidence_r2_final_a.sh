# round-2 final evidence, part A: GPU tests (incl. wl3 at full size), smoke, every bench line +
# the reference arm on the same box
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/f2_pytest.log 2>&1; tail -25 gpurun_out/f2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; tail -1 gpurun_out/f2_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f2_bench_$c.log 2>&1; tail -1 gpurun_out/f2_bench_$c.log | cut -c1-120
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/f2_ref_$c.log 2>&1; tail -1 gpurun_out/f2_ref_$c.log | cut -c1-120
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f2_bench_default.log 2>&1; tail -1 gpurun_out/f2_bench_default.log | cut -c1-200
