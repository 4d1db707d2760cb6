# round-2 closing evidence at HEAD (after the helper-CTA split): GPU tests, smoke, every bench line + the reference arm on the
# same box, the default bench and its ncu launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f11_pytest.log 2>&1; tail -2 gpurun_out/f11_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f11_smoke.log 2>&1; tail -1 gpurun_out/f11_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f11_bench_$c.log 2>&1; tail -1 gpurun_out/f11_bench_$c.log | cut -c1-150
  timeout 1500 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/f11_ref_$c.log 2>&1; tail -1 gpurun_out/f11_ref_$c.log | cut -c1-150
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f11_bench_default.log 2>&1; tail -1 gpurun_out/f11_bench_default.log | cut -c1-200
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f11_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f11_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f11_ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/f11_launches_ts1.csv > gpurun_out/f11_launches_ts1.txt 2>&1; head -4 gpurun_out/f11_launches_ts1.txt
