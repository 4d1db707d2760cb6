# full evidence pass: tests, smoke, all bench lines, ncu launch list of the default bench, full captures
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/g_pytest.log 2>&1; tail -4 gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; tail -2 gpurun_out/g_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/g_bench_$c.log 2>&1; tail -1 gpurun_out/g_bench_$c.log | cut -c1-300; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_bench_ref.log 2>&1; tail -1 gpurun_out/g_bench_ref.log | cut -c1-300
python bench.py --steps 3 --warmup 3 > gpurun_out/g_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/g_ncu_bench.log 2>&1
python tools/profile_run.py wl3 40 > gpurun_out/g_wl3_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 39 -c 1 -o gpurun_out/g_prof_wl3_trace3 \
    python tools/profile_run.py wl3 40 > gpurun_out/g_wl3_ncu.log 2>&1
python tools/profile_run.py ts1 > gpurun_out/g_ts1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -c 1 -o gpurun_out/g_prof_ts1_run1d \
    python tools/profile_run.py ts1 > gpurun_out/g_ts1_ncu.log 2>&1
ls gpurun_out
