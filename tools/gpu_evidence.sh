# evidence pass: tests, smoke, all bench lines, reference arm, launch list, full ncu captures
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/v_pytest.log 2>&1; tail -4 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/v_bench_$c.log 2>&1; tail -1 gpurun_out/v_bench_$c.log | cut -c1-200; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_bench_ref.log 2>&1; tail -1 gpurun_out/v_bench_ref.log | cut -c1-200
python bench.py --steps 3 --warmup 3 > gpurun_out/v_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/v_ncu_bench.log 2>&1
for spec in "ts1 run_1d_kernel 0" "sl1 run_1d_kernel 0" "wl1 run_1d_kernel 0"; do set -- $spec
  python tools/profile_run.py $1 > gpurun_out/v_$1_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/v_prof_$1 \
      python tools/profile_run.py $1 > gpurun_out/v_$1_ncu.log 2>&1
done
python tools/profile_run.py wl3 40 > gpurun_out/v_wl3_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 39 -c 1 -o gpurun_out/v_prof_wl3 \
    python tools/profile_run.py wl3 40 > gpurun_out/v_wl3_ncu.log 2>&1
python tools/profile_run.py wl2 80 > gpurun_out/v_wl2_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 79 -c 1 -o gpurun_out/v_prof_wl2 \
    python tools/profile_run.py wl2 80 > gpurun_out/v_wl2_ncu.log 2>&1
ls gpurun_out | grep "^v_"
