# round-2 evidence pass: GPU tests, smoke, every bench line + the reference arm, launch list,
# full ncu captures of the dominant kernels (each command first run plain, then under ncu)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/v2_pytest.log 2>&1; tail -3 gpurun_out/v2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2_smoke.log 2>&1; tail -1 gpurun_out/v2_smoke.log
for c in ts1 wl1 sl1 wl2 wl3; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/v2_bench_$c.log 2>&1; tail -1 gpurun_out/v2_bench_$c.log | cut -c1-150
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/v2_ref_$c.log 2>&1; tail -1 gpurun_out/v2_ref_$c.log | cut -c1-150
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v2_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v2_ncu_bench.log 2>&1
for c in ts1 sl1 wl1; do
  python tools/profile_run.py $c > gpurun_out/v2_${c}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -c 1 -o gpurun_out/v2_prof_$c \
      python tools/profile_run.py $c > gpurun_out/v2_${c}_ncu.log 2>&1
done
python tools/profile_run.py wl2 80 > gpurun_out/v2_wl2_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 79 -c 1 -o gpurun_out/v2_prof_wl2 \
    python tools/profile_run.py wl2 80 > gpurun_out/v2_wl2_ncu.log 2>&1
python tools/profile_run.py wl3 40 > gpurun_out/v2_wl3_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 39 -c 1 -o gpurun_out/v2_prof_wl3 \
    python tools/profile_run.py wl3 40 > gpurun_out/v2_wl3_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:field_update_kernel -s 39 -c 1 -o gpurun_out/v2_prof_wl3_field \
    python tools/profile_run.py wl3 40 > gpurun_out/v2_wl3f_ncu.log 2>&1
ls gpurun_out | grep "^v2_"
