# ncu evidence for the d = 1 run kernels + the launch list of the default bench command
set -x
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/v_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/v_ncu_bench.log 2>&1
for c in ts1 sl1 wl1; do
  python tools/profile_run.py $c > gpurun_out/v_${c}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -s 0 -c 1 -o gpurun_out/v_prof_$c \
      python tools/profile_run.py $c > gpurun_out/v_${c}_ncu.log 2>&1
done
ls gpurun_out | grep "^v_"
