# round-2 final evidence, part B: launch list of the default bench, full ncu captures of the
# dominant kernels (each command first run plain), summarised on the box; scaling projection;
# d = 1 phase stamps
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f2_ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/f2_launches_ts1.csv > gpurun_out/f2_launches_ts1.txt 2>&1
cap() {  # name kernel-regex skip args...
  name=$1; k=$2; s=$3; shift 3
  python tools/profile_run.py "$@" > gpurun_out/f2_${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/f2_prof_$name \
      python tools/profile_run.py "$@" > gpurun_out/f2_${name}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/f2_prof_$name.ncu-rep > gpurun_out/f2_prof_$name.txt 2>&1
}
cap ts1 run_1d_kernel 0 ts1
cap sl1 run_1d_kernel 0 sl1
cap wl1 run_1d_kernel 0 wl1
cap wl2 trace_rho_kernel 79 wl2 80
cap wl3 trace_rho_kernel 39 wl3 40
cap wl3field field_update_kernel 39 wl3 40
cp /tmp/f2_prof_ts1.ncu-rep /tmp/f2_prof_wl3.ncu-rep gpurun_out/ 2>/dev/null
for c in wl3 wl2; do timeout 900 python tools/scaling_projection.py $c 20 50 > gpurun_out/f2_scal_$c.json 2>/dev/null; done
for c in ts1 wl1 sl1; do timeout 300 python tools/stamps.py $c > gpurun_out/f2_stamps_$c.txt 2>&1; done
ls -la gpurun_out | grep "f2_"
