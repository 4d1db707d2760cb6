# round-2 evidence refresh after the shifted-state d = 1 lookup: GPU tests, smoke, the d = 1
# bench lines + reference arm, default bench, launch list, ncu of the d = 1 run kernels
# (each command first run plain), stamps, parity margins
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f6_pytest.log 2>&1; tail -2 gpurun_out/f6_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; tail -1 gpurun_out/f6_smoke.log
for c in ts1 wl1 sl1; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f6_bench_$c.log 2>&1; tail -1 gpurun_out/f6_bench_$c.log | cut -c1-120
  timeout 1500 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/f6_ref_$c.log 2>&1; tail -1 gpurun_out/f6_ref_$c.log | cut -c1-120
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f6_bench_default.log 2>&1; tail -1 gpurun_out/f6_bench_default.log | cut -c1-200
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f6_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f6_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f6_ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/f6_launches_ts1.csv > gpurun_out/f6_launches_ts1.txt 2>&1
cap() {  # name kernel-regex skip args...
  name=$1; k=$2; s=$3; shift 3
  python tools/profile_run.py "$@" > gpurun_out/f6_${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/f6_prof_$name \
      python tools/profile_run.py "$@" > gpurun_out/f6_${name}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/f6_prof_$name.ncu-rep > gpurun_out/f6_prof_$name.txt 2>&1
}
cap ts1 run_1d_kernel 0 ts1
cap wl1 run_1d_kernel 0 wl1
cap sl1 run_1d_kernel 0 sl1
for c in ts1 wl1 sl1; do timeout 300 python tools/stamps.py $c > gpurun_out/f6_stamps_$c.txt 2>&1; done
timeout 900 python tools/parity_margins.py wl1 ts1 sl1 > gpurun_out/f6_parity_margins.txt 2>&1; cat gpurun_out/f6_parity_margins.txt
