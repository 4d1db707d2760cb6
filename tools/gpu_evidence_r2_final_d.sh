# round-2 evidence refresh after the d >= 2 stage-counter change: GPU tests, smoke, the d >= 2
# bench lines + reference arm on the same box, ncu captures (each command first run plain),
# scaling projections, parity margins
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f4_pytest.log 2>&1; tail -2 gpurun_out/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -1 gpurun_out/f4_smoke.log
for c in wl2 wl3; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f4_bench_$c.log 2>&1; tail -1 gpurun_out/f4_bench_$c.log | cut -c1-120
  timeout 1500 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/f4_ref_$c.log 2>&1; tail -1 gpurun_out/f4_ref_$c.log | cut -c1-120
done
cap() {  # name kernel-regex skip args...
  name=$1; k=$2; s=$3; shift 3
  python tools/profile_run.py "$@" > gpurun_out/f4_${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/f4_prof_$name \
      python tools/profile_run.py "$@" > gpurun_out/f4_${name}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/f4_prof_$name.ncu-rep > gpurun_out/f4_prof_$name.txt 2>&1
}
cap wl2 trace_rho_kernel 79 wl2 80
cap wl3 trace_rho_kernel 39 wl3 40
cp /tmp/f4_prof_wl3.ncu-rep gpurun_out/ 2>/dev/null
for c in wl3 wl2; do timeout 900 python tools/scaling_projection.py $c 20 50 > gpurun_out/f4_scal_$c.json 2>/dev/null; done
timeout 900 python tools/parity_margins.py wl2 wl3 > gpurun_out/f4_parity_margins.txt 2>&1; cat gpurun_out/f4_parity_margins.txt
ls gpurun_out | grep -c "f4_"
