mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_async_dropin.py tests/test_gpu_properties.py tests/test_history.py -m gpu -q -rf -x > gpurun_out/i_pytest.log 2>&1; tail -3 gpurun_out/i_pytest.log
for pf in 0 1; do
if [ $pf = 1 ]; then export NUFI_NOPREFETCH=1; else unset NUFI_NOPREFETCH; fi
for c in ts1 wl1 sl1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/i_bench_${c}_$pf.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/i_bench_${c}_$pf.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c noprefetch=$pf", round(d["ms_per_step"],3), "frac", round(r["frac"],4))
PY
done; done
unset NUFI_NOPREFETCH
timeout 300 python tools/stamps.py ts1
timeout 300 python tools/stamps.py wl1
