mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_async_dropin.py -m gpu -q -rf -x > gpurun_out/r_pytest.log 2>&1; tail -2 gpurun_out/r_pytest.log
for sp in 0 1; do
if [ $sp = 1 ]; then export NUFI_NOSPEC=1; else unset NUFI_NOSPEC; fi
for c in ts1 wl1 sl1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/r_bench_${c}_$sp.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/r_bench_${c}_$sp.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c nospec=$sp", round(d["ms_per_step"],3), "frac", round(r["frac"],4))
PY
done; done
unset NUFI_NOSPEC
timeout 300 python tools/stamps.py ts1 | head -2
