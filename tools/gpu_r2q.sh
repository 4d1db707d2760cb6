mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_async_dropin.py -m gpu -q -rf -x > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
for b in 0 1; do
if [ $b = 1 ]; then export NUFI_NOBULKSTAGE=1; else unset NUFI_NOBULKSTAGE; fi
for c in ts1 wl1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/q_bench_${c}_$b.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/q_bench_${c}_$b.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c nobulk=$b", round(d["ms_per_step"],3), "frac", round(r["frac"],4))
PY
done; done
unset NUFI_NOBULKSTAGE
timeout 300 python tools/stamps.py ts1 | head -3
