mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/k_pytest.log 2>&1; tail -3 gpurun_out/k_pytest.log
bash tools/fs.sh > gpurun_out/k_fs.txt 2>&1; cat gpurun_out/k_fs.txt
for c in wl2 wl3; do timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/k_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/k_bench_$c.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c", round(d["ms_per_step"],2), "trace/launch", round(r["trace_ms_per_launch"],4), "reduce", r["reduce_ms_per_launch"], "field", r["field_ms_per_launch"], "frac", round(r["frac"],3))
PY
done
