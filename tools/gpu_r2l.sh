mkdir -p gpurun_out
for ps in 1 2 4; do NUFI_PASSES=$ps timeout 900 python bench.py --config wl2 --steps 2 --warmup 1 --no-cpu-baseline --no-api-step > gpurun_out/l_wl2_$ps.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/l_wl2_$ps.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("wl2 passes=$ps", round(d["ms_per_step"],2), "trace/launch", round(r["trace_ms_per_launch"],4), "field", r["field_ms_per_launch"], "frac", round(r["frac"],3))
PY
done
for ps in 4 8 16; do NUFI_PASSES=$ps timeout 900 python bench.py --config wl3 --steps 1 --warmup 1 --no-cpu-baseline --no-api-step > gpurun_out/l_wl3_$ps.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/l_wl3_$ps.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("wl3 passes=$ps", round(d["ms_per_step"],2), "trace/launch", round(r["trace_ms_per_launch"],4), "field", r["field_ms_per_launch"], "frac", round(r["frac"],3))
PY
done
