mkdir -p gpurun_out
for c in ts1 wl1 wl2; do timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/d_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/d_bench_$c.log").read().strip().splitlines()[-1])
print("$c", d["ms_per_step"], d["value"], d["e2e"]["value"], d["api_step"])
PY
done
