# timing A/B of a compile-time kick variant on the d = 1 N = 64 runs (results not checked)
V=${1:-ax}
for lib in "" $V "" $V; do
for c in ts1 wl1; do
  NUFI_LIB_VARIANT=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/y_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/y_${c}.log").read().strip().splitlines()[-1])
print("$c ${lib:-base}", round(d["ms_per_step"],3))
PY
done; done
