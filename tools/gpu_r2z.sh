# A/B of the d = 1 two-level combine and ring depth knobs on ts1 / wl1
for knob in "" "NUFI_TWO_LEVEL=1" "" "NUFI_TWO_LEVEL=1"; do
for c in ts1 wl1; do
  env $knob timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/z_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/z_${c}.log").read().strip().splitlines()[-1])
print("$c ${knob:-default}", round(d["ms_per_step"],3))
PY
done; done
