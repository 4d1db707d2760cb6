# timing A/B of compile-time variants on ts1 / wl1 (interleaved, 2 rounds)
for r in 1 2; do for lib in "" "$@"; do for c in ts1 wl1; do
  NUFI_LIB_VARIANT=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/s2_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/s2_${c}.log").read().strip().splitlines()[-1])
print("$c ${lib:-base}", round(d["ms_per_step"],3))
PY
done; done; done
