# timing A/B of a compile-time variant on sl1 / ts1 (interleaved, 2 rounds)
for r in 1 2; do for lib in "" "$@"; do for c in sl1 ts1; do
  NUFI_LIB_VARIANT=$lib timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/t2_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/t2_${c}.log").read().strip().splitlines()[-1])
print("$c ${lib:-base}", round(d["ms_per_step"],3))
PY
done; done; done
