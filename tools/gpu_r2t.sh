# A/B of a compile-time kick variant (NUFI_LIB_VARIANT=<tag> loads libnufi_b200_<tag>.so)
mkdir -p gpurun_out
V=${1:-w}
for lib in "" $V; do
for c in ts1 sl1 wl1; do
  NUFI_LIB_VARIANT=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/t_${c}_${lib:-base}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/t_${c}_${lib:-base}.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c ${lib:-base}", round(d["ms_per_step"],3), "frac", round(r["frac"],4))
PY
done; done
NUFI_LIB_VARIANT=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -q -x -k "ts1 or sl1 or wl1 or kat" > gpurun_out/t_pytest.log 2>&1; tail -2 gpurun_out/t_pytest.log
