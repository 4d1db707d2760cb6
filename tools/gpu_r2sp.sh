# the d = 1 split (helper CTAs trace every tile's last row): GPU tests, then ts1 / wl1 timing
# against the previous build (libnufi_b200_old.so) and with the split turned off
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/sp_pytest.log 2>&1; tail -2 gpurun_out/sp_pytest.log
for r in 1 2; do for v in "base" "old" "nosplit"; do for c in ts1 wl1; do
  lib=""; [ $v = old ] && lib=old; ns=1; [ $v = nosplit ] && ns=0
  NUFI_D1_SPLIT=$ns NUFI_LIB_VARIANT=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/sp_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/sp_${c}.log").read().strip().splitlines()[-1])
print("$c $v", round(d["ms_per_step"],3))
PY
done; done; done
