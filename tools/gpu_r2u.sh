# full GPU suite + d=1 bench lines after a kernel change
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/u_pytest.log 2>&1; tail -3 gpurun_out/u_pytest.log
for c in ts1 sl1 wl1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-api-step > gpurun_out/u_${c}.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/u_${c}.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c", round(d["ms_per_step"],3), "frac", round(r["frac"],4), d["clocks"])
PY
done
for c in ts1 wl1; do timeout 300 python tools/stamps.py $c 2>/dev/null | grep -v "^  n=" ; done
