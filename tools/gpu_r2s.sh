mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -q -rf -x > gpurun_out/s_pytest.log 2>&1; tail -2 gpurun_out/s_pytest.log
for r in 1 2 3; do for c in ts1 wl1; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/s_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/s_bench_$c.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c", round(d["ms_per_step"],3), "frac", round(r["frac"],4))
PY
done; done
