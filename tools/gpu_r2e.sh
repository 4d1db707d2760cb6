mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async_dropin.py tests/test_gpu_api_surface.py tests/test_gpu_parity.py tests/test_kernels_plugin.py -m gpu -q -rf -x > gpurun_out/e_pytest.log 2>&1; tail -30 gpurun_out/e_pytest.log
for c in ts1 wl1 wl2; do timeout 600 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/e_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/e_bench_$c.log").read().strip().splitlines()[-1])
print("$c", d["ms_per_step"], d["value"], d["e2e"]["value"], d["api_step"])
PY
done
