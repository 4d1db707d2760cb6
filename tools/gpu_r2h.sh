mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_async_dropin.py tests/test_gpu_properties.py -m gpu -q -rf -x > gpurun_out/h_pytest.log 2>&1; tail -3 gpurun_out/h_pytest.log
for c in ts1 wl1 sl1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/h_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/h_bench_$c.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c", round(d["ms_per_step"],3), "frac", round(r["frac"],4), "api", round(d["api_step"]["read_each_step"]["wall_s_to_t_end"]*1e3,2), round(d["api_step"]["read_at_end"]["wall_s_to_t_end"]*1e3,2))
PY
done
timeout 300 python tools/stamps.py ts1
