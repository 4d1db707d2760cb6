mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async_dropin.py tests/test_gpu_api_surface.py tests/test_gpu_parity.py -m gpu -q -rf -x > gpurun_out/m_pytest.log 2>&1; tail -3 gpurun_out/m_pytest.log
for c in ts1 wl1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/m_bench_$c.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/m_bench_$c.log").read().strip().splitlines()[-1]); a=d["api_step"]
print("$c", round(d["ms_per_step"],2), round(a["read_each_step"]["wall_s_to_t_end"]*1e3,2), round(a["read_at_end"]["wall_s_to_t_end"]*1e3,2))
PY
done
