mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_multiprocess.py tests/test_gpu_async_dropin.py tests/test_diagnostics.py -m gpu -q -rf -x > gpurun_out/g_pytest.log 2>&1; tail -5 gpurun_out/g_pytest.log
for c in wl2 wl3; do for f in 0 1; do
 if [ $f = 1 ]; then export NUFI_NOFUSE_REDUCE=1; else unset NUFI_NOFUSE_REDUCE; fi
 timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-api-step > gpurun_out/g_bench_${c}_$f.log 2>&1; python - <<PY
import json; d=json.loads(open("gpurun_out/g_bench_${c}_$f.log").read().strip().splitlines()[-1]); r=d["roofline"]
print("$c nofuse=$f", round(d["ms_per_step"],2), "trace/launch", round(r["trace_ms_per_launch"],4), "reduce", r["reduce_ms_per_launch"], "field", r["field_ms_per_launch"], "frac", round(r["frac"],3))
PY
done; done
unset NUFI_NOFUSE_REDUCE
bash tools/fs.sh > gpurun_out/g_fs.txt 2>&1; cat gpurun_out/g_fs.txt
