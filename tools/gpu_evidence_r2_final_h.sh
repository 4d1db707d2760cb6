# ts1 evidence after the helper-CTA split: GPU tests, smoke, ts1 bench + reference arm, default
# bench, launch list, ncu capture of the run kernel (command first run plain), stamps, margins
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f10_pytest.log 2>&1; tail -1 gpurun_out/f10_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f10_smoke.log 2>&1; tail -1 gpurun_out/f10_smoke.log
timeout 1500 python bench.py --config ts1 --steps 3 --warmup 3 > gpurun_out/f10_bench_ts1.log 2>&1; tail -1 gpurun_out/f10_bench_ts1.log | cut -c1-120
timeout 1500 python bench.py --impl reference --config ts1 --steps 3 --warmup 1 > gpurun_out/f10_ref_ts1.log 2>&1; tail -1 gpurun_out/f10_ref_ts1.log | cut -c1-120
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f10_bench_default.log 2>&1; tail -1 gpurun_out/f10_bench_default.log | cut -c1-200
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f10_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f10_launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f10_ncu_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/f10_launches_ts1.csv > gpurun_out/f10_launches_ts1.txt 2>&1
python tools/profile_run.py ts1 > gpurun_out/f10_ts1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -s 0 -c 1 -o /tmp/f10_prof_ts1 \
    python tools/profile_run.py ts1 > gpurun_out/f10_ts1_ncu.log 2>&1
python tools/ncu_summary.py /tmp/f10_prof_ts1.ncu-rep > gpurun_out/f10_prof_ts1.txt 2>&1
timeout 300 python tools/stamps.py ts1 > gpurun_out/f10_stamps_ts1.txt 2>&1; head -1 gpurun_out/f10_stamps_ts1.txt
timeout 900 python tools/parity_margins.py ts1 > gpurun_out/f10_parity_margins.txt 2>&1; cat gpurun_out/f10_parity_margins.txt
