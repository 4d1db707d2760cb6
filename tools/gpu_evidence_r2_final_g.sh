# sl1 evidence after two tiles per pass in the WIDE d = 1 kernel: GPU tests, bench + reference
# arm, ncu capture of the run kernel (command first run plain), stamps, parity margins
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f8_pytest.log 2>&1; tail -1 gpurun_out/f8_pytest.log
timeout 1500 python bench.py --config sl1 --steps 3 --warmup 3 > gpurun_out/f8_bench_sl1.log 2>&1; tail -1 gpurun_out/f8_bench_sl1.log | cut -c1-120
timeout 1500 python bench.py --impl reference --config sl1 --steps 3 --warmup 1 > gpurun_out/f8_ref_sl1.log 2>&1; tail -1 gpurun_out/f8_ref_sl1.log | cut -c1-120
python tools/profile_run.py sl1 > gpurun_out/f8_sl1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -s 0 -c 1 -o /tmp/f8_prof_sl1 \
    python tools/profile_run.py sl1 > gpurun_out/f8_sl1_ncu.log 2>&1
python tools/ncu_summary.py /tmp/f8_prof_sl1.ncu-rep > gpurun_out/f8_prof_sl1.txt 2>&1
timeout 300 python tools/stamps.py sl1 > gpurun_out/f8_stamps_sl1.txt 2>&1; head -1 gpurun_out/f8_stamps_sl1.txt
timeout 900 python tools/parity_margins.py sl1 > gpurun_out/f8_parity_margins.txt 2>&1; cat gpurun_out/f8_parity_margins.txt
