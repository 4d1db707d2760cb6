# ncu evidence for the round: launch list of the bench command + full captures of the top kernels.
set -x
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/p_bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ts1.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/p_bench_ncu.log 2>&1
python tools/profile_run.py ts1 > gpurun_out/p_ts1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -c 1 -o gpurun_out/prof_ts1_run1d \
    python tools/profile_run.py ts1 > gpurun_out/p_ts1_ncu.log 2>&1
python tools/profile_run.py wl3 40 > gpurun_out/p_wl3_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 39 -c 1 -o gpurun_out/prof_wl3_trace3 \
    python tools/profile_run.py wl3 40 > gpurun_out/p_wl3_ncu.log 2>&1
python tools/profile_run.py wl2 80 > gpurun_out/p_wl2_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:trace_rho_kernel -s 79 -c 1 -o gpurun_out/prof_wl2_trace2 \
    python tools/profile_run.py wl2 80 > gpurun_out/p_wl2_ncu.log 2>&1
python tools/profile_run.py sl1 > gpurun_out/p_sl1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:run_1d_kernel -c 1 -o gpurun_out/prof_sl1_run1d \
    python tools/profile_run.py sl1 > gpurun_out/p_sl1_ncu.log 2>&1
ls -la gpurun_out
