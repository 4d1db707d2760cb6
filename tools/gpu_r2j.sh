mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_api_surface.py -m gpu -q -rf -x > gpurun_out/j_pytest.log 2>&1; tail -3 gpurun_out/j_pytest.log
bash tools/fs.sh > gpurun_out/j_fs.txt 2>&1; cat gpurun_out/j_fs.txt
python tools/profile_run.py wl3r 8 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:field_update_kernel -s 4 -c 1 -o gpurun_out/j_prof_field_wl3r python tools/profile_run.py wl3r 8 > gpurun_out/j_ncu.log 2>&1; tail -2 gpurun_out/j_ncu.log
