mkdir -p gpurun_out
for c in ts1 wl1 sl1; do timeout 300 python tools/stamps.py $c > gpurun_out/c_stamps_$c.txt 2>&1; cat gpurun_out/c_stamps_$c.txt; done
