mkdir -p gpurun_out
for c in wl3 wl2 sl1 ts1; do timeout 900 python tools/scaling_projection.py $c 20 50 > gpurun_out/o_scal_$c.json 2> gpurun_out/o_scal_$c.err; tail -c 600 gpurun_out/o_scal_$c.json; echo; tail -2 gpurun_out/o_scal_$c.err; done
