mkdir -p gpurun_out
for c in ts1 wl1; do NUFI_STAMPS=/tmp/st_$c.txt timeout 300 python tools/profile_run.py $c > /dev/null 2>&1; grep micro /tmp/st_$c.txt > gpurun_out/micro_$c.txt; grep -v "^#" /tmp/st_$c.txt | sed -n '10,12p;100,102p;800,802p' >> gpurun_out/micro_$c.txt; done
