#!/bin/bash
out=gpurun_out/r2c32; mkdir -p $out
for n in 256 384 512 640 768; do KBENCH_STEPS=40 timeout 300 python tools/kbench.py $n f64 auto c5; KBENCH_STEPS=40 timeout 300 python tools/kbench.py $n f32 auto c5; done > $out/kbench.txt 2>&1
KBENCH_STEPS=100 timeout 300 python tools/kbench.py 256 f64 auto c3 >> $out/kbench.txt 2>&1
cat $out/kbench.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct
timeout 600 python tools/profile_step.py f64 4 768 > $out/plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:"pair_|leapfrog_" -s 2 -c 4 --csv python tools/profile_step.py f64 4 768 > $out/ncu.csv 2>&1
grep -E '"(gpu__time|dram__bytes|lts__t_sector_op_read_hit)' $out/ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/"//g' | cut -c1-20,150-
