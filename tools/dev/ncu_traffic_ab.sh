#!/bin/bash
# DRAM bytes per launch of K1r / K2 at 768^3 under env variants (ncu, 3 metrics only)
out=gpurun_out/r2tr; mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct
for v in "X=1" "PARAEXP_NO_LOOKAHEAD=1" "PARAEXP_ZCHUNK=74" "PARAEXP_ZCHUNK=74 PARAEXP_NO_LOOKAHEAD=1" "PARAEXP_ZCHUNK=24"; do
  env $v timeout 600 python tools/profile_step.py f64 4 768 > $out/plain.log 2>&1 && \
  env $v timeout 900 ncu --metrics $M --clock-control none -k regex:"pair_|leapfrog_" -s 2 -c 4 --csv \
    python tools/profile_step.py f64 4 768 > $out/ncu.csv 2>&1
  echo "== $v rc=$?" >> $out/res.txt
  grep -E '"(gpu__time|dram__bytes|lts__t_sector_op_read_hit)' $out/ncu.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/"//g' >> $out/res.txt
done
cat $out/res.txt
