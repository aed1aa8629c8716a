#!/bin/bash
# ncu --set full of one non-init K2 launch (C3-like grid), summarised on the box
tag=$1; dt=${2:-f64}; n=${3:-256}; kre=${4:-pair_}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 python tools/profile_step.py $dt 2 $n > $out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 1 -c 1 \
  -o $out/pair_${dt}_${n} python tools/profile_step.py $dt 2 $n > $out/ncu.log 2>&1
echo "rc=$?" | tee $out/rc.txt
python tools/ncu_summary.py $out/pair_${dt}_${n}.ncu-rep > $out/summary.json 2>&1
ncu -i $out/pair_${dt}_${n}.ncu-rep --page source --csv 2>/dev/null | gzip > $out/source.csv.gz
ncu -i $out/pair_${dt}_${n}.ncu-rep --page raw --csv 2>/dev/null | gzip > $out/raw.csv.gz
gzip -f $out/pair_${dt}_${n}.ncu-rep
