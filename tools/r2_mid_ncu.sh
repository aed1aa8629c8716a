#!/bin/bash
# ncu --set full of the mid-size resident leapfrog (C2, 64^3 fp64 and fp32), after a plain run
tag=${1:-midncu}
out=gpurun_out/$tag; mkdir -p $out
for dt in f64 f32; do
  timeout 120 python tools/mid_profile.py $dt > $out/plain_$dt.txt 2>&1; echo "plain $dt rc=$?"; cat $out/plain_$dt.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"leapfrog_mid_kernel" -c 1 \
    -o $out/mid_$dt python tools/mid_profile.py $dt > $out/ncu_$dt.log 2>&1; echo "ncu $dt rc=$?"; tail -2 $out/ncu_$dt.log
done
