#!/bin/bash
tag=${1:-midncu}
out=gpurun_out/$tag; mkdir -p $out
timeout 120 python tools/mid_profile.py > $out/plain.txt 2>&1; echo "plain rc=$?"; cat $out/plain.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mid_kernel" -c 2 -o $out/mid_f64 python tools/mid_profile.py > $out/ncu.log 2>&1; echo "ncu rc=$?"; tail -5 $out/ncu.log
