#!/bin/bash
# ncu --set full of the default fused kernels (leapfrog + Newton pair) on C3-like grids.
# Each capture is preceded by the same command without ncu (must exit 0).
# Usage: bash tools/ncu_kernels.sh <tag> <dtype:n> [<dtype:n> ...]     e.g. f64:256 f32:256 f64:768
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for spec in "$@"; do
  dt=${spec%%:*}; n=${spec##*:}
  timeout 600 python tools/profile_step.py $dt 6 $n > $out/plain_${dt}_${n}.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"pair_|leapfrog_" -s 2 -c 4 \
    -o $out/full_${dt}_${n} python tools/profile_step.py $dt 6 $n > $out/ncu_${dt}_${n}.log 2>&1
  echo "$spec rc=$?" | tee -a $out/rc.txt
done
