#!/bin/bash
# ncu --set full of the default fused kernels (leapfrog + Newton pair) on C3-like grids.
# Each capture is preceded by the same command without ncu (must exit 0).  The reports are
# summarised on the box (tools/ncu_summary.py + the raw page as CSV) and only the first one is
# kept (gzipped), so gpurun_out/ stays under gpurun's 64 MiB copy-back limit.
# Usage: bash tools/ncu_kernels.sh <tag> <dtype:n> [<dtype:n> ...]     e.g. f64:256 f32:256 f64:768
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
keep=1
for spec in "$@"; do
  dt=${spec%%:*}; n=${spec##*:}
  timeout 600 python tools/profile_step.py $dt 4 $n > $out/plain_${dt}_${n}.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"pair_|leapfrog_" -s 2 -c 4 \
    -o $out/full_${dt}_${n} python tools/profile_step.py $dt 4 $n > $out/ncu_${dt}_${n}.log 2>&1
  echo "$spec rc=$?" | tee -a $out/rc.txt
  if [ -f $out/full_${dt}_${n}.ncu-rep ]; then
    python tools/ncu_summary.py $out/full_${dt}_${n}.ncu-rep > $out/summary_${dt}_${n}.json 2>&1
    ncu -i $out/full_${dt}_${n}.ncu-rep --page raw --csv > $out/raw_${dt}_${n}.csv 2>/dev/null
    ncu -i $out/full_${dt}_${n}.ncu-rep --page source --csv > $out/source_${dt}_${n}.csv 2>/dev/null
    gzip -f $out/raw_${dt}_${n}.csv $out/source_${dt}_${n}.csv
    if [ $keep = 1 ]; then gzip -f $out/full_${dt}_${n}.ncu-rep; keep=0; else rm -f $out/full_${dt}_${n}.ncu-rep; fi
  fi
done
du -sh $out
