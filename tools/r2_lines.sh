#!/bin/bash
# secondary bench lines (one B200): the other BASELINE workloads, the C5 sweep, the config table
tag=${1:-r2l}
out=gpurun_out/$tag; mkdir -p $out
run() { name=$1; shift; timeout 1200 python bench.py "$@" > $out/$name.json 2> $out/$name.err; echo "$name rc=$?" | tee -a $out/rc.txt; tail -1 $out/$name.json | cut -c1-200; }
run c3p64 --workload c3 --p 64
run c2 --workload c2
run c1 --workload c1
run c4 --workload c4 --warmup 3 --steps 1 --no-e2e --no-cpu-baseline
for p in 8 16 64; do run c5s768_p$p --workload c5s-768-f64 --p $p --warmup 3 --steps 1 --no-e2e --no-cpu-baseline; done
[ -z "$SKIP_EXTRA" ] && timeout 1500 python tools/sweep_c5.py > $out/sweep_c5.csv 2> $out/sweep.err; echo "sweep rc=$?" | tee -a $out/rc.txt
[ -z "$SKIP_EXTRA" ] && timeout 900 python tools/config_table.py c1 c2 c3 c3-f32 c4 > $out/config_table.jsonl 2> $out/config_table.err; echo "ct rc=$?" | tee -a $out/rc.txt
