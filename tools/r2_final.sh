#!/bin/bash
# round-2 measurement set: bench lines, ncu launch list of the bench's solve, ncu --set full of
# the default kernels, C5 sweep, oracle whole-run times, per-config table
tag=${1:-r2f}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" | tee -a $out/rc.txt
timeout 900 python bench.py --workload c3-f32 > $out/bench32.json 2> $out/bench32.err; echo "bench32 rc=$?" | tee -a $out/rc.txt
LL="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-serial --no-e2e"
timeout 900 $LL > $out/ll_plain.json 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $out/launches.csv $LL > $out/ncu_ll.log 2>&1
echo "launches rc=$?" | tee -a $out/rc.txt
python tools/launch_summary.py $out/launches.csv --window solve:2 > $out/launch_summary.csv 2>&1
gzip -f $out/launches.csv
bash tools/ncu_kernels.sh $tag f64:256 f32:256 f64:768
timeout 1500 python tools/sweep_c5.py > $out/sweep_c5.csv 2> $out/sweep.err; echo "sweep rc=$?" | tee -a $out/rc.txt
timeout 1200 python tools/oracle_solve_time.py c1 c2 > $out/oracle_solve.jsonl 2> $out/oracle_solve.err; echo "oracle rc=$?" | tee -a $out/rc.txt
timeout 900 python tools/config_table.py c1 c2 c3 c3-f32 c4 > $out/config_table.jsonl 2> $out/config_table.err; echo "ct rc=$?" | tee -a $out/rc.txt
du -sh $out
