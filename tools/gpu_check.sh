#!/bin/bash
# One gpurun call: GPU tests, bench (with clocks), ncu launch list of a short bench run,
# ncu --set full of the two fused kernels.  Usage: bash tools/gpu_check.sh <tag> [what...]
tag=${1:-r1}; shift
what=${*:-"tests bench launches full"}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $out/rc.txt
for w in $what; do case $w in
tests) timeout 2400 python -m pytest tests -q -m gpu --durations=15 > $out/pytest_gpu.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt;;
tfile=*) timeout 2400 python -m pytest tests/${w#tfile=} -q -m gpu --durations=15 > $out/pytest_${w#tfile=}.log 2>&1; echo "$w rc=$?" | tee -a $out/rc.txt;;
bench) timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" | tee -a $out/rc.txt; tail -1 $out/bench.json;;
bench32) timeout 900 python bench.py --workload c3-f32 > $out/bench32.json 2> $out/bench32.err; echo "bench32 rc=$?" | tee -a $out/rc.txt; tail -1 $out/bench32.json;;
launches) timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-serial > $out/plain_short.json 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-serial > $out/ncu_launch.log 2>&1; echo "launches rc=$?" | tee -a $out/rc.txt;;
full) timeout 300 python tools/profile_step.py f64 > $out/prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pair_fused|leapfrog_fused" -s 2 -c 4 \
  -o $out/prof_f64 python tools/profile_step.py f64 > $out/ncu_full.log 2>&1; echo "full rc=$?" | tee -a $out/rc.txt;;
fullpair) timeout 300 python tools/profile_step.py f64 > $out/prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pair_fused" -s 4 -c 2 \
  -o $out/prof_pair_f64 python tools/profile_step.py f64 > $out/ncu_fullpair.log 2>&1; echo "fullpair rc=$?" | tee -a $out/rc.txt;;
esac; done
