#!/bin/bash
# Full GPU validation of a round: build, smoke, GPU test suite, bench (default + fp32 + C5
# sweep lines), ncu launch list of the bench's timed solve, ncu --set full of the fused kernels.
# Usage: bash tools/gpu_round.sh <tag>
tag=${1:-r1}
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $out/rc.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=20 > $out/pytest_gpu.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt
tail -1 $out/pytest_gpu.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" | tee -a $out/rc.txt
timeout 900 python bench.py --workload c3-f32 > $out/bench_f32.json 2> $out/bench_f32.err; echo "bench_f32 rc=$?" | tee -a $out/rc.txt
# launch list of the timed solve: skip K5 + the warm-up solve
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-serial > $out/plain_short.json 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -s 9150 -c 8900 --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-serial > $out/ncu_launch.log 2>&1; echo "launches rc=$?" | tee -a $out/rc.txt
timeout 300 python tools/profile_step.py f64 > $out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pair_fused|leapfrog_r" -s 4 -c 4 \
  -o $out/prof_f64 python tools/profile_step.py f64 > $out/ncu_full.log 2>&1; echo "full rc=$?" | tee -a $out/rc.txt
