#!/bin/bash
# A/B of the cross-unit prefetch on one box (alternating runs)
mkdir -p gpurun_out/r2ab
for r in 1 2 3; do for la in 0 1; do
  for spec in "256 f64 auto c3" "256 f32 auto c3" "768 f64 auto c5"; do
    PARAEXP_NO_LOOKAHEAD=$la KBENCH_STEPS=100 python tools/kbench.py $spec | sed "s/^/nolookahead=$la /"
  done
done; done > gpurun_out/r2ab/ab.txt 2>&1
cat gpurun_out/r2ab/ab.txt
