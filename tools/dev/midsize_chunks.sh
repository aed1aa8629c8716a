#!/bin/bash
out=gpurun_out/r2mid; mkdir -p $out
for n in 64 96; do for ch in auto 1 2 3 4 6 8 16; do
  if [ $ch = auto ]; then KBENCH_STEPS=400 python tools/kbench.py $n f64 auto c3; else PARAEXP_ZCHUNK=$ch KBENCH_STEPS=400 python tools/kbench.py $n f64 auto c3; fi
done; done > $out/chunks.txt 2>&1
cat $out/chunks.txt
