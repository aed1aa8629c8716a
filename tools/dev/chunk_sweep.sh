mkdir -p gpurun_out/r2m
for n in 640 384; do for ch in auto 8 16 24 32 48 64 96; do
 if [ $ch = auto ]; then KBENCH_STEPS=40 python tools/kbench.py $n f64 auto c5; else PARAEXP_ZCHUNK=$ch KBENCH_STEPS=40 python tools/kbench.py $n f64 auto c5; fi
done; done > gpurun_out/r2m/chunks.txt 2>&1
PARAEXP_STATIC_SCHED=1 KBENCH_STEPS=40 python tools/kbench.py 640 f64 auto c5 >> gpurun_out/r2m/chunks.txt 2>&1
cat gpurun_out/r2m/chunks.txt
