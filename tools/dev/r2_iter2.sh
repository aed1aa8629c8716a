#!/bin/bash
tag=${1:-r2n}
out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_small.py -q -x > $out/pytest.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt
tail -2 $out/pytest.log
for n in 256 384 512 640 768; do KBENCH_STEPS=40 timeout 300 python tools/kbench.py $n f64 auto c5; KBENCH_STEPS=40 timeout 300 python tools/kbench.py $n f32 auto c5; done > $out/kbench.txt 2>&1
KBENCH_STEPS=100 timeout 300 python tools/kbench.py 256 f64 auto c3 >> $out/kbench.txt 2>&1
cat $out/kbench.txt
