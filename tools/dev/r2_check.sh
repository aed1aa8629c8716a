#!/bin/bash
# one gpurun call: new multi-rank tests, the whole GPU suite, kernel micro-bench, ncu captures
tag=${1:-r2b}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi > $out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > $out/pytest_multirank.log 2>&1; echo "multirank rc=$?" | tee -a $out/rc.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > $out/pytest_gpu.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt
tail -3 $out/pytest_gpu.log
for n in 256 640 768; do timeout 300 python tools/kbench.py $n f64; done > $out/kbench.txt 2>&1
bash tools/ncu_kernels.sh $tag f64:256 f32:256 f64:768
