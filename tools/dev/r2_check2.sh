#!/bin/bash
tag=${1:-r2c}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q > $out/pytest_multirank.log 2>&1; echo "multirank rc=$?" | tee -a $out/rc.txt
timeout 1800 python -m pytest tests/test_gpu_horizon.py -q --durations=5 > $out/pytest_horizon.log 2>&1; echo "horizon rc=$?" | tee -a $out/rc.txt
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" | tee -a $out/rc.txt
bash tools/ncu_kernels.sh $tag f64:256 f32:256
