#!/bin/bash
# kernel iteration: parity subset, kernel micro-bench, per-config table
tag=${1:-r2i}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py tests/test_gpu_small.py -q -x > $out/pytest.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt
tail -2 $out/pytest.log
for spec in 256:f64 256:f32 768:f64 768:f32; do n=${spec%%:*}; d=${spec##*:}; timeout 300 python tools/kbench.py $n $d; done > $out/kbench.txt 2>&1
cat $out/kbench.txt
timeout 900 python tools/config_table.py c1 c2 c4 > $out/config_table.jsonl 2> $out/config_table.err; echo "ct rc=$?"
cat $out/config_table.jsonl
