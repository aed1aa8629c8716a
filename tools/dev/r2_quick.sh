#!/bin/bash
# quick kernel iteration: [parity subset] + kernel micro-bench.  Usage: r2_quick.sh tag [notest] [n:dtype ...]
tag=${1:-r2q}; shift
out=gpurun_out/$tag; mkdir -p $out
if [ "$1" = notest ]; then shift; else
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py -q -x > $out/pytest.log 2>&1; echo "tests rc=$?" | tee -a $out/rc.txt
tail -2 $out/pytest.log
fi
specs="$*"; [ -z "$specs" ] && specs="256:f64 256:f32 768:f64 512:f32"
for spec in $specs; do n=${spec%%:*}; d=${spec##*:}; timeout 300 python tools/kbench.py $n $d; done > $out/kbench.txt 2>&1
cat $out/kbench.txt
