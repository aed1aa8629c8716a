#!/bin/bash
tag=${1:-r2y}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "longer_horizon or c4" > $out/pytest_c4.log 2>&1; echo "c4 tests rc=$?" | tee -a $out/rc.txt; tail -2 $out/pytest_c4.log
timeout 900 python tools/config_table.py c1 c2 c3 c3-f32 c4 > $out/config_table.jsonl 2> $out/config_table.err; echo "ct rc=$?" | tee -a $out/rc.txt
SKIP_EXTRA=1 bash tools/r2_lines.sh $tag.l > /dev/null 2>&1; echo "lines rc=$?" | tee -a $out/rc.txt
