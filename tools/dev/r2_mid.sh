#!/bin/bash
# mid-size kernels: parity tests, timing against the TMA kernels, C2 config-table row
tag=${1:-mid1}
out=gpurun_out/$tag; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_mid.py -x -q > $out/pytest_mid.log 2>&1; echo "mid tests rc=$?" | tee -a $out/rc.txt
tail -30 $out/pytest_mid.log
timeout 300 python tools/mid_bench.py 32 48 64 > $out/mid_bench.txt 2>&1; echo "mid bench rc=$?" | tee -a $out/rc.txt
cat $out/mid_bench.txt
timeout 300 python tools/config_table.py c2 > $out/config_c2.jsonl 2> $out/config_c2.err; echo "ct rc=$?" | tee -a $out/rc.txt
cat $out/config_c2.jsonl; tail -3 $out/config_c2.err
