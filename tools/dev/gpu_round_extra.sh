#!/bin/bash
# gpu_round.sh plus the per-config table and the C5 sweep.  Usage: bash tools/gpu_round_extra.sh <tag>
bash tools/gpu_round.sh ${1:-r1}
timeout 900 python tools/config_table.py > gpurun_out/${1:-r1}/config_table.jsonl 2> gpurun_out/${1:-r1}/config_table.err; echo "ct rc=$?"
timeout 1200 python tools/sweep_c5.py > gpurun_out/${1:-r1}/sweep_c5.csv 2> gpurun_out/${1:-r1}/sweep.err; echo "sweep rc=$?"
