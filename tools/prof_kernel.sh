#!/bin/bash
# usage: tools/prof_kernel.sh <kernel-regex> <out-name> [skip]  — one ncu --set full capture at cfg3
ncu --set full --clock-control none --import-source on -k regex:$1 -s ${3:-0} -c 1 -o gpurun_out/$2 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/$2.ncu-rep > gpurun_out/$2.txt 2>&1
ncu -i gpurun_out/$2.ncu-rep --page raw --csv > gpurun_out/$2_raw.csv 2>/dev/null
cat gpurun_out/$2.txt
