#!/bin/bash
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de -s 9 -c 1 -o gpurun_out/prof_de5 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_v3 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
