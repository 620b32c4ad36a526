#!/bin/bash
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de -s 9 -c 1 -o gpurun_out/prof_de6 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_dh -s 13 -c 1 -o gpurun_out/prof_dh6 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
