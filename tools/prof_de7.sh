#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q --timeout 200 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de -s 1 -c 1 -o gpurun_out/prof_de7 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
