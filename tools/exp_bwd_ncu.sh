#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q --timeout 200 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_bwd --csv --log-file gpurun_out/bw.csv timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/bw.csv
