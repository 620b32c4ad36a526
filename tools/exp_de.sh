#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/l_a.csv timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
SPARTON_DE_STAGGER=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/l_b.csv timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de -s 12 -c 1 -o gpurun_out/prof_de timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_dh -s 20 -c 1 -o gpurun_out/prof_dh timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/l_a.csv; echo STAGGER; python tools/ncu_launches.py gpurun_out/l_b.csv
