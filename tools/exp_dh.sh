#!/bin/bash
for v in 2 3 4; do
SPARTON_DH_VARIANT=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_bwd_dh -c 11 --csv --log-file gpurun_out/dh_$v.csv timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
echo variant $v; python tools/ncu_launches.py gpurun_out/dh_$v.csv
done
