#!/bin/bash
for st in 0 1; do
SPARTON_DE_STAGGER=$st ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_bwd_de --csv --log-file gpurun_out/st$st.csv timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
echo stagger $st; python tools/ncu_launches.py gpurun_out/st$st.csv
done
