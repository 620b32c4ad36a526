#!/bin/bash
for cfg in "48 40" "100000 40" "24 80" "48 120" "32 60"; do
  set -- $cfg
  SPARTON_DE_CHUNK_MB=$1 SPARTON_DH_CHUNK_MB=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_bwd --csv --log-file gpurun_out/c_$1_$2.csv timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
done
