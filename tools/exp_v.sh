#!/bin/bash
for V in 30522 61044 122088 250002; do
for S in 512 256; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/v.csv timeout 300 python tools/fwd_probe.py 512 $S 768 $V > /dev/null 2>&1
  echo "V=$V S=$S"; python tools/ncu_launches.py gpurun_out/v.csv
done
done
