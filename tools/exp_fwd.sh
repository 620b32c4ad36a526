#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
mkdir -p gpurun_out
for g in 4096 8192 16384 24576; do
  SPARTON_FWD_GROUP_KB=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/f_${g}.csv timeout 300 python tools/fwd_probe.py 512 512 768 250002 > /dev/null 2>&1
  echo "group_kb=$g"; python tools/ncu_launches.py gpurun_out/f_${g}.csv
done
