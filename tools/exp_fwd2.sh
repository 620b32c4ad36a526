#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
for shape in "512 512 768 256" "64 512 768 250002" "8 512 768 250002" "512 512 768 30522" "128 512 768 250002"; do
  set -- $shape
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/p.csv timeout 300 python tools/fwd_probe.py $1 $2 $3 $4 > /dev/null 2>&1
  echo "shape=$shape"; python tools/ncu_launches.py gpurun_out/p.csv
  SPARTON_FWD_SCHED=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/p.csv timeout 300 python tools/fwd_probe.py $1 $2 $3 $4 > /dev/null 2>&1
  echo "shape=$shape sched=0"; python tools/ncu_launches.py gpurun_out/p.csv
done
