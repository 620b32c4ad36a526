#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
# E policy | H policy<<2 : 0 normal, 1 last, 2 first
for code in 1 0 4 5 8 9 2; do
  SPARTON_E_EVICT_LAST=$code ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/pol_$code.csv timeout 300 python tools/fwd_probe.py 512 512 768 250002 > /dev/null 2>&1
  echo "policy=$code"; python tools/ncu_launches.py gpurun_out/pol_$code.csv
done
