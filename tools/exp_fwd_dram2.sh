#!/bin/bash
# Forward DRAM traffic vs E-group size at cfg3, policy 5 (E and H evict_last),
# two ncu-measured launches per size (see exp_fwd_dram.sh).
export SPARTON_DEV=1 SPARTON_E_EVICT_LAST=5
mkdir -p gpurun_out
for g in 8192 12288 16384 20480 24576 28672 32768 40960 49152; do
  SPARTON_FWD_GROUP_KB=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none -k regex:sparton_fwd -s 1 -c 2 --csv --log-file gpurun_out/fg_${g}.csv timeout 300 python tools/fwd_probe.py 512 512 768 250002 3 > /dev/null 2>&1
  echo "group_kb=$g $(python tools/ncu_launches.py gpurun_out/fg_${g}.csv | tail -1 | cut -c70-)"
done
