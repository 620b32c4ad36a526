#!/bin/bash
# Forward DRAM traffic vs L2 policy and E-group size at cfg3 (one ncu-measured
# launch after a warm-up; --cache-control none so L2 starts as the previous
# launch left it, as inside the step).  SPARTON_E_EVICT_LAST = E | H<<2
# (0 normal, 1 evict_last, 2 evict_first); SPARTON_FWD_GROUP_KB = E group.
export SPARTON_DEV=1
mkdir -p gpurun_out
for g in 49152 32768 65536 98304; do
  for code in 5 1 9; do
    SPARTON_FWD_GROUP_KB=$g SPARTON_E_EVICT_LAST=$code ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/fd_${g}_${code}.csv timeout 300 python tools/fwd_probe.py 512 512 768 250002 > /dev/null 2>&1
    echo "group_kb=$g policy=$code $(python tools/ncu_launches.py gpurun_out/fd_${g}_${code}.csv | tail -1 | cut -c70-)"
  done
done
