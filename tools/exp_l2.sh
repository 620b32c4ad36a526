#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
# Forward DRAM-traffic probes at cfg3 (ncu, one launch each).
run() {  # label, env..., then shape
  local label=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/x.csv timeout 300 python tools/fwd_probe.py $SHAPE > /dev/null 2>&1
  echo "$label"; python tools/ncu_launches.py gpurun_out/x.csv
}
SHAPE="512 512 768 250002"
run persist40_pol1 SPARTON_L2_PERSIST_MB=40 SPARTON_E_EVICT_LAST=1
run persist80_pol1 SPARTON_L2_PERSIST_MB=80 SPARTON_E_EVICT_LAST=1
run persist80_pol5 SPARTON_L2_PERSIST_MB=80 SPARTON_E_EVICT_LAST=5
run sched1 SPARTON_FWD_SCHED=1
run sched1_pol5 SPARTON_FWD_SCHED=1 SPARTON_E_EVICT_LAST=5
run group32 SPARTON_FWD_GROUP_KB=32768
run group48 SPARTON_FWD_GROUP_KB=49152
run group48_pol5 SPARTON_FWD_GROUP_KB=49152 SPARTON_E_EVICT_LAST=5
run group64_pol5 SPARTON_FWD_GROUP_KB=65536 SPARTON_E_EVICT_LAST=5
SHAPE="256 512 768 250002"
run B256 SPARTON_E_EVICT_LAST=1
SHAPE="512 512 768 250002"
run cg1 SPARTON_FWD_CLUSTER=1
