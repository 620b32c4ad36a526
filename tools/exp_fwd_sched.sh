#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
# Forward schedule/L2-policy variants at cfg3: ncu DRAM bytes (one launch) + natural-clock time.
run() {
  local label=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control base -k regex:sparton_fwd -s 1 -c 1 --csv --log-file gpurun_out/x.csv python tools/fwd_probe.py 512 512 768 250002 > /dev/null 2>&1
  echo "== $label"; python tools/ncu_launches.py gpurun_out/x.csv
  env "$@" python tools/fwd_time.py 512 512 768 250002 "$label"
}
run default
run group96 SPARTON_FWD_GROUP_KB=98304
run group24 SPARTON_FWD_GROUP_KB=24576
run pol1 SPARTON_E_EVICT_LAST=1
run sched1 SPARTON_FWD_SCHED=1
run default
