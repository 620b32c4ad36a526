#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
mkdir -p gpurun_out
# A/B two builds on the forward: locked base clocks (ncu) and natural clocks (CUDA events, fwd loop).
for rep in 1 2; do
  for lib in "$1" "$2"; do
    SPARTON_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control base -k regex:sparton_fwd -s 1 -c 2 --csv --log-file gpurun_out/ab.csv python tools/fwd_probe.py 512 512 768 250002 > /dev/null 2>&1
    echo "== base clocks $lib"; python tools/ncu_launches.py gpurun_out/ab.csv
    SPARTON_LIB=$lib python tools/fwd_time.py 512 512 768 250002 "natural $lib"
    sleep 2
  done
done
