#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
mkdir -p gpurun_out
# A/B two library builds at locked base clocks (ncu --clock-control ${NCU_CLOCK:-base} gives
# run-to-run stable kernel times): tools/ab_kernels.sh <libA> <libB> [regex]
RX=${3:-"sparton"}
for rep in 1 2; do
  for lib in "$1" "$2"; do
    SPARTON_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control ${NCU_CLOCK:-base} -k regex:"$RX" --csv --log-file gpurun_out/ab.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
    echo "== $lib"; python tools/ncu_launches.py gpurun_out/ab.csv
  done
done
