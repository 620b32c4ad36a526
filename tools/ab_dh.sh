#!/bin/bash
export SPARTON_DEV=1   # the library honours SPARTON_* switches only under this gate
mkdir -p gpurun_out
# A/B dH builds at locked base clocks: tools/ab_dh.sh lib1 lib2 ...
for rep in 1 2; do
for lib in "$@"; do
  SPARTON_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control base -k regex:"dh" --csv --log-file gpurun_out/ab.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  echo "== $lib"; python tools/ncu_launches.py gpurun_out/ab.csv
done
done
