#!/bin/bash
mkdir -p gpurun_out
# A/B environment switches at locked base clocks:
#   tools/ab_env.sh <kernel regex> "VAR=a" "VAR=b" ...   ("-" = no switch)
RX=$1; shift
for rep in 1 2; do
  for kv in "$@"; do
    if [ "$kv" = "-" ]; then set_env=(); else set_env=("$kv"); fi
    env "${set_env[@]}" ncu --metrics gpu__time_duration.sum --clock-control base -k regex:"$RX" --csv \
      --log-file gpurun_out/ab.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
    echo "== $kv"; python tools/ncu_launches.py gpurun_out/ab.csv
  done
done
