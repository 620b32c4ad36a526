#!/bin/bash
# GPU round trip: the given test selection (default: whole -m gpu suite, no -x),
# junit + tail into gpurun_out/, then a short cfg3 bench line.
set -u
mkdir -p gpurun_out
SEL=${SEL:-tests/}
timeout ${TT:-1500} python -m pytest $SEL -m gpu -q --timeout 600 -rf --junitxml=gpurun_out/junit.xml > gpurun_out/tests.txt 2>&1
tail -40 gpurun_out/tests.txt
if [ -z "${NOBENCH:-}" ]; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg3.txt 2>&1
  tail -1 gpurun_out/bench_cfg3.txt | cut -c1-600
fi
