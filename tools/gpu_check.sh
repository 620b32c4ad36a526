#!/bin/bash
# One GPU round trip: parity tests, cfg3/cfg2 bench, per-kernel launch list.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 400 2>&1 | tail -15 > gpurun_out/tests.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg3.txt 2>&1
timeout 200 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_cfg2.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
cat gpurun_out/tests.txt
for f in gpurun_out/bench_cfg3.txt gpurun_out/bench_cfg2.txt; do
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], 'TF/s=%.1f ms=%.2f fwd=%.2f bwd=%.2f' % (d['value'], d['ms_per_step'], d['fwd_ms'], d['bwd_ms']), d['clocks'])" $f || tail -5 $f
done
python tools/ncu_launches.py gpurun_out/launches_cfg3.csv
