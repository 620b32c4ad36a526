#!/bin/bash
# Profile capture for profiles/: launch list of the bench command + one
# `ncu --set full` capture per kernel family (cfg3), then bench lines.
# Summaries: python tools/make_profiles.py <tag>
mkdir -p gpurun_out
B="timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-plugin --no-sparse --no-cfg1 --no-naive"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-plugin --no-sparse --no-cfg1 --no-naive > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_fwd -s 1 -c 1 -f -o gpurun_out/full_fwd $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de_staged -s 1 -c 1 -f -o gpurun_out/full_de $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_route -s 1 -c 1 -f -o gpurun_out/full_route $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_dh -s 11 -c 1 -f -o gpurun_out/full_dh $B > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
if [ -z "${NOBENCH:-}" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg3_full.txt 2>&1
  timeout 300 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu --no-plugin > gpurun_out/bench_cfg2_full.txt 2>&1
  timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-plugin > gpurun_out/bench_cfg4.txt 2>&1
  for f in bench_cfg3_full bench_cfg2_full bench_cfg4; do tail -1 gpurun_out/$f.txt | cut -c1-400; done
fi
