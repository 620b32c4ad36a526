#!/bin/bash
# Profile capture for profiles/: launch list of the bench command + one
# `ncu --set full` capture per kernel family (cfg3), then bench lines.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_fwd -s 1 -c 1 -o gpurun_out/full_fwd timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_de_staged -s 1 -c 1 -o gpurun_out/full_de timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_route -s 1 -c 1 -o gpurun_out/full_route timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sparton_bwd_dh -s 11 -c 1 -o gpurun_out/full_dh timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg3_full.txt 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 > gpurun_out/bench_cfg2_full.txt 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
timeout 600 python tools/naive_bench.py > gpurun_out/naive.txt 2>&1
tail -1 gpurun_out/bench_cfg3_full.txt; tail -1 gpurun_out/bench_cfg2_full.txt; tail -1 gpurun_out/bench_ref.txt; tail -3 gpurun_out/naive.txt
timeout 900 python tools/splade_bench.py 64 256 > gpurun_out/splade.txt 2>&1
timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg4.txt 2>&1
tail -1 gpurun_out/bench_cfg4.txt
