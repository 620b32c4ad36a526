#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q --timeout 400 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg3_e2e.txt 2>&1; tail -1 gpurun_out/bench_cfg3_e2e.txt
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_cfg4.txt 2>&1; tail -1 gpurun_out/bench_cfg4.txt
timeout 900 python tools/naive_bench.py > gpurun_out/naive.txt 2>&1; cat gpurun_out/naive.txt | tail -5
