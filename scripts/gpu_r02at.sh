#!/bin/bash
mkdir -p gpurun_out/r02at
timeout 600 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r02at/bench_sp2_c2.log 2>&1
timeout 600 python bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r02at/bench_sp4_c2.log 2>&1
