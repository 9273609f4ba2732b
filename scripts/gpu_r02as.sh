#!/bin/bash
mkdir -p gpurun_out/r02as
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02as/bench_C5.log 2>&1
echo "rc=$?" >> gpurun_out/r02as/bench_C5.log
