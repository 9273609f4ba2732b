#!/bin/bash
# Quick GPU iteration: parity subset + 1-GPU bench (run under gpurun).
# usage: scripts/gpu_quick.sh TAG [extra pytest -k expr]
TAG=${1:-q}
K=${2:-"small or C2_full or chunk or rank or batch or multi_item"}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -s -x -k "$K" > gpurun_out/parity_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/parity_$TAG.log
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
tail -2 gpurun_out/parity_$TAG.log
