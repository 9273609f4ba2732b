#!/bin/bash
mkdir -p gpurun_out/r02al
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k graph > gpurun_out/r02al/graph_test.log 2>&1
echo "rc=$?" >> gpurun_out/r02al/graph_test.log
timeout 1200 python bench.py --mode sweep --steps 5 --warmup 3 > gpurun_out/r02al/bench_sweep_c2.log 2>&1
