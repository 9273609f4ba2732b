#!/bin/bash
# round 2: f4 integrated (forward on compressed tokens) + compression kernels after the GEMM rewrite
mkdir -p gpurun_out/r02ab
ORBIT2_SYNC_CHECK=1 timeout 900 python -m pytest tests/test_gpu_compress.py -x -q -s > gpurun_out/r02ab/compress_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ab/compress_tests.log
timeout 600 python bench.py --mode compress --steps 10 --warmup 3 > gpurun_out/r02ab/bench_compress_c2.log 2>&1
