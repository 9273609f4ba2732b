#!/bin/bash
mkdir -p gpurun_out/r02ai
timeout 900 python bench.py --mode compress --steps 10 --warmup 3 > gpurun_out/r02ai/bench_compress_c2.log 2>&1
