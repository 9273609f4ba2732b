#!/bin/bash
mkdir -p gpurun_out/r02ar
timeout 900 python bench.py --gpus 4 --mode train --train-tiles --steps 5 --warmup 3 > gpurun_out/r02ar/bench_train_tiles4_c2.log 2>&1
timeout 900 python bench.py --gpus 4 --mode train --train-tiles --config C3 --steps 3 --warmup 3 > gpurun_out/r02ar/bench_train_tiles4_c3.log 2>&1
timeout 900 python bench.py --mode train --config C3 --steps 3 --warmup 3 > gpurun_out/r02ar/bench_train_c3_1gpu.log 2>&1
