#!/bin/bash
# round 2: full GPU suite; default bench (inference C2); training bench (C2 B=64); compression bench;
# ncu launch lists of the training step and of the compression step
mkdir -p gpurun_out/r02aa
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02aa/pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02aa/pytest.log
timeout 600 python bench.py > gpurun_out/r02aa/bench_c2.log 2>&1
timeout 900 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r02aa/bench_train_c2.log 2>&1
timeout 600 python bench.py --mode compress --steps 10 --warmup 3 > gpurun_out/r02aa/bench_compress_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02aa/launches_train_b16.csv \
   python scripts/train_once.py C2 16 1 > gpurun_out/r02aa/ncu_train.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02aa/launches_compress.csv \
   python bench.py --mode compress --steps 1 --warmup 1 > gpurun_out/r02aa/ncu_compress.log 2>&1
