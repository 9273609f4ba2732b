#!/bin/bash
# round 2: training-step bench at C2 (auto batch), per-kernel classes; ncu launch list of a short run
mkdir -p gpurun_out/r02s
timeout 600 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r02s/bench_train_c2.log 2>&1
echo "rc=$?" >> gpurun_out/r02s/bench_train_c2.log
timeout 600 python bench.py --mode train --steps 5 --warmup 3 --batch 16 > gpurun_out/r02s/bench_train_c2_b16.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02s/launches_train_b16.csv \
   python bench.py --mode train --steps 1 --warmup 1 --batch 16 --no-profile > gpurun_out/r02s/ncu_train.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02s/ncu_train.log
