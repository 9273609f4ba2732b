#!/bin/bash
# r02m: 4-GPU strong scaling with sample groups (C2) + peer tests at R = 4.
OUT=gpurun_out/r02m
mkdir -p $OUT
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c2_n1.log 2>&1
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/bench_c2_n2.log 2>&1
timeout 300 python bench.py --gpus 4 --steps 10 --warmup 3 > $OUT/bench_c2_n4.log 2>&1
timeout 300 python bench.py --gpus 4 --steps 10 --warmup 3 --sp-groups 1 > $OUT/bench_c2_n4_g1.log 2>&1
timeout 300 python bench.py --gpus 4 --steps 10 --warmup 3 --sp-groups 8 > $OUT/bench_c2_n4_g8.log 2>&1
timeout 900 python -m pytest tests/test_peer_sp.py -m gpu -q -s > $OUT/pytest_peer4.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_peer4.log
