#!/bin/bash
# r02g: 4-GPU strong scaling (peer-memory SP) for C2 and C4 + 1-GPU baselines + peer tests at R = 4.
OUT=gpurun_out/r02g
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c2_n1.log 2>&1
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/bench_c2_n2.log 2>&1
timeout 300 python bench.py --gpus 4 --steps 10 --warmup 3 > $OUT/bench_c2_n4.log 2>&1
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_n1.log 2>&1
timeout 600 python bench.py --config C4 --gpus 2 --steps 3 --warmup 3 > $OUT/bench_c4_n2.log 2>&1
timeout 600 python bench.py --config C4 --gpus 4 --steps 3 --warmup 3 > $OUT/bench_c4_n4.log 2>&1
timeout 900 python -m pytest tests/test_peer_sp.py -m gpu -q -s > $OUT/pytest_peer4.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_peer4.log
