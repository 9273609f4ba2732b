#!/bin/bash
# r02l: decoder / residual convolutions: parity + invariance (1 GPU) and peer SP with convs (2 GPUs).
OUT=gpurun_out/r02l
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_peer_sp.py -m gpu -q -s -k "residual_conv or small or C2_full or peer_sp_multi or chunk or rank or both_attention or zero_head or coordinate" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=8 --set dec_hidden=8 > $OUT/bench_c2_convs.log 2>&1
