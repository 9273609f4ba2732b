#!/bin/bash
OUT=gpurun_out/r02o
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -x -k "variable_aggregation or residual_conv or small or C2_full" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set var_agg=1 > $OUT/bench_c2_varagg.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=8 --set dec_hidden=8 > $OUT/bench_c2_convs8.log 2>&1
