#!/bin/bash
OUT=gpurun_out/r02n
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi_host.py -m "gpu" -q -s -k "residual_conv" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=8 --set dec_hidden=8 > $OUT/bench_c2_convs8.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=8 > $OUT/bench_c2_res8.log 2>&1
