#!/bin/bash
# r02a: full GPU test suite (new sampled C3/C4/C5 bf16 + fp32 parity) + bench line.
OUT=gpurun_out/r02a
mkdir -p $OUT
nproc > $OUT/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -s -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
