#!/bin/bash
# GPU suite + smoke + default bench after the BF16 head-row validation / decompression change
OUT=gpurun_out/r02aw
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
