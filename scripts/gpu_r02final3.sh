#!/bin/bash
# certification run at the last commit: full GPU suite, smoke, default bench, training line
OUT=gpurun_out/r02final3
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
timeout 900 python bench.py --mode train --steps 5 --warmup 3 > $OUT/bench_train_C2.log 2>&1
timeout 900 python bench.py --mode train --config C3 --steps 3 --warmup 3 > $OUT/bench_train_C3.log 2>&1
