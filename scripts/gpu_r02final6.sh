#!/bin/bash
# certification run at the last code commit (after the stitch-backward and loss-kernel changes): full GPU suite, smoke, C2 / C3 / C4 / reference / training lines, launch list
OUT=gpurun_out/r02final6
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
timeout 900 python bench.py --mode train --steps 5 --warmup 3 > $OUT/bench_train_C2.log 2>&1
timeout 900 python bench.py --mode train --config C3 --steps 3 --warmup 3 > $OUT/bench_train_C3.log 2>&1
timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $OUT/bench_C4.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.log 2>&1
LCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $LCMD > $OUT/ncu_list.log 2>&1
