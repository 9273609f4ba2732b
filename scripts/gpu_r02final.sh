#!/bin/bash
# round-2 final evidence at one commit: full GPU suite, smoke, bench lines (default C2, C3, C4), the
# reference arm, training (C2, C3), compression, tile sweep, ncu launch list of the default bench and
# ncu --set full of the attention forward / backward
OUT=gpurun_out/r02final
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $OUT/bench_C4.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.log 2>&1
timeout 900 python bench.py --mode train --steps 5 --warmup 3 > $OUT/bench_train_C2.log 2>&1
timeout 900 python bench.py --mode train --config C3 --steps 3 --warmup 3 > $OUT/bench_train_C3.log 2>&1
timeout 900 python bench.py --mode compress --steps 10 --warmup 3 > $OUT/bench_compress.log 2>&1
timeout 1200 python bench.py --mode sweep --steps 5 --warmup 3 > $OUT/bench_sweep.log 2>&1
LCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $LCMD > $OUT/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 2 -c 1 -o $OUT/attn_fwd python scripts/infer_once.py C2 16 2 > $OUT/ncu_attn_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 6 -c 1 -o $OUT/attn_bwd python scripts/train_once.py C2 16 2 > $OUT/ncu_attn_bwd.log 2>&1
ls -la $OUT
