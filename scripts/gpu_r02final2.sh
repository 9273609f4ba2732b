#!/bin/bash
# round-2 final evidence (after the CTA-pair GEMMs and the weight-gradient changes): full GPU suite, smoke, bench lines (default C2, C3, C4), the
# reference arm, training (C2, C3), compression, tile sweep, ncu launch list of the default bench and
# ncu --set full of the C3 pair GEMMs and weight gradients
OUT=gpurun_out/r02final2
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
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 4 -o $OUT/gemm_c3_pair python scripts/infer_once.py C3 16 1 > $OUT/ncu_gemm_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -c 4 -o $OUT/wgrad_c3 python scripts/train_once.py C3 16 1 > $OUT/ncu_wgrad_c3.log 2>&1
ls -la $OUT
