#!/bin/bash
# r02k: full validation + evidence on one GPU: pytest -m gpu, smoke, bench lines (C2 default,
# C3, C4), reference arm, ncu launch list of the default bench, ncu --set full of one forward.
OUT=gpurun_out/r02k
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --no-cpu-baseline > $OUT/bench_C4.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.log 2>&1
LCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $LCMD > $OUT/ncu_list.log 2>&1
FCMD="python bench.py --steps 1 --warmup 1 --batch 16 --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn|block_tc|gemm_tc_kernel|layernorm|stitch|gather" -s 23 -c 23 -o $OUT/full $FCMD > $OUT/ncu_full.log 2>&1
ls -la $OUT
