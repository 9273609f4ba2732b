#!/bin/bash
# Round evidence (run under gpurun, 1 GPU): bench line, ncu launch list of the
# same bench command, ncu --set full of the top kernels, attention timeline.
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
CMD="python bench.py --steps 10 --warmup 3"
$CMD > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
LCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
$LCMD > $OUT/plain_list.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $LCMD > $OUT/ncu_list.log 2>&1
FCMD="python bench.py --steps 1 --warmup 1 --batch 16 --no-cpu-baseline --no-profile"
$FCMD > $OUT/plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"attn_tc|mlp_tc|block_tc|gemm_tc_kernel|layernorm|stitch|gather" -s 23 -c 23 -o $OUT/full $FCMD > $OUT/ncu_full.log 2>&1
# timeline variants (built beforehand: build.py --variant tl -D ORBIT2_ATTN_TIMELINE, --variant mtl -D ORBIT2_MLP_TIMELINE)
P=paper_2505_04802_b200
[ -f $P/liborbit2_tl.so ] && ORBIT2_LIB=$P/liborbit2_tl.so python scripts/attn_timeline.py > $OUT/timeline.log 2>&1
[ -f $P/liborbit2_btl.so ] && ORBIT2_LIB=$P/liborbit2_btl.so python scripts/block_timeline.py > $OUT/block_timeline.log 2>&1
ls -la $OUT
