#!/bin/bash
# ncu --set full of one layer's four weight-gradient launches in the C3 training step
OUT=gpurun_out/r02bd
mkdir -p $OUT
timeout 300 python scripts/train_once.py C3 16 1 > $OUT/plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -c 4 -o $OUT/wgrad_c3 python scripts/train_once.py C3 16 1 > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
