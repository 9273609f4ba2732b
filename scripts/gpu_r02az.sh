#!/bin/bash
# ncu --set full of the generic GEMMs at C3 (layer 0 of the first forward: qkv, oproj, mlp_up, mlp_down)
OUT=gpurun_out/r02az
mkdir -p $OUT
timeout 300 python scripts/infer_once.py C3 16 1 > $OUT/plain.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 1 -c 4 -o $OUT/gemm_c3 python scripts/infer_once.py C3 16 1 > $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
