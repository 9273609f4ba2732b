#!/bin/bash
# round 2: ncu --set full of the training step's attention backward and weight-gradient GEMM (C2, B=16)
mkdir -p gpurun_out/r02w
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 6 -c 1 \
   -o gpurun_out/r02w/attn_bwd python scripts/train_once.py C2 16 2 > gpurun_out/r02w/ncu_attn_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wgrad -s 4 -c 1 \
   -o gpurun_out/r02w/wgrad python scripts/train_once.py C2 16 2 > gpurun_out/r02w/ncu_wgrad.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ln_bwd -s 2 -c 1 \
   -o gpurun_out/r02w/ln_bwd python scripts/train_once.py C2 16 2 > gpurun_out/r02w/ncu_ln_bwd.log 2>&1
