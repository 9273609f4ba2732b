#!/bin/bash
mkdir -p gpurun_out/r02y
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 6 -c 1 \
   -o gpurun_out/r02y/attn_bwd python scripts/train_once.py C2 16 2 > gpurun_out/r02y/ncu_attn_bwd.log 2>&1
