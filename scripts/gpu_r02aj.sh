#!/bin/bash
mkdir -p gpurun_out/r02aj
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 2 -c 1 \
   -o gpurun_out/r02aj/attn_fwd python scripts/infer_once.py C2 16 2 > gpurun_out/r02aj/ncu_attn_fwd.log 2>&1
