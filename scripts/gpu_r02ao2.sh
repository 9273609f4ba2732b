#!/bin/bash
mkdir -p gpurun_out/r02ao
for g in 2 4 8; do ORBIT2_E2E_GROUPS=$g timeout 600 python bench.py --no-cpu-baseline --no-profile > gpurun_out/r02ao/bench_g$g.log 2>&1; done
