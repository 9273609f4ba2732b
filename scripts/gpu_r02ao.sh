#!/bin/bash
mkdir -p gpurun_out/r02ao
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "forward_host or graph" > gpurun_out/r02ao/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ao/tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02ao/bench.log 2>&1
