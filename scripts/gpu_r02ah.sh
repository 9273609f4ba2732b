#!/bin/bash
mkdir -p gpurun_out/r02ah
ORBIT2_SYNC_CHECK=1 timeout 900 python -m pytest tests/test_gpu_compress.py -x -q -s > gpurun_out/r02ah/compress_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ah/compress_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ah/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02ah/smoke.log
