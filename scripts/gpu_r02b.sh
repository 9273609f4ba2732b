#!/bin/bash
# r02b: peer-memory SP -- processes on one GPU (pytest) and real 2-GPU runs.
OUT=gpurun_out/r02b
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 600 python -m pytest tests/test_peer_sp.py -m gpu -q -s -x > $OUT/pytest_peer.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_peer.log
timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/sp_peer_demo.py C2 2 oracle > $OUT/demo_c2b2.log 2>&1; echo "exit $?" >> $OUT/demo_c2b2.log
timeout 300 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 scripts/sp_peer_demo.py C2 64 > $OUT/demo_c2b64.log 2>&1; echo "exit $?" >> $OUT/demo_c2b64.log
timeout 300 python bench.py --gpus 2 --steps 10 --warmup 3 > $OUT/bench2.log 2>&1; echo "exit $?" >> $OUT/bench2.log
timeout 300 python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench1.log 2>&1; echo "exit $?" >> $OUT/bench1.log
