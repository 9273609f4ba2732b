#!/bin/bash
# multi-GPU re-confirmation at the last code commit (run under gpurun --gpus 4): the peer-SP tests, the
# driver's torchrun launch of the default bench at N = 2 / 4, C4 at 4 GPUs, tile-parallel training
OUT=gpurun_out/r02bw
mkdir -p $OUT
timeout 900 python -m pytest tests/test_peer_sp.py -m gpu -q -rA > $OUT/pytest_peer.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_peer.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_torchrun_n$N.log 2>&1
done
timeout 900 python bench.py --gpus 4 --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_C4_n4.log 2>&1
timeout 900 python bench.py --gpus 4 --mode train --train-tiles --steps 5 --warmup 3 > $OUT/bench_train_tiles_n4.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,power.draw --format=csv >> $OUT/smi.txt
