# Multi-GPU evidence at HEAD (run under gpurun --gpus N): dp weak scaling and TILES SP strong scaling.
N=${1:-4}
OUT=gpurun_out/r01e/multigpu
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 600 $R bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_dp$N.log 2>&1
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_C4_n1.log 2>&1
timeout 600 $R bench.py --gpus $N --mode sp --config C4 --steps 5 --warmup 3 > $OUT/bench_sp_C4_n$N.log 2>&1
ls -la $OUT
