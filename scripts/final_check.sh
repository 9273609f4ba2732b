OUT=gpurun_out/r01e
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench exit $?" >> $OUT/bench.log
LCMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-profile"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $LCMD > $OUT/ncu_list.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.log 2>&1
ls -la $OUT
