#!/bin/bash
OUT=gpurun_out/r02p
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "variable_aggregation or residual_conv" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set var_agg=1 > $OUT/bench_c2_varagg.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=8 --set dec_hidden=8 > $OUT/bench_c2_convs8.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --set res_hidden=16 --set dec_hidden=16 > $OUT/bench_c2_convs16.log 2>&1
python - > $OUT/pcie.log 2>&1 <<'PY'
import torch, time
x = torch.empty(800 * 2**20 // 4, dtype=torch.float32).pin_memory(); d = torch.empty_like(x, device="cuda")
for name, f in (("H2D", lambda: d.copy_(x, non_blocking=True)), ("D2H", lambda: x.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    print(name, 5 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9, "GB/s")
PY
