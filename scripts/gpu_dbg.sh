#!/bin/bash
OUT=gpurun_out/dbg
mkdir -p $OUT
cat > /tmp/dbg1.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from workloads import get_config, make_input, make_weights
from tests.gpu_helpers import run_cuda, oracle_full, rel_err
name, over = sys.argv[1], eval(sys.argv[2])
w = get_config(name, batch=int(sys.argv[3]), **over)
x = make_input(w); blob = make_weights(w)
got = run_cuda(w, x, blob, 0)
print("ran", name, over, np.isfinite(got).all())
if w.batch <= 2 and w.H <= 64:
    print("rel", rel_err(got, oracle_full(w, x, blob)[0]))
PY
export ORBIT2_SYNC_CHECK=1 ORBIT2_TRACE=1 ORBIT2_DEBUG_TMAP=1
timeout 120 python /tmp/dbg1.py C1 "dict(tiles_y=3, tiles_x=5, halo=1)" 1 > $OUT/c1_3x5.log 2>&1
timeout 120 python /tmp/dbg1.py C2 "dict()" 2 > $OUT/c2.log 2>&1
timeout 120 compute-sanitizer --tool memcheck python /tmp/dbg1.py C1 "dict(tiles_y=3, tiles_x=5, halo=1)" 1 > $OUT/c1_3x5_san.log 2>&1
