#!/bin/bash
# r02h: 3-Q-tile / 64-key attention (attn3_tc.cu): parity subset + A/B vs the 2-tile kernel.
OUT=gpurun_out/r02h
mkdir -p $OUT
P=paper_2505_04802_b200
export ORBIT2_LIB=$P/liborbit2_attn3.so
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
from workloads import get_config, make_input, make_weights
from tests.gpu_helpers import run_cuda, oracle_full, rel_err
w = get_config('C2', batch=1, H=48, W=96, tiles_y=2, tiles_x=3, depth=2)
x = make_input(w); blob = make_weights(w)
got = run_cuda(w, x, blob, 0)
print('quick C2-small rel', rel_err(got, oracle_full(w, x, blob)[0]), np.isfinite(got).all())
" > $OUT/quick.log 2>&1; echo "exit $?" >> $OUT/quick.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "small or C2_full or chunk or rank or packing or repeated or multi_item or bench_configuration or batch_independence" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
AB_LIBS="$ORBIT2_LIB" timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_attn3.log 2>&1
AB_LIBS="$ORBIT2_LIB" ORBIT2_ATTN2=1 timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_attn2.log 2>&1
AB_LIBS="$ORBIT2_LIB" timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3_attn3.log 2>&1
AB_LIBS="$ORBIT2_LIB" ORBIT2_ATTN2=1 timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3_attn2.log 2>&1
