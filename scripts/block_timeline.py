"""Debug: clock64 timeline of CTA 0 of the D = 256 block-tail kernel (C2, B=16).

Needs a library built with -DORBIT2_BLOCK_TIMELINE:
    python -m paper_2505_04802_b200.build --variant btl -D ORBIT2_BLOCK_TIMELINE
    ORBIT2_LIB=paper_2505_04802_b200/liborbit2_btl.so python scripts/block_timeline.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

w = get_config(sys.argv[1] if len(sys.argv) > 1 else "C2", batch=int(sys.argv[2]) if len(sys.argv) > 2 else 16)
ctx = o2.Context(o2.config_from(w))
x = torch.from_numpy(make_input(w)).cuda()
packed = ctx.prepare_weights(torch.from_numpy(make_weights(w)).cuda())
ctx.forward(packed, x)
buf = torch.zeros(3 * 64 * 8, dtype=torch.int64, device="cuda")
f = o2.lib.orbit2_debug_mlp_timeline
f.argtypes = [ctypes.c_void_p]
f(buf.data_ptr())
ctx.forward(packed, x)   # every launch overwrites: the last layer's launch remains
torch.cuda.synchronize()
f(None)
t = buf.cpu().numpy().reshape(3, 64, 8).astype(np.int64)
t0 = t[t > 0].min()
ev = {0: "MMA: x_full, oproj_issued, xn_full, last_gemm2_issued",
      1: "EPI(warp4): op_full, pass1, stats, xn_arrive, gelu0_start, o_full, z_stored, ln1_done",
      2: "EPI(warp4): s_full done of hidden chunk 0..7"}
for role in (0, 1, 2):
    print(f"== {ev[role]}")
    for c in range(12):
        row = t[role, c]
        if (row > 0).any():
            print(f"  block {c:2d}: " + " ".join(f"{(v - t0):8d}" if v > 0 else "       -" for v in row[:8]))
