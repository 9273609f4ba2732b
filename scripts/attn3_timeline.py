"""Debug: clock64 timeline of CTA 0 of attn3_tc_kernel (C2, B=16); build with
python -m paper_2505_04802_b200.build --variant a3tl -D ORBIT2_ATTN3_TIMELINE."""
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
buf = torch.zeros(7 * 64 * 8, dtype=torch.int64, device="cuda")
f = o2.lib.orbit2_debug_attn_timeline
f.argtypes = [ctypes.c_void_p]
f(buf.data_ptr())
ctx.forward(packed, x)
torch.cuda.synchronize()
f(None)
t = buf.cpu().numpy().astype(np.int64).reshape(7, 64, 8)
t0 = t[t > 0].min()
names = ["softmax tile0", "softmax tile1", "softmax tile2", "mma tile0", "mma tile1", "mma tile2"]
ev = ["loop,s_full,s_loaded,max_done,pv_done,p_arrived", "s_issue_wait,s_free_done,pv_wait,p_full_done"]
for role in range(6):
    print(f"== {names[role]}: {ev[0 if role < 3 else 1]}")
    for b in range(48):
        row = t[role, b]
        if (row > 0).any():
            print(f"  blk {b:2d}: " + " ".join(f"{(v - t0):8d}" if v > 0 else "       -" for v in row[:6]))
