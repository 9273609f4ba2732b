"""Debug: clock64 timeline of CTA 0 of the attention kernel (C2, B=16)."""
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
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:3584].reshape(7, 64, 8)
t0 = t[t > 0].min()
names = {0: "softmax tile0", 1: "softmax tile1", 2: "mma tile0", 3: "mma tile1", 4: "producer",
         5: "epilogue tile0 (per item)", 6: "epilogue tile1 (per item)"}
ev = {0: "loop,s_full_done,s_loaded,max_done,pfree_done,exp_done,p_arrive,after_pingpong_bar",
      2: "k_full_done,s_free_done,v_full_done,p_full_done,pv_issued",
      4: "k_empty_done,v_empty_done", 5: "start,pv_done,o_read,stored,arrived,fenced,(next)loop_top,(next)item_taken"}
for role in range(7):
    print(f"== {names[role]}: {ev.get(role if role in (0, 2, 4, 5) else role - 1, '')}")
    for b in range(40):
        row = t[role, b]
        if (row > 0).any():
            print(f"  blk {b:2d}: " + " ".join(f"{(v - t0):8d}" if v > 0 else "       -" for v in row[:8]))

