"""Debug: run the forward repeatedly with per-launch sync checks (ORBIT2_SYNC_CHECK=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = get_config("C2", batch=B)
ctx = o2.Context(o2.config_from(w))
x = torch.from_numpy(make_input(w)).cuda()
packed = ctx.prepare_weights(torch.from_numpy(make_weights(w)).cuda())
for i in range(reps):
    try:
        out = ctx.forward(packed, x)
        torch.cuda.synchronize()
        print(f"rep {i} ok", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"rep {i} FAILED: {e}", flush=True)
        break
