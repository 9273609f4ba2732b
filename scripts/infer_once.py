"""Run a few inference forwards at one config (for ncu captures): python scripts/infer_once.py C2 16 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

cfg_name, B = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = get_config(cfg_name).replace(batch=B)
ctx = o2.Context(o2.config_from(w, batch=B, precision=o2.BF16))
packed = ctx.prepare_weights(torch.from_numpy(make_weights(w)).cuda())
x = torch.from_numpy(make_input(w, batch=B)).cuda()
for _ in range(steps):
    out = ctx.forward(packed, x)
torch.cuda.synchronize()
print("ok", float(out.float().abs().mean()))
