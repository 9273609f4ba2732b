"""Run a few training steps at one config (for ncu captures): python scripts/train_once.py C2 16 [steps]"""
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
ctx.train_bind()
blob = torch.from_numpy(make_weights(w)).cuda()
packed = ctx.prepare_weights(blob)
ctx.train_prepare(blob)
x = torch.from_numpy(make_input(w, batch=B)).cuda()
y = torch.randn(B, w.K, w.scale * w.H, w.scale * w.W, device="cuda")
bufs = ctx.train_buffers()
for _ in range(steps):
    loss, _, _ = ctx.train_step(packed, x, y, 1e-3, 1e-3, True, bufs)
torch.cuda.synchronize()
print("loss", loss.mean().item())
