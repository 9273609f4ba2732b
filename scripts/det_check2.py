"""Bisect the packing dependence: C2 (B=4) with depth 0,1,2; chunk1 vs all."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

for depth in (0, 1, 2):
    for H, W, ty, tx, B in [(180, 360, 4, 4, 4), (180, 360, 4, 4, 1), (48, 96, 2, 3, 4)]:
        w = get_config("C2", batch=B, depth=depth, H=H, W=W, tiles_y=ty, tiles_x=tx)
        x = torch.from_numpy(make_input(w, batch=B)).cuda()
        blob = torch.from_numpy(make_weights(w)).cuda()
        res = []
        for ch in (0, 1):
            ctx = o2.Context(o2.config_from(w, chunk_tiles=ch))
            res.append(ctx.forward(ctx.prepare_weights(blob), x))
        torch.cuda.synchronize()
        d = (res[0] - res[1]).abs()
        print(f"depth {depth} grid {H}x{W} tiles {ty}x{tx} B={B}: exact={torch.equal(res[0], res[1])} max={d.max().item():.3e} "
              f"count={(d > 0).sum().item()}")
