"""Bit-reproducibility checks on one GPU: full C2 (B=4) forward vs chunked /
rank-emulated / repeated runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

w = get_config("C2", batch=4)
x = torch.from_numpy(make_input(w, batch=4)).cuda()
blob = torch.from_numpy(make_weights(w)).cuda()


def run(**kw):
    out = torch.full((4, w.K, w.scale * w.H, w.scale * w.W), float("nan"), device="cuda")
    R = kw.get("world_size", 1)
    for r in range(R):
        ctx = o2.Context(o2.config_from(w, rank=r, **kw))
        ctx.forward(ctx.prepare_weights(blob), x, out=out)
    torch.cuda.synchronize()
    return out


ref = run()
for name, kw in [("repeat", {}), ("chunk1", dict(chunk_tiles=1)), ("chunk5", dict(chunk_tiles=5)),
                 ("ranks2", dict(world_size=2)), ("ranks3", dict(world_size=3))]:
    for env in ([None] if name != "repeat" else [None, "1"]):
        if env:
            os.environ["ORBIT2_UNFUSED_MLP"] = env
        o = run(**kw)
        d = (o - ref).abs().max().item()
        print(f"{name} unfused={env}: bit-exact={torch.equal(o, ref)} maxdiff={d:.3e}")
        os.environ.pop("ORBIT2_UNFUSED_MLP", None)
