"""TILES sequence parallelism over real ranks (torchrun, NCCL): one sample's
tiles spread over the GPUs, halo exchange + output gather, checked against a
single-GPU forward on rank 0 (bit-exact) and timed with CUDA events."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2, sequence_parallel as sp  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
w = get_config(name, batch=batch)
full = torch.from_numpy(make_input(w, batch=batch)).cuda()
blob = torch.from_numpy(make_weights(w)).cuda()
ctx = o2.Context(o2.config_from(w, world_size=world, rank=rank))
packed = ctx.prepare_weights(blob)
x = torch.full_like(full, float("nan"))
cores, _ = o2.orbit2_xfer_plan(ctx.cfg, o2.XFER_CORES, (rank + 1) % world, o2.SEND)
for y0, y1, x0, x1 in cores:
    x[:, :, y0:y1, x0:x1] = full[:, :, y0:y1, x0:x1]
out = torch.empty((batch, w.K, w.scale * w.H, w.scale * w.W), device="cuda") if rank == 0 else None
res = sp.forward_sequence_parallel(ctx, packed, x.clone(), out, dist)
torch.cuda.synchronize()
times = []
for _ in range(3):
    xx = x.clone()
    dist.barrier(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sp.forward_sequence_parallel(ctx, packed, xx, out, dist)
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    times.append(t.item())
if rank == 0:
    ref_ctx = o2.Context(o2.config_from(w))
    ref = ref_ctx.forward(ref_ctx.prepare_weights(blob), full.clone())
    torch.cuda.synchronize()
    print(f"SP {name} B={batch} R={world}: bit-exact={torch.equal(res, ref)} ms={min(times):.2f}")
    if not torch.equal(res, ref):
        d = (res - ref).abs()
        print("max diff", d.max().item(), "nan", torch.isnan(res).sum().item())
        P = w.scale * w.patch
        for t in ctx.tiles:
            blk = d[:, :, t.core_y0 * P:t.core_y1 * P, t.core_x0 * P:t.core_x1 * P]
            print(f"tile {t.tile_id} owner {t.owner_rank}: max {blk.max().item():.3e} nan {torch.isnan(blk).sum().item()}")
dist.destroy_process_group()
