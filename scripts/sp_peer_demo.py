"""Peer-memory TILES SP over real GPUs (torchrun, one process per GPU): one
batch's tiles over the ranks, bit-exact against the 1-GPU forward on rank 0
and within the bf16 tolerance of the fp64 oracle (small configs only).

    torchrun --nproc-per-node N scripts/sp_peer_demo.py CONFIG BATCH [oracle] [field=int ...]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04802_b200 import orbit2 as o2  # noqa: E402
from paper_2505_04802_b200.sequence_parallel import PeerSP  # noqa: E402
from workloads import get_config, make_input, make_weights  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
over = {k: int(v) for k, v in (a.split("=") for a in sys.argv[1:] if "=" in a)}   # e.g. tiles_y=1 halo=0
groups = over.pop("groups", 1)     # sample groups per rank (PeerSP work_ctx)
name = args[0] if len(args) > 0 else "C2"
batch = int(args[1]) if len(args) > 1 else 1
check_oracle = len(args) > 2 and args[2] == "oracle"
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
w = get_config(name, batch=batch, **over)
x_host = make_input(w, batch=batch)
full = torch.from_numpy(x_host).cuda()
blob = torch.from_numpy(make_weights(w)).cuda()
ctx = o2.Context(o2.config_from(w, world_size=world, rank=rank, chunk_tiles=0))
n = ctx.info.n_local_tiles
ctx = o2.Context(o2.config_from(w, world_size=world, rank=rank, chunk_tiles=max(1, -(-n // 4))))
packed = ctx.prepare_weights(blob)
x = torch.full_like(full, float("nan"))
for t in ctx.tiles:
    if t.owner_rank == rank:
        sl = (slice(None), slice(None), slice(t.core_y0 * w.patch, t.core_y1 * w.patch),
              slice(t.core_x0 * w.patch, t.core_x1 * w.patch))
        x[sl] = full[sl]
out = torch.full((batch, w.K, w.scale * w.H, w.scale * w.W), float("nan"), device="cuda") if rank == 0 else None
wctx = o2.Context(o2.config_from(w, batch=batch // groups, world_size=world, rank=rank,
                                 chunk_tiles=ctx.info.chunk_tiles)) if groups > 1 else None
sp = PeerSP(ctx, x, out, dist, gather_root=0, work_ctx=wctx)
sp.step(packed)
torch.cuda.synchronize()
ctx.comm_status()
times = []
for _ in range(5):
    dist.barrier(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sp.step(packed)
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    times.append(t.item())
ctx.comm_status()
if rank == 0:
    ref_ctx = o2.Context(o2.config_from(w))
    ref = ref_ctx.forward(ref_ctx.prepare_weights(blob), full.clone())
    torch.cuda.synchronize()
    exact = torch.equal(out, ref)
    msg = f"peer SP {name} {over} B={batch} R={world}: bit-exact={exact} ms={min(times):.2f}"
    if check_oracle:
        from oracle import reslim_tiles as O
        from tests.gpu_helpers import rel_err
        want = O.tiles_forward(x_host, blob.cpu().numpy(), O.Problem.from_config(w))
        e = rel_err(out.cpu().numpy(), want)
        msg += f" rel_err_vs_oracle={e:.3e}"
        exact = exact and e <= 2e-2
    print(msg, flush=True)
    print("RESULT", "PASS" if exact else "FAIL", flush=True)
    if not exact:
        d = (out - ref).abs()
        print("max diff", d.nan_to_num(1e30).max().item(), "nan", torch.isnan(out).sum().item())
dist.destroy_process_group()
