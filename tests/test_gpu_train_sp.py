"""Tile-parallel training (paper_2505_04802_b200.training.TilesTrainSP) on the GPU: R ranks as
processes sharing cuda:0 over gloo (CUDA tensors), each computing its LPT-assigned tiles; the
summed gradient equals the one-rank gradient (fp32 atomics order only) and the loss is the
same on every rank."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_04802_b200 import orbit2 as o2
        from paper_2505_04802_b200.training import TilesTrainSP
        from workloads import get_config, make_input, make_weights
        w = get_config("C2", batch=2, H=48, W=80, tiles_y=2, tiles_x=3, halo=2, depth=2)
        blob = torch.from_numpy(make_weights(w, seed=3)).cuda()
        x = torch.from_numpy(make_input(w, batch=2, seed=4)).cuda()
        y = torch.randn(2, w.K, w.scale * w.H, w.scale * w.W, generator=torch.Generator().manual_seed(5)).cuda()
        ctx = o2.Context(o2.config_from(w, precision=o2.BF16, world_size=world, rank=rank))
        packed = ctx.prepare_weights(blob)
        sp = TilesTrainSP(ctx, dist)
        sp.prepare(blob)
        loss, grad, _ = sp.step(packed, x, y, 0.05, 0.02)
        torch.cuda.synchronize()
        if rank == 0:
            one = o2.Context(o2.config_from(w, precision=o2.BF16))
            p1 = one.prepare_weights(blob)
            one.train_bind()
            one.train_prepare(blob)
            l1, g1, _ = one.train_step(p1, x, y, 0.05, 0.02, True)
            torch.cuda.synchronize()
            g, g1 = grad.double().cpu().numpy(), g1.double().cpu().numpy()
            q.put(("ok", float(np.linalg.norm(g - g1) / np.linalg.norm(g1)),
                   float(abs(loss.sum().item() - l1.sum().item()) / abs(l1.sum().item())), ctx.info.n_local_tiles))
        else:
            q.put(("ok", 0.0, 0.0, ctx.info.n_local_tiles))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("err", traceback.format_exc(), 0.0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tiles_train_sp_equals_one_rank(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[0] == "ok", r[1]
    assert sum(r[3] for r in res) == 6
    gerr, lerr = max(r[1] for r in res), max(r[2] for r in res)
    assert gerr <= 1e-5 and lerr <= 1e-6, (gerr, lerr)
