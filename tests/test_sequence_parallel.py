"""TILES sequence parallelism: transfer-plan geometry (CPU), the NCCL-style
orchestration with world_size 2 over gloo (CPU, fake kernels), and rank
emulation of halo exchange + per-rank forward + root stitch on one GPU
(bit-identical to a single rank)."""
import os
import socket

import numpy as np
import pytest
import torch

from workloads import get_config, make_input, make_weights


@pytest.fixture(scope="module")
def o2():
    from paper_2505_04802_b200 import build
    build.build()
    from paper_2505_04802_b200 import orbit2
    return orbit2


def _mask(shape, rects):
    m = np.zeros(shape, bool)
    for y0, y1, x0, x1 in rects:
        m[y0:y1, x0:x1] = True
    return m


@pytest.mark.parametrize("mode", [0, 1])
def test_xfer_plan_geometry(o2, mode):
    """Owned cores partition the grid; every padded rectangle of a rank is
    covered by its own cores plus the halo it receives; what a rank receives
    from a peer is exactly what the peer sends it, and lies in the peer's cores."""
    w = get_config("C1", H=36, W=60, tiles_y=3, tiles_x=4, halo=2, halo_mode=mode)
    p = w.patch
    for R in (2, 3, 4):
        cores = {}
        for r in range(R):
            cfg = o2.config_from(w, world_size=R, rank=r)
            for s in range(R):
                if s != r:
                    cores[r], _ = o2.orbit2_xfer_plan(cfg, o2.XFER_CORES, s, o2.SEND)
                    break
        owner = np.zeros((w.H, w.W), int)
        for r in range(R):
            owner += _mask((w.H, w.W), cores[r])
        assert (owner == 1).all()
        for r in range(R):
            cfg = o2.config_from(w, world_size=R, rank=r)
            tiles, _ = o2.orbit2_tiles_plan(cfg)
            have = _mask((w.H, w.W), cores[r])
            for s in range(R):
                if s == r:
                    continue
                recv, nr = o2.orbit2_xfer_plan(cfg, o2.XFER_HALO, s, o2.RECV)
                sent, ns = o2.orbit2_xfer_plan(o2.config_from(w, world_size=R, rank=s), o2.XFER_HALO, r, o2.SEND)
                assert recv == sent and nr == ns
                assert nr == w.batch * w.V * sum((a[1] - a[0]) * (a[3] - a[2]) for a in recv)
                assert not (_mask((w.H, w.W), recv) & ~_mask((w.H, w.W), cores[s])).any()
                have |= _mask((w.H, w.W), recv)
            for t in tiles:
                if t.owner_rank != r:
                    continue
                y0, y1 = max(0, t.pad_y0 * p), min(w.H, t.pad_y1 * p)
                x0, x1 = max(0, t.pad_x0 * p), min(w.W, t.pad_x1 * p)
                assert have[y0:y1, x0:x1].all()


# ---------------------------------------------------------------- gloo orchestration
class FakeCtx:
    """CPU stand-in for orbit2.Context implementing the kernels' data movement
    in torch (test code), with the real planner's rectangles and plan."""

    def __init__(self, o2, cfg):
        self.o2, self.cfg = o2, cfg
        self.tiles, self.info = o2.orbit2_tiles_plan(cfg)

    def _rects(self, kind, peer, direction):
        return self.o2.orbit2_xfer_plan(self.cfg, kind, peer, direction)[0]

    def orbit2_xfer_pack(self, kind, peer, x, buf, stream=None):
        parts = [x[:, :, y0:y1, x0:x1].reshape(-1) for y0, y1, x0, x1 in self._rects(kind, peer, self.o2.SEND)]
        buf.copy_(torch.cat(parts))

    def orbit2_xfer_unpack(self, kind, peer, buf, x, stream=None):
        off = 0
        B, V = x.shape[:2]
        for y0, y1, x0, x1 in self._rects(kind, peer, self.o2.RECV):
            n = B * V * (y1 - y0) * (x1 - x0)
            x[:, :, y0:y1, x0:x1] = buf[off:off + n].reshape(B, V, y1 - y0, x1 - x0)
            off += n

    def rank_tile_out(self):
        return torch.zeros((self.cfg.batch * self.info.local_core_tokens, 1), dtype=torch.float64)

    def forward_rank(self, packed, x, tile_out, stream=None):
        """tile_out[b, core token] = sum of the tile's padded pixels (needs the halo)."""
        p = self.cfg.patch
        mine = [t for t in self.tiles if t.owner_rank == self.cfg.rank]
        n = self.info.local_core_tokens
        off = 0
        for t in mine:
            y0, y1 = max(0, t.pad_y0 * p), min(self.cfg.H, t.pad_y1 * p)
            x0, x1 = max(0, t.pad_x0 * p), min(self.cfg.W, t.pad_x1 * p)
            v = x[:, :, y0:y1, x0:x1].double().sum(dim=(1, 2, 3))
            for b in range(self.cfg.batch):
                tile_out[b * n + off:b * n + off + t.n_core_tokens, 0] = v[b]
            off += t.n_core_tokens
        return tile_out

    def orbit2_stitch_peer(self, peer, tile_out, x, out, stream=None):
        p = self.cfg.patch
        mine = [t for t in self.tiles if t.owner_rank == peer]
        n = sum(t.n_core_tokens for t in mine)
        off = 0
        for t in mine:
            for b in range(self.cfg.batch):
                out[b, t.core_y0 * p:t.core_y1 * p, t.core_x0 * p:t.core_x1 * p] = tile_out[b * n + off, 0]
            off += t.n_core_tokens


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_04802_b200 import orbit2 as o2
        from paper_2505_04802_b200 import sequence_parallel as sp
        w = get_config("C1", batch=2, H=36, W=60, tiles_y=3, tiles_x=4, halo=2)
        cfg = o2.config_from(w, world_size=world, rank=rank)
        ctx = FakeCtx(o2, cfg)
        full = torch.from_numpy(make_input(w, batch=2))
        x = torch.full_like(full, float("nan"))
        cores = ctx._rects(o2.XFER_CORES, 1 - rank, o2.SEND)
        for y0, y1, x0, x1 in cores:          # each rank starts with its owned pixels only
            x[:, :, y0:y1, x0:x1] = full[:, :, y0:y1, x0:x1]
        out = torch.zeros((2, w.H, w.W), dtype=torch.float64)
        res = sp.forward_sequence_parallel(ctx, None, x, out, dist, root=0)
        if rank == 0:
            # reference: the same fake forward on the full input, one rank
            ref_ctx = FakeCtx(o2, o2.config_from(w))
            t1 = ref_ctx.forward_rank(None, full, ref_ctx.rank_tile_out())
            ref = torch.zeros_like(out)
            ref_ctx.orbit2_stitch_peer(0, t1, full, ref)
            q.put(("ok", bool(torch.equal(res, ref)), bool(torch.isfinite(x).all())))
        else:
            q.put(("ok", True, True))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), False))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_exchange_and_gather():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
        assert r[1] and r[2], r


# ---------------------------------------------------------------- GPU rank emulation
@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 4])
def test_gpu_rank_emulation_halo_exchange_bit_exact(o2, R):
    """R ranks emulated on one GPU: each starts with only its owned pixels
    (NaN elsewhere), exchanges halos through the library's pack/unpack kernels
    (device copies stand in for NCCL), runs its tiles, and the root gathers the
    input cores and every tile_out and stitches them: bit-identical to R = 1."""
    w = get_config("C2", batch=2, H=48, W=96, tiles_y=2, tiles_x=3, depth=2)
    full = torch.from_numpy(make_input(w, batch=2)).cuda()
    blob = torch.from_numpy(make_weights(w)).cuda()
    ref_ctx = o2.Context(o2.config_from(w))
    ref = ref_ctx.forward(ref_ctx.prepare_weights(blob), full.clone())
    ctxs = [o2.Context(o2.config_from(w, world_size=R, rank=r)) for r in range(R)]
    xs = []
    for r, c in enumerate(ctxs):
        x = torch.full_like(full, float("nan"))
        cores, _ = o2.orbit2_xfer_plan(c.cfg, o2.XFER_CORES, (r + 1) % R, o2.SEND)
        for y0, y1, x0, x1 in cores:
            x[:, :, y0:y1, x0:x1] = full[:, :, y0:y1, x0:x1]
        xs.append(x)
    for r, c in enumerate(ctxs):                 # halo exchange
        for s in range(R):
            if s == r:
                continue
            _, n = o2.orbit2_xfer_plan(ctxs[s].cfg, o2.XFER_HALO, r, o2.SEND)
            if n == 0:
                continue
            buf = torch.empty(n, device="cuda")
            ctxs[s].orbit2_xfer_pack(o2.XFER_HALO, r, xs[s], buf)
            c.orbit2_xfer_unpack(o2.XFER_HALO, s, buf, xs[r])
    touts = []
    for r, c in enumerate(ctxs):                 # per-rank forward
        packed = c.prepare_weights(blob)
        touts.append(c.forward_rank(packed, xs[r], c.rank_tile_out()))
    root = ctxs[0]
    for s in range(1, R):                        # input cores to root
        _, n = o2.orbit2_xfer_plan(ctxs[s].cfg, o2.XFER_CORES, 0, o2.SEND)
        buf = torch.empty(n, device="cuda")
        ctxs[s].orbit2_xfer_pack(o2.XFER_CORES, 0, xs[s], buf)
        root.orbit2_xfer_unpack(o2.XFER_CORES, s, buf, xs[0])
    out = torch.full_like(ref, float("nan"))
    for s in range(R):
        root.orbit2_stitch_peer(s, touts[s], xs[0], out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # and against the fp64 oracle itself (P:527-532 TILES definition), not only R = 1
    from oracle import reslim_tiles as O
    from tests.gpu_helpers import BF16_TOL, rel_err
    want = O.tiles_forward(full.cpu().numpy(), blob.cpu().numpy(), O.Problem.from_config(w))
    assert rel_err(out.cpu().numpy(), want) <= BF16_TOL
