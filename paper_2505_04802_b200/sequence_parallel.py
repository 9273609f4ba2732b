"""TILES sequence parallelism over the GPUs of one box ("assigning each
tile to a separate GPU"; P:530 halo; "stitched together").

One process per GPU.  The product path is `PeerSP`: the library moves every
byte itself through NVLink peer mappings (CUDA IPC), so there is no separate
communication step and no host synchronisation inside a step:

  1. halo exchange  -- orbit2_halo_exchange: each rank stores the pixels of its
                       owned cores that peers' tiles need straight into the
                       peers' input fields (push kernel), then a device-side
                       barrier (release/acquire flags, system scope).
  2. forward        -- orbit2_reslim_forward over the rank's LPT-assigned tiles,
                       chunk by chunk into two alternating tile_out buffers.
  3. output gather  -- orbit2_stitch of each chunk writes the root's output
                       field directly through NVLink (fused crop + stitch +
                       residual + gather), on a side stream, so it overlaps
                       the next chunk's forward; gather_root = -1 keeps the
                       output sharded (each rank stitches into its own field).
  4. end barrier    -- orbit2_comm_barrier: every rank's stores are visible.

torch.distributed is plumbing only: one all_gather_object of the export
handles at setup.  The NCCL point-to-point functions further down
(`forward_sequence_parallel`) are the round-1 baseline transport (torch
batch_isend_irecv of packed rectangles), kept for comparison.
"""
from __future__ import annotations

from . import orbit2 as o2


class PeerSP:
    """Peer-memory TILES SP for one rank (see the module docstring).

    ctx    : orbit2.Context with world_size = R, rank = this rank
    x_dev  : this rank's input field [B,V,H,W] (owned core pixels valid)
    out_dev: this rank's output field [B,K,sH,sW] (root / sharded), else None
    """

    def __init__(self, ctx, x_dev, out_dev, dist, gather_root=0, group=None, work_ctx=None):
        """work_ctx: optional Context of the same problem with batch B / G (G sample
        groups): the forward and stitch run group by group (a smaller last stitch into
        the root's field is exposed at the end of the step); halo exchange and
        barriers stay on `ctx` (the whole batch)."""
        import torch
        self.ctx, self.x = ctx, x_dev
        self.wctx = work_ctx if work_ctx is not None else ctx
        world = ctx.cfg.world_size
        mine = ctx.ipc_handles(x_dev, out_dev)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.target = ctx.comm_init(gather_root, x_dev, out_dev, allh)
        dist.barrier(group=group)             # every rank's flags zeroed before anyone signals
        wc = self.wctx
        if ctx.cfg.batch % wc.cfg.batch:
            raise ValueError("work_ctx batch must divide the batch")
        self.groups = ctx.cfg.batch // wc.cfg.batch
        n, ch = wc.info.n_local_tiles, max(wc.info.chunk_tiles, 1)
        self.chunks = [(g, tb, min(ch, n - tb)) for g in range(self.groups) for tb in range(0, n, ch)]
        self.tile_out = [wc.tile_out_buffer() for _ in range(min(2, len(self.chunks)))]
        c = wc.cfg
        self.x_step = c.batch * c.V * c.H * c.W                        # elements per sample group
        self.out_step = c.batch * c.K * (c.scale * c.H) * (c.scale * c.W) * 4   # bytes per sample group
        self.side = torch.cuda.Stream(ctx.device) if hasattr(torch.cuda, "Stream") and x_dev.is_cuda else None
        self.ev_fwd = [None, None]
        self.ev_st = [None, None]

    def step(self, packed, stream=None):
        """One TILES-SP step of this rank; stream-ordered, no host sync."""
        import torch
        ctx = self.ctx
        cuda = self.x.is_cuda
        if stream is None and cuda:
            stream = torch.cuda.current_stream(ctx.device)
        ctx.halo_exchange(stream)
        side = self.side if self.side is not None else stream
        wc = self.wctx
        for i, (g, tb, tc) in enumerate(self.chunks):
            b = i & 1
            if cuda and self.ev_st[b] is not None:
                stream.wait_event(self.ev_st[b])           # tile_out[b] stitched (chunk i - 2)
            xg = self.x if self.groups == 1 else self.x.view(-1)[g * self.x_step:(g + 1) * self.x_step].view(
                (wc.cfg.batch,) + tuple(self.x.shape[1:]))
            wc.orbit2_reslim_forward(packed, xg, tb, tc, self.tile_out[b], stream)
            if cuda:
                self.ev_fwd[b] = torch.cuda.Event()
                self.ev_fwd[b].record(stream)
                side.wait_event(self.ev_fwd[b])
            wc._stitch_to(self.tile_out[b], xg, tb, tc, self.target + g * self.out_step, side)
            if cuda:
                self.ev_st[b] = torch.cuda.Event()
                self.ev_st[b].record(side)
        if cuda:
            stream.wait_stream(side)
        ctx.comm_barrier(stream)


def _sync(x_dev, stream):
    """Make packed buffers complete before NCCL (a different stream) reads them."""
    if x_dev.is_cuda:
        import torch
        (torch.cuda.current_stream() if stream is None else stream).synchronize()


def _exchange(pairs, dist, group):
    """pairs: list of (peer, send_tensor or None, recv_tensor or None)."""
    ops = []
    for peer, sbuf, rbuf in pairs:
        if sbuf is not None and sbuf.numel():
            ops.append(dist.P2POp(dist.isend, sbuf, peer, group))
        if rbuf is not None and rbuf.numel():
            ops.append(dist.P2POp(dist.irecv, rbuf, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def halo_exchange(ctx, x_dev, dist, group=None, stream=None):
    """Fill the padded-rectangle pixels this rank does not own from their owners."""
    import torch
    cfg = ctx.cfg
    pairs, recvs = [], []
    for peer in range(cfg.world_size):
        if peer == cfg.rank:
            continue
        _, ns = o2.orbit2_xfer_plan(cfg, o2.XFER_HALO, peer, o2.SEND)
        _, nr = o2.orbit2_xfer_plan(cfg, o2.XFER_HALO, peer, o2.RECV)
        sbuf = torch.empty(ns, dtype=torch.float32, device=x_dev.device) if ns else None
        rbuf = torch.empty(nr, dtype=torch.float32, device=x_dev.device) if nr else None
        if sbuf is not None:
            ctx.orbit2_xfer_pack(o2.XFER_HALO, peer, x_dev, sbuf, stream)
        pairs.append((peer, sbuf, rbuf))
        if rbuf is not None:
            recvs.append((peer, rbuf))
    _sync(x_dev, stream)
    _exchange(pairs, dist, group)
    for peer, rbuf in recvs:
        ctx.orbit2_xfer_unpack(o2.XFER_HALO, peer, rbuf, x_dev, stream)


def gather_to_root(ctx, tile_out, x_dev, out, dist, root=0, group=None, stream=None):
    """Root receives each rank's tile_out and owned input cores, then stitches
    every rank's tiles into out (valid on root only)."""
    import torch
    cfg = ctx.cfg
    r = cfg.rank
    _sync(x_dev, stream)
    if r != root:
        _, ns = o2.orbit2_xfer_plan(cfg, o2.XFER_CORES, root, o2.SEND)
        cbuf = torch.empty(ns, dtype=torch.float32, device=x_dev.device)
        ctx.orbit2_xfer_pack(o2.XFER_CORES, root, x_dev, cbuf, stream)
        _sync(x_dev, stream)
        _exchange([(root, tile_out, None), (root, cbuf, None)], dist, group)
        return None
    peers = {}
    pairs = []
    for peer in range(cfg.world_size):
        if peer == root:
            continue
        pcfg = o2.config_from_cfg(cfg, rank=peer)
        _, pinfo = o2.orbit2_tiles_plan(pcfg)
        nh = tile_out.shape[1]
        tbuf = torch.empty((cfg.batch * max(pinfo.local_core_tokens, 1), nh), dtype=tile_out.dtype,
                           device=x_dev.device)
        _, nr = o2.orbit2_xfer_plan(cfg, o2.XFER_CORES, peer, o2.RECV)
        cbuf = torch.empty(nr, dtype=torch.float32, device=x_dev.device)
        peers[peer] = (tbuf, cbuf)
        pairs.append((peer, None, tbuf))
        pairs.append((peer, None, cbuf))
    _exchange(pairs, dist, group)
    for peer, (tbuf, cbuf) in peers.items():
        ctx.orbit2_xfer_unpack(o2.XFER_CORES, peer, cbuf, x_dev, stream)
    for peer in range(cfg.world_size):
        ctx.orbit2_stitch_peer(peer, tile_out if peer == root else peers[peer][0], x_dev, out, stream)
    return out


def forward_sequence_parallel(ctx, packed, x_dev, out, dist, root=0, group=None, stream=None):
    """Steps 1-3 of the module docstring for this rank; returns out on root."""
    halo_exchange(ctx, x_dev, dist, group, stream)
    tile_out = ctx.rank_tile_out()
    ctx.forward_rank(packed, x_dev, tile_out, stream)
    return gather_to_root(ctx, tile_out, x_dev, out, dist, root, group, stream)
