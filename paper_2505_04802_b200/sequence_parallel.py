"""TILES sequence parallelism over the GPUs of one box ("assigning each
tile to a separate GPU"; "stitched together").

One process per GPU.  Every data movement is a library kernel (rectangle
pack/unpack, stitch); NCCL (through torch.distributed point-to-point ops)
only moves the packed buffers over NVLink:

  1. halo exchange   -- each rank starts with its owned core pixels; it
                        receives the pixels of its padded tile rectangles that
                        neighbouring ranks own (orbit2_xfer_* HALO).
  2. forward         -- steps (1)-(3) + head over the rank's LPT-assigned tiles.
  3. output gather   -- the root receives every rank's tile_out (bf16 decoder
                        outputs of the core tokens) and the owned input cores
                        (for the residual), then stitches all tiles
                        (orbit2_stitch_peer).  gather_root=None leaves the
                        output sharded (each rank stitches its own tiles).
"""
from __future__ import annotations

from . import orbit2 as o2


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
