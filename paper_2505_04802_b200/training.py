"""Tile-parallel training step over the GPUs of one box (P:527
"assigning each tile to a separate GPU", "gradients from all GPUs are averaged to
maintain the model consistency").

One process per GPU, every rank computing the tiles the planner assigns it (LPT):

  1. forward        -- orbit2_train_forward over the rank's tiles (input replicated on
                       every rank), orbit2_stitch of their cores + residual into a zeroed
                       field
  2. field          -- one NCCL all-reduce (sum) of the fields: the cores are disjoint, so
                       every rank holds the whole output field (the loss's TV prior reaches
                       across tile borders)
  3. loss           -- orbit2_loss over the whole field (the same value on every rank)
  4. backward       -- orbit2_train_backward over the rank's tiles: their share of the
                       gradient of the batch loss
  5. gradient       -- one NCCL all-reduce (sum) of the gradients: the tiles partition the
                       output cores, so the sum is the gradient of the batch loss, identical
                       on every rank (reading R36: the per-rank shares are summed, the
                       equivalent of averaging per-rank gradients of per-rank mean losses)

torch.distributed (NCCL) carries the two collectives; every step of the path runs in the
library's kernels.
"""
from __future__ import annotations


class TilesTrainSP:
    """ctx: orbit2.Context with world_size = R, rank = this rank (BF16, chunk_tiles = 0)."""

    def __init__(self, ctx, dist, group=None):
        self.ctx, self.dist, self.group = ctx, dist, group
        self.has_tiles = ctx.info.n_local_tiles > 0
        ctx.train_bind()                    # also for a rank without tiles: the loss's latitude weights
        self.bufs = ctx.train_buffers()

    def prepare(self, canonical_dev, stream=None):
        if self.has_tiles:
            self.ctx.train_prepare(canonical_dev, stream)

    def step(self, packed, x_dev, truth_dev, lam=1e-3, delta=1e-3, geo=True, stream=None):
        """-> (loss per sample [B] float64, gradient of the batch loss [canonical count] fp32,
        the whole output field).  x_dev: the full input field on every rank."""
        import torch
        ctx, dist = self.ctx, self.dist
        tile_out, out, dout, loss, grad = self.bufs
        s = torch.cuda.current_stream(ctx.device) if stream is None else stream
        with torch.cuda.stream(s):
            out.zero_()
            if self.has_tiles:
                ctx.train_forward(packed, x_dev, tile_out, s)
                ctx.orbit2_stitch(tile_out, x_dev, 0, ctx.info.n_local_tiles, out, s)
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)
            ctx.loss(out, truth_dev, lam, delta, geo, loss, dout, s)
            if self.has_tiles:
                ctx.train_backward(packed, dout, grad, s)
            else:
                grad.zero_()
            dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=self.group)
        return loss, grad, out

