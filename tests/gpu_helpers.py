"""Shared helpers of the GPU parity tests (CUDA path through the C ABI vs the fp64 oracle)."""
import numpy as np

from oracle import reslim_tiles as O

BF16_TOL = 2e-2     # north_star: max relative error <= 2e-2 (bf16 path)
FP32_TOL = 1e-4     # north_star: <= 1e-4 (fp32 path)


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """DESIGN.md metric (reading R21): per output variable k,
    max|y - y_ref| / max|y_ref|, then max over k.  Arrays [..., K, Y, X]."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    k_axis = got.ndim - 3
    worst = 0.0
    for k in range(got.shape[k_axis]):
        g = np.take(got, k, axis=k_axis)
        r = np.take(ref, k, axis=k_axis)
        den = np.abs(r).max()
        worst = max(worst, float(np.abs(g - r).max() / (den if den > 0 else 1.0)))
    return worst


def run_cuda(w, x: np.ndarray, blob: np.ndarray, precision: int, chunk_tiles: int = 0,
             world_size: int = 1, ranks=None, out=None):
    """Forward + stitch of every tile through the C ABI; returns out [B,K,sH,sW] (numpy)."""
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    wd = torch.from_numpy(np.ascontiguousarray(blob)).cuda()
    B = x.shape[0]
    if out is None:
        out = torch.full((B, w.K, w.scale * w.H, w.scale * w.W), float("nan"), dtype=torch.float32, device="cuda")
    for r in (range(world_size) if ranks is None else ranks):
        cfg = o2.config_from(w, batch=B, precision=precision, chunk_tiles=chunk_tiles,
                             world_size=world_size, rank=r)
        ctx = o2.Context(cfg)
        packed = ctx.prepare_weights(wd)
        ctx.forward(packed, xd, out=out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def oracle_full(w, x, blob):
    return O.tiles_forward(x, blob, O.Problem.from_config(w), return_parts=True)


def sampled_tiles(w):
    """1 corner, 1 edge, 2 interior tiles (SURVEY §8(c) parity gates)."""
    ty, tx = w.tiles_y, w.tiles_x
    ids = [0]
    if tx > 2:
        ids.append(tx // 2)
    if ty > 2 and tx > 2:
        ids += [(ty // 2) * tx + tx // 2, (ty - 2) * tx + 1]
    return sorted(set(i for i in ids if i < ty * tx))
