"""fp64 CPU ORACLE of the ORBIT-2 training step.

TEST INFRASTRUCTURE ONLY -- the same rules as oracle/reslim_tiles.py: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import this module; it imports nothing from the
product path and shares no code with it.

What is computed, step by step:
  T1 latitude weights   -- the loss's "D is a latitude weighting matrix to account
                           for the decrease in longitudinal spacing toward the
                           poles", reading R35: diagonal per output row,
                           w_r = cos(lat_r) / mean_r cos(lat_r),
                           lat_r = 90 - 180 (r + 1/2) / sH degrees (row 0 = north)
  T2 Bayesian loss      -- P:500-507 (unnumbered equation [Bayesian Training Loss]):
                           ||y - x||_D^2 + sum_k sum_i sum_{j in C(i)} b_ij ||x_ki - x_kj||,
                           reading R34: C(i) = the 8 surrounding pixels inside the
                           field, b_ij = 1 / euclidean distance (1 axial, 1/sqrt 2
                           diagonal), ||.|| smoothed as the Huber function
                           h(r) = r^2 / (2 delta) for |r| <= delta, |r| - delta/2
                           otherwise (-> |r| as delta -> 0), weighted by lambda; both
                           terms normalised by K*N (a mean over variables and
                           pixels), the batch loss the mean over samples
  T3 backward           -- the gradient of the batch loss with respect to every
                           weight of the canonical blob (same order), by reverse-mode
                           differentiation of reslim_tiles.tile_forward written out
                           step by step (chain rule through head, LN_f, the blocks
                           in reverse, attention per head, the embedding)
  T4 gradient averaging -- P:532 "gradients from all GPUs are averaged to maintain
                           the model consistency", once per batch; reading R36: with
                           the batch split over ranks each rank's gradient is of the
                           mean loss over ITS samples, the all-reduced gradient the
                           mean over ranks (equal shares) = the full-batch gradient

Training scope (reading R36): the configuration without the optional O3b / O5b /
O8 stages (var_agg = dec_hidden = res_hidden = 0); the bilinear residual has no
weights, so dL/dout flows only into the ViT branch.

Pins (tests/test_train_oracle.py): central finite differences of the loss over
random blob coordinates (brute force, fp64) on tiled problems with halos; torch
autograd of the untiled torch library model (full halo => tiled == global);
the SPEC's 3x3 worked example and closed forms for T1/T2.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

from . import reslim_tiles as O


# ---------------------------------------------------------------------------
# T1 latitude weights (R35)
# ---------------------------------------------------------------------------
def lat_weights(sH: int, geo: bool = True) -> np.ndarray:
    if not geo:
        return np.ones(sH)
    lat = 90.0 - 180.0 * (np.arange(sH, dtype=np.float64) + 0.5) / sH
    c = np.cos(np.deg2rad(lat))
    return c / c.mean()


# ---------------------------------------------------------------------------
# T2 Bayesian loss (R34)
# ---------------------------------------------------------------------------
NEIGHBOURS = [(dy, dx, 1.0 / math.hypot(dy, dx)) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
              if (dy, dx) != (0, 0)]


def huber(r: np.ndarray, delta: float) -> np.ndarray:
    a = np.abs(r)
    return np.where(a <= delta, r * r / (2.0 * delta), a - 0.5 * delta)


def huber_grad(r: np.ndarray, delta: float) -> np.ndarray:
    return np.where(np.abs(r) <= delta, r / delta, np.sign(r))


def bayesian_loss(pred: np.ndarray, truth: np.ndarray, latw: np.ndarray, lam: float,
                  delta: float) -> float:
    """One sample: pred, truth [K, sH, sW]."""
    pred = np.asarray(pred, np.float64)
    K, sH, sW = pred.shape
    n = K * sH * sW
    t1 = (latw[None, :, None] * (truth - pred) ** 2).sum() / n
    t2 = 0.0
    for dy, dx, b in NEIGHBOURS:        # pixel i = (Y, X), neighbour j = (Y + dy, X + dx)
        ys, yd = slice(max(0, -dy), sH - max(0, dy)), slice(max(0, dy), sH - max(0, -dy))
        xs, xd = slice(max(0, -dx), sW - max(0, dx)), slice(max(0, dx), sW - max(0, -dx))
        t2 += b * huber(pred[:, ys, xs] - pred[:, yd, xd], delta).sum()
    return t1 + lam * t2 / n


def bayesian_loss_grad(pred: np.ndarray, truth: np.ndarray, latw: np.ndarray, lam: float,
                       delta: float) -> np.ndarray:
    """d bayesian_loss / d pred (one sample).  Each ordered pair (i, j) contributes
    b h'(x_i - x_j) to pixel i and its negative to pixel j."""
    pred = np.asarray(pred, np.float64)
    K, sH, sW = pred.shape
    n = K * sH * sW
    g = -2.0 * latw[None, :, None] * (truth - pred) / n
    for dy, dx, b in NEIGHBOURS:
        ys, yd = slice(max(0, -dy), sH - max(0, dy)), slice(max(0, dy), sH - max(0, -dy))
        xs, xd = slice(max(0, -dx), sW - max(0, dx)), slice(max(0, dx), sW - max(0, -dx))
        h = lam * b * huber_grad(pred[:, ys, xs] - pred[:, yd, xd], delta) / n
        g[:, ys, xs] += h
        g[:, yd, xd] -= h
    return g


# ---------------------------------------------------------------------------
# T3 backward through one tile (reverse of reslim_tiles.tile_forward)
# ---------------------------------------------------------------------------
def _ln_fwd(z, g, b):
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + O.LN_EPS)
    xh = (z - mu) * rstd
    return xh * g + b, (xh, rstd)


def _ln_bwd(dy, cache, g):
    """y = xh g + b, xh = (z - mu) rstd:  dz = rstd (dxh - mean(dxh) - xh mean(dxh xh))."""
    xh, rstd = cache
    dxh = dy * g
    dz = rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xh * (dxh * xh).mean(axis=-1, keepdims=True))
    return dz, (dy * xh).sum(axis=0), dy.sum(axis=0)


def _gelu_grad(x):
    """d/dx [x Phi(x)] = Phi(x) + x phi(x)  (erf GELU, R9)."""
    return 0.5 * (1.0 + erf(x / math.sqrt(2.0))) + x * np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def _attn_fwd(q, k, v):
    d = q.shape[-1]
    P = O.softmax_rows(q @ k.T / math.sqrt(d))
    return P @ v, P


def _attn_bwd(do, q, k, v, P):
    """O = P v, P = softmax(S), S = q k^T / sqrt(d):
    dv = P^T dO; dP = dO v^T; dS = P (dP - rowsum(dP P)); dq = dS k / sqrt d; dk = dS^T q / sqrt d."""
    d = q.shape[-1]
    dv = P.T @ do
    dP = do @ v.T
    dS = P * (dP - (dP * P).sum(axis=1, keepdims=True))
    return dS @ k / math.sqrt(d), dS.T @ q / math.sqrt(d), dv


def _block_fwd(z, Lw, heads):
    D = z.shape[1]
    d = D // heads
    c = {"z_in": z}
    xn1, c["ln1"] = _ln_fwd(z, Lw["ln1_g"], Lw["ln1_b"])
    qkv = xn1 @ Lw["W_qkv"].T + Lw["b_qkv"]
    c["xn1"], c["qkv"] = xn1, qkv
    outs, Ps = [], []
    for h in range(heads):
        o, P = _attn_fwd(qkv[:, h * d:(h + 1) * d], qkv[:, D + h * d:D + (h + 1) * d],
                         qkv[:, 2 * D + h * d:2 * D + (h + 1) * d])
        outs.append(o)
        Ps.append(P)
    ao = np.concatenate(outs, axis=1)
    c["ao"], c["P"] = ao, Ps
    zm = z + ao @ Lw["W_o"].T + Lw["b_o"]
    xn2, c["ln2"] = _ln_fwd(zm, Lw["ln2_g"], Lw["ln2_b"])
    hpre = xn2 @ Lw["W_1"].T + Lw["b_1"]
    hact = O.gelu(hpre)
    c["xn2"], c["hpre"], c["hact"] = xn2, hpre, hact
    return zm + hact @ Lw["W_2"].T + Lw["b_2"], c


def _block_bwd(dz, c, Lw, heads):
    """Returns (d z_in, {name: grad}) for one block (reverse of _block_fwd)."""
    D = dz.shape[1]
    d = D // heads
    gw = {}
    # z_out = zm + hact W_2^T + b_2
    gw["W_2"], gw["b_2"] = dz.T @ c["hact"], dz.sum(axis=0)
    dhpre = (dz @ Lw["W_2"]) * _gelu_grad(c["hpre"])
    gw["W_1"], gw["b_1"] = dhpre.T @ c["xn2"], dhpre.sum(axis=0)
    dzm, gw["ln2_g"], gw["ln2_b"] = _ln_bwd(dhpre @ Lw["W_1"], c["ln2"], Lw["ln2_g"])
    dzm = dzm + dz
    # zm = z_in + ao W_o^T + b_o
    gw["W_o"], gw["b_o"] = dzm.T @ c["ao"], dzm.sum(axis=0)
    dao = dzm @ Lw["W_o"]
    qkv = c["qkv"]
    dqkv = np.zeros_like(qkv)
    for h in range(heads):
        sq, sk, sv = (slice(o + h * d, o + (h + 1) * d) for o in (0, D, 2 * D))
        dq, dk, dv = _attn_bwd(dao[:, h * d:(h + 1) * d], qkv[:, sq], qkv[:, sk], qkv[:, sv], c["P"][h])
        dqkv[:, sq], dqkv[:, sk], dqkv[:, sv] = dq, dk, dv
    gw["W_qkv"], gw["b_qkv"] = dqkv.T @ c["xn1"], dqkv.sum(axis=0)
    dzin, gw["ln1_g"], gw["ln1_b"] = _ln_bwd(dqkv @ Lw["W_qkv"], c["ln1"], Lw["ln1_g"])
    return dzin + dzm, gw


def tile_backward(x_b: np.ndarray, tile: O.Tile, pr: O.Problem, Wt: dict, dg: np.ndarray,
                  grads: dict) -> None:
    """Adds d(loss)/d(weights) of ONE tile of ONE sample to `grads`, given
    dg = d loss / d g for the tile's head output g [n_core, K P^2] (O5)."""
    p = pr.patch
    a = O.patch_tokens(O.gather_tile(x_b, tile, p), p)
    z = O.embed_tile(O.gather_tile(x_b, tile, p), tile, p, Wt, pr.heads)
    caches = []
    for Lw in Wt["layers"]:
        z, cch = _block_fwd(z, Lw, pr.heads)
        caches.append(cch)
    rows = O.core_rows(tile)
    hin, lnf = _ln_fwd(z[rows], Wt["lnf_g"], Wt["lnf_b"])
    # g = hin W_h^T + b_h
    grads["W_h"] += dg.T @ hin
    grads["b_h"] += dg.sum(axis=0)
    dcore, dgf, dbf = _ln_bwd(dg @ Wt["W_h"], lnf, Wt["lnf_g"])
    grads["lnf_g"] += dgf
    grads["lnf_b"] += dbf
    dz = np.zeros_like(z)
    dz[rows] = dcore                     # halo rows of the last block feed nothing (R16)
    for l in range(len(Wt["layers"]) - 1, -1, -1):
        dz, gw = _block_bwd(dz, caches[l], Wt["layers"][l], pr.heads)
        for k_, v_ in gw.items():
            grads["layers"][l][k_] += v_
    # z0 = a W_e^T + b_e + e_s + pi
    grads["W_e"] += dz.T @ a
    grads["b_e"] += dz.sum(axis=0)
    grads["e_s"] += dz.sum(axis=0)


def _zeros_like_weights(Wt: dict) -> dict:
    g = {k: np.zeros_like(v) for k, v in Wt.items() if k != "layers"}
    g["layers"] = [{k: np.zeros_like(v) for k, v in Lw.items()} for Lw in Wt["layers"]]
    return g


def pack_grads(g: dict, pr: O.Problem) -> np.ndarray:
    """Gradient dict -> flat fp64 vector in the canonical blob order (include/orbit2.h)."""
    parts = [g["W_e"], g["b_e"], g["e_s"]]
    for Lg in g["layers"]:
        parts += [Lg[k] for k in ("ln1_g", "ln1_b", "W_qkv", "b_qkv", "W_o", "b_o", "ln2_g", "ln2_b",
                                  "W_1", "b_1", "W_2", "b_2")]
    parts += [g["lnf_g"], g["lnf_b"], g["W_h"], g["b_h"]]
    return np.concatenate([np.ravel(q) for q in parts])


def check_train_scope(pr: O.Problem) -> None:
    if pr.var_agg or pr.dec_hidden or pr.res_hidden:
        raise ValueError("training step: var_agg / dec_hidden / res_hidden stages are out of scope (R36)")


def train_loss(x: np.ndarray, y: np.ndarray, blob: np.ndarray, pr: O.Problem, lam: float, delta: float,
               geo: bool = True) -> float:
    """Mean over the batch of the T2 loss of the TILES forward (T4's per-rank loss)."""
    check_train_scope(pr)
    out = O.tiles_forward(x, blob, pr)
    latw = lat_weights(out.shape[2], geo)
    return float(np.mean([bayesian_loss(out[b], y[b], latw, lam, delta) for b in range(x.shape[0])]))


def train_step_grads(x: np.ndarray, y: np.ndarray, blob: np.ndarray, pr: O.Problem, lam: float,
                     delta: float, geo: bool = True):
    """(loss, grad) with grad = d loss / d blob in the canonical order (fp64)."""
    check_train_scope(pr)
    Wt = pr.weights(blob)
    tiles = pr.tiles()
    out = O.tiles_forward(x, blob, pr)
    B, K, sH, sW = out.shape
    P = pr.P
    latw = lat_weights(sH, geo)
    grads = _zeros_like_weights(Wt)
    loss = 0.0
    for b in range(B):
        loss += bayesian_loss(out[b], y[b], latw, lam, delta) / B
        dout = bayesian_loss_grad(out[b], y[b], latw, lam, delta) / B
        for t in tiles:
            # O6 read backwards: g[token(u,w), (k P + al) P + be] <- dout[k, P u + al, P w + be]
            ch, cw = t.core_y1 - t.core_y0, t.core_x1 - t.core_x0
            blk = dout[:, t.core_y0 * P:t.core_y1 * P, t.core_x0 * P:t.core_x1 * P]
            dg = blk.reshape(K, ch, P, cw, P).transpose(1, 3, 0, 2, 4).reshape(ch * cw, K * P * P)
            tile_backward(x[b], t, pr, Wt, dg, grads)
    return loss, pack_grads(grads, pr)



# ---------------------------------------------------------------------------
# T5 the weight update (R43)
# ---------------------------------------------------------------------------
def adamw(w: np.ndarray, g: np.ndarray, m: np.ndarray, v: np.ndarray, step: int, lr: float, beta1: float = 0.9,
          beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0):
    """AdamW (decoupled weight decay, bias-corrected moments), one step t = step >= 1:
    m <- b1 m + (1 - b1) g;  v <- b2 v + (1 - b2) g^2;
    w <- w - lr (wd w + (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)).  Returns (w, m, v)."""
    w, g, m, v = (np.asarray(a, np.float64) for a in (w, g, m, v))
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mh = m / (1.0 - beta1 ** step)
    vh = v / (1.0 - beta2 ** step)
    return w - lr * (weight_decay * w + mh / (np.sqrt(vh) + eps)), m, v
