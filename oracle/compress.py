"""CPU ORACLE of the adaptive spatial compression module.

TEST INFRASTRUCTURE ONLY -- the same rules as oracle/reslim_tiles.py: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` leg may
import this module; it imports nothing from the product path and shares no code with it.

P:483 [Adaptive Spatial Compression]: "the model projects the embedding back into image
space and recursively partitions it into spatial quadrants using a quad-tree structure.
Partitioning continues for any quadrant where the estimated feature density -- computed
via Canny edge detection -- exceeds a predefined threshold, terminating when a minimum
patch size is reached or below predefined threshold."  P:485: "finer-grained learning in
feature-rich regions through smaller patches ... After ViT training blocks, the
decompression module reconstructs the high-resolution output from the compressed
embeddings."  The paper fixes no Canny parameters, density formula, token construction or
decompression; readings R37-R40 take the SPEC's:

  K1 canny(img)          -- Gaussian blur (sigma, radius ceil(3 sigma), edge replication),
                            Sobel 3x3 (edge replication), magnitude sqrt(gx^2 + gy^2),
                            non-maximum suppression along the gradient direction quantized
                            to 4 bins, double threshold low/high_frac * max magnitude,
                            hysteresis over 8-connected weak pixels (R37)
  K2 quadtree(edges)     -- from the max_side grid, split a square while its edge density
                            (edge pixels / area) is STRICTLY above the threshold and its side
                            exceeds min_side (R38); leaves in row-major order of their
                            top-left corner
  K3 tokenize(feat)      -- every leaf average-pooled to min_side x min_side per channel,
                            flattened (c, y, x), token = W_tok a + b_tok + E_scale[log2(side /
                            min_side)] (R39)
  K4 detokenize(tokens)  -- proj = W_dec t + b_dec as [C][m][m], nearest-neighbour broadcast
                            over the leaf, then one same-padded (zeros) 3x3 convolution
                            C -> C (R40)

Precision: K1 decides booleans from floating point, so it runs in float32 with the
kernel's operation order (every product and sum rounded separately, no fused
multiply-add; correctly rounded sqrt) -- both sides take the decision in the same
precision.  K2 is integer (density compared in double: count > thr * area).  K3 / K4 are
float64.
Pins: tests/test_compress_oracle.py (scipy.ndimage Gaussian / Sobel / label, torch
conv2d, the SPEC's worked examples and closed forms, exhaustive invariants).
"""
from __future__ import annotations

import math

import numpy as np

F32 = np.float32


# ---------------------------------------------------------------------------
# K1 Canny (R37)
# ---------------------------------------------------------------------------
def gaussian_taps(sigma: float) -> np.ndarray:
    """Normalised taps w_i = exp(-i^2 / (2 sigma^2)) / sum, i = -r..r, r = ceil(3 sigma),
    computed in double and rounded to float32 (the kernel receives the same taps)."""
    r = int(math.ceil(3.0 * sigma))
    i = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(i * i) / (2.0 * sigma * sigma))
    return (w / w.sum()).astype(F32)


def _shift_rep(a: np.ndarray, dy: int, dx: int) -> np.ndarray:
    """b[y, x] = a[clamp(y + dy), clamp(x + dx)] (edge replication)."""
    H, W = a.shape
    ys = np.clip(np.arange(H) + dy, 0, H - 1)
    xs = np.clip(np.arange(W) + dx, 0, W - 1)
    return a[ys][:, xs]


def blur(img: np.ndarray, sigma: float) -> np.ndarray:
    """Separable blur in float32: rows (x taps, left to right) then columns; each step
    acc = acc + w_i * v (product rounded, then the sum rounded)."""
    w = gaussian_taps(sigma)
    r = (len(w) - 1) // 2
    a = np.asarray(img, F32)
    acc = np.zeros_like(a)
    for i in range(-r, r + 1):
        acc = (acc + (w[i + r] * _shift_rep(a, 0, i)).astype(F32)).astype(F32)
    b = np.zeros_like(acc)
    for i in range(-r, r + 1):
        b = (b + (w[i + r] * _shift_rep(acc, i, 0)).astype(F32)).astype(F32)
    return b


def sobel(b: np.ndarray):
    """gx = (p[-1,+1] + 2 p[0,+1] + p[+1,+1]) - (p[-1,-1] + 2 p[0,-1] + p[+1,-1]), gy likewise
    (rows), float32, the sums in this order; edge replication."""
    s = lambda dy, dx: _shift_rep(b, dy, dx)
    two = F32(2.0)
    right = ((s(-1, 1) + (two * s(0, 1)).astype(F32)).astype(F32) + s(1, 1)).astype(F32)
    left = ((s(-1, -1) + (two * s(0, -1)).astype(F32)).astype(F32) + s(1, -1)).astype(F32)
    down = ((s(1, -1) + (two * s(1, 0)).astype(F32)).astype(F32) + s(1, 1)).astype(F32)
    up = ((s(-1, -1) + (two * s(-1, 0)).astype(F32)).astype(F32) + s(-1, 1)).astype(F32)
    return (right - left).astype(F32), (down - up).astype(F32)


TAN22 = F32(0.41421356237309503)   # tan(22.5 deg) in float32


def direction_bins(gx: np.ndarray, gy: np.ndarray) -> np.ndarray:
    """0: gradient ~horizontal (neighbours left/right), 1: ~vertical (up/down),
    2: gx gy > 0 (neighbours (y-1, x-1) / (y+1, x+1)), 3: gx gy < 0 ((y-1, x+1) / (y+1, x-1)).
    |gy| <= tan22.5 |gx| -> 0; |gx| <= tan22.5 |gy| -> 1 (products rounded in float32)."""
    ax, ay = np.abs(gx), np.abs(gy)
    d = np.where(gx * gy > 0, 2, 3)
    d = np.where((TAN22 * ay).astype(F32) >= ax, 1, d)
    d = np.where((TAN22 * ax).astype(F32) >= ay, 0, d)
    return d


def magnitude(gx, gy):
    return np.sqrt(((gx * gx).astype(F32) + (gy * gy).astype(F32)).astype(F32)).astype(F32)


def nms(mag: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Keep a pixel when its magnitude is > 0 and >= both neighbours along its direction
    bin (neighbours outside the image count as 0); suppressed pixels -> 0."""
    H, W = mag.shape
    p = np.zeros((H + 2, W + 2), F32)
    p[1:-1, 1:-1] = mag
    n = lambda dy, dx: p[1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
    a = np.select([d == 0, d == 1, d == 2], [n(0, -1), n(-1, 0), n(-1, -1)], n(-1, 1))
    b = np.select([d == 0, d == 1, d == 2], [n(0, 1), n(1, 0), n(1, 1)], n(1, -1))
    keep = (mag > 0) & (mag >= a) & (mag >= b)
    return np.where(keep, mag, F32(0))


def hysteresis(m: np.ndarray, low: np.float32, high: np.float32) -> np.ndarray:
    """Edges = pixels with m >= high, plus pixels with m >= low 8-connected to them through
    pixels with m >= low (breadth-first search)."""
    H, W = m.shape
    cand = m >= low
    edge = np.zeros((H, W), bool)
    stack = [tuple(p) for p in np.argwhere(cand & (m >= high))]
    for y, x in stack:
        edge[y, x] = True
    while stack:
        y, x = stack.pop()
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                yy, xx = y + dy, x + dx
                if 0 <= yy < H and 0 <= xx < W and cand[yy, xx] and not edge[yy, xx]:
                    edge[yy, xx] = True
                    stack.append((yy, xx))
    return edge


def canny(img: np.ndarray, sigma: float = 1.0, low_frac: float = 0.1, high_frac: float = 0.2):
    """K1: boolean edge map of a 2-D field (R37)."""
    img = np.asarray(img, F32)
    if img.ndim != 2 or min(img.shape) < 3:
        raise ValueError("canny: a 2-D image of at least 3 x 3")
    gx, gy = sobel(blur(img, sigma))
    mag = magnitude(gx, gy)
    m = nms(mag, direction_bins(gx, gy))
    gmax = mag.max()
    if gmax <= 0:
        return np.zeros(img.shape, bool)
    return hysteresis(m, F32(F32(low_frac) * gmax), F32(F32(high_frac) * gmax))


# ---------------------------------------------------------------------------
# K2 quad-tree partition (R38)
# ---------------------------------------------------------------------------
def quadtree(edges: np.ndarray, min_side: int, max_side: int, threshold: float) -> list:
    """Leaves (row, col, side) in row-major order of (row, col).  Requires the field to be
    a multiple of max_side and max_side = min_side * 2^k."""
    H, W = edges.shape
    if max_side % min_side or (max_side // min_side) & (max_side // min_side - 1):
        raise ValueError("max_side must be a power-of-two multiple of min_side")
    if H % max_side or W % max_side:
        raise ValueError("field not a multiple of max_side (pad first)")
    e = np.asarray(edges, bool)
    thr = float(np.float32(threshold))
    out = []

    def visit(r, c, s):
        cnt = int(e[r:r + s, c:c + s].sum())
        if s > min_side and float(cnt) > thr * float(s * s):
            h = s // 2
            for rr, cc in ((r, c), (r, c + h), (r + h, c), (r + h, c + h)):
                visit(rr, cc, h)
        else:
            out.append((r, c, s))

    for r in range(0, H, max_side):
        for c in range(0, W, max_side):
            visit(r, c, max_side)
    out.sort()
    return out


def compression_ratio(patches: list, H: int, W: int, min_side: int) -> float:
    return (H * W / (min_side * min_side)) / len(patches)


def pad_replicate(img: np.ndarray, max_side: int) -> np.ndarray:
    """Edge-replicate the last axes up to multiples of max_side."""
    H, W = img.shape[-2:]
    Hp, Wp = -(-H // max_side) * max_side, -(-W // max_side) * max_side
    pad = [(0, 0)] * (img.ndim - 2) + [(0, Hp - H), (0, Wp - W)]
    return np.pad(img, pad, mode="edge")


# ---------------------------------------------------------------------------
# K3 / K4 tokens (R39, R40)
# ---------------------------------------------------------------------------
def pool_patch(feat: np.ndarray, r: int, c: int, s: int, m: int) -> np.ndarray:
    """[C, m, m]: mean over each (s/m) x (s/m) block of the leaf."""
    C = feat.shape[0]
    f = s // m
    blk = np.asarray(feat[:, r:r + s, c:c + s], np.float64)
    return blk.reshape(C, m, f, m, f).mean(axis=(2, 4))


def tokenize(feat: np.ndarray, patches: list, m: int, W_tok: np.ndarray, b_tok: np.ndarray,
             E_scale: np.ndarray) -> np.ndarray:
    """K3: [n, D] tokens; E_scale[level] with level = log2(side / m)."""
    rows = []
    for r, c, s in patches:
        a = pool_patch(feat, r, c, s, m).reshape(-1)
        lvl = int(round(math.log2(s // m)))
        rows.append(np.asarray(W_tok, np.float64) @ a + b_tok + E_scale[lvl])
    return np.array(rows).reshape(len(patches), -1)


def conv3x3_same(x: np.ndarray, Wc: np.ndarray, b: np.ndarray) -> np.ndarray:
    Cin, Y, X = x.shape
    xp = np.zeros((Cin, Y + 2, X + 2))
    xp[:, 1:-1, 1:-1] = x
    out = np.zeros((Wc.shape[0], Y, X)) + np.asarray(b, np.float64)[:, None, None]
    for dy in range(3):
        for dx in range(3):
            out += np.einsum("oi,iyx->oyx", Wc[:, :, dy, dx], xp[:, dy:dy + Y, dx:dx + X])
    return out


def detokenize(tokens: np.ndarray, patches: list, m: int, C: int, H: int, W: int, W_dec: np.ndarray,
               b_dec: np.ndarray, W_sm: np.ndarray, b_sm: np.ndarray) -> np.ndarray:
    """K4: [C, H, W].  proj[c, i, j] = (W_dec t + b_dec)[(c m + i) m + j]; pixel (y, x) of a
    leaf (r, c0, s) takes proj[:, (y - r) m // s, (x - c0) m // s]; then the 3x3 smoothing."""
    img = np.zeros((C, H, W))
    for t, (r, c, s) in zip(np.asarray(tokens, np.float64), patches):
        proj = (np.asarray(W_dec, np.float64) @ t + b_dec).reshape(C, m, m)
        idx = (np.arange(s) * m) // s
        img[:, r:r + s, c:c + s] = proj[:, idx][:, :, idx]
    return conv3x3_same(img, np.asarray(W_sm, np.float64), b_sm)


# ---------------------------------------------------------------------------
# K5 the Reslim forward on compressed tokens (R41)
# ---------------------------------------------------------------------------
def compression_field(z0: np.ndarray, Hp: int, Wp: int) -> np.ndarray:
    """R41: the embedding projected back into image space by the channel-averaging
    projection: f[u, w] = mean_d z0[u Wp + w, d] (float64 here; the kernel's is fp32)."""
    return np.asarray(z0, np.float64).mean(axis=1).reshape(Hp, Wp)


def partition_tokens(z0: np.ndarray, Hp: int, Wp: int, max_side: int, threshold: float, sigma: float = 1.0,
                     low_frac: float = 0.1, high_frac: float = 0.2) -> list:
    """Leaves (u0, w0, side) over the patch grid (min_side = 1 patch): Canny on the field
    edge-padded to a multiple of max_side, quad-tree, leaves rooted in the padding dropped."""
    f = pad_replicate(compression_field(z0, Hp, Wp), max_side).astype(F32)
    leaves = quadtree(canny(f, sigma, low_frac, high_frac), 1, max_side, threshold)
    return [(u, w, s) for (u, w, s) in leaves if u < Hp and w < Wp]


def compressed_forward(x_b: np.ndarray, pr, Wt: dict, E_scale: np.ndarray, leaves: list) -> np.ndarray:
    """K5 for one sample, T = 1 tile, halo 0 (R41): z0 = the O3 embedding of every patch;
    token of a leaf = mean of z0 over its patches inside the grid + E_scale[log2 side]; the
    ViT blocks attend over the sample's compressed tokens; the head (O5) per token; every
    patch takes its leaf's head output (nearest decompression); stitch (O6) and the
    bilinear residual (O7).  Returns out [K, sH, sW]."""
    from . import reslim_tiles as O
    p, P, K = pr.patch, pr.P, pr.K
    Hp, Wp = pr.H // p, pr.W // p
    tile = O.plan_tiles(Hp, Wp, 1, 1, 0)[0]
    z0 = O.embed_tile(O.gather_tile(x_b, tile, p), tile, p, Wt, pr.heads)
    zg = z0.reshape(Hp, Wp, -1)
    toks = []
    for u, w, s in leaves:
        blk = zg[u:min(u + s, Hp), w:min(w + s, Wp)].reshape(-1, zg.shape[2])
        toks.append(blk.mean(axis=0) + E_scale[int(round(math.log2(s)))])
    z = np.array(toks)
    for Lw in Wt["layers"]:
        z = O.block(z, Lw, pr.heads)
    g = O.head(z, Wt)                                   # [n, K P^2]
    gp = np.zeros((Hp, Wp, g.shape[1]))
    for (u, w, s), gi in zip(leaves, g):
        gp[u:min(u + s, Hp), w:min(w + s, Wp)] = gi
    out_vit = np.zeros((K, P * Hp, P * Wp))
    O.stitch_tile(out_vit, gp.reshape(Hp * Wp, -1), tile, K, P)
    return out_vit + O.residual_up(x_b, pr)


# ---------------------------------------------------------------------------
# K6 compressed tokens inside TILES tiles (R42)
# ---------------------------------------------------------------------------
def tile_field_shape(tiles, max_side: int):
    """(Hq, Wq): the largest padded rectangle over the tiles, rounded up to max_side (every
    tile's field is edge-padded to this one shape)."""
    hq = max(t.pad_h for t in tiles)
    wq = max(t.pad_w for t in tiles)
    return -(-hq // max_side) * max_side, -(-wq // max_side) * max_side


def tile_leaves(z0: np.ndarray, tile, Hq: int, Wq: int, max_side: int, threshold: float, sigma: float = 1.0,
                low_frac: float = 0.1, high_frac: float = 0.2) -> list:
    """Leaves (u0, w0, side) of one tile in its padded-rectangle coordinates: Canny on the
    channel-mean field of its z0 edge-padded to Hq x Wq, quad-tree, leaves rooted outside the
    rectangle dropped."""
    f = compression_field(z0, tile.pad_h, tile.pad_w)
    f = np.pad(f, ((0, Hq - tile.pad_h), (0, Wq - tile.pad_w)), mode="edge").astype(F32)
    leaves = quadtree(canny(f, sigma, low_frac, high_frac), 1, max_side, threshold)
    return [(u, w, s) for (u, w, s) in leaves if u < tile.pad_h and w < tile.pad_w]


def tiles_compressed_forward(x_b: np.ndarray, pr, Wt: dict, E_scale: np.ndarray, leaves_by_tile=None,
                             max_side: int = 8, threshold: float = 0.1, sigma: float = 1.0):
    """K6 for one sample (R42): every tile's padded rectangle compressed on its own (K5 within
    the tile: field, quad-tree, pooled tokens + scale embedding), the blocks attend within the
    tile over its compressed tokens, the head per token, decompression to the tile's CORE
    patches only (the halo is discarded), stitch and residual.  Returns (out, leaves)."""
    from . import reslim_tiles as O
    p, P, K = pr.patch, pr.P, pr.K
    tiles = pr.tiles()
    Hq, Wq = tile_field_shape(tiles, max_side)
    sH, sW = pr.scale * pr.H, pr.scale * pr.W
    out_vit = np.zeros((K, sH, sW))
    got = []
    for ti, t in enumerate(tiles):
        z0 = O.embed_tile(O.gather_tile(x_b, t, p), t, p, Wt, pr.heads)
        lv = tile_leaves(z0, t, Hq, Wq, max_side, threshold, sigma) if leaves_by_tile is None else leaves_by_tile[ti]
        got.append(lv)
        zg = z0.reshape(t.pad_h, t.pad_w, -1)
        z = np.array([zg[u:min(u + s, t.pad_h), w:min(w + s, t.pad_w)].reshape(-1, zg.shape[2]).mean(axis=0)
                      + E_scale[int(round(math.log2(s)))] for (u, w, s) in lv])
        for Lw in Wt["layers"]:
            z = O.block(z, Lw, pr.heads)
        g = O.head(z, Wt)
        gp = np.zeros((t.pad_h, t.pad_w, g.shape[1]))
        for (u, w, s), gi in zip(lv, g):
            gp[u:min(u + s, t.pad_h), w:min(w + s, t.pad_w)] = gi
        core = gp[t.core_y0 - t.pad_y0:t.core_y1 - t.pad_y0, t.core_x0 - t.pad_x0:t.core_x1 - t.pad_x0]
        O.stitch_tile(out_vit, core.reshape(-1, g.shape[1]), t, K, P)
    return out_vit + O.residual_up(x_b, pr), got
