"""fp64 CPU ORACLE of the ORBIT-2 TILES tile-wise Reslim forward pass.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` leg may import this module.
The product path (`paper_2505_04802_b200/`, `include/`, the CUDA library)
never imports, links or executes anything under `oracle/`, and this module
imports nothing from the product path.  It shares no code with it: the
planner, gather, embedding, blocks, head, stitch and bilinear residual below
are written out independently from the paper.

Citations: `P:n` = /root/reference/PAPER.md line n (section in brackets);
readings `R#` = DESIGN.md "Readings of the paper" (the SURVEY.md §8(c)
ambiguity register, same numbering).

What is computed (the method, step by step, in the paper's order):
  O1 plan      -- tiles + halo rectangles     P:527-530 [Innovation/TILES], R3-R6
  O2 gather    -- padded tile pixels           P:530 (Fig.4 caption P:515)
  O3 embed     -- patch tokens + res-embedding + sincos position
                  P:475-479 [Reslim main path], P:150 (p=2), R1, R2, R7, R8
  O3b variable aggregation (optional, var_agg = 1) -- P:479 "the main path uses a
                  cross-attention module to aggregate multi-variable embeddings into
                  a unified representation, effectively collapsing the variable
                  dimension", reading R33: per-variable tokens t_v = W_t[v] a_v +
                  e_var[v]; one learned query attends over the V tokens of each
                  patch (multi-head, keys / values W_ak t + b_ak, W_av t + b_av);
                  z0 = W_ao o + b_ao + e_s + pi(u, w)  (replaces W_e a + b_e)
  O4 blocks    -- pre-norm MHSA + GELU MLP, attention restricted to the tile
                  P:54, P:404, P:527 ("self-attention is restricted within
                  each tile"), R9, R17, R18
  O5 head      -- LN_f + linear decoder head   P:480, R10, R11
  O6 stitch    -- halo outputs discarded, cores placed   P:532, R16
  O7 residual  -- bilinear upsample added      P:487-498 [Residual Learning], R12, R13
  O5b decoder convolutions (optional, dec_hidden > 0) -- P:480 "a decoder comprising
                  convolutional layers and linear projections", reading R32: the
                  linear head (O5) runs on the tile's core tokens plus a ring of
                  ceil(2/P) patches (clipped to the grid), is unpatchified, and
                  conv_db(GELU(conv_da(.))) (3x3, zero padding outside that region)
                  gives the core output; the ring is then discarded with the halo
  O8 residual convolutional path (optional, res_hidden > 0) -- P:498 "the residual
                  convolutional path reintroduces upsampling outside the main ViT
                  path, using lightweight convolutional layers", reading R31:
                  res = up + conv_b(GELU(conv_a(up))), 3x3 convolutions, zero
                  padding outside the high-resolution field

Everything is float64.  fp32 inputs and weights are promoted exactly.
Library primitives used as single steps: numpy matmul, numpy exp, scipy erf.

Pins (tests/test_oracle_pins.py): every function here is pinned against
something other than itself -- torch fp64 library modules (conv2d,
TransformerEncoderLayer, layer_norm, pixel_shuffle, interpolate), closed forms,
brute force and the paper's printed token counts.  The only part not pinned
by the paper is the numeric value of a full-size output: the paper prints no
worked example and ships no weights -- "parity unpinned" for
absolute full-config values; trust rests on the pins listed in DESIGN.md.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
from scipy.special import erf

LN_EPS = 1e-5          # R9
POS_BASE = 10000.0     # R7

HALO_CLAMP = 0
HALO_REPLICATE = 1


# ---------------------------------------------------------------------------
# O1  Plan  ("partitions both inputs and downscaled outputs into spatial
#            tiles"; "each tile is extended with a fixed-width halo")
# ---------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Tile:
    tile_id: int
    ty: int
    tx: int
    core_y0: int    # patch units, half-open
    core_y1: int
    core_x0: int
    core_x1: int
    pad_y0: int     # patch units; may leave the grid only in REPLICATE mode
    pad_y1: int
    pad_x0: int
    pad_x1: int

    @property
    def pad_h(self) -> int:
        return self.pad_y1 - self.pad_y0

    @property
    def pad_w(self) -> int:
        return self.pad_x1 - self.pad_x0

    @property
    def n_tokens(self) -> int:
        return self.pad_h * self.pad_w

    @property
    def n_core(self) -> int:
        return (self.core_y1 - self.core_y0) * (self.core_x1 - self.core_x0)


def split_extent(n: int, parts: int) -> list[int]:
    """R5: r_i = floor(n/parts) + [i < n mod parts]  (earlier tiles get +1)."""
    return [n // parts + (1 if i < n % parts else 0) for i in range(parts)]


def plan_tiles(Hp: int, Wp: int, tiles_y: int, tiles_x: int, halo: int,
               mode: int = HALO_CLAMP) -> list[Tile]:
    """Row-major tile list over the Hp x Wp patch grid (R6)."""
    if tiles_y < 1 or tiles_x < 1 or tiles_y > Hp or tiles_x > Wp:
        raise ValueError("tile count must be in [1, patch-grid extent]")
    if halo < 0:
        raise ValueError("halo must be >= 0")
    rows, cols = split_extent(Hp, tiles_y), split_extent(Wp, tiles_x)
    tiles = []
    y0 = 0
    for i in range(tiles_y):
        x0 = 0
        for j in range(tiles_x):
            cy0, cy1, cx0, cx1 = y0, y0 + rows[i], x0, x0 + cols[j]
            if mode == HALO_CLAMP:   # R4: no halo beyond the grid
                py0, py1 = max(0, cy0 - halo), min(Hp, cy1 + halo)
                px0, px1 = max(0, cx0 - halo), min(Wp, cx1 + halo)
            else:                    # REPLICATE: full halo, edge-replicated pixels
                py0, py1, px0, px1 = cy0 - halo, cy1 + halo, cx0 - halo, cx1 + halo
            tiles.append(Tile(i * tiles_x + j, i, j, cy0, cy1, cx0, cx1, py0, py1, px0, px1))
            x0 += cols[j]
        y0 += rows[i]
    return tiles


# ---------------------------------------------------------------------------
# O2  Gather: the tile's padded pixels (Fig.4(b))
# ---------------------------------------------------------------------------
def gather_tile(x_b: np.ndarray, tile: Tile, p: int) -> np.ndarray:
    """x_b [V,H,W] -> padded tile pixels [V, p*pad_h, p*pad_w].

    x~[v,a,c] = x[v, clamp(p*u0+a, 0, H-1), clamp(p*w0+c, 0, W-1)];
    the clamp only acts in REPLICATE mode (R4).
    """
    V, H, W = x_b.shape
    rows = np.clip(p * tile.pad_y0 + np.arange(p * tile.pad_h), 0, H - 1)
    cols = np.clip(p * tile.pad_x0 + np.arange(p * tile.pad_w), 0, W - 1)
    return x_b[:, rows][:, :, cols].astype(np.float64)


# ---------------------------------------------------------------------------
# O3  Patch embedding + sincos position (R7) + resolution embedding (R8)
# ---------------------------------------------------------------------------
def sincos_pos(u: np.ndarray, w: np.ndarray, D: int) -> np.ndarray:
    """pi(u,w) in R^D with Q = D/4, omega_m = 10000^(-m/Q):
    [sin(u*om) | cos(u*om) | sin(w*om) | cos(w*om)]  (R7, global patch coords)."""
    Q = D // 4
    om = POS_BASE ** (-np.arange(Q, dtype=np.float64) / Q)
    au = np.outer(np.asarray(u, np.float64), om)
    aw = np.outer(np.asarray(w, np.float64), om)
    return np.concatenate([np.sin(au), np.cos(au), np.sin(aw), np.cos(aw)], axis=1)


def patch_tokens(xt: np.ndarray, p: int) -> np.ndarray:
    """[V, p*ph, p*pw] -> a [ph*pw, V*p*p], token row-major (u,w), column (v*p+dy)*p+dx."""
    V, hh, ww = xt.shape
    ph, pw = hh // p, ww // p
    a = xt.reshape(V, ph, p, pw, p)            # v, u, dy, w, dx
    a = a.transpose(1, 3, 0, 2, 4)             # u, w, v, dy, dx
    return a.reshape(ph * pw, V * p * p)


def aggregate_variables(a: np.ndarray, Wt: dict, heads: int, p: int) -> np.ndarray:
    """O3b (R33): a [n, V*p*p] patch rows -> [n, D].  Per-variable tokens
    t_v = W_t[v] a_v + e_var[v]; per head h a learned query q_h scores the V
    tokens, s_{h,v} = <q_h, (W_ak t_v + b_ak)_h> / sqrt(d); softmax over v;
    o_h = sum_v alpha_{h,v} (W_av t_v + b_av)_h; result W_ao o + b_ao."""
    n = a.shape[0]
    V, D = Wt["W_t"].shape[0], Wt["W_t"].shape[1]
    d = D // heads
    pp = p * p
    t = np.stack([a[:, v * pp:(v + 1) * pp] @ Wt["W_t"][v].T + Wt["e_var"][v] for v in range(V)], axis=1)  # [n,V,D]
    k = t @ Wt["W_ak"].T + Wt["b_ak"]
    val = t @ Wt["W_av"].T + Wt["b_av"]
    o = np.zeros((n, D))
    for h in range(heads):
        sl = slice(h * d, (h + 1) * d)
        sc = k[:, :, sl] @ Wt["q_agg"][sl] / math.sqrt(d)              # [n, V]
        al = softmax_rows(sc)
        o[:, sl] = np.einsum("nv,nvd->nd", al, val[:, :, sl])
    return o @ Wt["W_ao"].T + Wt["b_ao"]


def embed_tile(xt: np.ndarray, tile: Tile, p: int, Wt: dict, heads: int = 1) -> np.ndarray:
    """z0 = W_e a + b_e + e_s + pi(u,w)   (resolution embedding 'added to
    the feature embedding'); with the variable aggregation (O3b) the joint
    linear W_e a + b_e is replaced by aggregate_variables(a)."""
    a = patch_tokens(xt, p)
    D = Wt["W_e"].shape[0]
    uu, ww = np.meshgrid(np.arange(tile.pad_y0, tile.pad_y1),
                         np.arange(tile.pad_x0, tile.pad_x1), indexing="ij")
    pos = sincos_pos(uu.ravel(), ww.ravel(), D)
    feat = aggregate_variables(a, Wt, heads, p) if "W_t" in Wt else a @ Wt["W_e"].T + Wt["b_e"]
    return feat + Wt["e_s"] + pos


# ---------------------------------------------------------------------------
# O4  Transformer blocks ("self-attention ... among all tokens"; P:527
#     attention restricted to the tile; R9 pre-norm, LN eps 1e-5, erf GELU)
# ---------------------------------------------------------------------------
def layer_norm(z: np.ndarray, g: np.ndarray, b: np.ndarray) -> np.ndarray:
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)     # biased variance
    return (z - mu) / np.sqrt(var + LN_EPS) * g + b


def gelu(x: np.ndarray) -> np.ndarray:
    return x * 0.5 * (1.0 + erf(x / math.sqrt(2.0)))


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """R18: max-subtracted softmax over the last axis."""
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """softmax(q k^T / sqrt(d)) v for one head over one tile's tokens."""
    d = q.shape[-1]
    return softmax_rows(q @ k.T / math.sqrt(d)) @ v


def block(z: np.ndarray, Lw: dict, heads: int) -> np.ndarray:
    """One pre-norm ViT block over the tokens of ONE tile of ONE sample."""
    D = z.shape[1]
    d = D // heads
    qkv = layer_norm(z, Lw["ln1_g"], Lw["ln1_b"]) @ Lw["W_qkv"].T + Lw["b_qkv"]
    q, k, v = qkv[:, :D], qkv[:, D:2 * D], qkv[:, 2 * D:]
    o = np.concatenate([attention(q[:, h * d:(h + 1) * d], k[:, h * d:(h + 1) * d],
                                  v[:, h * d:(h + 1) * d]) for h in range(heads)], axis=1)
    z = z + o @ Lw["W_o"].T + Lw["b_o"]
    hdn = gelu(layer_norm(z, Lw["ln2_g"], Lw["ln2_b"]) @ Lw["W_1"].T + Lw["b_1"])
    return z + hdn @ Lw["W_2"].T + Lw["b_2"]


# ---------------------------------------------------------------------------
# O5  Head (P:480 decoder "linear projections"; R10, R11)
# ---------------------------------------------------------------------------
def head(z: np.ndarray, Wt: dict) -> np.ndarray:
    return layer_norm(z, Wt["lnf_g"], Wt["lnf_b"]) @ Wt["W_h"].T + Wt["b_h"]


def core_rows(tile: Tile) -> np.ndarray:
    """Indices (into the tile's padded token list) of its core tokens, row-major."""
    uu, ww = np.meshgrid(np.arange(tile.core_y0, tile.core_y1),
                         np.arange(tile.core_x0, tile.core_x1), indexing="ij")
    return ((uu - tile.pad_y0) * tile.pad_w + (ww - tile.pad_x0)).ravel()


# ---------------------------------------------------------------------------
# O6  Stitch ("the halo regions are discarded, and the non-padded tile
#     outputs are stitched together")
# ---------------------------------------------------------------------------
def stitch_tile(out_vit: np.ndarray, g: np.ndarray, tile: Tile, K: int, P: int) -> None:
    """out_vit[k, P*u+al, P*w+be] = g[token(u,w), (k*P+al)*P+be] for core (u,w)."""
    ch, cw = tile.core_y1 - tile.core_y0, tile.core_x1 - tile.core_x0
    blk = g.reshape(ch, cw, K, P, P).transpose(2, 0, 3, 1, 4).reshape(K, ch * P, cw * P)
    out_vit[:, tile.core_y0 * P:tile.core_y1 * P, tile.core_x0 * P:tile.core_x1 * P] = blk


# ---------------------------------------------------------------------------
# O7  Residual bilinear upsample (R12: align_corners=False, edge clamp)
# ---------------------------------------------------------------------------
def _bilinear_axis(n_in: int, s: int):
    Y = np.arange(n_in * s, dtype=np.float64)
    src = np.maximum((Y + 0.5) / s - 0.5, 0.0)
    y0 = np.floor(src).astype(np.int64)
    y0 = np.minimum(y0, n_in - 1)
    y1 = np.minimum(y0 + 1, n_in - 1)
    lam = src - y0
    return y0, y1, lam


def upsample_bilinear_region(plane: np.ndarray, s: int, ys: slice, xs: slice) -> np.ndarray:
    """The same O7 formula evaluated only at output rows ys and columns xs
    (for sampled-tile parity at sizes where the full field does not fit)."""
    H, W = plane.shape
    y0, y1, ly = (a[ys] for a in _bilinear_axis(H, s))
    x0, x1, lx = (a[xs] for a in _bilinear_axis(W, s))
    ly = ly[:, None]
    lx = lx[None, :]
    pr = plane[np.union1d(y0, y1)].astype(np.float64)   # only the rows needed
    rmap = {r: i for i, r in enumerate(np.union1d(y0, y1))}
    iy0 = np.array([rmap[r] for r in y0])
    iy1 = np.array([rmap[r] for r in y1])
    r0 = (1 - lx) * pr[iy0][:, x0] + lx * pr[iy0][:, x1]
    r1 = (1 - lx) * pr[iy1][:, x0] + lx * pr[iy1][:, x1]
    return (1 - ly) * r0 + ly * r1


def upsample_bilinear(plane: np.ndarray, s: int) -> np.ndarray:
    """[H,W] -> [sH,sW]:
    up = (1-ly)((1-lx)x[y0,x0] + lx x[y0,x1]) + ly((1-lx)x[y1,x0] + lx x[y1,x1])."""
    plane = plane.astype(np.float64)
    H, W = plane.shape
    y0, y1, ly = _bilinear_axis(H, s)
    x0, x1, lx = _bilinear_axis(W, s)
    ly = ly[:, None]
    lx = lx[None, :]
    r0 = (1 - lx) * plane[y0][:, x0] + lx * plane[y0][:, x1]
    r1 = (1 - lx) * plane[y1][:, x0] + lx * plane[y1][:, x1]
    return (1 - ly) * r0 + ly * r1


# ---------------------------------------------------------------------------
# O8  Residual convolutional path (reading R31)
# ---------------------------------------------------------------------------
def conv3x3(x: np.ndarray, Wc: np.ndarray, b: np.ndarray) -> np.ndarray:
    """y[o, Y, X] = b[o] + sum_{i, dy, dx} Wc[o, i, dy, dx] x[i, Y + dy - 1, X + dx - 1],
    x taken as 0 outside its extent (zero padding)."""
    Cin, Y, X = x.shape
    xp = np.zeros((Cin, Y + 2, X + 2))
    xp[:, 1:-1, 1:-1] = x
    out = np.zeros((Wc.shape[0], Y, X)) + np.asarray(b, np.float64)[:, None, None]
    for dy in range(3):
        for dx in range(3):
            out += np.einsum("oi,iyx->oyx", Wc[:, :, dy, dx], xp[:, dy:dy + Y, dx:dx + X])
    return out


def residual_conv(up: np.ndarray, Wt: dict) -> np.ndarray:
    """res = up + conv_b(GELU(conv_a(up))) over a [K, Y, X] field (R31)."""
    return up + conv3x3(gelu(conv3x3(up, Wt["W_ra"], Wt["b_ra"])), Wt["W_rb"], Wt["b_rb"])


# ---------------------------------------------------------------------------
# Canonical weight blob -> named fp64 arrays (order: include/orbit2.h, restated here)
# ---------------------------------------------------------------------------
def unpack_weights(blob: np.ndarray, D: int, L: int, din: int, n_head: int, K: int = 0,
                   res_hidden: int = 0, dec_hidden: int = 0, var_agg: int = 0, V: int = 0) -> dict:
    blob = np.asarray(blob, dtype=np.float64)
    F = 4 * D
    off = 0

    def take(*shape):
        nonlocal off
        n = int(np.prod(shape))
        a = blob[off:off + n].reshape(shape)
        off += n
        return a

    Wt = {"W_e": take(D, din), "b_e": take(D), "e_s": take(D), "layers": []}
    for _ in range(L):
        Lw = {}
        Lw["ln1_g"], Lw["ln1_b"] = take(D), take(D)
        Lw["W_qkv"], Lw["b_qkv"] = take(3 * D, D), take(3 * D)
        Lw["W_o"], Lw["b_o"] = take(D, D), take(D)
        Lw["ln2_g"], Lw["ln2_b"] = take(D), take(D)
        Lw["W_1"], Lw["b_1"] = take(F, D), take(F)
        Lw["W_2"], Lw["b_2"] = take(D, F), take(D)
        Wt["layers"].append(Lw)
    Wt["lnf_g"], Wt["lnf_b"] = take(D), take(D)
    Wt["W_h"], Wt["b_h"] = take(n_head, D), take(n_head)
    if res_hidden:   # O8: W_ra[C_r][K][3][3], b_ra[C_r], W_rb[K][C_r][3][3], b_rb[K]
        Wt["W_ra"], Wt["b_ra"] = take(res_hidden, K, 3, 3), take(res_hidden)
        Wt["W_rb"], Wt["b_rb"] = take(K, res_hidden, 3, 3), take(K)
    if dec_hidden:   # O5b: W_da[C_d][K][3][3], b_da[C_d], W_db[K][C_d][3][3], b_db[K]
        Wt["W_da"], Wt["b_da"] = take(dec_hidden, K, 3, 3), take(dec_hidden)
        Wt["W_db"], Wt["b_db"] = take(K, dec_hidden, 3, 3), take(K)
    if var_agg:      # O3b: W_t[V][D][p*p], e_var[V][D], q_agg[D], W_ak, b_ak, W_av, b_av, W_ao, b_ao
        pp = din // V
        Wt["W_t"], Wt["e_var"], Wt["q_agg"] = take(V, D, pp), take(V, D), take(D)
        Wt["W_ak"], Wt["b_ak"] = take(D, D), take(D)
        Wt["W_av"], Wt["b_av"] = take(D, D), take(D)
        Wt["W_ao"], Wt["b_ao"] = take(D, D), take(D)
    if off != blob.size:
        raise ValueError(f"weight blob has {blob.size} values, layout needs {off}")
    return Wt


# ---------------------------------------------------------------------------
# The whole pass
# ---------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Problem:
    """The paper's problem statement: coarse grid of V variables, downscale
    factor, tiles, halo, ViT width/depth/heads (north star)."""
    H: int
    W: int
    V: int
    K: int
    scale: int
    patch: int
    tiles_y: int
    tiles_x: int
    halo: int
    embed: int
    depth: int
    heads: int
    halo_mode: int = HALO_CLAMP
    channel_map: tuple | None = None
    res_hidden: int = 0      # O8 hidden channels (0: no residual convolutions)
    dec_hidden: int = 0      # O5b hidden channels (0: linear decoder head only)
    var_agg: int = 0         # O3b per-variable tokens + cross-attention aggregation (R33)

    @classmethod
    def from_config(cls, cfg) -> "Problem":
        return cls(cfg.H, cfg.W, cfg.V, cfg.K, cfg.scale, cfg.patch, cfg.tiles_y, cfg.tiles_x,
                   cfg.halo, cfg.embed, cfg.depth, cfg.heads, cfg.halo_mode,
                   tuple(cfg.out_channel_map) if cfg.out_channel_map is not None else None,
                   getattr(cfg, "res_hidden", 0), getattr(cfg, "dec_hidden", 0), getattr(cfg, "var_agg", 0))

    @property
    def P(self) -> int:
        return self.scale * self.patch

    def cmap(self) -> tuple:
        return self.channel_map if self.channel_map is not None else tuple(range(self.K))

    def tiles(self) -> list[Tile]:
        return plan_tiles(self.H // self.patch, self.W // self.patch, self.tiles_y,
                          self.tiles_x, self.halo, self.halo_mode)

    def weights(self, blob) -> dict:
        return unpack_weights(blob, self.embed, self.depth, self.V * self.patch ** 2,
                              self.K * self.P * self.P, self.K, self.res_hidden, self.dec_hidden, self.var_agg,
                              self.V)


def decoder_rect(tile: Tile, pr: Problem):
    """O5b: the tile's core grown by r = ceil(2/P) patches (the two 3x3 convolutions'
    reach at the output resolution), clipped to the patch grid (patch units)."""
    r = -(-2 // pr.P)
    Hp, Wp = pr.H // pr.patch, pr.W // pr.patch
    return (max(0, tile.core_y0 - r), min(Hp, tile.core_y1 + r),
            max(0, tile.core_x0 - r), min(Wp, tile.core_x1 + r))


def tile_forward(x_b: np.ndarray, tile: Tile, pr: Problem, Wt: dict) -> np.ndarray:
    """Steps O2-O5 (+ O5b) for one tile of one sample: returns g [n_core, K*P*P]."""
    z = embed_tile(gather_tile(x_b, tile, pr.patch), tile, pr.patch, Wt, pr.heads)
    for Lw in Wt["layers"]:
        z = block(z, Lw, pr.heads)
    if not pr.dec_hidden:
        return head(z[core_rows(tile)], Wt)
    # O5b: head over the decoder rectangle, unpatchify, two 3x3 convolutions, keep the core
    K, P = pr.K, pr.P
    oy0, oy1, ox0, ox1 = decoder_rect(tile, pr)
    uu, ww = np.meshgrid(np.arange(oy0, oy1), np.arange(ox0, ox1), indexing="ij")
    rows = ((uu - tile.pad_y0) * tile.pad_w + (ww - tile.pad_x0)).ravel()
    g = head(z[rows], Wt)
    oh, ow = oy1 - oy0, ox1 - ox0
    field = g.reshape(oh, ow, K, P, P).transpose(2, 0, 3, 1, 4).reshape(K, oh * P, ow * P)
    dec = conv3x3(gelu(conv3x3(field, Wt["W_da"], Wt["b_da"])), Wt["W_db"], Wt["b_db"])
    ch, cw = tile.core_y1 - tile.core_y0, tile.core_x1 - tile.core_x0
    core = dec[:, (tile.core_y0 - oy0) * P:(tile.core_y1 - oy0) * P, (tile.core_x0 - ox0) * P:(tile.core_x1 - ox0) * P]
    return core.reshape(K, ch, P, cw, P).transpose(1, 3, 0, 2, 4).reshape(ch * cw, K * P * P)


def residual_up(x_b: np.ndarray, pr: Problem, Wt: dict | None = None) -> np.ndarray:
    """The residual path over the whole field: O7 upsample (+ O8 convolutions)."""
    up = np.stack([upsample_bilinear(x_b[m], pr.scale) for m in pr.cmap()])
    return residual_conv(up, Wt) if pr.res_hidden else up


def tiles_forward(x: np.ndarray, blob: np.ndarray, pr: Problem, tile_order=None,
                  return_parts: bool = False):
    """Full TILES Reslim forward: x [B,V,H,W] -> out [B,K,sH,sW] (fp64).

    `tile_order` permutes the order tiles are processed in (invariant I3).
    With return_parts=True also returns (out_vit, up)."""
    Wt = pr.weights(blob)
    tiles = pr.tiles()
    order = range(len(tiles)) if tile_order is None else tile_order
    B = x.shape[0]
    sH, sW = pr.scale * pr.H, pr.scale * pr.W
    out_vit = np.zeros((B, pr.K, sH, sW))
    up = np.zeros((B, pr.K, sH, sW))
    for b in range(B):
        for t in order:
            stitch_tile(out_vit[b], tile_forward(x[b], tiles[t], pr, Wt), tiles[t], pr.K, pr.P)
        up[b] = residual_up(x[b], pr, Wt)
    out = out_vit + up
    return (out, out_vit, up) if return_parts else out


def tiles_forward_sampled(x_b: np.ndarray, blob: np.ndarray, pr: Problem, tile_ids) -> dict:
    """Per-tile outputs for selected tiles only (exact: tiles are independent).
    Returns {tile_id: (rows slice, cols slice, out_block [K, ch*P, cw*P],
    vit_block)} over the tile's core output rectangle."""
    Wt = pr.weights(blob)
    tiles = pr.tiles()
    res = {}
    for t in tile_ids:
        tile = tiles[t]
        g = tile_forward(x_b, tile, pr, Wt)
        ch, cw = tile.core_y1 - tile.core_y0, tile.core_x1 - tile.core_x0
        vit = g.reshape(ch, cw, pr.K, pr.P, pr.P).transpose(2, 0, 3, 1, 4).reshape(
            pr.K, ch * pr.P, cw * pr.P)
        ys = slice(tile.core_y0 * pr.P, tile.core_y1 * pr.P)
        xs = slice(tile.core_x0 * pr.P, tile.core_x1 * pr.P)
        if pr.res_hidden:
            # O8 needs up within 2 output pixels of the rectangle: evaluate O7 on the
            # rectangle grown by 2 (clipped to the field, where zero padding applies),
            # convolve, keep the centre
            sH, sW = pr.scale * pr.H, pr.scale * pr.W
            y0, y1 = max(0, ys.start - 2), min(sH, ys.stop + 2)
            x0, x1 = max(0, xs.start - 2), min(sW, xs.stop + 2)
            upx = np.stack([upsample_bilinear_region(x_b[m], pr.scale, slice(y0, y1), slice(x0, x1))
                            for m in pr.cmap()])
            up = residual_conv(upx, Wt)[:, ys.start - y0:ys.stop - y0, xs.start - x0:xs.stop - x0]
        else:
            up = np.stack([upsample_bilinear_region(x_b[m], pr.scale, ys, xs) for m in pr.cmap()])
        res[t] = (ys, xs, vit + up, vit)
    return res


def global_forward(x: np.ndarray, blob: np.ndarray, pr: Problem) -> np.ndarray:
    """The UNTILED Reslim forward over the whole patch grid (attention over all
    tokens), written separately from the tile loop for invariants I2/I6."""
    Wt = pr.weights(blob)
    p, P, K = pr.patch, pr.P, pr.K
    Hp, Wp = pr.H // p, pr.W // p
    B = x.shape[0]
    out = np.zeros((B, K, pr.scale * pr.H, pr.scale * pr.W))
    for b in range(B):
        a = patch_tokens(x[b].astype(np.float64), p)
        uu, ww = np.meshgrid(np.arange(Hp), np.arange(Wp), indexing="ij")
        feat = aggregate_variables(a, Wt, pr.heads, p) if pr.var_agg else a @ Wt["W_e"].T + Wt["b_e"]
        z = feat + Wt["e_s"] + sincos_pos(uu.ravel(), ww.ravel(), pr.embed)
        for Lw in Wt["layers"]:
            z = block(z, Lw, pr.heads)
        g = head(z, Wt)
        out[b] = g.reshape(Hp, Wp, K, P, P).transpose(2, 0, 3, 1, 4).reshape(K, Hp * P, Wp * P)
        if pr.dec_hidden:
            out[b] = conv3x3(gelu(conv3x3(out[b], Wt["W_da"], Wt["b_da"])), Wt["W_db"], Wt["b_db"])
        out[b] += residual_up(x[b], pr, Wt)
    return out


# ---------------------------------------------------------------------------
# Analytic counts (SURVEY.md §8(d) definitions, restated)
# ---------------------------------------------------------------------------
def token_counts(pr: Problem) -> dict:
    tiles = pr.tiles()
    n = np.array([t.n_tokens for t in tiles], dtype=np.int64)
    c = np.array([t.n_core for t in tiles], dtype=np.int64)
    return {"n_pad": int(n.sum()), "n_core": int(c.sum()), "sum_n2": int((n * n).sum()),
            "sum_nc": int((n * c).sum()), "n": n, "c": c}


def paper_sequence_length(out_h: int, out_w: int, channels: int, p: int) -> int:
    """P:150 convention: sequence length = output pixels x channels / p^2."""
    return out_h * out_w * channels // (p * p)
