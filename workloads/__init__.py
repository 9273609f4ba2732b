"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no embedding, attention, tiling,
stitching or interpolation).  It only defines
  * the five BASELINE.json configurations C1..C5 as plain data (SURVEY.md §8
    "Config resolution"; DESIGN.md "Readings" R3, R23-R26),
  * a seeded generator for ERA5-shaped coarse input fields (DESIGN.md
    "Input recipe"),
  * a seeded generator for the canonical fp32 weight blob, drawn parameter by
    parameter in the canonical order documented in include/orbit2.h,
  * special inputs used by pins (constant field, affine ramp).
Both `oracle/` and the CUDA path consume these arrays as DATA; neither imports
the other.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Config", "CONFIGS", "get_config", "make_input", "make_weights",
    "weight_count", "bf16_round", "constant_input", "ramp_input",
]


@dataclasses.dataclass(frozen=True)
class Config:
    """One workload: coarse grid, downscale factor, tiling and ViT size.

    Field names follow the paper's problem statement (PAPER.md L404 model
    sizes; L527-532 tiles/halo) and include/orbit2.h `orbit2_config`.
    """
    name: str
    H: int            # coarse rows (pixels)
    W: int            # coarse cols (pixels)
    V: int            # input variables
    K: int            # output variables
    scale: int        # downscale factor s
    patch: int        # patch size p (pixels)
    tiles_y: int
    tiles_x: int
    halo: int         # halo width in PATCHES (reading R3)
    embed: int        # D
    depth: int        # L
    heads: int
    batch: int        # bench batch B
    halo_mode: int = 0          # 0 = CLAMP (reading R4), 1 = REPLICATE
    out_channel_map: tuple | None = None   # K entries in [0,V); None = identity
    res_hidden: int = 0         # residual-path conv hidden channels (reading R31); 0 = none
    dec_hidden: int = 0         # decoder conv hidden channels (reading R32); 0 = linear head only
    var_agg: int = 0            # per-variable tokens + cross-attention aggregation (reading R33)

    @property
    def mlp_hidden(self) -> int:
        return 4 * self.embed

    @property
    def head_dim(self) -> int:
        return self.embed // self.heads

    @property
    def Hp(self) -> int:
        return self.H // self.patch

    @property
    def Wp(self) -> int:
        return self.W // self.patch

    @property
    def P(self) -> int:
        """Output pixels per patch side: s*p."""
        return self.scale * self.patch

    @property
    def din(self) -> int:
        return self.V * self.patch * self.patch

    @property
    def head_out(self) -> int:
        return self.K * self.P * self.P

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)

    def channel_map(self) -> tuple:
        if self.out_channel_map is not None:
            return tuple(self.out_channel_map)
        return tuple(range(self.K))


# BASELINE.json "configs" resolved to concrete shapes.
CONFIGS = {
    "C1": Config("C1-toy", 32, 64, 3, 3, 4, 2, 2, 2, 2, 64, 1, 2, batch=1),
    "C2": Config("C2-era5-1.0deg-0.25deg-9.5M", 180, 360, 20, 3, 4, 2, 4, 4, 4, 256, 6, 4, batch=64),
    "C3": Config("C3-us-28km-7km-126M", 180, 360, 23, 3, 4, 2, 8, 8, 2, 1024, 8, 16, batch=16),
    "C4": Config("C4-global-0.25deg-3.5km-1B", 720, 1440, 23, 18, 8, 2, 16, 16, 4, 2048, 16, 32, batch=1),
    "C5": Config("C5-hyperres-0.9km", 5400, 10800, 23, 18, 4, 2, 36, 36, 4, 256, 6, 4, batch=1),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return cfg.replace(**overrides) if overrides else cfg


# ---------------------------------------------------------------------------
# Input fields
# ---------------------------------------------------------------------------
N_MODES = 32
MAX_WAVENUMBER = 16
NOISE_STD = 0.1


def _field_plane(rng: np.random.Generator, H: int, W: int) -> np.ndarray:
    """One [H,W] plane: sum of 32 periodic plane waves with a kappa^-3 power
    spectrum plus white noise, then standardised (zero mean, unit variance).

    cos(a_y + b_x) = cos a_y cos b_x - sin a_y sin b_x, so the sum of modes is
    a rank-2*N_MODES outer product, evaluated with one matmul.
    """
    k = rng.integers(-MAX_WAVENUMBER, MAX_WAVENUMBER + 1, size=N_MODES)
    l = rng.integers(-MAX_WAVENUMBER, MAX_WAVENUMBER + 1, size=N_MODES)
    zero = (k == 0) & (l == 0)
    k[zero] = 1
    kappa = np.sqrt(k.astype(np.float64) ** 2 + l.astype(np.float64) ** 2)
    amp = kappa ** -1.5
    phi = rng.uniform(0.0, 2.0 * math.pi, size=N_MODES)
    ay = 2.0 * math.pi * np.outer(np.arange(H) / H, k) + phi        # [H, M]
    bx = 2.0 * math.pi * np.outer(np.arange(W) / W, l)              # [W, M]
    U = np.concatenate([np.cos(ay) * amp, -np.sin(ay) * amp], axis=1)   # [H, 2M]
    Vm = np.concatenate([np.cos(bx), np.sin(bx)], axis=1)               # [W, 2M]
    plane = U @ Vm.T
    plane += NOISE_STD * rng.standard_normal((H, W))
    plane -= plane.mean()
    sd = plane.std()
    if sd > 0:
        plane /= sd
    return plane


def make_input(cfg: Config, batch: int | None = None, seed: int | None = None) -> np.ndarray:
    """fp32 [B,V,H,W] synthetic ERA5-shaped coarse field, row 0 = north."""
    B = cfg.batch if batch is None else batch
    if seed is None:
        seed = 1000 + int(cfg.name[1]) if cfg.name[0] == "C" and cfg.name[1].isdigit() else 1000
    x = np.empty((B, cfg.V, cfg.H, cfg.W), dtype=np.float32)
    for b in range(B):
        for v in range(cfg.V):
            rng = np.random.default_rng([seed, b, v])
            x[b, v] = _field_plane(rng, cfg.H, cfg.W)
    return x


def constant_input(cfg: Config, value: float = 1.25, batch: int = 1) -> np.ndarray:
    return np.full((batch, cfg.V, cfg.H, cfg.W), value, dtype=np.float32)


def ramp_input(cfg: Config, batch: int = 1) -> np.ndarray:
    """x[b,v,y,x] = 0.5 + 0.25*y - 0.125*x + v (exact in fp32 for small grids)."""
    yy = np.arange(cfg.H, dtype=np.float32)[:, None]
    xx = np.arange(cfg.W, dtype=np.float32)[None, :]
    x = np.empty((batch, cfg.V, cfg.H, cfg.W), dtype=np.float32)
    for v in range(cfg.V):
        x[:, v] = 0.5 + 0.25 * yy - 0.125 * xx + v
    return x


# ---------------------------------------------------------------------------
# Canonical weight blob (order documented in include/orbit2.h)
# ---------------------------------------------------------------------------
def weight_count(cfg: Config) -> int:
    D, L, F = cfg.embed, cfg.depth, cfg.mlp_hidden
    per_layer = 2 * D + 3 * D * D + 3 * D + D * D + D + 2 * D + F * D + F + D * F + D
    n = cfg.din * D + 2 * D + L * per_layer + 2 * D + cfg.head_out * D + cfg.head_out
    for c in (cfg.res_hidden, cfg.dec_hidden):
        if c:
            n += 2 * 9 * c * cfg.K + c + cfg.K
    if cfg.var_agg:
        n += cfg.V * D * cfg.patch ** 2 + cfg.V * D + D + 3 * (D * D + D)
    return n


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def make_weights(cfg: Config, seed: int | None = None, sharp: bool = True,
                 head_gain: float = 1.0, round_bf16: bool = True, res_gain: float = 1.0) -> np.ndarray:
    """Flat fp32 canonical blob.

    W ~ N(0, 1/fan_in); biases ~ N(0, 0.02^2); LN gamma ~ 1+U(-0.1,0.1),
    beta ~ U(-0.1,0.1); resolution embedding e_s ~ N(0, 0.02^2);
    head W_h ~ N(0, head_gain^2/D).  `sharp` doubles the W_q rows so attention
    logits have std ~2 (exercises the softmax range).  All values are rounded
    to bf16-representable fp32 so weight quantisation is not charged to the
    bf16 tolerance.
    """
    if seed is None:
        seed = 2000 + int(cfg.name[1]) if cfg.name[0] == "C" and cfg.name[1].isdigit() else 2000
    rng = np.random.default_rng(seed)
    D, L, F, Din, Nh = cfg.embed, cfg.depth, cfg.mlp_hidden, cfg.din, cfg.head_out
    parts = []

    def lin(out_f, in_f, gain=1.0):
        parts.append((rng.standard_normal((out_f, in_f)) * (gain / math.sqrt(in_f))).ravel())

    def bias(n, std=0.02):
        parts.append(rng.standard_normal(n) * std)

    def ln(n):
        parts.append(1.0 + rng.uniform(-0.1, 0.1, n))
        parts.append(rng.uniform(-0.1, 0.1, n))

    lin(D, Din); bias(D); bias(D)                     # W_e, b_e, e_s
    for _ in range(L):
        ln(D)                                         # ln1 gamma, beta
        wqkv = rng.standard_normal((3 * D, D)) / math.sqrt(D)
        if sharp:
            wqkv[:D] *= 2.0
        parts.append(wqkv.ravel())                    # W_qkv rows Q|K|V
        bias(3 * D)                                   # b_qkv
        lin(D, D); bias(D)                            # W_o, b_o
        ln(D)                                         # ln2
        lin(F, D); bias(F)                            # W_1, b_1
        lin(D, F); bias(D)                            # W_2, b_2
    ln(D)                                             # lnf
    lin(Nh, D, head_gain); bias(Nh)                   # W_h, b_h
    if cfg.res_hidden:                                # residual convs W_ra, b_ra, W_rb, b_rb
        lin(cfg.res_hidden, cfg.K * 9); bias(cfg.res_hidden)
        lin(cfg.K, cfg.res_hidden * 9, res_gain); bias(cfg.K)
    if cfg.dec_hidden:                                # decoder convs W_da, b_da, W_db, b_db
        lin(cfg.dec_hidden, cfg.K * 9); bias(cfg.dec_hidden)
        lin(cfg.K, cfg.dec_hidden * 9); bias(cfg.K)
    if cfg.var_agg:                                   # variable aggregation (R33)
        pp = cfg.patch ** 2
        parts.append((rng.standard_normal((cfg.V, D, pp)) / math.sqrt(pp)).ravel())   # W_t[v]
        parts.append(rng.standard_normal(cfg.V * D) * 0.5)                            # e_var
        parts.append(rng.standard_normal(D) * 2.0)                                    # q_agg (sharp-ish)
        for _ in range(3):                                                             # W_ak, W_av, W_ao + biases
            lin(D, D); bias(D)
    blob = np.concatenate(parts).astype(np.float32)
    assert blob.size == weight_count(cfg)
    return bf16_round(blob) if round_bf16 else blob
