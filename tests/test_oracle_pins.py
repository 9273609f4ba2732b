"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names the passage / reading it pins and what would break it.
Pins used: torch fp64 library modules the oracle does not call (conv2d,
TransformerEncoderLayer, scaled_dot_product_attention, layer_norm,
pixel_shuffle, interpolate), closed forms, brute force over small grids,
the paper's printed token counts, and the invariants I1-I10.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import reslim_tiles as O
from workloads import get_config, make_input, make_weights, constant_input, ramp_input



@pytest.fixture(autouse=True)
def _fp64_default():
    """The torch library pins run in fp64; restored afterwards (a process-wide
    float64 default would leak into the GPU tests' float32 buffers)."""
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def small_problem(**kw):
    base = dict(H=24, W=40, V=3, K=2, scale=4, patch=2, tiles_y=2, tiles_x=3, halo=1,
                embed=16, depth=2, heads=2)
    base.update(kw)
    return O.Problem(**base)


def blob_for(pr, seed=7, head_gain=1.0, sharp=True, res_gain=1.0):
    cfg = get_config("C1", H=pr.H, W=pr.W, V=pr.V, K=pr.K, scale=pr.scale, patch=pr.patch,
                     tiles_y=pr.tiles_y, tiles_x=pr.tiles_x, halo=pr.halo, embed=pr.embed,
                     depth=pr.depth, heads=pr.heads, halo_mode=pr.halo_mode, res_hidden=pr.res_hidden,
                     dec_hidden=pr.dec_hidden, var_agg=pr.var_agg)
    return make_weights(cfg, seed=seed, head_gain=head_gain, sharp=sharp, res_gain=res_gain), cfg


def input_for(cfg, batch=1, seed=11):
    return make_input(cfg, batch=batch, seed=seed)


# ---------------------------------------------------------------- O1 plan
@pytest.mark.parametrize("mode", [O.HALO_CLAMP, O.HALO_REPLICATE])
def test_plan_brute_force(mode):
    """P:527-530, R3-R6: cores partition the grid; sizes differ by <=1 with
    earlier tiles larger; a patch is in the padded rect iff its Chebyshev
    distance to the core (per axis) is <= halo (and inside the grid in CLAMP).
    Brute force over every patch of every small layout."""
    for Hp in range(1, 9):
        for Wp in range(1, 9):
            for ty in range(1, min(Hp, 4) + 1):
                for tx in range(1, min(Wp, 4) + 1):
                    for h in range(0, 4):
                        tiles = O.plan_tiles(Hp, Wp, ty, tx, h, mode)
                        assert [t.tile_id for t in tiles] == list(range(ty * tx))
                        owner = -np.ones((Hp, Wp), int)
                        for t in tiles:
                            assert t.tile_id == t.ty * tx + t.tx
                            blk = owner[t.core_y0:t.core_y1, t.core_x0:t.core_x1]
                            assert (blk == -1).all()
                            blk[...] = t.tile_id
                        assert (owner >= 0).all()
                        hs = [tiles[i * tx].core_y1 - tiles[i * tx].core_y0 for i in range(ty)]
                        ws = [tiles[j].core_x1 - tiles[j].core_x0 for j in range(tx)]
                        assert max(hs) - min(hs) <= 1 and hs == sorted(hs, reverse=True)
                        assert max(ws) - min(ws) <= 1 and ws == sorted(ws, reverse=True)
                        for t in tiles:
                            rng_y = range(-h - 1, Hp + h + 1)
                            rng_x = range(-h - 1, Wp + h + 1)
                            for u in rng_y:
                                dy = max(t.core_y0 - u, u - (t.core_y1 - 1), 0)
                                iny = dy <= h and (mode == O.HALO_REPLICATE or 0 <= u < Hp)
                                assert iny == (t.pad_y0 <= u < t.pad_y1)
                            for w in rng_x:
                                dx = max(t.core_x0 - w, w - (t.core_x1 - 1), 0)
                                inx = dx <= h and (mode == O.HALO_REPLICATE or 0 <= w < Wp)
                                assert inx == (t.pad_x0 <= w < t.pad_x1)


def test_plan_spec_examples():
    """SPEC S:453 T=1,h=0 -> one tile = whole image; S:454 4x4 tiles on 720x1440
    -> per-tile token share 1/16; R5: C2 tile rows 23,23,22,22 patches."""
    t = O.plan_tiles(10, 7, 1, 1, 0)
    assert len(t) == 1 and (t[0].core_y0, t[0].core_y1, t[0].core_x0, t[0].core_x1) == (0, 10, 0, 7)
    assert (t[0].pad_y0, t[0].pad_y1, t[0].pad_x0, t[0].pad_x1) == (0, 10, 0, 7)
    tiles = O.plan_tiles(360, 720, 4, 4, 0)
    assert all(x.n_core * 16 == 360 * 720 for x in tiles)
    c2 = O.plan_tiles(90, 180, 4, 4, 4)
    assert [c2[i * 4].core_y1 - c2[i * 4].core_y0 for i in range(4)] == [23, 23, 22, 22]


def test_paper_token_anchors():
    """P:150 (24,576 for [128,256,3]), P:434 (298M for [5760,11520,18]),
    P:436 (1.1B for [11520,23040,18]), P:437 (4.2B for [21600,43200,18]).
    P:150 prints 777,660 for [720,1440,3]; the formula gives 777,600 (R22)."""
    assert O.paper_sequence_length(128, 256, 3, 2) == 24576
    assert O.paper_sequence_length(5760, 11520, 18, 2) == 298_598_400
    assert O.paper_sequence_length(11520, 23040, 18, 2) == 1_194_393_600
    assert O.paper_sequence_length(21600, 43200, 18, 2) == 4_199_040_000
    assert O.paper_sequence_length(720, 1440, 3, 2) == 777_600


def test_complexity_law():
    """attention cost O(N^2/T): with h=0 and an even split, sum n_t^2 = N^2/T."""
    for (Hp, Wp, ty, tx) in [(16, 32, 2, 2), (90, 180, 3, 4), (64, 64, 8, 8)]:
        pr = O.Problem(2 * Hp, 2 * Wp, 1, 1, 2, 2, ty, tx, 0, 8, 1, 1)
        c = O.token_counts(pr)
        N, T = Hp * Wp, ty * tx
        assert c["sum_n2"] * T == N * N and c["n_pad"] == N


def test_survey_config_counts():
    """N_pad/sample for C1-C5 (computed by the oracle planner)."""
    want = {"C1": (720, 512), "C2": (23256, 16200), "C3": (24544, 16200),
            "C4": (403200, 259200), "C5": (16926400, 14580000)}
    for name, (npad, ncore) in want.items():
        c = O.token_counts(O.Problem.from_config(get_config(name)))
        assert (c["n_pad"], c["n_core"]) == (npad, ncore), name


# ---------------------------------------------------------------- O2 gather
def test_gather_clamp_is_slice_and_replicate_is_edge_pad():
    """R4: CLAMP gather = plain slice of the padded rect; REPLICATE = np.pad(edge)."""
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 12, 20)).astype(np.float32)
    p = 2
    for t in O.plan_tiles(6, 10, 2, 3, 2, O.HALO_CLAMP):
        got = O.gather_tile(x, t, p)
        assert np.array_equal(got, x[:, p * t.pad_y0:p * t.pad_y1, p * t.pad_x0:p * t.pad_x1])
    h = 2
    xp = np.pad(x, ((0, 0), (p * h, p * h), (p * h, p * h)), mode="edge")
    for t in O.plan_tiles(6, 10, 2, 3, h, O.HALO_REPLICATE):
        got = O.gather_tile(x, t, p)
        want = xp[:, p * (t.pad_y0 + h):p * (t.pad_y1 + h), p * (t.pad_x0 + h):p * (t.pad_x1 + h)]
        assert np.array_equal(got, want)


# ---------------------------------------------------------------- O3 embed
def test_patch_embed_matches_conv2d():
    """R1: the joint patch embed is a conv with kernel = stride = p; column
    order (v*p+dy)*p+dx equals torch's [D][V][p][p] weight flattening."""
    rng = np.random.default_rng(1)
    V, p, D, H, W = 3, 2, 10, 8, 12
    x = rng.standard_normal((V, H, W))
    We = rng.standard_normal((D, V * p * p))
    a = O.patch_tokens(x, p)                                   # [Hp*Wp, Din]
    got = a @ We.T
    want = F.conv2d(torch.from_numpy(x)[None], torch.from_numpy(We).reshape(D, V, p, p), stride=p)
    want = want[0].permute(1, 2, 0).reshape(-1, D).numpy()
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)


def test_sincos_closed_form():
    """R7 closed forms: pi(0,0) = [0..,1..,0..,1..]; sin^2+cos^2 = 1 per pair;
    omega_0 = 1 so pi[0] = sin(u), pi[3Q] = cos(w); omega_{Q/2} = 10000^-1/2 = 0.01."""
    D = 16
    Q = D // 4
    p0 = O.sincos_pos(np.array([0]), np.array([0]), D)[0]
    assert np.array_equal(p0, np.r_[np.zeros(Q), np.ones(Q), np.zeros(Q), np.ones(Q)])
    u = np.array([3, -2, 7]); w = np.array([5, 11, -1])
    pe = O.sincos_pos(u, w, D)
    np.testing.assert_allclose(pe[:, :Q] ** 2 + pe[:, Q:2 * Q] ** 2, 1.0, atol=1e-15)
    np.testing.assert_allclose(pe[:, 2 * Q:3 * Q] ** 2 + pe[:, 3 * Q:] ** 2, 1.0, atol=1e-15)
    assert pe[0, 0] == math.sin(3.0) and pe[0, 3 * Q] == math.cos(5.0)
    np.testing.assert_allclose(pe[:, Q // 2], np.sin(0.01 * u), rtol=1e-14)
    np.testing.assert_allclose(pe[:, 2 * Q + Q // 2], np.sin(0.01 * w), rtol=1e-14)


# ---------------------------------------------------------------- O4 blocks
def test_attention_textbook_cases():
    """S:171-175 / I1: rows sum to 1; n=1 -> o = v; identical q,k rows ->
    uniform weights -> mean of v; matches torch SDPA (math) in fp64."""
    rng = np.random.default_rng(2)
    q, k, v = (rng.standard_normal((9, 4)) * 3 for _ in range(3))
    A = O.softmax_rows(q @ k.T / 2.0)
    assert np.abs(A.sum(1) - 1).max() <= 1e-12 and (A >= 0).all()
    v1 = rng.standard_normal((1, 4))
    assert np.array_equal(O.attention(q[:1], k[:1], v1), v1)
    qq = np.tile(q[:1], (9, 1)); kk = np.tile(k[:1], (9, 1))
    np.testing.assert_allclose(O.attention(qq, kk, v), np.tile(v.mean(0), (9, 1)), atol=1e-14)
    want = F.scaled_dot_product_attention(*(torch.from_numpy(t)[None] for t in (q, k, v)))[0].numpy()
    np.testing.assert_allclose(O.attention(q, k, v), want, rtol=1e-12, atol=1e-13)


def test_layer_norm_and_gelu_vs_torch():
    rng = np.random.default_rng(3)
    z = rng.standard_normal((7, 12)) * 4 + 1
    g, b = rng.standard_normal(12), rng.standard_normal(12)
    want = F.layer_norm(torch.from_numpy(z), (12,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5)
    np.testing.assert_allclose(O.layer_norm(z, g, b), want.numpy(), rtol=1e-12, atol=1e-12)
    xg = np.linspace(-6, 6, 101)
    np.testing.assert_allclose(O.gelu(xg), F.gelu(torch.from_numpy(xg)).numpy(), rtol=1e-14, atol=1e-15)


def _torch_layer(Lw, D, heads):
    layer = torch.nn.TransformerEncoderLayer(D, heads, dim_feedforward=4 * D, dropout=0.0,
                                             activation="gelu", layer_norm_eps=1e-5,
                                             batch_first=True, norm_first=True, dtype=torch.float64)
    sd = {
        "self_attn.in_proj_weight": Lw["W_qkv"], "self_attn.in_proj_bias": Lw["b_qkv"],
        "self_attn.out_proj.weight": Lw["W_o"], "self_attn.out_proj.bias": Lw["b_o"],
        "linear1.weight": Lw["W_1"], "linear1.bias": Lw["b_1"],
        "linear2.weight": Lw["W_2"], "linear2.bias": Lw["b_2"],
        "norm1.weight": Lw["ln1_g"], "norm1.bias": Lw["ln1_b"],
        "norm2.weight": Lw["ln2_g"], "norm2.bias": Lw["ln2_b"],
    }
    layer.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()})
    return layer.eval()


def test_block_matches_torch_transformer_layer():
    """R9: pre-norm block (LN eps 1e-5, qkv bias, 1/sqrt(d), MLP 4D, erf GELU,
    heads = contiguous d-slices of Q|K|V) == torch TransformerEncoderLayer
    (norm_first, gelu) in fp64.  A swapped head split, a missing bias or a
    post-norm block fails this."""
    pr = small_problem(embed=24, heads=3, depth=1)
    blob, _ = blob_for(pr)
    Wt = pr.weights(blob)
    z = np.random.default_rng(4).standard_normal((37, 24))
    got = O.block(z, Wt["layers"][0], 3)
    with torch.no_grad():
        want = _torch_layer(Wt["layers"][0], 24, 3)(torch.from_numpy(z)[None])[0].numpy()
    np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-11)


# ---------------------------------------------------------------- O7 residual
@pytest.mark.parametrize("s", [1, 2, 4, 8, 16])
def test_bilinear_matches_interpolate(s):
    """R12: align_corners=False bilinear with edge clamp == F.interpolate."""
    x = np.random.default_rng(5).standard_normal((7, 11))
    want = F.interpolate(torch.from_numpy(x)[None, None], scale_factor=s, mode="bilinear",
                         align_corners=False)[0, 0].numpy()
    np.testing.assert_allclose(O.upsample_bilinear(x, s), want, rtol=1e-14, atol=1e-14)
    c = np.full((5, 6), 2.5)
    assert np.array_equal(O.upsample_bilinear(c, s), np.full((5 * s, 6 * s), 2.5))


def test_bilinear_region_equals_full_slice():
    """The region evaluation of O7 (used for sampled C4/C5 parity) is the full
    upsample restricted to the region, bit for bit."""
    x = np.random.default_rng(6).standard_normal((9, 13))
    for s in (2, 4, 8):
        full = O.upsample_bilinear(x, s)
        for ys, xs in [(slice(0, 5), slice(3, 17)), (slice(7, 9 * s), slice(0, 13 * s)), (slice(11, 12), slice(5, 6))]:
            assert np.array_equal(O.upsample_bilinear_region(x, s, ys, xs), full[ys, xs])


# ---------------------------------------------------------------- O6 stitch
def test_stitch_coordinate_codes():
    """every core token's head output lands at its own output pixels.
    g[(k*P+al)*P+be] for core (u,w) carries code(k, P*u+al, P*w+be); after
    stitching out_vit[k,Y,X] == code(k,Y,X) everywhere (bit-exact), so each
    output pixel is written exactly once by the right tile."""
    K, P, Hp, Wp = 3, 4, 7, 9
    code = lambda k, Y, X: (k * 1000 + Y) * 1000 + X
    for mode in (O.HALO_CLAMP, O.HALO_REPLICATE):
        out = np.full((K, Hp * P, Wp * P), -1.0)
        for t in O.plan_tiles(Hp, Wp, 3, 2, 2, mode):
            uu, ww = np.meshgrid(np.arange(t.core_y0, t.core_y1), np.arange(t.core_x0, t.core_x1),
                                 indexing="ij")
            k, al, be = np.meshgrid(np.arange(K), np.arange(P), np.arange(P), indexing="ij")
            g = code(k[None], P * uu.ravel()[:, None, None, None] + al[None],
                     P * ww.ravel()[:, None, None, None] + be[None]).reshape(len(uu.ravel()), -1)
            O.stitch_tile(out, g.astype(np.float64), t, K, P)
        kk, YY, XX = np.meshgrid(np.arange(K), np.arange(Hp * P), np.arange(Wp * P), indexing="ij")
        assert np.array_equal(out, code(kk, YY, XX).astype(np.float64))


# ---------------------------------------------------------------- whole pass
def torch_global_model(x, blob, pr):
    """Independent untiled Reslim from torch fp64 library modules: conv2d
    embed, TransformerEncoderLayer blocks, layer_norm + linear head,
    pixel_shuffle decoder, F.interpolate residual."""
    Wt = pr.weights(blob)
    D, p, P = pr.embed, pr.patch, pr.P
    Hp, Wp = pr.H // p, pr.W // p
    xt = torch.from_numpy(x.astype(np.float64))
    with torch.no_grad():
        z = F.conv2d(xt, torch.from_numpy(Wt["W_e"]).reshape(D, pr.V, p, p),
                     torch.from_numpy(Wt["b_e"] + Wt["e_s"]), stride=p)     # [B,D,Hp,Wp]
        z = z.flatten(2).transpose(1, 2)
        uu, ww = np.meshgrid(np.arange(Hp), np.arange(Wp), indexing="ij")
        z = z + torch.from_numpy(O.sincos_pos(uu.ravel(), ww.ravel(), D))[None]
        for Lw in Wt["layers"]:
            z = _torch_layer(Lw, D, pr.heads)(z)
        g = F.linear(F.layer_norm(z, (D,), torch.from_numpy(Wt["lnf_g"]),
                                  torch.from_numpy(Wt["lnf_b"]), eps=1e-5),
                     torch.from_numpy(Wt["W_h"]), torch.from_numpy(Wt["b_h"]))
        g = g.transpose(1, 2).reshape(x.shape[0], pr.K * P * P, Hp, Wp)
        vit = F.pixel_shuffle(g, P)
        up = F.interpolate(xt[:, list(pr.cmap())], scale_factor=pr.scale, mode="bilinear",
                           align_corners=False)
    return (vit + up).numpy()


def test_untiled_oracle_matches_torch_library_model():
    """I2 (part 1): the oracle's T=1, h=0 TILES forward equals an untiled
    Reslim assembled from torch library modules, to fp64 rounding."""
    pr = small_problem(tiles_y=1, tiles_x=1, halo=0, channel_map=(2, 0))
    blob, cfg = blob_for(pr)
    x = input_for(cfg, batch=2)
    got = O.tiles_forward(x, blob, pr)
    want = torch_global_model(x, blob, pr)
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(O.global_forward(x, blob, pr), want, rtol=1e-10, atol=1e-10)


def test_I6_full_halo_equals_global():
    """I6: CLAMP with h >= max(Hp,Wp): every padded tile is the whole grid, so
    the tiled pass equals the untiled global model."""
    pr = small_problem(halo=50)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    np.testing.assert_allclose(O.tiles_forward(x, blob, pr), O.global_forward(x, blob, pr),
                               rtol=1e-12, atol=1e-12)


def test_I4_zero_head_gives_upsample_exactly():
    """I4 / S:379 initialization contract: W_h = 0, b_h = 0 -> out == bilinear up, bitwise."""
    pr = small_problem()
    blob, cfg = blob_for(pr, head_gain=0.0)
    nh = pr.K * pr.P ** 2
    blob[-nh:] = 0.0
    x = input_for(cfg)
    out, vit, up = O.tiles_forward(x, blob, pr, return_parts=True)
    assert np.array_equal(vit, np.zeros_like(vit)) and np.array_equal(out, up)


def test_I5_locality():
    """I5 (S:480 'locality'): perturbing input pixels outside tile t's padded
    rect leaves t's core output bit-identical (h >= 1 so the bilinear support
    stays inside the padded rect)."""
    pr = small_problem(tiles_y=3, tiles_x=3, H=36, W=36, halo=1)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)[0]
    t = 4   # interior tile
    tile = pr.tiles()[t]
    base = O.tiles_forward_sampled(x, blob, pr, [t])[t]
    x2 = x.copy()
    mask = np.ones(x.shape[1:], bool)
    mask[2 * tile.pad_y0:2 * tile.pad_y1, 2 * tile.pad_x0:2 * tile.pad_x1] = False
    x2[:, mask] += 3.0
    pert = O.tiles_forward_sampled(x2, blob, pr, [t])[t]
    assert np.array_equal(base[2], pert[2])
    # and a perturbation INSIDE the halo does change it (the test can fail)
    x3 = x.copy()
    x3[:, 2 * tile.pad_y0, 2 * tile.pad_x0] += 3.0
    assert not np.array_equal(base[2], O.tiles_forward_sampled(x3, blob, pr, [t])[t][2])


def test_I7_no_blocks_is_tiling_independent():
    """I7: with L=0 every token's output depends only on its own patch (global
    position embedding), so out is independent of T, h and halo mode."""
    ref = None
    for (ty, tx, h, mode) in [(1, 1, 0, 0), (2, 3, 1, 0), (3, 2, 2, 1), (4, 5, 0, 1)]:
        pr = small_problem(depth=0, tiles_y=ty, tiles_x=tx, halo=h, halo_mode=mode)
        blob, cfg = blob_for(pr)
        out = O.tiles_forward(input_for(cfg), blob, pr)
        if ref is None:
            ref = out
        np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-13)


def test_I8_batch_independence():
    pr = small_problem()
    blob, cfg = blob_for(pr)
    x = input_for(cfg, batch=3)
    full = O.tiles_forward(x, blob, pr)
    assert np.array_equal(full[1], O.tiles_forward(x[1:2], blob, pr)[0])


def test_I9_head_linearity():
    """I9: (out - up) scales by c when (W_h, b_h) scale by c."""
    pr = small_problem()
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    nh = pr.K * pr.P ** 2
    n_head = nh * pr.embed + nh
    b2 = blob.astype(np.float64).copy()
    b2[-n_head:] *= 2.5
    _, v1, _ = O.tiles_forward(x, blob, pr, return_parts=True)
    _, v2, _ = O.tiles_forward(x, b2, pr, return_parts=True)
    np.testing.assert_allclose(v2, 2.5 * v1, rtol=1e-12, atol=1e-12)


def test_I10_replicate_equals_clamp_on_interior_tiles():
    pr_c = small_problem(tiles_y=3, tiles_x=3, H=36, W=36, halo=1, halo_mode=0)
    pr_r = small_problem(tiles_y=3, tiles_x=3, H=36, W=36, halo=1, halo_mode=1)
    blob, cfg = blob_for(pr_c)
    x = input_for(cfg)[0]
    a = O.tiles_forward_sampled(x, blob, pr_c, [4])[4]
    b = O.tiles_forward_sampled(x, blob, pr_r, [4])[4]
    assert np.array_equal(a[2], b[2])
    # a border tile differs (halo content differs), so the test can fail
    a0 = O.tiles_forward_sampled(x, blob, pr_c, [0])[0]
    b0 = O.tiles_forward_sampled(x, blob, pr_r, [0])[0]
    assert not np.array_equal(a0[2], b0[2])


def test_I3_tile_order_permutation():
    pr = small_problem()
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    n = pr.tiles_y * pr.tiles_x
    perm = np.random.default_rng(9).permutation(n)
    assert np.array_equal(O.tiles_forward(x, blob, pr), O.tiles_forward(x, blob, pr, tile_order=perm))


def test_tiling_changes_output_but_stays_close():
    """Sanity that TILES is an approximation: with h>0 the tiled output
    differs from global attention, so the parity tests can tell them apart."""
    pr = small_problem(halo=1)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    a, b = O.tiles_forward(x, blob, pr), O.global_forward(x, blob, pr)
    assert not np.allclose(a, b, atol=1e-6)


def test_constant_and_ramp_inputs_residual():
    """O7 closed forms: constant field -> constant upsample; an affine ramp is
    reproduced exactly away from the clamped border."""
    cfg = get_config("C1")
    pr = O.Problem.from_config(cfg)
    up = O.residual_up(constant_input(cfg)[0], pr)
    assert np.array_equal(up, np.full_like(up, 1.25))
    x = ramp_input(cfg)[0]
    up = O.residual_up(x, pr)
    s = cfg.scale
    Y = (np.arange(cfg.H * s) + 0.5) / s - 0.5
    X = (np.arange(cfg.W * s) + 0.5) / s - 0.5
    want = 0.5 + 0.25 * Y[:, None] - 0.125 * X[None, :]
    inner = (slice(s, -s), slice(s, -s))
    np.testing.assert_allclose(up[0][inner], want[inner], rtol=0, atol=1e-12)


def test_golden_paper_sequence_lengths():
    """tests/golden/paper_sequence_lengths.txt: every sequence length the paper prints
    (P:150), reproduced by the oracle's count at the paper's printed precision."""
    import pathlib
    path = pathlib.Path(__file__).parent / "golden" / "paper_sequence_lengths.txt"
    rows = [ln.split() for ln in path.read_text().splitlines()
            if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 6
    for r in rows:
        h, w, c, p = (int(x) for x in r[:4])
        printed, unit = float(r[4]), float(r[5])
        exact = O.paper_sequence_length(h, w, c, p)
        digits = len(r[4].split(".")[1]) if "." in r[4] else 0
        # the paper mixes truncation (298.6M -> "298M", 1.19B -> "1.1B") and rounding
        # (4.199B -> "4.2B"): the exact count lies within one unit of the last printed digit
        scale = unit / 10 ** digits
        assert abs(exact - printed * unit) < scale, (r, exact)
        assert round(exact / scale) * scale == printed * unit or \
            int(exact // scale) * scale == printed * unit, (r, exact)


# ---------------------------------------------------------------- sampled-tile oracle
@pytest.mark.parametrize("res_hidden,dec_hidden", [(0, 0), (4, 0), (4, 3)])
@pytest.mark.parametrize("mode", [O.HALO_CLAMP, O.HALO_REPLICATE])
def test_sampled_tiles_equal_full_forward_restricted(mode, res_hidden, dec_hidden):
    """tiles_forward_sampled (which supplies every C3/C4/C5 expected value) is
    tiles_forward restricted to the tile's core output rectangle, bit for bit,
    for EVERY tile of a 3 x 3 problem (the core outputs of a tile are
    stitched into exactly its core rectangle; the residual is the same O7
    formula evaluated on that rectangle).  A wrong core slice, reshape or
    bilinear window in the sampled path fails here."""
    pr = small_problem(H=36, W=44, tiles_y=3, tiles_x=3, halo=2, halo_mode=mode, channel_map=(2, 0),
                       res_hidden=res_hidden, dec_hidden=dec_hidden)
    blob, cfg = blob_for(pr)
    x = input_for(cfg, batch=2)
    full, full_vit, _ = O.tiles_forward(x, blob, pr, return_parts=True)
    tiles = pr.tiles()
    covered = np.zeros(full.shape[1:], bool)
    for b in range(2):
        res = O.tiles_forward_sampled(x[b], blob, pr, range(len(tiles)))
        assert sorted(res) == list(range(len(tiles)))
        for t, (ys, xs, blk, vit) in res.items():
            tile = tiles[t]
            assert (ys.start, ys.stop) == (tile.core_y0 * pr.P, tile.core_y1 * pr.P)
            assert (xs.start, xs.stop) == (tile.core_x0 * pr.P, tile.core_x1 * pr.P)
            if res_hidden:   # O8 on a grown window: same sums, different array extents
                np.testing.assert_allclose(blk, full[b][:, ys, xs], rtol=0, atol=1e-12)
            else:
                assert np.array_equal(blk, full[b][:, ys, xs])
            assert np.array_equal(vit, full_vit[b][:, ys, xs])
            if b == 0:
                assert not covered[:, ys, xs].any()
                covered[:, ys, xs] = True
    assert covered.all()


# ---------------------------------------------------------------- canonical weight blob
def test_unpack_weights_marker_blob():
    """The oracle's blob walk against the layout include/orbit2.h documents
    (orbit2_prepare_weights comment), with closed-form offsets: value i at
    canonical offset i, so every named array must hold exactly the offsets
    the header assigns it.  W_e[D][V*p*p], b_e, e_s; per layer l at
    base_l = Din*D + 2D + l*(12D^2 + 13D): ln1_g, ln1_b, W_qkv[3D][D], b_qkv[3D],
    W_o[D][D], b_o, ln2_g, ln2_b, W_1[4D][D], b_1[4D], W_2[D][4D], b_2; then
    lnf_g, lnf_b, W_h[K P^2][D], b_h[K P^2]; total Din*D + 2D + L(12D^2+13D) +
    2D + D*K*P^2 + K*P^2."""
    D, L, Din, Nh = 8, 3, 12, 5
    total = Din * D + 2 * D + L * (12 * D * D + 13 * D) + 2 * D + D * Nh + Nh
    blob = np.arange(total, dtype=np.float64)
    Wt = O.unpack_weights(blob, D, L, Din, Nh)

    def rng(off, *shape):
        return off + np.arange(int(np.prod(shape)), dtype=np.float64).reshape(shape)

    assert np.array_equal(Wt["W_e"], rng(0, D, Din))
    assert Wt["W_e"][3, 7] == 3 * Din + 7          # row = output feature, column (v p + dy) p + dx
    assert np.array_equal(Wt["b_e"], rng(Din * D, D))
    assert np.array_equal(Wt["e_s"], rng(Din * D + D, D))
    for l in range(L):
        base = Din * D + 2 * D + l * (12 * D * D + 13 * D)
        Lw = Wt["layers"][l]
        want = {"ln1_g": rng(base, D), "ln1_b": rng(base + D, D),
                "W_qkv": rng(base + 2 * D, 3 * D, D), "b_qkv": rng(base + 2 * D + 3 * D * D, 3 * D),
                "W_o": rng(base + 5 * D + 3 * D * D, D, D), "b_o": rng(base + 5 * D + 4 * D * D, D),
                "ln2_g": rng(base + 6 * D + 4 * D * D, D), "ln2_b": rng(base + 7 * D + 4 * D * D, D),
                "W_1": rng(base + 8 * D + 4 * D * D, 4 * D, D), "b_1": rng(base + 8 * D + 8 * D * D, 4 * D),
                "W_2": rng(base + 12 * D + 8 * D * D, D, 4 * D), "b_2": rng(base + 12 * D + 12 * D * D, D)}
        assert sorted(Lw) == sorted(want)
        for k, v in want.items():
            assert np.array_equal(Lw[k], v), (l, k)
        # rows Q | K | V, head h = rows [h d, (h+1) d) of each: K row 0 of layer l
        assert Lw["W_qkv"][D, 0] == base + 2 * D + D * D
    tail = Din * D + 2 * D + L * (12 * D * D + 13 * D)
    assert np.array_equal(Wt["lnf_g"], rng(tail, D))
    assert np.array_equal(Wt["lnf_b"], rng(tail + D, D))
    assert np.array_equal(Wt["W_h"], rng(tail + 2 * D, Nh, D))
    assert np.array_equal(Wt["b_h"], rng(tail + 2 * D + Nh * D, Nh))
    with pytest.raises(ValueError):
        O.unpack_weights(np.zeros(total + 1), D, L, Din, Nh)


# ---------------------------------------------------------------- O8 residual convolutions (R31)
def test_conv3x3_matches_torch_conv2d():
    """O8's 3x3 convolution (zero padding) is torch.nn.functional.conv2d(padding=1) in fp64."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 11, 17))
    Wc = rng.standard_normal((5, 3, 3, 3))
    b = rng.standard_normal(5)
    want = F.conv2d(torch.from_numpy(x)[None], torch.from_numpy(Wc), torch.from_numpy(b), padding=1)[0].numpy()
    np.testing.assert_allclose(O.conv3x3(x, Wc, b), want, rtol=1e-12, atol=1e-12)
    # one-hot kernel = shift: output[o, y, x] = x[i, y + 1, x - 1] inside, 0 past the edge
    Wd = np.zeros((1, 3, 3, 3))
    Wd[0, 1, 2, 0] = 1.0
    got = O.conv3x3(x, Wd, np.zeros(1))[0]
    assert np.array_equal(got[:-1, 1:], x[1, 1:, :-1]) and not got[-1].any() and not got[:, 0].any()


def test_residual_conv_path_torch_model_and_init_contract():
    """The whole pass with the residual convolutional path (T = 1, h = 0) equals an
    untiled torch model (conv2d -> gelu -> conv2d on the interpolated field + identity
    skip); zero second convolution -> the path is exactly the bilinear upsample (the
    initialization contract: P:498 'high-resolution approximation' = the upsample)."""
    pr = small_problem(tiles_y=1, tiles_x=1, halo=0, res_hidden=4)
    blob, cfg = blob_for(pr)
    x = input_for(cfg, batch=2)
    Wt = pr.weights(blob)
    got = O.tiles_forward(x, blob, pr)
    import dataclasses
    n_conv = 2 * 9 * 4 * pr.K + 4 + pr.K
    base = torch_global_model(x, blob[:-n_conv], dataclasses.replace(pr, res_hidden=0))
    xt = torch.from_numpy(x.astype(np.float64))
    with torch.no_grad():
        up = F.interpolate(xt[:, list(pr.cmap())], scale_factor=pr.scale, mode="bilinear", align_corners=False)
        h = F.gelu(F.conv2d(up, torch.from_numpy(Wt["W_ra"]), torch.from_numpy(Wt["b_ra"]), padding=1))
        conv = F.conv2d(h, torch.from_numpy(Wt["W_rb"]), torch.from_numpy(Wt["b_rb"]), padding=1)
    np.testing.assert_allclose(got, base + conv.numpy(), rtol=1e-10, atol=1e-10)
    z = blob.copy()
    z[-(9 * 4 * pr.K + pr.K):] = 0.0          # W_rb, b_rb = 0
    out, vit, res = O.tiles_forward(x, z, pr, return_parts=True)
    up = np.stack([np.stack([O.upsample_bilinear(x[b][m], pr.scale) for m in pr.cmap()]) for b in range(2)])
    assert np.array_equal(res, up)


def test_residual_conv_locality():
    """I5 with the convolutions: perturbing input pixels outside a tile's padded
    rectangle leaves its core output unchanged (halo 1 patch = 2 px covers the
    conv + bilinear support of ceil(2/s) + 1 = 2 coarse px at s = 4)."""
    pr = small_problem(tiles_y=2, tiles_x=3, halo=1, res_hidden=4)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    t = pr.tiles()[4]
    a = O.tiles_forward_sampled(x[0], blob, pr, [4])[4]
    x2 = x.copy()
    mask = np.ones(x.shape[2:], bool)
    mask[max(0, t.pad_y0 * pr.patch):t.pad_y1 * pr.patch, max(0, t.pad_x0 * pr.patch):t.pad_x1 * pr.patch] = False
    x2[0][:, mask] += 5.0
    b2 = O.tiles_forward_sampled(x2[0], blob, pr, [4])[4]
    assert np.array_equal(a[2], b2[2])


# ---------------------------------------------------------------- O5b decoder convolutions (R32)
def test_decoder_convs_untiled_match_torch():
    """T = 1, h = 0: the decoder rectangle is the whole grid, so the tiled pass with
    decoder convolutions equals an untiled torch model (linear head, pixel_shuffle,
    conv2d -> gelu -> conv2d with zero padding at the field border), and the oracle's
    separate untiled global_forward too."""
    import dataclasses
    pr = small_problem(tiles_y=1, tiles_x=1, halo=0, dec_hidden=3)
    blob, cfg = blob_for(pr)
    x = input_for(cfg, batch=2)
    Wt = pr.weights(blob)
    n_dec = 2 * 9 * 3 * pr.K + 3 + pr.K
    base = dataclasses.replace(pr, dec_hidden=0)
    xt = torch.from_numpy(x.astype(np.float64))
    with torch.no_grad():
        vit = torch.from_numpy(torch_global_model(x, blob[:-n_dec], base)) - F.interpolate(
            xt[:, list(pr.cmap())], scale_factor=pr.scale, mode="bilinear", align_corners=False)
        h = F.gelu(F.conv2d(vit, torch.from_numpy(Wt["W_da"]), torch.from_numpy(Wt["b_da"]), padding=1))
        dec = F.conv2d(h, torch.from_numpy(Wt["W_db"]), torch.from_numpy(Wt["b_db"]), padding=1)
        up = F.interpolate(xt[:, list(pr.cmap())], scale_factor=pr.scale, mode="bilinear", align_corners=False)
    want = (dec + up).numpy()
    np.testing.assert_allclose(O.tiles_forward(x, blob, pr), want, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(O.global_forward(x, blob, pr), want, rtol=1e-10, atol=1e-10)


def test_decoder_convs_full_halo_equals_global_and_locality():
    """I6 with the decoder convolutions: a halo covering the grid gives every tile all
    tokens, so its ring outputs are the global ones and tiled == untiled; I5: a tile's
    output is unchanged by input pixels outside its padded rectangle."""
    pr = small_problem(halo=50, dec_hidden=3, res_hidden=2)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    np.testing.assert_allclose(O.tiles_forward(x, blob, pr), O.global_forward(x, blob, pr), rtol=1e-11, atol=1e-11)
    pr = small_problem(tiles_y=2, tiles_x=3, halo=1, dec_hidden=3)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    t = pr.tiles()[1]
    a = O.tiles_forward_sampled(x[0], blob, pr, [1])[1]
    x2 = x.copy()
    mask = np.ones(x.shape[2:], bool)
    mask[max(0, t.pad_y0 * pr.patch):t.pad_y1 * pr.patch, max(0, t.pad_x0 * pr.patch):t.pad_x1 * pr.patch] = False
    x2[0][:, mask] -= 3.0
    assert np.array_equal(a[3], O.tiles_forward_sampled(x2[0], blob, pr, [1])[1][3])


# ---------------------------------------------------------------- O3b variable aggregation (R33)
def test_variable_aggregation_matches_torch_multihead_attention():
    """O3b against torch.nn.functional.multi_head_attention_forward (fp64): one learned
    query per patch (identity query projection), keys / values = the V per-variable
    tokens t_v = W_t[v] a_v + e_var[v] with in-projections W_ak / W_av, output
    projection W_ao -- the library routine the paper's citation (ClimaX) uses."""
    pr = small_problem(var_agg=1, V=5, embed=16, heads=4)
    blob, cfg = blob_for(pr)
    Wt = pr.weights(blob)
    rng = np.random.default_rng(5)
    n, pp, D = 7, pr.patch ** 2, pr.embed
    a = rng.standard_normal((n, pr.V * pp))
    got = O.aggregate_variables(a, Wt, pr.heads, pr.patch)
    t = np.stack([a[:, v * pp:(v + 1) * pp] @ Wt["W_t"][v].T + Wt["e_var"][v] for v in range(pr.V)], axis=0)  # [V,n,D]
    q = np.broadcast_to(Wt["q_agg"], (1, n, D)).copy()
    in_w = np.concatenate([np.eye(D), Wt["W_ak"], Wt["W_av"]])
    in_b = np.concatenate([np.zeros(D), Wt["b_ak"], Wt["b_av"]])
    T = lambda z: torch.from_numpy(np.ascontiguousarray(z))
    want, _ = F.multi_head_attention_forward(T(q), T(t), T(t), D, pr.heads, T(in_w), T(in_b), None, None, False,
                                             0.0, T(Wt["W_ao"]), T(Wt["b_ao"]), training=False, need_weights=False)
    np.testing.assert_allclose(got, want[0].numpy(), rtol=1e-11, atol=1e-11)
    # identical variable tokens -> uniform weights: the result is the value path of one token
    a1 = np.tile(a[:, :pp], (1, pr.V))
    W1 = dict(Wt, W_t=np.repeat(Wt["W_t"][:1], pr.V, 0), e_var=np.repeat(Wt["e_var"][:1], pr.V, 0))
    one = (a1[:, :pp] @ W1["W_t"][0].T + W1["e_var"][0]) @ Wt["W_av"].T + Wt["b_av"]
    np.testing.assert_allclose(O.aggregate_variables(a1, W1, pr.heads, pr.patch), one @ Wt["W_ao"].T + Wt["b_ao"],
                               rtol=1e-12, atol=1e-12)


def test_variable_aggregation_permutation_and_tiling():
    """Permuting the input variables together with their tokenizer weights and
    variable embeddings leaves the pass unchanged (the aggregation is a set
    function of the variables); the sampled-tile path equals the full pass."""
    pr = small_problem(var_agg=1, V=4, tiles_y=2, tiles_x=2, halo=1)
    blob, cfg = blob_for(pr)
    x = input_for(cfg)
    out = O.tiles_forward(x, blob, pr)
    perm = [2, 0, 3, 1]
    Wt = pr.weights(blob)
    n_agg = pr.V * pr.embed * pr.patch ** 2 + pr.V * pr.embed + pr.embed + 3 * (pr.embed ** 2 + pr.embed)
    tail = blob[-n_agg:].copy()
    D, pp = pr.embed, pr.patch ** 2
    wt = tail[:pr.V * D * pp].reshape(pr.V, D, pp)[perm]
    ev = tail[pr.V * D * pp:pr.V * D * pp + pr.V * D].reshape(pr.V, D)[perm]
    tail2 = np.concatenate([wt.ravel(), ev.ravel(), tail[pr.V * D * pp + pr.V * D:]])
    blob2 = np.concatenate([blob[:-n_agg], tail2]).astype(blob.dtype)
    x2 = x[:, perm]
    pr2 = O.Problem(**{**pr.__dict__, "channel_map": tuple(perm.index(k) for k in range(pr.K))})
    np.testing.assert_allclose(O.tiles_forward(x2, blob2, pr2), out, rtol=1e-10, atol=1e-10)
    res = O.tiles_forward_sampled(x[0], blob, pr, [3])[3]
    assert np.array_equal(res[2], out[0][:, res[0], res[1]])
