"""Pins of the adaptive-compression oracle (oracle/compress.py), CPU only.

K1 (Canny) is pinned by scipy.ndimage (gaussian_filter, sobel, label -- library routines the
oracle does not call) and by analytic edge locations of step images; K2 (quad-tree) by the
SPEC's worked examples and by invariants checked on 2000 random maps that do not
use the recursion (exact coverage by rasterization, the split rule read off every leaf and its
parent, threshold monotonicity); K3 / K4 reduce to conventional patch embedding /
unpatchify + conv2d (torch) on a uniform layout.
"""
import numpy as np
import pytest
import scipy.ndimage as ndi
import torch
import torch.nn.functional as F

from oracle import compress as K


@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


# ---------------------------------------------------------------- K1
@pytest.mark.parametrize("sigma", [1.0, 2.0])
def test_blur_matches_scipy_gaussian_filter(sigma):
    """R37: radius ceil(3 sigma), normalised taps, edge replication == scipy gaussian_filter
    (mode='nearest', truncate=3) to float32 rounding."""
    img = np.random.default_rng(0).standard_normal((23, 31)).astype(np.float32)
    want = ndi.gaussian_filter(img.astype(np.float64), sigma, mode="nearest", truncate=3.0)
    np.testing.assert_allclose(K.blur(img, sigma), want, rtol=0, atol=2e-6)


def test_sobel_matches_scipy():
    b = np.random.default_rng(1).standard_normal((17, 19)).astype(np.float32)
    gx, gy = K.sobel(b)
    np.testing.assert_allclose(gx, ndi.sobel(b.astype(np.float64), axis=1, mode="nearest"), atol=1e-5)
    np.testing.assert_allclose(gy, ndi.sobel(b.astype(np.float64), axis=0, mode="nearest"), atol=1e-5)


def test_hysteresis_matches_scipy_label():
    """Edges = the 8-connected components of {m >= low} that hold a pixel >= high."""
    rng = np.random.default_rng(2)
    m = rng.random((40, 50)).astype(np.float32) * (rng.random((40, 50)) < 0.45)
    low, high = np.float32(0.3), np.float32(0.8)
    lab, n = ndi.label(m >= low, structure=np.ones((3, 3)))
    keep = set(np.unique(lab[m >= high])) - {0}
    want = np.isin(lab, list(keep))
    assert np.array_equal(K.hysteresis(m, low, high), want)


def test_constant_image_has_no_edges():
    assert not K.canny(np.full((20, 30), 3.5, np.float32)).any()


@pytest.mark.parametrize("orient", ["vertical", "horizontal", "diagonal"])
def test_step_edges_are_located_at_the_step(orient):
    """a step image gives edge pixels within 1 pixel of the step, one per row
    (vertical), per column (horizontal), along the diagonal (diagonal step: direction bins
    2 / 3), and nowhere else."""
    H, W = 32, 40
    yy, xx = np.mgrid[0:H, 0:W]
    if orient == "vertical":
        img, dist = (xx >= 17).astype(np.float32), np.abs(xx - 16.5)
    elif orient == "horizontal":
        img, dist = (yy >= 11).astype(np.float32), np.abs(yy - 10.5)
    else:
        img, dist = (xx - yy >= 5).astype(np.float32), np.abs(xx - yy - 4.5) / np.sqrt(2)
    e = K.canny(img)
    assert e.any()
    assert (dist[e] <= 1.5).all()
    if orient == "vertical":
        assert e.any(axis=1).all()
    if orient == "horizontal":
        assert e.any(axis=0).all()


def test_canny_rejects_degenerate_input():
    with pytest.raises(ValueError):
        K.canny(np.zeros((2, 9), np.float32))


# ---------------------------------------------------------------- K2
def test_quadtree_spec_examples():
    """all-false -> one max_side patch per max cell; all-true -> every patch
    min_side; one edge pixel at the corner, threshold 0, min 2, max 16, 16 x 16 -> the chain
    1 -> 4 -> 7 -> 10 patches."""
    e = np.zeros((32, 48), bool)
    p = K.quadtree(e, 2, 16, 0.05)
    assert p == [(r, c, 16) for r in range(0, 32, 16) for c in range(0, 48, 16)]
    p = K.quadtree(~e, 2, 16, 0.05)
    assert len(p) == 16 * 24 and all(s == 2 for _, _, s in p)
    e = np.zeros((16, 16), bool)
    e[0, 0] = True
    p = K.quadtree(e, 2, 16, 0.0)
    assert len(p) == 10
    assert sorted(s for _, _, s in p) == [2] * 4 + [4] * 3 + [8] * 3


def _rasterize(patches, H, W):
    cover = np.zeros((H, W), np.int32)
    for r, c, s in patches:
        cover[r:r + s, c:c + s] += 1
    return cover


def test_quadtree_invariants_random_maps():
    """2000 random 8x8 / 16x32 maps (min 2, max 8 / 16): exact coverage; row-major order;
    sides power-of-two multiples of min; a leaf larger than min has density <= thr; every leaf
    smaller than max has a parent square of density > thr; lowering the threshold never
    decreases the count."""
    rng = np.random.default_rng(3)
    for t in range(2000):
        H, W, mx = (8, 8, 8) if t % 2 == 0 else (16, 32, 16)
        e = rng.random((H, W)) < rng.random()
        thr = float(np.float32(rng.choice([0.0, 0.05, 0.1, 0.25, 0.5])))
        p = K.quadtree(e, 2, mx, thr)
        assert (_rasterize(p, H, W) == 1).all()
        assert p == sorted(p)
        for r, c, s in p:
            assert s in {2 ** k for k in range(1, 5)} and s <= mx and r % s == 0 and c % s == 0
            dens = e[r:r + s, c:c + s].mean()
            if s > 2:
                assert dens <= thr
            if s < mx:
                pr, pc = r - r % (2 * s), c - c % (2 * s)
                assert e[pr:pr + 2 * s, pc:pc + 2 * s].mean() > thr
        if thr > 0:
            assert len(K.quadtree(e, 2, mx, 0.0)) >= len(p)


def test_compression_ratio_closed_forms():
    e = np.zeros((16, 16), bool)
    assert K.compression_ratio(K.quadtree(e, 4, 16, 0.05), 16, 16, 4) == 16.0
    assert K.compression_ratio(K.quadtree(~e, 4, 16, 0.05), 16, 16, 4) == 1.0
    with pytest.raises(ValueError):
        K.quadtree(e, 4, 12, 0.05)


# ---------------------------------------------------------------- K3 / K4
def _weights(C, m, D, levels, seed=4):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((D, C * m * m)), rng.standard_normal(D), rng.standard_normal((levels, D)),
            rng.standard_normal((C * m * m, D)), rng.standard_normal(C * m * m),
            rng.standard_normal((C, C, 3, 3)), rng.standard_normal(C))


def test_tokenize_uniform_layout_is_patch_embedding():
    """a uniform min_side layout == conventional ViT patch embedding (conv2d, stride m)
    plus the level-0 scale embedding, tokens row-major."""
    C, H, W, m, D = 3, 12, 16, 2, 5
    feat = np.random.default_rng(5).standard_normal((C, H, W))
    Wt, bt, E, *_ = _weights(C, m, D, 3)
    p = K.quadtree(np.ones((H, W), bool), m, 4, 0.05)
    tok = K.tokenize(feat, p, m, Wt, bt, E)
    want = F.conv2d(torch.from_numpy(feat)[None], torch.from_numpy(Wt).reshape(D, C, m, m),
                    torch.from_numpy(bt), stride=m)[0].reshape(D, -1).T.numpy() + E[0]
    np.testing.assert_allclose(tok, want, rtol=1e-12, atol=1e-12)


def test_tokenize_pools_and_levels():
    """A constant field: every token of one level is the same vector; levels differ by the
    scale embedding difference."""
    C, m, D = 2, 2, 4
    feat = np.full((C, 16, 16), 0.7)
    Wt, bt, E, *_ = _weights(C, m, D, 3)
    e = np.zeros((16, 16), bool)
    e[0:4, 0:4] = True
    p = K.quadtree(e, 2, 8, 0.1)
    tok = K.tokenize(feat, p, m, Wt, bt, E)
    by = {}
    for t, (_, _, s) in zip(tok, p):
        by.setdefault(s, []).append(t)
    assert len(by) >= 2
    for s, ts in by.items():
        np.testing.assert_allclose(np.array(ts), np.repeat(ts[:1], len(ts), 0), atol=1e-12)
    s0, s1 = sorted(by)[:2]
    np.testing.assert_allclose(by[s1][0] - by[s0][0], E[int(np.log2(s1 // m))] - E[int(np.log2(s0 // m))],
                               atol=1e-12)


def test_detokenize_uniform_layout_is_unpatchify_plus_conv():
    """a uniform layout == linear projection, unpatchify (pixel placement (c, i, j)),
    then the same-padded 3x3 convolution (torch conv2d)."""
    C, H, W, m, D = 2, 8, 12, 2, 6
    *_, Wd, bd, Ws, bs = _weights(C, m, D, 2)
    p = K.quadtree(np.ones((H, W), bool), m, 4, 0.05)
    tok = np.random.default_rng(6).standard_normal((len(p), D))
    got = K.detokenize(tok, p, m, C, H, W, Wd, bd, Ws, bs)
    proj = tok @ Wd.T + bd                                   # [n, C m m]
    img = torch.from_numpy(proj).reshape(H // m, W // m, C, m, m).permute(2, 0, 3, 1, 4).reshape(C, H, W)
    want = F.conv2d(img[None], torch.from_numpy(Ws), torch.from_numpy(bs), padding=1)[0].numpy()
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_detokenize_single_patch_is_nearest_broadcast():
    """One leaf covering the field: before smoothing every (s/m) x (s/m) block holds one
    projected value (identity smoothing kernel)."""
    C, m, D, s = 1, 2, 3, 8
    *_, Wd, bd, _, _ = _weights(C, m, D, 1)
    Ws = np.zeros((C, C, 3, 3))
    Ws[0, 0, 1, 1] = 1.0
    tok = np.random.default_rng(7).standard_normal((1, D))
    got = K.detokenize(tok, [(0, 0, s)], m, C, s, s, Wd, bd, Ws, np.zeros(C))
    proj = (Wd @ tok[0] + bd).reshape(C, m, m)
    np.testing.assert_allclose(got[0], np.kron(proj[0], np.ones((s // m, s // m))), atol=1e-12)


# ---------------------------------------------------------------- K5
def _k5_problem(**kw):
    from oracle import reslim_tiles as O
    base = dict(H=16, W=24, V=2, K=2, scale=2, patch=2, tiles_y=1, tiles_x=1, halo=0, embed=16, depth=2, heads=2)
    base.update(kw)
    return O.Problem(**base)


def _k5_data(pr, seed=3):
    from workloads import get_config, make_input, make_weights
    cfg = get_config("C1", H=pr.H, W=pr.W, V=pr.V, K=pr.K, scale=pr.scale, patch=pr.patch, tiles_y=1, tiles_x=1,
                     halo=0, embed=pr.embed, depth=pr.depth, heads=pr.heads)
    return make_input(cfg, batch=1, seed=seed)[0].astype(np.float64), make_weights(cfg, seed=seed).astype(np.float64)


def test_compressed_forward_full_refinement_is_the_uncompressed_forward():
    """R41: with every leaf one patch (threshold -1: every density > -1 splits) and a zero
    level-0 scale embedding the compressed forward IS the T = 1 TILES forward."""
    from oracle import reslim_tiles as O
    pr = _k5_problem()
    x, blob = _k5_data(pr)
    Wt = pr.weights(blob)
    Hp, Wp = pr.H // pr.patch, pr.W // pr.patch
    tile = O.plan_tiles(Hp, Wp, 1, 1, 0)[0]
    z0 = O.embed_tile(O.gather_tile(x, tile, pr.patch), tile, pr.patch, Wt, pr.heads)
    leaves = K.partition_tokens(z0, Hp, Wp, 4, -1.0)
    assert leaves == [(u, w, 1) for u in range(Hp) for w in range(Wp)]
    E = np.zeros((3, pr.embed))
    np.testing.assert_allclose(K.compressed_forward(x, pr, Wt, E, leaves), O.tiles_forward(x[None], blob, pr)[0],
                               rtol=1e-12, atol=1e-12)


def test_compressed_forward_coarse_leaves_decompress_piecewise():
    """One leaf per max cell (threshold above every density): every patch of a leaf holds the
    same head output (decompression is a nearest broadcast), so out - residual repeats the
    same P x P pattern over the leaf's patches; the leaf clipped at the grid edge averages
    only real patches (grid 8 x 12 patches, max_side 8: padded to 8 x 16)."""
    from oracle import reslim_tiles as O
    pr = _k5_problem()
    x, blob = _k5_data(pr, seed=5)
    Wt = pr.weights(blob)
    Hp, Wp = pr.H // pr.patch, pr.W // pr.patch
    tile = O.plan_tiles(Hp, Wp, 1, 1, 0)[0]
    z0 = O.embed_tile(O.gather_tile(x, tile, pr.patch), tile, pr.patch, Wt, pr.heads)
    leaves = K.partition_tokens(z0, Hp, Wp, 8, 2.0)
    assert leaves == [(0, 0, 8), (0, 8, 8)]
    E = np.random.default_rng(0).standard_normal((4, pr.embed))
    out = K.compressed_forward(x, pr, Wt, E, leaves) - O.residual_up(x, pr)
    P = pr.P
    for (u, w, s) in leaves:
        nu, nw = min(u + s, Hp) - u, min(w + s, Wp) - w
        blk = out[:, u * P:(u + nu) * P, w * P:(w + nw) * P].reshape(pr.K, nu, P, nw, P)
        np.testing.assert_allclose(blk, np.broadcast_to(blk[:, :1, :, :1, :], blk.shape), atol=1e-12)


# ---------------------------------------------------------------- K6
def test_tiles_compressed_forward_reductions():
    """R42: (a) one tile, halo 0 == K5; (b) full refinement with a zero level-0 scale
    embedding == the uncompressed TILES forward (2 x 2 tiles, halo 1: every tile's tokens
    are its padded patches, the halo discarded after the blocks)."""
    from oracle import reslim_tiles as O
    pr1 = _k5_problem()
    x, blob = _k5_data(pr1, seed=7)
    Wt = pr1.weights(blob)
    E = np.random.default_rng(2).standard_normal((4, pr1.embed))
    out6, lv6 = K.tiles_compressed_forward(x, pr1, Wt, E, max_side=8, threshold=0.05)
    np.testing.assert_allclose(out6, K.compressed_forward(x, pr1, Wt, E, lv6[0]), rtol=1e-12, atol=1e-12)
    pr = _k5_problem(tiles_y=2, tiles_x=2, halo=1)
    out, lv = K.tiles_compressed_forward(x, pr, Wt, np.zeros((4, pr.embed)), max_side=4, threshold=-1.0)
    assert all(all(s == 1 for _, _, s in l) for l in lv)
    np.testing.assert_allclose(out, O.tiles_forward(x[None], blob, pr)[0], rtol=1e-12, atol=1e-12)


def test_tiles_compressed_leaves_cover_each_padded_rectangle():
    pr = _k5_problem(tiles_y=2, tiles_x=3, halo=2)
    x, blob = _k5_data(pr, seed=9)
    _, lv = K.tiles_compressed_forward(x, pr, pr.weights(blob), np.zeros((4, pr.embed)), max_side=4, threshold=0.2)
    for t, l in zip(pr.tiles(), lv):
        cover = np.zeros((t.pad_h, t.pad_w), np.int32)
        for u, w, s in l:
            cover[u:u + s, w:w + s] += 1
        assert (cover == 1).all()
