"""GPU parity of the adaptive spatial compression against
oracle/compress.py, through the C ABI (orbit2_compress_*).

The edge map and the leaf list are integer / boolean results: bit-exact (the Canny
arithmetic is float32 in the same operation order on both sides, R37).  Tokens and the
decompressed field are fp32 sums of products: 1e-5 of the field's scale.
"""
import numpy as np
import pytest

from oracle import compress as K
from workloads import get_config, make_input

pytestmark = pytest.mark.gpu


def _fields(B, H, W, seed):
    """ERA5-shaped synthetic fields (workloads.make_input channel 0 of C2, cropped / edge
    padded) plus a step and a diagonal step: smooth regions and sharp fronts."""
    w = get_config("C2")
    x = make_input(w, batch=B, seed=seed)[:, 0].astype(np.float32)     # [B, 180, 360]
    x = np.pad(x, ((0, 0), (0, max(0, H - x.shape[1])), (0, max(0, W - x.shape[2]))), mode="edge")[:, :H, :W]
    yy, xx = np.mgrid[0:H, 0:W]
    if B > 1:
        x[1] = np.where(xx >= W // 3, 1.0, 0.0) + 0.1 * x[1] / (np.abs(x[1]).max() + 1e-6)
    if B > 2:
        x[2] = np.where(xx - yy >= 7, 2.0, -1.0).astype(np.float32)
    return np.ascontiguousarray(x, np.float32)


def _run(B, H, W, mn, mx, thr, C=3, D=16, seed=0, sigma=1.0):
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    img = _fields(B, H, W, seed)
    comp = o2.Compressor(batch=B, H=H, W=W, C=C, min_side=mn, max_side=mx, embed=D, threshold=thr, sigma=sigma)
    patches, offsets, n, edges = comp.partition(torch.from_numpy(img).cuda(), edges=True)
    torch.cuda.synchronize()
    return comp, img, patches, offsets.cpu().numpy(), n, edges.cpu().numpy().astype(bool)


@pytest.mark.parametrize("shape,mn,mx,thr,sigma", [((64, 96), 2, 16, 0.05, 1.0), ((48, 48), 4, 16, 0.0, 1.0),
                                                 ((96, 160), 2, 32, 0.1, 2.0)])
def test_partition_bit_exact(shape, mn, mx, thr, sigma):
    """Edge maps and leaf lists (order, offsets) equal the oracle's exactly, per image."""
    H, W = shape
    B = 3
    comp, img, patches, offsets, n, edges = _run(B, H, W, mn, mx, thr, sigma=sigma)
    p = patches.cpu().numpy()
    assert offsets[0] == 0 and offsets[B] == n
    for b in range(B):
        e_ref = K.canny(img[b], sigma)
        assert np.array_equal(edges[b], e_ref), (b, int((edges[b] != e_ref).sum()))
        ref = K.quadtree(e_ref, mn, mx, thr)
        got = [tuple(int(v) for v in r[1:]) for r in p[offsets[b]:offsets[b + 1]]]
        assert (p[offsets[b]:offsets[b + 1], 0] == b).all()
        assert got == ref


def test_tokenize_and_detokenize_match_oracle():
    import torch
    B, H, W, C, mn, mx, D = 2, 64, 96, 3, 2, 16, 24
    comp, img, patches, offsets, n, edges = _run(B, H, W, mn, mx, 0.05, C=C, D=D, seed=3)
    rng = np.random.default_rng(4)
    feat = rng.standard_normal((B, C, H, W)).astype(np.float32)
    levels = int(np.log2(mx // mn)) + 1
    Wt, bt, E = (rng.standard_normal((D, C * mn * mn)).astype(np.float32), rng.standard_normal(D).astype(np.float32),
                 rng.standard_normal((levels, D)).astype(np.float32))
    Wd, bd = rng.standard_normal((C * mn * mn, D)).astype(np.float32), rng.standard_normal(C * mn * mn).astype(np.float32)
    Ws, bs = (0.2 * rng.standard_normal((C, C, 3, 3))).astype(np.float32), rng.standard_normal(C).astype(np.float32)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tok = comp.tokenize(cu(feat), patches, n, cu(Wt), cu(bt), cu(E))
    out = comp.detokenize(tok, patches, n, cu(Wd), cu(bd), cu(Ws), cu(bs))
    torch.cuda.synchronize()
    tok, out = tok.cpu().numpy(), out.cpu().numpy()
    p = patches.cpu().numpy()
    for b in range(B):
        leaves = [tuple(int(v) for v in r[1:]) for r in p[offsets[b]:offsets[b + 1]]]
        ref_t = K.tokenize(feat[b].astype(np.float64), leaves, mn, Wt, bt, E)
        np.testing.assert_allclose(tok[offsets[b]:offsets[b + 1]], ref_t, rtol=0, atol=1e-5 * np.abs(ref_t).max())
        # decompress the oracle's tokens of the GPU's own tokens (isolates K4)
        ref_o = K.detokenize(tok[offsets[b]:offsets[b + 1]].astype(np.float64), leaves, mn, C, H, W, Wd, bd, Ws, bs)
        np.testing.assert_allclose(out[b], ref_o, rtol=0, atol=1e-5 * np.abs(ref_o).max())


def test_partition_full_c2_field_batch():
    """The C2 coarse field size (180 x 360, edge padded to 192 x 368 for max_side 16), B = 8:
    the leaf lists of images 0 and 7 equal the oracle's; every image's leaves tile its field;
    the compression ratio is > 1 on these smooth fields."""
    B, H, W = 8, 192, 368
    comp, img, patches, offsets, n, edges = _run(B, H, W, 2, 16, 0.05, seed=5)
    p = patches.cpu().numpy()
    for b in (0, B - 1):
        ref = K.quadtree(K.canny(img[b]), 2, 16, 0.05)
        got = [tuple(int(v) for v in r[1:]) for r in p[offsets[b]:offsets[b + 1]]]
        assert got == ref
    for b in range(B):
        cover = np.zeros((H, W), np.int32)
        for _, r, c, s in p[offsets[b]:offsets[b + 1]]:
            cover[r:r + s, c:c + s] += 1
        assert (cover == 1).all()
    assert n < B * (H // 2) * (W // 2)


def _cf_setup(B=2, depth=2, embed=256, heads=4, seed=8):
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    from oracle import reslim_tiles as O
    from workloads import make_weights
    w = get_config("C2", batch=B, H=48, W=80, tiles_y=1, tiles_x=1, halo=0, depth=depth, embed=embed, heads=heads)
    pr = O.Problem.from_config(w)
    x = make_input(w, batch=B, seed=seed)
    blob = make_weights(w, seed=seed)
    ctx = o2.Context(o2.config_from(w, precision=o2.BF16))
    packed = ctx.prepare_weights(torch.from_numpy(blob).cuda())
    return w, pr, x, blob, ctx, packed


def test_compressed_forward_matches_oracle_on_its_leaves():
    """R41 end to end: the GPU forward on compressed tokens (24 x 40 patch grid, max_side 8)
    against oracle K5 given the same leaves (the leaves are an integer result of the GPU's bf16 embedding; the partition
    kernels are pinned bit-exact above), bf16 tolerance 2e-2 of the field per variable."""
    import torch
    from oracle import reslim_tiles as O
    from tests.gpu_helpers import rel_err
    w, pr, x, blob, ctx, packed = _cf_setup()
    levels = 4
    E = (0.1 * np.random.default_rng(1).standard_normal((levels, w.embed))).astype(np.float32)
    out, leaves, n = ctx.compressed_forward(packed, torch.from_numpy(x).cuda(), torch.from_numpy(E).cuda(),
                                            max_side=8, threshold=0.12, sigma=1.0)
    torch.cuda.synchronize()
    out, lv = out.cpu().numpy(), leaves.cpu().numpy()
    Hp, Wp = w.H // w.patch, w.W // w.patch
    assert n < w.batch * Hp * Wp                       # something was compressed
    Wt = pr.weights(blob)
    for b in range(w.batch):
        lb = [tuple(int(v) for v in r[1:]) for r in lv if r[0] == b]
        cover = np.zeros((Hp, Wp), np.int32)
        for u, v, s in lb:
            cover[u:u + s, v:v + s] += 1
        assert (cover == 1).all()
        ref = K.compressed_forward(x[b].astype(np.float64), pr, Wt, E.astype(np.float64), lb)
        assert rel_err(out[b], ref) <= 2e-2, rel_err(out[b], ref)


def test_compressed_forward_full_refinement_equals_uncompressed():
    """Threshold -1 (every density > -1: every leaf one patch) and E_scale[0] = 0: the
    compressed forward equals the uncompressed one-tile forward (both on the GPU, bf16;
    the only differences are rounding order: 1e-2 of the field)."""
    import torch
    from tests.gpu_helpers import rel_err
    w, pr, x, blob, ctx, packed = _cf_setup(seed=9)
    E = np.zeros((4, w.embed), np.float32)
    xd = torch.from_numpy(x).cuda()
    out_c, leaves, n = ctx.compressed_forward(packed, xd, torch.from_numpy(E).cuda(), max_side=8, threshold=-1.0)
    out_u = ctx.forward(packed, xd)
    torch.cuda.synchronize()
    assert n == w.batch * (w.H // w.patch) * (w.W // w.patch)
    assert rel_err(out_c.cpu().numpy(), out_u.cpu().numpy()) <= 1e-2


def test_compressed_forward_inside_tiles_matches_oracle():
    """R42: compressed tokens inside TILES tiles (2 x 3 tiles, halo 2, ragged 12 x 13-patch
    rectangles) against oracle K6 given the GPU's leaves per (sample, tile); and full
    refinement == the uncompressed TILES forward (GPU, bf16 rounding order only)."""
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    from oracle import reslim_tiles as O
    from tests.gpu_helpers import rel_err
    from workloads import make_weights
    B = 2
    w = get_config("C2", batch=B, H=48, W=80, tiles_y=2, tiles_x=3, halo=2, depth=2)
    pr = O.Problem.from_config(w)
    x = make_input(w, batch=B, seed=12)
    blob = make_weights(w, seed=12)
    ctx = o2.Context(o2.config_from(w, precision=o2.BF16))
    packed = ctx.prepare_weights(torch.from_numpy(blob).cuda())
    E = (0.1 * np.random.default_rng(2).standard_normal((3, w.embed))).astype(np.float32)
    xd, Ed = torch.from_numpy(x).cuda(), torch.from_numpy(E).cuda()
    out, leaves, n = ctx.compressed_forward(packed, xd, Ed, max_side=4, threshold=0.15)
    torch.cuda.synchronize()
    out, lv = out.cpu().numpy(), leaves.cpu().numpy()
    T = w.tiles_y * w.tiles_x
    assert n < B * ctx.info.local_tokens
    Wt = pr.weights(blob)
    for b in range(B):
        by_tile = [[tuple(int(v) for v in r[1:]) for r in lv if r[0] == b * T + t] for t in range(T)]
        ref, _ = K.tiles_compressed_forward(x[b].astype(np.float64), pr, Wt, E.astype(np.float64), by_tile)
        assert rel_err(out[b], ref) <= 2e-2, rel_err(out[b], ref)
    E0 = torch.zeros_like(Ed)
    out_c, _, n = ctx.compressed_forward(packed, xd, E0, max_side=4, threshold=-1.0)
    out_u = ctx.forward(packed, xd)
    torch.cuda.synchronize()
    assert n == B * ctx.info.local_tokens
    assert rel_err(out_c.cpu().numpy(), out_u.cpu().numpy()) <= 1e-2
