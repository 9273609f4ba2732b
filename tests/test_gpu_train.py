"""GPU parity of the training step against the fp64 oracle
(oracle/train.py), through the C ABI (orbit2_train_* / orbit2_loss).

Tolerances: the loss within 1e-2 relative (bf16 ViT
branch, the north star's 2e-2 forward bar halved for a mean over pixels), the
gradient within 3e-2 of the oracle in relative Frobenius norm per weight tensor
(bf16 activations and operands are rounded at ~4 stages per block of the
backward, unit roundoff 2^-9 each; fp32 accumulation) and the whole gradient with
cosine similarity >= 0.999.
"""
import numpy as np
import pytest

from oracle import reslim_tiles as O
from oracle import train as T
from workloads import get_config, make_input, make_weights

pytestmark = pytest.mark.gpu

GRAD_TOL = 3e-2
LOSS_TOL = 1e-2


def _names(pr):
    D, din, Nh = pr.embed, pr.V * pr.patch ** 2, pr.K * pr.P ** 2
    F = 4 * D
    out = [("W_e", D * din), ("b_e", D), ("e_s", D)]
    for l in range(pr.depth):
        out += [(f"{l}.{n}", c) for n, c in (("ln1_g", D), ("ln1_b", D), ("W_qkv", 3 * D * D), ("b_qkv", 3 * D),
                                              ("W_o", D * D), ("b_o", D), ("ln2_g", D), ("ln2_b", D),
                                              ("W_1", F * D), ("b_1", F), ("W_2", D * F), ("b_2", D))]
    out += [("lnf_g", D), ("lnf_b", D), ("W_h", Nh * D), ("b_h", Nh)]
    return out


def _gpu_step(w, x, y, blob, lam, delta, geo=True):
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    cfg = o2.config_from(w, batch=x.shape[0], precision=o2.BF16)
    ctx = o2.Context(cfg)
    wd = torch.from_numpy(np.ascontiguousarray(blob, dtype=np.float32)).cuda()
    packed = ctx.prepare_weights(wd)
    ctx.train_bind()
    ctx.train_prepare(wd)
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    yd = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).cuda()
    loss, grad, out = ctx.train_step(packed, xd, yd, lam, delta, geo)
    torch.cuda.synchronize()
    return ctx, loss.cpu().numpy(), grad.cpu().numpy().astype(np.float64), out.cpu().numpy()


def _problem_and_data(name="toy", batch=2, seed=3, **kw):
    base = dict(H=24, W=32, V=3, K=2, scale=2, patch=2, tiles_y=2, tiles_x=2, halo=2, embed=128, depth=2, heads=2)
    base.update(kw)
    w = get_config("C1", **base)
    pr = O.Problem.from_config(w)
    blob = make_weights(w, seed=seed)
    x = make_input(w, batch=batch, seed=seed + 1)
    rng = np.random.default_rng(seed + 2)
    # truth = the bilinear residual plus structure, so (y - out) has the scale of real fields
    y = (O.tiles_forward(x, blob, pr) + 0.5 * rng.standard_normal((batch, pr.K, pr.scale * pr.H, pr.scale * pr.W)))
    return w, pr, blob, x, y.astype(np.float32)


def _check_grads(pr, got, ref):
    assert got.shape == ref.shape
    off = 0
    worst = (0.0, "")
    for name, n in _names(pr):
        g, r = got[off:off + n], ref[off:off + n]
        off += n
        den = np.linalg.norm(r)
        err = np.linalg.norm(g - r) / (den if den > 0 else 1.0)
        worst = max(worst, (err, name))
        assert err <= GRAD_TOL, (name, err)
    assert off == ref.size
    cos = float(got @ ref / (np.linalg.norm(got) * np.linalg.norm(ref)))
    assert cos >= 0.999, cos
    return worst, cos


@pytest.mark.parametrize("mode", [O.HALO_CLAMP, O.HALO_REPLICATE])
def test_train_step_matches_oracle(mode):
    """Loss and every weight tensor's gradient vs oracle/train.py (2x2 tiles, halo 2,
    ragged query / key blocks: 10x12 = 120-token and 10x10 padded tiles, B = 2)."""
    w, pr, blob, x, y = _problem_and_data(halo_mode=mode)
    lam, delta = 0.05, 0.02
    _, loss, grad, out = _gpu_step(w, x, y, blob, lam, delta)
    ref_loss, ref_grad = T.train_step_grads(x.astype(np.float64), y.astype(np.float64), blob.astype(np.float64),
                                            pr, lam, delta)
    assert abs(loss.mean() - ref_loss) <= LOSS_TOL * abs(ref_loss)
    worst, cos = _check_grads(pr, grad, ref_grad)
    print(f"worst tensor {worst[1]} rel {worst[0]:.3e}, cosine {cos:.6f}")


def test_train_step_multiblock_tiles_and_no_geo():
    """Tiles of 300+ tokens (three 128-key blocks, ragged tail), one tile row of 3,
    non-geographic weights (all ones), 1 block."""
    w, pr, blob, x, y = _problem_and_data(H=40, W=96, tiles_y=1, tiles_x=3, halo=1, depth=1, batch=1, seed=9)
    lam, delta = 0.1, 0.05
    _, loss, grad, _ = _gpu_step(w, x, y, blob, lam, delta, geo=False)
    ref_loss, ref_grad = T.train_step_grads(x.astype(np.float64), y.astype(np.float64), blob.astype(np.float64),
                                            pr, lam, delta, geo=False)
    assert abs(loss.mean() - ref_loss) <= LOSS_TOL * abs(ref_loss)
    _check_grads(pr, grad, ref_grad)


def test_loss_kernel_matches_oracle_elementwise():
    """orbit2_loss alone on a given field: per-sample loss and d loss / d out vs the
    oracle's T2 (fp32 kernel, double accumulation: 1e-5 relative)."""
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    w = get_config("C1", H=16, W=20, V=2, K=2, scale=3, patch=2, tiles_y=1, tiles_x=1, halo=0, embed=128, depth=0,
                   heads=2)
    cfg = o2.config_from(w, batch=2, precision=o2.BF16)
    ctx = o2.Context(cfg)
    ctx.train_bind()
    rng = np.random.default_rng(1)
    out = rng.standard_normal((2, 2, 48, 60)).astype(np.float32)
    out[:, :, 10:20, 10:20] = 0.3            # flat patch: Huber's quadratic branch
    y = rng.standard_normal(out.shape).astype(np.float32)
    od, yd = torch.from_numpy(out).cuda(), torch.from_numpy(y).cuda()
    loss = torch.empty(2, dtype=torch.float64, device="cuda")
    dout = torch.empty_like(od)
    lam, delta = 0.2, 0.1
    ctx.loss(od, yd, lam, delta, True, loss, dout)
    torch.cuda.synchronize()
    latw = T.lat_weights(48)
    for b in range(2):
        ref = T.bayesian_loss(out[b].astype(np.float64), y[b].astype(np.float64), latw, lam, delta)
        assert abs(loss[b].item() - ref) <= 1e-5 * abs(ref)
        g = T.bayesian_loss_grad(out[b].astype(np.float64), y[b].astype(np.float64), latw, lam, delta) / 2
        np.testing.assert_allclose(dout[b].cpu().numpy(), g, rtol=1e-4, atol=1e-6 * np.abs(g).max())


def test_train_step_c2_full_size_properties():
    """C2 at its bench shape (B = 4 to bound memory; every tile): the loss of sample 0
    and its d loss / d out against the oracle's T2 on the GPU's own output; the head
    bias gradient equals its closed form sum over core pixels of dout (the stitch read
    backwards + the bias column sums); the gradient is finite."""
    import torch
    w = get_config("C2")
    pr = O.Problem.from_config(w)
    B = 4
    blob = make_weights(w, seed=5)
    x = make_input(w, batch=B, seed=6)
    rng = np.random.default_rng(7)
    y = rng.standard_normal((B, w.K, w.scale * w.H, w.scale * w.W)).astype(np.float32)
    lam, delta = 1e-3, 1e-3
    ctx, loss, grad, out = _gpu_step(w, x, y, blob, lam, delta)
    latw = T.lat_weights(w.scale * w.H)
    ref0 = T.bayesian_loss(out[0].astype(np.float64), y[0].astype(np.float64), latw, lam, delta)
    assert abs(loss[0] - ref0) <= 1e-5 * abs(ref0)
    assert np.isfinite(grad).all()
    # b_h: sum over samples and core tokens of dout at the token's pixels
    dout = np.concatenate([T.bayesian_loss_grad(out[b].astype(np.float64), y[b].astype(np.float64), latw, lam,
                                                delta)[None] / B for b in range(B)])
    P, K = pr.P, pr.K
    Hp, Wp = pr.H // pr.patch, pr.W // pr.patch
    want_bh = dout.reshape(B, K, Hp, P, Wp, P).sum(axis=(0, 2, 4)).reshape(-1)   # [(k, al, be)]
    names = _names(pr)
    off = sum(n for _, n in names[:-1])
    got_bh = grad[off:off + K * P * P]
    # dG is rounded to bf16 before the column sums: 2^-9 relative per term
    np.testing.assert_allclose(got_bh, want_bh, rtol=5e-3, atol=5e-3 * np.abs(want_bh).max())


def test_train_step_wide_model_matches_oracle():
    """The C3 / C4 model width (D = 1024, 16 heads of 64: the LayerNorm backward's 8-float4
    rows, weight-gradient tiles of 256 columns over K = 1024) on a small grid, one block."""
    w, pr, blob, x, y = _problem_and_data(H=16, W=24, embed=1024, heads=16, depth=1, batch=1, seed=11)
    lam, delta = 0.05, 0.02
    _, loss, grad, _ = _gpu_step(w, x, y, blob, lam, delta)
    ref_loss, ref_grad = T.train_step_grads(x.astype(np.float64), y.astype(np.float64), blob.astype(np.float64),
                                            pr, lam, delta)
    assert abs(loss.mean() - ref_loss) <= LOSS_TOL * abs(ref_loss)
    _check_grads(pr, grad, ref_grad)


def test_train_step_cta_pair_gemms_match_oracle(monkeypatch):
    """D = 512 (8 heads of 64) on a 48 x 96 grid, B = 6 (~10.7k token rows): every GEMM of
    the step with K >= 512 and >= 74 256 x 256 tiles runs as a CTA pair (cta_group::2) --
    the forward QKV / MLP-up (bf16 out), the residual GEMMs (transposed fp32 epilogue), the
    MLP-down input gradient (EPI_DGELU) and the fp32 input gradients.  Loss and every
    gradient within tolerance of the oracle, with the pairs and with single-CTA tiles
    (ORBIT2_SINGLE_CTA_GEMM=1)."""
    w, pr, blob, x, y = _problem_and_data(H=48, W=96, embed=512, heads=8, depth=1, batch=6, seed=13)
    lam, delta = 0.05, 0.02
    ref_loss, ref_grad = T.train_step_grads(x.astype(np.float64), y.astype(np.float64), blob.astype(np.float64),
                                            pr, lam, delta)
    _, loss, grad, _ = _gpu_step(w, x, y, blob, lam, delta)
    assert abs(loss.mean() - ref_loss) <= LOSS_TOL * abs(ref_loss)
    _check_grads(pr, grad, ref_grad)
    monkeypatch.setenv("ORBIT2_SINGLE_CTA_GEMM", "1")
    _, loss1, grad1, _ = _gpu_step(w, x, y, blob, lam, delta)
    assert abs(loss1.mean() - ref_loss) <= LOSS_TOL * abs(ref_loss)
    _check_grads(pr, grad1, ref_grad)


def test_adamw_step_matches_oracle():
    """orbit2_adamw_step (R43) over three steps == oracle T5 (fp32 kernel vs fp64)."""
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    rng = np.random.default_rng(5)
    n = 10007
    w0 = rng.standard_normal(n)
    gs = [rng.standard_normal(n) for _ in range(3)]
    w = torch.from_numpy(w0.astype(np.float32)).cuda()
    m, v = torch.zeros_like(w), torch.zeros_like(w)
    wr, mr, vr = w0.astype(np.float32).astype(np.float64), np.zeros(n), np.zeros(n)
    for t, g in enumerate(gs, start=1):
        gd = torch.from_numpy(g.astype(np.float32)).cuda()
        o2.adamw_step(w, gd, m, v, t, 1e-2, 0.9, 0.95, 1e-8, 0.1)
        wr, mr, vr = T.adamw(wr, g.astype(np.float32), mr, vr, t, 1e-2, 0.9, 0.95, 1e-8, 0.1)
    torch.cuda.synchronize()
    np.testing.assert_allclose(w.cpu().numpy(), wr, rtol=0, atol=1e-5)
    np.testing.assert_allclose(m.cpu().numpy(), mr, rtol=0, atol=1e-5)
