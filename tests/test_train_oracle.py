"""Pins of the training-step oracle (oracle/train.py), CPU only.

T1/T2 are pinned by closed forms and the SPEC's 3x3 worked example;
T3 (the backward) by brute force -- central finite differences of the loss,
which is computed by the already-pinned forward oracle -- and by torch autograd
of an untiled model assembled from torch library modules (full halo => tiled ==
global, invariant I6).  A dropped term, a wrong sign, a transposed operand or a
missing halo/core restriction anywhere in the backward fails one of them.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import reslim_tiles as O
from oracle import train as T
from workloads import get_config, make_input, make_weights


@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def problem(**kw):
    base = dict(H=12, W=16, V=2, K=2, scale=2, patch=2, tiles_y=2, tiles_x=2, halo=1,
                embed=8, depth=2, heads=2)
    base.update(kw)
    return O.Problem(**base)


def data_for(pr, batch=2, seed=3):
    cfg = get_config("C1", H=pr.H, W=pr.W, V=pr.V, K=pr.K, scale=pr.scale, patch=pr.patch,
                     tiles_y=pr.tiles_y, tiles_x=pr.tiles_x, halo=pr.halo, embed=pr.embed,
                     depth=pr.depth, heads=pr.heads, halo_mode=pr.halo_mode)
    blob = make_weights(cfg, seed=seed).astype(np.float64)
    x = make_input(cfg, batch=batch, seed=seed + 1).astype(np.float64)
    rng = np.random.default_rng(seed + 2)
    y = rng.standard_normal((batch, pr.K, pr.scale * pr.H, pr.scale * pr.W))
    return x, y, blob


# ---------------------------------------------------------------- T1
def test_lat_weights_closed_forms():
    """R35: mean 1; symmetric about the equator; equator > pole; sH = 2 -> lat +-45 -> [1, 1];
    sH = 4 -> lat 67.5, 22.5, ... -> cos ratio."""
    for sH in (2, 3, 7, 128, 721):
        w = T.lat_weights(sH)
        assert abs(w.mean() - 1.0) < 1e-12
        np.testing.assert_allclose(w, w[::-1], rtol=0, atol=1e-13)
        assert (w > 0).all()
    np.testing.assert_allclose(T.lat_weights(2), [1.0, 1.0], atol=1e-15)
    c1, c2 = math.cos(math.radians(67.5)), math.cos(math.radians(22.5))
    np.testing.assert_allclose(T.lat_weights(4), np.array([c1, c2, c2, c1]) / ((c1 + c2) / 2), rtol=1e-14)
    w = T.lat_weights(9)
    assert w[4] == w.max() and w[0] == w.min()
    assert np.array_equal(T.lat_weights(5, geo=False), np.ones(5))


# ---------------------------------------------------------------- T2
def test_spec_3x3_worked_example():
    """1x3x3 field [[0,0,0],[0,1,0],[0,0,0]] vs zero truth, all-ones weights,
    lambda = 1, delta -> 0: term1 = 1/9; term2 counts every ordered neighbour pair
    with |x_i - x_j| = 1: the centre's 4 axial + 4 diagonal neighbours (4 + 4/sqrt2)
    and the same pairs seen from the 8 border pixels -> (8 + 4 sqrt2) / 9."""
    pred = np.zeros((1, 3, 3))
    pred[0, 1, 1] = 1.0
    ones = np.ones(3)
    assert abs(T.bayesian_loss(pred, np.zeros_like(pred), ones, 0.0, 1e-12) - 1.0 / 9.0) < 1e-15
    got = T.bayesian_loss(pred, np.zeros_like(pred), ones, 1.0, 1e-12)
    assert abs(got - (1.0 + 8.0 + 4.0 * math.sqrt(2.0)) / 9.0) < 1e-11


def test_loss_trivial_cases_and_neighbour_counts():
    """pred = truth constant -> 0 (both terms); a single ramp along X has axial
    differences 1 and diagonal differences 1 -> closed form for the TV term."""
    c = np.full((2, 5, 6), 3.25)
    assert T.bayesian_loss(c, c, T.lat_weights(5), 0.7, 1e-3) == 0.0
    K, Hh, Ww = 1, 4, 5
    ramp = np.tile(np.arange(Ww, dtype=np.float64), (K, Hh, 1))
    # ordered pairs with |dx| = 1: horizontal 2*Hh*(Ww-1) (b=1); diagonal 4*(Hh-1)*(Ww-1) (b=1/sqrt2);
    # vertical pairs have difference 0.  delta -> 0: h = |r| = 1
    want = (2 * Hh * (Ww - 1) + 4 * (Hh - 1) * (Ww - 1) / math.sqrt(2)) / (K * Hh * Ww)
    got = T.bayesian_loss(ramp, ramp, np.ones(Hh), 1.0, 1e-12)
    assert abs(got - want) < 1e-10


def test_huber_branches():
    """h is C1 at |r| = delta, -> |r| as delta -> 0, quadratic r^2/(2 delta) inside."""
    d = 0.1
    r = np.array([-0.3, -d, -0.05, 0.0, 0.05, d, 0.3])
    np.testing.assert_allclose(T.huber(r, d), [0.25, 0.05, 0.0125, 0.0, 0.0125, 0.05, 0.25], rtol=1e-14)
    eps = 1e-7
    for r0 in (d - 1e-3, d + 1e-3, -0.2, 0.01):
        fd = (T.huber(np.array(r0 + eps), d) - T.huber(np.array(r0 - eps), d)) / (2 * eps)
        assert abs(fd - T.huber_grad(np.array(r0), d)) < 1e-6


def test_loss_grad_finite_differences():
    """d loss / d pred against central differences at every pixel of a small field,
    with delta in the range of the neighbour differences (both Huber branches)."""
    rng = np.random.default_rng(0)
    pred, truth = rng.standard_normal((2, 5, 6)), rng.standard_normal((2, 5, 6))
    latw = T.lat_weights(5)
    lam, delta = 0.3, 0.4
    g = T.bayesian_loss_grad(pred, truth, latw, lam, delta)
    eps = 1e-6
    for idx in np.ndindex(*pred.shape):
        e = np.zeros_like(pred)
        e[idx] = eps
        fd = (T.bayesian_loss(pred + e, truth, latw, lam, delta)
              - T.bayesian_loss(pred - e, truth, latw, lam, delta)) / (2 * eps)
        assert abs(fd - g[idx]) < 1e-7 * max(1.0, abs(fd)), idx


# ---------------------------------------------------------------- T3
def _fd_check(pr, lam=0.05, delta=0.02, n_coords=60, seed=0, tol=2e-6):
    x, y, blob = data_for(pr)
    loss, grad = T.train_step_grads(x, y, blob, pr, lam, delta)
    assert abs(loss - T.train_loss(x, y, blob, pr, lam, delta)) < 1e-12
    assert grad.shape == blob.shape
    rng = np.random.default_rng(seed)
    # every weight group gets coordinates: sample uniformly plus the first entry of each group
    idx = set(rng.choice(blob.size, n_coords, replace=False).tolist())
    idx |= {0, blob.size - 1}
    eps = 1e-5
    for i in sorted(idx):
        bp, bm = blob.copy(), blob.copy()
        bp[i] += eps
        bm[i] -= eps
        fd = (T.train_loss(x, y, bp, pr, lam, delta) - T.train_loss(x, y, bm, pr, lam, delta)) / (2 * eps)
        assert abs(fd - grad[i]) <= tol * max(1e-2, abs(fd)), (i, fd, grad[i])
    return grad


@pytest.mark.parametrize("mode", [O.HALO_CLAMP, O.HALO_REPLICATE])
def test_backward_finite_differences_tiled(mode):
    """Brute force: the analytic gradient of the tiled loss equals central differences of
    the forward oracle's loss (2x2 tiles, halo 1, 2 blocks, 2 heads, B = 2)."""
    _fd_check(problem(halo_mode=mode))


def test_backward_finite_differences_ragged_no_halo_channel_map():
    """Ragged tiles (Hp = 7 over 3 rows of tiles), halo 0, a channel map, 1 block."""
    _fd_check(problem(H=14, W=10, tiles_y=3, tiles_x=2, halo=0, depth=1, channel_map=(1, 0)), seed=1)


def _torch_loss_grads(x, y, blob, pr, lam, delta):
    """Untiled model from torch library modules + the loss written with torch ops
    (lat weights from the cos formula, the 8 shifted differences), differentiated
    by autograd; returns the gradient flattened in canonical order."""
    Wt = pr.weights(blob)
    D, p, P, K = pr.embed, pr.patch, pr.P, pr.K
    Hp, Wp = pr.H // p, pr.W // p
    params = {}

    def leaf(name, a):
        t = torch.tensor(np.asarray(a, np.float64), requires_grad=True)
        params[name] = t
        return t

    W_e, b_e, e_s = leaf("W_e", Wt["W_e"]), leaf("b_e", Wt["b_e"]), leaf("e_s", Wt["e_s"])
    xt = torch.from_numpy(x)
    z = F.conv2d(xt, W_e.reshape(D, pr.V, p, p), b_e + e_s, stride=p).flatten(2).transpose(1, 2)
    uu, ww = np.meshgrid(np.arange(Hp), np.arange(Wp), indexing="ij")
    z = z + torch.from_numpy(O.sincos_pos(uu.ravel(), ww.ravel(), D))[None]
    names = ("ln1_g", "ln1_b", "W_qkv", "b_qkv", "W_o", "b_o", "ln2_g", "ln2_b", "W_1", "b_1", "W_2", "b_2")
    for l, Lw in enumerate(Wt["layers"]):
        t = {n: leaf(f"{l}.{n}", Lw[n]) for n in names}
        h = F.layer_norm(z, (D,), t["ln1_g"], t["ln1_b"], eps=1e-5)
        a, _ = F.multi_head_attention_forward(
            h.transpose(0, 1), h.transpose(0, 1), h.transpose(0, 1), D, pr.heads, t["W_qkv"], t["b_qkv"],
            None, None, False, 0.0, t["W_o"], t["b_o"], need_weights=False)
        z = z + a.transpose(0, 1)
        h = F.layer_norm(z, (D,), t["ln2_g"], t["ln2_b"], eps=1e-5)
        z = z + F.linear(F.gelu(F.linear(h, t["W_1"], t["b_1"])), t["W_2"], t["b_2"])
    lnf_g, lnf_b = leaf("lnf_g", Wt["lnf_g"]), leaf("lnf_b", Wt["lnf_b"])
    W_h, b_h = leaf("W_h", Wt["W_h"]), leaf("b_h", Wt["b_h"])
    g = F.linear(F.layer_norm(z, (D,), lnf_g, lnf_b, eps=1e-5), W_h, b_h)
    vit = F.pixel_shuffle(g.transpose(1, 2).reshape(x.shape[0], K * P * P, Hp, Wp), P)
    up = F.interpolate(xt[:, list(pr.cmap())], scale_factor=pr.scale, mode="bilinear", align_corners=False)
    out = vit + up
    sH, sW = out.shape[2], out.shape[3]
    lat = torch.deg2rad(90.0 - 180.0 * (torch.arange(sH, dtype=torch.float64) + 0.5) / sH)
    w = torch.cos(lat) / torch.cos(lat).mean()
    yt = torch.from_numpy(y)
    t1 = (w[None, None, :, None] * (yt - out) ** 2).mean(dim=(1, 2, 3))
    t2 = torch.zeros(x.shape[0])
    pad = F.pad(out, (1, 1, 1, 1), value=float("nan"))
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            if dy == 0 and dx == 0:
                continue
            nb = pad[:, :, 1 + dy:1 + dy + sH, 1 + dx:1 + dx + sW]
            r = out - nb
            valid = ~torch.isnan(r)
            r = torch.where(valid, r, torch.zeros_like(r))
            hub = F.huber_loss(r, torch.zeros_like(r), reduction="none", delta=delta) / delta
            t2 = t2 + torch.where(valid, hub, torch.zeros_like(hub)).sum(dim=(1, 2, 3)) / math.hypot(dy, dx)
    loss = (t1 + lam * t2 / (K * sH * sW)).mean()
    loss.backward()
    order = ["W_e", "b_e", "e_s"] + [f"{l}.{n}" for l in range(pr.depth) for n in names] + \
            ["lnf_g", "lnf_b", "W_h", "b_h"]
    return float(loss), np.concatenate([params[n].grad.numpy().ravel() for n in order])


@pytest.mark.parametrize("halo", [0, 50])
def test_backward_matches_torch_autograd_global(halo):
    """T = 1 (halo 0) and 2x2 tiles with a full halo (I6: tiled == global) against torch
    autograd of the untiled library model with the loss in torch ops (F.huber_loss / delta
    is the R34 Huber; F.multi_head_attention_forward the attention)."""
    tiles = (1, 1) if halo == 0 else (2, 2)
    pr = problem(tiles_y=tiles[0], tiles_x=tiles[1], halo=halo, channel_map=(1, 0))
    x, y, blob = data_for(pr, seed=5)
    lam, delta = 0.05, 0.02
    loss, grad = T.train_step_grads(x, y, blob, pr, lam, delta)
    tl, tg = _torch_loss_grads(x, y, blob, pr, lam, delta)
    assert abs(loss - tl) < 1e-12 * max(1.0, abs(tl))
    np.testing.assert_allclose(grad, tg, rtol=1e-9, atol=1e-12)


def test_backward_scope_and_linearity_in_batch():
    """Out-of-scope stages raise; the batch gradient is the mean of per-sample gradients."""
    with pytest.raises(ValueError):
        T.train_step_grads(np.zeros((1, 2, 12, 16)), np.zeros((1, 2, 24, 32)), np.zeros(1),
                           problem(res_hidden=4), 0.0, 1e-3)
    pr = problem()
    x, y, blob = data_for(pr)
    _, g = T.train_step_grads(x, y, blob, pr, 0.05, 0.02)
    _, g0 = T.train_step_grads(x[:1], y[:1], blob, pr, 0.05, 0.02)
    _, g1 = T.train_step_grads(x[1:], y[1:], blob, pr, 0.05, 0.02)
    np.testing.assert_allclose(g, 0.5 * (g0 + g1), rtol=1e-12, atol=1e-15)


def _avg_worker(rank, world, port, q):
    """One rank: the oracle gradient of ITS half of the batch, then the once-per-batch
    gradient averaging as bench.py --mode train runs it (all_reduce AVG over gloo)."""
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr = problem(depth=1)
        x, y, blob = data_for(pr, batch=2 * world)
        sl = slice(2 * rank, 2 * rank + 2)
        _, g = T.train_step_grads(x[sl], y[sl], blob, pr, 0.05, 0.02)
        gt = torch.from_numpy(g)
        dist.all_reduce(gt, op=dist.ReduceOp.AVG)
        if rank == 0:
            _, full = T.train_step_grads(x, y, blob, pr, 0.05, 0.02)
            q.put(("ok", float(np.abs(gt.numpy() - full).max() / np.abs(full).max())))
        else:
            q.put(("ok", 0.0))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_gradient_averaging_gloo_world2_equals_full_batch():
    """T4 / R36 ("gradients from all GPUs are averaged"): two ranks with two samples
    each, one all-reduce (average) of their gradients == the gradient of the 4-sample batch."""
    import multiprocessing as mp
    import socket
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_avg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[0] == "ok", r
        assert r[1] <= 1e-12, r


def test_adamw_matches_torch_optimizer():
    """T5 / R43: three AdamW steps == torch.optim.AdamW (library, fp64) on the same gradients."""
    rng = np.random.default_rng(4)
    w0 = rng.standard_normal(37)
    gs = [rng.standard_normal(37) for _ in range(3)]
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    opt = torch.optim.AdamW([p], lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    w, m, v = w0.copy(), np.zeros(37), np.zeros(37)
    for t, g in enumerate(gs, start=1):
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        w, m, v = T.adamw(w, g, m, v, t, 1e-2, 0.9, 0.95, 1e-8, 0.1)
    np.testing.assert_allclose(w, p.detach().numpy(), rtol=1e-13, atol=1e-14)
