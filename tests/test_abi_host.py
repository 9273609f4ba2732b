"""Host-side tests of liborbit2.so (no GPU needed): the library loads and
exports every symbol include/orbit2.h declares; orbit2_tiles_plan is
bit-exact against the oracle's independent planner; validation errors name
the field; the analytic FLOP model matches brute-force counts."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import reslim_tiles as O
from workloads import CONFIGS, get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def o2():
    from paper_2505_04802_b200 import build
    build.build()
    from paper_2505_04802_b200 import orbit2
    return orbit2


def test_exports_every_declared_symbol(o2):
    hdr = open(os.path.join(ROOT, "include", "orbit2.h")).read()
    declared = set(re.findall(r"\b(orbit2_[a-z_0-9]+)\s*\(", hdr))
    assert {"orbit2_tiles_plan", "orbit2_reslim_forward", "orbit2_stitch"} <= declared
    lib = C.CDLL(o2.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(o2.EXPORTED)


def _plan_both(o2, **kw):
    w = get_config("C1", **kw)
    tiles, info = o2.orbit2_tiles_plan(o2.config_from(w))
    ref = O.plan_tiles(w.Hp, w.Wp, w.tiles_y, w.tiles_x, w.halo, w.halo_mode)
    return w, tiles, info, ref


@pytest.mark.parametrize("mode", [0, 1])
def test_plan_bit_exact_vs_oracle_planner(o2, mode):
    for H, W in [(8, 8), (12, 20), (32, 64), (18, 34)]:
        for ty in range(1, 5):
            for tx in range(1, 5):
                for h in range(0, 4):
                    if ty > H // 2 or tx > W // 2:
                        continue
                    w, tiles, info, ref = _plan_both(o2, H=H, W=W, tiles_y=ty, tiles_x=tx, halo=h,
                                                     halo_mode=mode)
                    assert info.n_tiles == len(ref)
                    off = core = 0
                    for a, b in zip(tiles, ref):
                        assert (a.tile_id, a.tile_y, a.tile_x) == (b.tile_id, b.ty, b.tx)
                        assert (a.core_y0, a.core_y1, a.core_x0, a.core_x1) == \
                               (b.core_y0, b.core_y1, b.core_x0, b.core_x1)
                        assert (a.pad_y0, a.pad_y1, a.pad_x0, a.pad_x1) == \
                               (b.pad_y0, b.pad_y1, b.pad_x0, b.pad_x1)
                        assert a.n_tokens == b.n_tokens and a.n_core_tokens == b.n_core
                        assert a.token_offset == off and a.core_token_offset == core
                        off += b.n_tokens
                        core += b.n_core


@pytest.mark.parametrize("name", list(CONFIGS))
def test_counts_and_flops_vs_oracle(o2, name):
    w = get_config(name)
    _, info = o2.orbit2_tiles_plan(o2.config_from(w))
    c = O.token_counts(O.Problem.from_config(w))
    assert info.tokens_per_sample == c["n_pad"] and info.core_tokens_per_sample == c["n_core"]
    assert info.sum_n2_per_sample == c["sum_n2"] and info.sum_nc_per_sample == c["sum_nc"]
    # brute-force FLOP count: sum over tiles of per-layer GEMM + attention work
    D, L, Din, Nh = w.embed, w.depth, w.din, w.head_out
    f = 0.0
    for n, cc in zip(c["n"], c["c"]):
        n, cc = float(n), float(cc)
        f += 2 * n * Din * D + 2 * cc * D * Nh
        for layer in range(L):
            last = layer == L - 1
            rows_q = cc if last else n
            f += 2 * n * D * 2 * D + 2 * rows_q * D * D          # K,V for all rows; Q for rows_q
            f += 2 * rows_q * n * D * 2                           # QK^T and PV over heads
            f += 2 * rows_q * D * D + 2 * rows_q * D * 4 * D * 2  # O-proj, MLP up+down
    assert info.flops_per_sample == pytest.approx(f, rel=1e-12)
    assert info.canonical_weight_count == __import__("workloads").weight_count(w)


def test_survey_flop_values(o2):
    """algorithmic FLOP/sample C1..C5."""
    want = {"C1": 9.10e7, "C2": 4.111e11, "C3": 5.074e12, "C4": 7.240e14, "C5": 1.493e15}
    for n, v in want.items():
        _, info = o2.orbit2_tiles_plan(o2.config_from(get_config(n)))
        assert info.flops_per_sample == pytest.approx(v, rel=2e-3)


@pytest.mark.parametrize("bad,field", [
    (dict(H=33), "H"), (dict(tiles_y=17), "tiles_y"), (dict(halo=-1), "halo"),
    (dict(heads=3), "embed"), (dict(scale=0), "scale"), (dict(K=4), "K"),
    (dict(batch=0), "batch"),
])
def test_validation_errors_name_the_field(o2, bad, field):
    w = get_config("C1")
    cfg = o2.config_from(w, **bad)
    with pytest.raises(o2.Orbit2Error) as e:
        o2.orbit2_tiles_plan(cfg)
    assert e.value.status in (o2.E_INVALID, o2.E_UNSUPPORTED)
    assert field in str(e.value)


def test_unsupported_head_dim(o2):
    cfg = o2.config_from(get_config("C1"), embed=48, heads=3)
    with pytest.raises(o2.Orbit2Error) as e:
        o2.orbit2_tiles_plan(cfg)
    assert e.value.status == o2.E_UNSUPPORTED


def test_bf16_head_rows_must_be_16_byte_aligned(o2):
    """K (s p)^2 = 9 bf16 head outputs per token: BF16 rejects it (E_UNSUPPORTED, naming K),
    FP32 plans it."""
    w = get_config("C1", K=1, scale=3, patch=1)
    with pytest.raises(o2.Orbit2Error) as e:
        o2.orbit2_tiles_plan(o2.config_from(w, precision=o2.BF16))
    assert e.value.status == o2.E_UNSUPPORTED and "K" in str(e.value)
    _, info = o2.orbit2_tiles_plan(o2.config_from(w, precision=o2.FP32))
    assert info.n_tiles == 4


def test_capacity_two_call_sizing(o2):
    cfg = o2.config_from(get_config("C2"))
    info = o2.orbit2_plan_info()
    small = (o2.orbit2_tile * 3)()
    st = o2.lib.orbit2_tiles_plan(C.byref(cfg), small, 3, C.byref(info))
    assert st == o2.E_CAPACITY and info.n_tiles == 16


def test_rank_partition_lpt(o2):
    """Every tile owned by exactly one rank; LPT keeps per-rank cost within 5%
    of the mean for C2..C4 at R = 2, 4, 8."""
    for name in ("C2", "C3", "C4"):
        w = get_config(name)
        for R in (2, 4, 8):
            loads = np.zeros(R)
            owners = None
            for r in range(R):
                tiles, info = o2.orbit2_tiles_plan(o2.config_from(w, world_size=R, rank=r))
                own = [t.owner_rank for t in tiles]
                owners = own if owners is None else owners
                assert own == owners
                loads[r] = info.local_flops_per_sample
                assert info.n_local_tiles == sum(1 for t in tiles if t.owner_rank == r)
            assert loads.sum() == pytest.approx(info.flops_per_sample, rel=1e-12)
            assert loads.max() / loads.mean() < 1.05, (name, R, loads)


def test_create_rejects_bad_workspace(o2):
    cfg = o2.config_from(get_config("C1"))
    h = C.c_void_p()
    st = o2.lib.orbit2_create(C.byref(cfg), None, 0, C.byref(h))
    assert st == o2.E_INVALID and b"workspace" in o2.lib.orbit2_last_error()


def test_residual_conv_config_counts_and_halo(o2):
    """res_hidden (ABI v2, reading R31): the canonical blob grows by the two 3x3
    convolutions (18 C_r K + C_r + K, the workloads generator agrees), out-of-range
    values are rejected, and with halo 0 the rectangles a rank receives cover every
    owned core + 1 + ceil(2 / s) coarse pixels (the convolutions' receptive field)."""
    from workloads import weight_count
    w = get_config("C1", res_hidden=8)
    _, info = o2.orbit2_tiles_plan(o2.config_from(w))
    assert info.canonical_weight_count == weight_count(w)
    assert info.canonical_weight_count == weight_count(w.replace(res_hidden=0)) + 18 * 8 * w.K + 8 + w.K
    for bad in (65, 6):
        with pytest.raises(o2.Orbit2Error, match="res_hidden"):
            o2.orbit2_tiles_plan(o2.config_from(w, res_hidden=bad))
    w0 = get_config("C1", H=36, W=60, tiles_y=3, tiles_x=4, halo=0, res_hidden=4)
    dil = 1 + -(-2 // w0.scale)
    for R in (2, 3):
        for r in range(R):
            cfg = o2.config_from(w0, world_size=R, rank=r)
            tiles, _ = o2.orbit2_tiles_plan(cfg)
            have = np.zeros((w0.H, w0.W), bool)
            for t in tiles:
                if t.owner_rank == r:
                    have[t.core_y0 * 2:t.core_y1 * 2, t.core_x0 * 2:t.core_x1 * 2] = True
            for s in range(R):
                if s != r:
                    for y0, y1, x0, x1 in o2.orbit2_xfer_plan(cfg, o2.XFER_HALO, s, o2.RECV)[0]:
                        have[y0:y1, x0:x1] = True
            for t in tiles:
                if t.owner_rank == r:
                    y0, y1 = max(0, t.core_y0 * 2 - dil), min(w0.H, t.core_y1 * 2 + dil)
                    x0, x1 = max(0, t.core_x0 * 2 - dil), min(w0.W, t.core_x1 * 2 + dil)
                    assert have[y0:y1, x0:x1].all()


def test_variable_aggregation_config_counts(o2):
    """var_agg (ABI v2, reading R33): the canonical blob grows by the tokenizer, the
    variable embeddings, the query and three D x D projections (+ biases); the
    workloads generator agrees; other values are rejected."""
    from workloads import weight_count
    w = get_config("C1", var_agg=1, embed=64, heads=2)
    _, info = o2.orbit2_tiles_plan(o2.config_from(w))
    D, V = w.embed, w.V
    assert info.canonical_weight_count == weight_count(w)
    assert info.canonical_weight_count == weight_count(w.replace(var_agg=0)) + V * D * 4 + V * D + D + 3 * (D * D + D)
    with pytest.raises(o2.Orbit2Error, match="var_agg"):
        o2.orbit2_tiles_plan(o2.config_from(w, var_agg=2))


def test_compress_plan_validation_and_sizes(o2):
    """orbit2_compress_plan (host only): sizes grow with the field; every invalid field is
    rejected with E_INVALID and a message naming it (R37 / R38 constraints)."""
    import ctypes as C
    ws, mp = C.c_int64(), C.c_int64()

    def plan(**kw):
        base = dict(batch=2, H=64, W=96, C=3, min_side=2, max_side=16, embed=32, threshold=0.05, sigma=1.0,
                    low_frac=0.1, high_frac=0.2)
        base.update(kw)
        cfg = o2.orbit2_compress_config(*[base[k] for k in ("batch", "H", "W", "C", "min_side", "max_side", "embed",
                                                             "threshold", "sigma", "low_frac", "high_frac")])
        return o2.lib.orbit2_compress_plan(C.byref(cfg), C.byref(ws), C.byref(mp)), o2.lib.orbit2_last_error().decode()

    st, _ = plan()
    assert st == o2.OK and mp.value == 2 * 32 * 48
    w0 = ws.value
    assert plan(H=128)[0] == o2.OK and ws.value > w0
    for kw, word in [(dict(max_side=12), "max_side"), (dict(max_side=2), "max_side"), (dict(H=60), "multiples"),
                     (dict(sigma=3.0), "sigma"), (dict(sigma=0.0), "sigma"), (dict(low_frac=0.3), "low_frac"),
                     (dict(low_frac=0.0), "low_frac"), (dict(batch=0), "batch"), (dict(max_side=256), "max_side"),
                     (dict(threshold=float("nan")), "threshold")]:
        st, msg = plan(**kw)
        assert st == o2.E_INVALID and word in msg, (kw, msg)
    assert plan(threshold=-1.0)[0] == o2.OK          # < 0: split down to min_side
