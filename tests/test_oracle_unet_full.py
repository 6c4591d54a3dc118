"""Pins for the whole-UNet oracle (oracle/unet_full.py, BASELINE config 5): the dense
parts against torch float64 library routines (conv2d, group_norm, nearest interpolation) and a
pure-Python brute-force ResBlock; the mask-aware step against the invariants the paper fixes
(a cache recorded from the same inputs reproduces the dense step on the masked rows; an empty
mask leaves the latent untouched; a cache from other inputs is really used)."""
import dataclasses
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

U = synth.UNET_FULL_TINY


def _np(t):
    return t.double().numpy()


@pytest.mark.parametrize("stride", [1, 2])
def test_conv3x3_matches_torch_conv2d(stride):
    g = torch.Generator().manual_seed(stride)
    x = torch.randn(2, 8, 6, 5, generator=g, dtype=torch.float64)       # N H W C
    w = torch.randn(7, 3, 3, 5, generator=g, dtype=torch.float64)       # Co ky kx Ci
    b = torch.randn(7, generator=g, dtype=torch.float64)
    ref = F.conv2d(x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, stride=stride, padding=1).permute(0, 2, 3, 1)
    got = oracle.conv3x3(_np(x), _np(w).reshape(7, 45), _np(b), stride=stride)
    np.testing.assert_allclose(got, _np(ref), rtol=1e-12, atol=1e-12)


def test_group_norm_and_upsample_match_torch():
    g = torch.Generator().manual_seed(3)
    x = torch.randn(2, 12, 64, generator=g, dtype=torch.float64) * 2 + 0.5  # N P C
    ga = torch.rand(64, generator=g, dtype=torch.float64) + 0.5
    be = torch.randn(64, generator=g, dtype=torch.float64)
    ref = F.group_norm(x.permute(0, 2, 1), 32, ga, be, eps=1e-5).permute(0, 2, 1)
    np.testing.assert_allclose(oracle.group_norm(_np(x), _np(ga), _np(be), 32, 1e-5), _np(ref), rtol=1e-12, atol=1e-12)
    y = torch.randn(1, 3, 4, 5, generator=g, dtype=torch.float64)
    ref = F.interpolate(y.permute(0, 3, 1, 2), scale_factor=2, mode="nearest").permute(0, 2, 3, 1)
    np.testing.assert_array_equal(oracle.upsample2(_np(y)), _np(ref))


def test_timestep_embedding_closed_form_at_zero():
    W = {k: _np(v) for k, v in synth.make_unet_full_weights(U, names={"time.lin1.w", "time.lin1.b", "time.lin2.w", "time.lin2.b"}).items()}
    e = np.concatenate([np.ones(U.ch[0] // 2), np.zeros(U.ch[0] // 2)])  # cos 0 = 1, sin 0 = 0
    h = e @ W["time.lin1.w"].T + W["time.lin1.b"]
    h = h / (1.0 + np.exp(-h))
    np.testing.assert_allclose(oracle.timestep_embedding(U, W, 0.0), h @ W["time.lin2.w"].T + W["time.lin2.b"], rtol=1e-13)


def _brute_resblock(u, W, p, x, temb):
    """Pure-Python loops (no NumPy algebra): GroupNorm, SiLU, two 3x3 convolutions with zero
    padding, the timestep projection and the linear skip."""
    N, H, Wd, Ci = x.shape
    Co = len(W[p + ".conv1.b"])
    G = u.gn_groups
    X = x.tolist()

    def gn_silu(T, C, g, b):
        out = [[[[0.0] * C for _ in range(Wd)] for _ in range(H)] for _ in range(N)]
        cg = C // G
        for n in range(N):
            for gi in range(G):
                vals = [T[n][y][xx][c] for y in range(H) for xx in range(Wd) for c in range(gi * cg, (gi + 1) * cg)]
                mu = sum(vals) / len(vals)
                var = sum((v - mu) ** 2 for v in vals) / len(vals)
                r = 1.0 / math.sqrt(var + u.gn_eps)
                for y in range(H):
                    for xx in range(Wd):
                        for c in range(gi * cg, (gi + 1) * cg):
                            v = (T[n][y][xx][c] - mu) * r * g[c] + b[c]
                            out[n][y][xx][c] = v / (1.0 + math.exp(-v))
        return out

    def conv(T, Cin, w, b):
        out = [[[[b[o] for o in range(Co)] for _ in range(Wd)] for _ in range(H)] for _ in range(N)]
        for n in range(N):
            for y in range(H):
                for xx in range(Wd):
                    for o in range(Co):
                        s = 0.0
                        for ky in range(3):
                            for kx in range(3):
                                yy, xs = y + ky - 1, xx + kx - 1
                                if 0 <= yy < H and 0 <= xs < Wd:
                                    for c in range(Cin):
                                        s += T[n][yy][xs][c] * w[o][(ky * 3 + kx) * Cin + c]
                        out[n][y][xx][o] += s
        return out

    Wl = {k: np.asarray(v).tolist() for k, v in W.items() if k.startswith(p)}
    h = conv(gn_silu(X, Ci, Wl[p + ".gn1.g"], Wl[p + ".gn1.b"]), Ci, Wl[p + ".conv1.w"], Wl[p + ".conv1.b"])
    tp = []
    for n in range(N):
        st = [v / (1.0 + math.exp(-v)) for v in temb[n]]
        tp.append([sum(st[k] * Wl[p + ".temb.w"][o][k] for k in range(len(st))) + Wl[p + ".temb.b"][o] for o in range(Co)])
    for n in range(N):
        for y in range(H):
            for xx in range(Wd):
                for o in range(Co):
                    h[n][y][xx][o] += tp[n][o]
    h = conv(gn_silu(h, Co, Wl[p + ".gn2.g"], Wl[p + ".gn2.b"]), Co, Wl[p + ".conv2.w"], Wl[p + ".conv2.b"])
    out = np.zeros((N, H, Wd, Co))
    for n in range(N):
        for y in range(H):
            for xx in range(Wd):
                for o in range(Co):
                    sk = X[n][y][xx][o] if Ci == Co else \
                        sum(X[n][y][xx][c] * Wl[p + ".skip.w"][o][c] for c in range(Ci)) + Wl[p + ".skip.b"][o]
                    out[n, y, xx, o] = sk + h[n][y][xx][o]
    return out


@pytest.mark.parametrize("ci,co", [(4, 4), (4, 6)])
def test_resblock_matches_brute_force(ci, co):
    u = dataclasses.replace(U, gn_groups=2, ch=(4, 4, 4))
    p = "r"
    rng = np.random.default_rng(ci + co)
    W = {p + ".gn1.g": 1 + 0.1 * rng.standard_normal(ci), p + ".gn1.b": 0.1 * rng.standard_normal(ci),
         p + ".conv1.w": rng.standard_normal((co, 9 * ci)) / 6, p + ".conv1.b": rng.standard_normal(co) / 6,
         p + ".temb.w": rng.standard_normal((co, 8)) / 3, p + ".temb.b": rng.standard_normal(co) / 3,
         p + ".gn2.g": 1 + 0.1 * rng.standard_normal(co), p + ".gn2.b": 0.1 * rng.standard_normal(co),
         p + ".conv2.w": rng.standard_normal((co, 9 * co)) / 6, p + ".conv2.b": rng.standard_normal(co) / 6}
    if ci != co:
        W[p + ".skip.w"] = rng.standard_normal((co, ci)) / 2
        W[p + ".skip.b"] = rng.standard_normal(co) / 2
    x = rng.standard_normal((2, 4, 3, ci))
    temb = rng.standard_normal((2, 8))
    np.testing.assert_allclose(oracle.resblock(u, W, p, x, temb), _brute_resblock(u, W, p, x, temb), rtol=1e-11, atol=1e-11)


# ------------------------------------------------------------------------------- whole step
@pytest.fixture(scope="module")
def tiny():
    W = {k: _np(v) for k, v in synth.make_unet_full_weights(U).items()}
    lat = _np(synth.make_unet_latent(U, 0))
    ctx = _np(synth.normal(0, "unet_full_ctx", (U.ctx_len, U.ctx_dim)))
    cond = _np(synth.normal(0, "unet_full_cond", (U.temb_dim,))) * 0.1
    return W, lat, ctx, cond


def _masks():
    rng = np.random.default_rng(5)
    n = U.grid * U.grid
    return {"rect": synth.rect_mask(synth.ModelDesc("g", 0, 1, 64, 1, 64, 64, 4, U.grid, U.grid, 0), 3, 9, 5, 12),
            "blob": (rng.random(n) < 0.2).astype(np.uint8)}


@pytest.mark.parametrize("kind", ["rect", "blob"])
def test_same_input_cache_reproduces_dense_step(tiny, kind):
    W, lat, ctx, cond = tiny
    sig = [0.9, 0.6, 0.3]
    traj, caches = oracle.unet_full_cache_template(U, W, lat, cond, ctx, sig)
    mask = _masks()[kind]
    idx = np.flatnonzero(mask)
    x = lat.copy()
    un = mask == 0
    for s in range(2):  # two steps along the recorded trajectory
        # the dense ResBlocks read every latent row: the caller blends the unmasked rows with the
        # template's trajectory before each step (standard inpainting, C-AMB 11)
        x[un] = traj[s][un]
        inp = x.copy()
        x = oracle.unet_full_edit_step(U, W, x, mask, caches[s], sig[s], sig[s + 1], cond, ctx)
        scale = np.abs(traj[s + 1]).max()
        assert np.max(np.abs(x[idx] - traj[s + 1][idx])) <= 1e-11 * scale
        assert np.array_equal(x[un], inp[un])


def test_degenerate_masks_and_foreign_cache(tiny):
    W, lat, ctx, cond = tiny
    sig = [0.8, 0.5]
    _, caches = oracle.unet_full_cache_template(U, W, _np(synth.make_unet_latent(U, 7)), cond, ctx, sig)
    n = U.grid * U.grid
    zero = np.zeros(n, np.uint8)
    assert np.array_equal(oracle.unet_full_edit_step(U, W, lat, zero, caches[0], 0.8, 0.5, cond, ctx), lat)
    ones = np.ones(n, np.uint8)
    dense = oracle.unet_full_dense_step(U, W, lat, 0.8, 0.5, cond, ctx)
    assert np.array_equal(oracle.unet_full_edit_step(U, W, lat, ones, caches[0], 0.8, 0.5, cond, ctx), dense)
    mask = _masks()["rect"]
    idx = np.flatnonzero(mask)
    a = oracle.unet_full_edit_step(U, W, lat, mask, caches[0], 0.8, 0.5, cond, ctx)
    assert np.max(np.abs(a[idx] - dense[idx])) > 1e-6  # the foreign template's cache is used


def test_level_masks_are_any_pools():
    mask = _masks()["blob"]
    m0, m1, m2 = oracle.level_masks(U, mask)
    g = U.grid
    mm = mask.reshape(g, g)
    for r in range(g // 2):
        for c in range(g // 2):
            assert m1.reshape(g // 2, g // 2)[r, c] == int(mm[2 * r:2 * r + 2, 2 * c:2 * c + 2].any())
    assert m2.sum() <= m1.sum() <= m0.sum() or m2.sum() * 16 >= m0.sum()


def test_transformer2d_masked_full_mask_is_dense(tiny):
    W, lat, ctx, cond = tiny
    p, lvl, c, dep = synth.unet_t2ds(U)[0]
    P = U.level_grid(lvl) ** 2
    x = np.random.default_rng(1).standard_normal((P, c))
    dense, kv = oracle.t2d_dense(U, W, p, lvl, dep, x, ctx, record=True)
    ones = np.ones(P, np.uint8)
    np.testing.assert_array_equal(oracle.t2d_masked(U, W, p, lvl, dep, x, ones, None, None, ctx), dense)
    mask = np.zeros(P, np.uint8)
    mask[5:30] = 1
    got = oracle.t2d_masked(U, W, p, lvl, dep, x, mask, kv, dense, ctx)  # same-input cache
    np.testing.assert_allclose(got, dense, rtol=1e-11, atol=1e-11)


def test_sweep_tool_flop_model_matches_oracle_macs():
    """tools/unet_full_sweep.py's FLOP model (its own arithmetic: the tool may not import the
    oracle) equals 2x the oracle's MAC counter for the dense step of the SDXL shape, and the
    Transformer2Ds' share of the dense step is in the paper's range (82% for SDXL)."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import unet_full_sweep as T
    u = synth.SDXL_UNET
    macs = oracle.unet_full_macs(u)
    assert T.dense_conv_macs(u) == macs["conv"]
    ones = np.ones(u.grid * u.grid, np.uint8)
    assert abs(T.flops(u, ones) - 2 * (macs["conv"] + macs["t2d"])) <= 1e-9 * T.flops(u, ones)
    share = macs["t2d"] / (macs["conv"] + macs["t2d"])
    assert 0.7 < share < 0.85
