"""Pins of the UNet attention-stack oracle (oracle/unet.py; BASELINE config 5)
against things other than itself: math.erf values, closed forms with zeroed sub-blocks, a
pure-Python brute-force block, and the exactness invariants the paper fixes (all-ones mask
== dense, empty mask untouched, cache from the same inputs == dense on the masked rows)."""
import math

import numpy as np
import pytest

import oracle
import synth

D = synth.UNET_TINY


def _weights(d=D, seed=0, **zero):
    W = {k: v.double().numpy() for k, v in synth.make_weights(d, seed).items()}
    for name in zero:
        W[name] = np.zeros_like(W[name])
    return W


def _state(d=D, rid=1):
    return synth.make_latent(d, rid).double().numpy()


def _ctx(d=D, rid=1):
    return synth.make_ctx(d, rid).double().numpy()


def test_gelu_erf_matches_math_erf_and_limits():
    xs = [-6.0, -1.0, -0.25, 0.0, 0.3, 1.0, 2.5, 8.0]
    got = oracle.gelu_erf(np.array(xs))
    for x, g in zip(xs, got):
        assert g == pytest.approx(0.5 * x * (1 + math.erf(x / math.sqrt(2))), rel=1e-15, abs=1e-300)
    assert oracle.gelu_erf(np.array([1.0]))[0] == pytest.approx(0.8413447460685429, rel=1e-15)
    assert oracle.gelu_erf(np.array([-1.0]))[0] == pytest.approx(-0.15865525393145707, rel=1e-15)


def test_layernorm_affine_row_statistics():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 8)) * 5 + 2
    g = np.ones(8)
    b = np.zeros(8)
    y = oracle.layernorm_affine(x, g, b, 0.0)
    for r in range(3):
        row = list(y[r])
        assert sum(row) / 8 == pytest.approx(0.0, abs=1e-12)
        assert sum(v * v for v in row) / 8 == pytest.approx(1.0, rel=1e-12)
    g2 = rng.uniform(0.5, 1.5, 8)
    b2 = rng.uniform(-1, 1, 8)
    y2 = oracle.layernorm_affine(x, g2, b2, 0.0)
    np.testing.assert_allclose(y2, y * g2 + b2, rtol=1e-13, atol=1e-13)


def test_geglu_hand_example():
    """hidden = first half, gate = second half: out = (a * gelu(g)) W2^T + b2."""
    class d:
        mlp_hidden = 2
    W = {"p.ff.geglu.w": np.array([[1.0, 0.0], [0.0, 1.0], [2.0, 0.0], [0.0, -1.0]]),
         "p.ff.geglu.b": np.array([0.0, 1.0, 0.0, 0.5]),
         "p.ff.out.w": np.array([[1.0, 1.0]]), "p.ff.out.b": np.array([0.25])}
    h = np.array([[1.0, 2.0]])
    a0, a1 = 1.0, 3.0           # h W^T + b, hidden half
    g0, g1 = 2.0, -1.5          # gate half
    ph = lambda z: 0.5 * z * (1 + math.erf(z / math.sqrt(2)))  # noqa: E731
    want = a0 * ph(g0) + a1 * ph(g1) + 0.25
    assert oracle.geglu_ff(d, W, "p", h)[0, 0] == pytest.approx(want, rel=1e-14)


def test_cross_attention_single_key_closed_form():
    """ctx_len = 1: softmax over one key is 1, so with the self-attention and FF outputs
    zeroed the block adds (ctx Wv^T) Wo^T + bo to every row, whatever the query."""
    d = synth._unet("u1", 1, 64, 4, 8, 1, 16)
    W = _weights(d, **{"unet.0.attn1.out.w": 1, "unet.0.attn1.out.b": 1, "unet.0.ff.out.w": 1, "unet.0.ff.out.b": 1})
    x = _state(d)
    ctx = _ctx(d)
    out = oracle.unet_dense_step(d, W, x, ctx)
    H = d.hidden
    v = ctx @ W["unet.0.attn2.kv.w"][H:].T
    add = v @ W["unet.0.attn2.out.w"].T + W["unet.0.attn2.out.b"]
    np.testing.assert_allclose(out, x + add, rtol=1e-12, atol=1e-12)


def test_cross_attention_key_value_halves():
    """Zero the key half of attn2.kv: all scores are equal, so cross-attention returns the
    mean of the value rows (a swapped K/V split would return zeros)."""
    d = synth._unet("u2", 1, 64, 4, 8, 5, 16)
    H = d.hidden
    W = _weights(d, **{"unet.0.attn1.out.w": 1, "unet.0.attn1.out.b": 1, "unet.0.ff.out.w": 1, "unet.0.ff.out.b": 1})
    W["unet.0.attn2.kv.w"][:H] = 0.0
    x = _state(d)
    ctx = _ctx(d)
    out = oracle.unet_dense_step(d, W, x, ctx)
    v = (ctx @ W["unet.0.attn2.kv.w"][H:].T).mean(axis=0)
    add = v @ W["unet.0.attn2.out.w"].T + W["unet.0.attn2.out.b"]
    np.testing.assert_allclose(out, x + add, rtol=1e-12, atol=1e-12)


def _brute_block(d, W, i, x, ctx):
    """Pure-Python loops: one BasicTransformerBlock over all tokens (no NumPy algebra)."""
    H, hd, eps, F = d.hidden, d.head_dim, d.ln_eps, d.mlp_hidden
    p = f"unet.{i}."
    w = {k[len(p):]: W[k].tolist() for k in W if k.startswith(p)}

    def ln(rows, g, b):
        out = []
        for r in rows:
            mu = sum(r) / H
            var = sum((v - mu) ** 2 for v in r) / H
            s = 1.0 / math.sqrt(var + eps)
            out.append([(r[c] - mu) * s * g[c] + b[c] for c in range(H)])
        return out

    def lin(rows, M, bias=None):
        return [[sum(r[k] * M[o][k] for k in range(len(r))) + (bias[o] if bias else 0.0) for o in range(len(M))]
                for r in rows]

    def attn(q, K, V):
        out = []
        for qi in q:
            row = [0.0] * H
            for h in range(d.heads):
                c0 = h * hd
                s = [sum(qi[c0 + t] * kj[c0 + t] for t in range(hd)) / math.sqrt(hd) for kj in K]
                m = max(s)
                e = [math.exp(v - m) for v in s]
                z = sum(e)
                for j, vj in enumerate(V):
                    for t in range(hd):
                        row[c0 + t] += e[j] / z * vj[c0 + t]
            out.append(row)
        return out

    X = [list(r) for r in x]
    h = ln(X, w["ln1.g"], w["ln1.b"])
    qkv = lin(h, w["attn1.qkv.w"])
    q = [r[:H] for r in qkv]
    k = [r[H:2 * H] for r in qkv]
    v = [r[2 * H:] for r in qkv]
    o = lin(attn(q, k, v), w["attn1.out.w"], w["attn1.out.b"])
    X = [[a + b for a, b in zip(r, s)] for r, s in zip(X, o)]
    h = ln(X, w["ln2.g"], w["ln2.b"])
    q2 = lin(h, w["attn2.q.w"])
    kv2 = lin([list(r) for r in ctx], w["attn2.kv.w"])
    o = lin(attn(q2, [r[:H] for r in kv2], [r[H:] for r in kv2]), w["attn2.out.w"], w["attn2.out.b"])
    X = [[a + b for a, b in zip(r, s)] for r, s in zip(X, o)]
    h = ln(X, w["ln3.g"], w["ln3.b"])
    u = lin(h, w["ff.geglu.w"], w["ff.geglu.b"])
    g = [[r[j] * 0.5 * r[F + j] * (1 + math.erf(r[F + j] / math.sqrt(2))) for j in range(F)] for r in u]
    o = lin(g, w["ff.out.w"], w["ff.out.b"])
    return np.array([[a + b for a, b in zip(r, s)] for r, s in zip(X, o)])


def test_block_matches_brute_force_loops():
    d = synth._unet("u3", 1, 16, 2, 4, 3, 8)  # 16 tokens, H=16, 2 heads of 8, F=64
    W = _weights(d)
    x = _state(d)
    ctx = _ctx(d)
    np.testing.assert_allclose(oracle.unet_dense_step(d, W, x, ctx), _brute_block(d, W, 0, x, ctx),
                               rtol=1e-11, atol=1e-11)


def test_all_ones_mask_equals_dense_and_empty_is_untouched():
    W = _weights()
    x = _state()
    ctx = _ctx()
    junk = synth.make_cache_kv(D, 3, 1).double().numpy()[0]
    dense = oracle.unet_dense_step(D, W, x, ctx)
    np.testing.assert_allclose(oracle.unet_edit_step(D, W, x, np.ones(D.L_img, np.uint8), junk, ctx), dense,
                               rtol=1e-13, atol=1e-13)
    out = oracle.unet_edit_step(D, W, x, np.zeros(D.L_img, np.uint8), junk, ctx)
    assert np.array_equal(out, x)


@pytest.mark.parametrize("kind", ["rect", "blob"])
def test_same_inputs_cache_reproduces_dense_on_masked_rows(kind):
    """A cache recorded along the dense trajectory from the same state: the edit step equals
    the dense step on the masked rows and keeps the unmasked rows (per block, the unmasked
    tokens' K/V are exactly the cached ones)."""
    W = _weights()
    ctx = _ctx()
    states, cache = oracle.unet_cache_template(D, W, _state(), ctx, 2)
    rng = np.random.default_rng(5)
    mask = (synth.rect_mask_count(D, 60, rng) if kind == "rect" else synth.blob_mask_count(D, 90, rng))
    for s in range(2):
        out = oracle.unet_edit_step(D, W, states[s], mask, cache[s], ctx)
        m = mask != 0
        np.testing.assert_allclose(out[m], states[s + 1][m], rtol=1e-12, atol=1e-12)
        assert np.array_equal(out[~m], states[s][~m])
    # and a cache from other inputs changes the masked rows (the cache is really read)
    other = oracle.unet_edit_step(D, W, states[0], mask, cache[1], ctx)
    assert not np.allclose(other[mask != 0], states[1][mask != 0])


def test_any_pool2_brute_force_and_properties():
    rng = np.random.default_rng(3)
    for _ in range(5):
        m = (rng.random(64 * 64) < 0.05).astype(np.uint8)
        p = oracle.any_pool2(m, 64, 64)
        g = m.reshape(64, 64)
        for r in range(32):
            for c in range(32):
                want = int(g[2 * r, 2 * c] or g[2 * r + 1, 2 * c] or g[2 * r, 2 * c + 1] or g[2 * r + 1, 2 * c + 1])
                assert p[r * 32 + c] == want
        assert p.sum() >= m.sum() / 4
    assert oracle.any_pool2(np.ones(16, np.uint8), 4, 4).tolist() == [1, 1, 1, 1]


def test_macs_per_row_counts_the_block():
    oracle.reset_macs()
    W = _weights()
    x = _state()
    ctx = _ctx()
    mask = synth.rect_mask_count(D, 40, np.random.default_rng(0))
    cache = synth.make_cache_kv(D, 3, 1).double().numpy()[0]
    oracle.unet_edit_step(D, W, x, mask, cache, ctx)
    per = oracle.unet_macs_per_row(D)
    cross = D.n_unet * D.ctx_len * 2 * D.hidden * D.ctx_dim   # the context's K/V, per request
    assert oracle.MACS["linear"] == 40 * D.n_unet * per["linear"] + cross
    assert oracle.MACS["attn"] == 40 * D.n_unet * per["attn"]


def test_levels_any_pool2_matches_oracle():
    """The product's host-side level-mask reduction equals the oracle's loop definition."""
    from paper_2505_20600_b200 import levels
    rng = np.random.default_rng(9)
    for n in (0, 1, 37, 900, 4096):
        m = synth.blob_mask_count(synth.SDXL_L64, n, rng)
        assert np.array_equal(levels.any_pool2(m, 64, 64), oracle.any_pool2(m, 64, 64))
    with pytest.raises(ValueError):
        levels.any_pool2(np.zeros(15, np.uint8), 3, 5)


def test_y_variant_pins():
    """Y variant: (1) with a Y cache recorded along the dense trajectory from the same state,
    the Y step equals the dense step on the masked rows (exactly: the recomputed K/V of the
    unmasked rows are the dense ones); (2) K/V recomputed from the recorded Y_{b-1} equal the
    recorded K/V of block b; (3) no Y blocks == the K/V step; (4) a hybrid split equals the
    dense step too, and the Y cache is really read (other Y rows change the result)."""
    W = _weights()
    ctx = _ctx()
    states, kv, ys = oracle.unet_cache_template(D, W, _state(), ctx, 2, record_y=True)
    mask = synth.blob_mask_count(D, 80, np.random.default_rng(8))
    m = mask != 0
    for s in range(2):
        out = oracle.unet_edit_step_y(D, W, states[s], mask, ys[s], states[s], ctx)
        np.testing.assert_allclose(out[m], states[s + 1][m], rtol=1e-12, atol=1e-12)
        assert np.array_equal(out[~m], states[s][~m])
        hyb = oracle.unet_edit_step_y(D, W, states[s], mask, ys[s], states[s], ctx, y_blocks=[1], kv_cache_step=kv[s])
        np.testing.assert_allclose(hyb[m], states[s + 1][m], rtol=1e-12, atol=1e-12)
    k1, v1 = oracle.unet_kv_from_y(D, W, 1, ys[0][0])
    np.testing.assert_allclose(k1, kv[0][1][0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(v1, kv[0][1][1], rtol=1e-12, atol=1e-12)
    junk = synth.make_cache_kv(D, 4, 1).double().numpy()[0]
    np.testing.assert_array_equal(oracle.unet_edit_step_y(D, W, states[0], mask, ys[0], states[0], ctx, y_blocks=[],
                                                          kv_cache_step=junk),
                                  oracle.unet_edit_step(D, W, states[0], mask, junk, ctx))
    other = oracle.unet_edit_step_y(D, W, states[0], mask, ys[1], states[0], ctx)
    assert not np.allclose(other[m], states[1][m])


def test_planned_step_pins():
    """Algorithm-1 dense prefix on the UNet stack: k = 0 is the K/V (resp. hybrid) step; k = N
    is the dense step on [masked rows of state | unmasked rows of tstate]; with a cache recorded
    from the same state every k stays on the dense trajectory."""
    W = _weights()
    ctx = _ctx()
    states, kv, ys = oracle.unet_cache_template(D, W, _state(), ctx, 1, record_y=True)
    mask = synth.rect_mask_count(D, 50, np.random.default_rng(13))
    m = mask != 0
    x = _state(rid=7)
    junk = synth.make_cache_kv(D, 5, 1).double().numpy()[0]
    np.testing.assert_array_equal(oracle.unet_edit_step_planned(D, W, x, mask, states[0], ctx, 0, kv_cache_step=junk),
                                  oracle.unet_edit_step(D, W, x, mask, junk, ctx))
    np.testing.assert_allclose(
        oracle.unet_edit_step_planned(D, W, x, mask, states[0], ctx, 0, kv_cache_step=junk, y_cache_step=ys[0], y_blocks=[0]),
        oracle.unet_edit_step_y(D, W, x, mask, ys[0], states[0], ctx, y_blocks=[0], kv_cache_step=junk), rtol=0, atol=0)
    comb = np.array(states[0])
    comb[m] = x[m]
    full = oracle.unet_dense_step(D, W, comb, ctx)
    got = oracle.unet_edit_step_planned(D, W, x, mask, states[0], ctx, D.n_unet, kv_cache_step=junk)
    np.testing.assert_allclose(got[m], full[m], rtol=1e-12, atol=1e-12)
    assert np.array_equal(got[~m], x[~m])
    for k in range(D.n_unet + 1):
        for yb in ((), (1,)):
            out = oracle.unet_edit_step_planned(D, W, states[0], mask, states[0], ctx, k, kv_cache_step=kv[0],
                                                y_cache_step=ys[0], y_blocks=yb)
            np.testing.assert_allclose(out[m], states[1][m], rtol=1e-12, atol=1e-12)


def test_sweep_flop_model_matches_oracle_macs():
    """tools/unet_sweep.py's algorithmic FLOPs (the config-5 roofline numerator) equal twice the
    oracle's counted multiply-accumulates of the same step."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "unet_sweep", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "unet_sweep.py"))
    sw = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sw)
    W = _weights()
    ctx = _ctx()
    cache = synth.make_cache_kv(D, 3, 1).double().numpy()[0]
    masks = [synth.rect_mask_count(D, 40, np.random.default_rng(0)), synth.blob_mask_count(D, 25, np.random.default_rng(1))]
    oracle.reset_macs()
    for mk in masks:
        oracle.unet_edit_step(D, W, _state(), mk, cache, ctx)
    macs = oracle.MACS["linear"] + oracle.MACS["attn"]
    assert sw.step_flops(D, 65, 2) == 2 * macs
