"""Pin of the oracle's Flux/SD3 block COMPOSITION against a pure-Python loop implementation.

`oracle/instgenie.py` builds `dense_step` and the masked path from shared helpers
(`_qkv_stream`, `_double_out`, `_single_pre`, `_single_out`, `modulation`, `conditioning`,
`final_velocity`, `image_positions`), so the masked == dense exactness grid cannot see an
error inside them.  This file re-derives one whole step from the readings alone, with
scalar Python loops and no NumPy algebra, sharing no helper with the oracle:

* conditioning: vec = MLP_t(sinusoid_256(1000 sigma)) + cond_vec, sinusoid cos-first with
  f_k = exp(-ln(10000) k / 128), MLP_t(e) = SiLU(e W1 + b1) W2 + b2 (SURVEY C-ALG 2, C-AMB 12);
* per-block modulation SiLU(vec) W_mod + b in chunk order (shift1, scale1, gate1, shift2,
  scale2, gate2) (double), (shift, scale, gate) (single), (scale, shift) (final and an SD3
  context-pre-only text stream) (C-ALG 2);
* adaLN h = LN(x)(1 + scale) + shift, LN without affine, eps 1e-6 (C-AMB 6);
* QK-RMSNorm per head (eps 1e-6, gain), 3-axis RoPE with image token i at
  (0, i div W, i mod W), text at (0, 0, 0), pair (2j, 2j+1) of axis a rotated by
  pos_a * theta^(-2j/d_a) (C-AMB 7);
* merged keys: text rows fresh, masked image rows fresh, unmasked rows from the cache
  (C-ALG 4 'Merge'); softmax(q k / sqrt(d)) per head (C-AMB 4);
* double block: x += g1 (o W_o + b); x += g2 (GELU_tanh(z W1 + b1) W2 + b2) with
  z = LN(x)(1+sc2)+sh2; single block: [q|k|v|u] = h W1 + b, x += g ([o | GELU_tanh(u)] W2 + b)
  (C-ALG 4-5);
* final: v = (LN(x)(1+sc)+sh) W_out + b; latent[i] += (sigma' - sigma) v[i] on masked rows
  only (C-ALG 6, C-AMB 11-12).

A deliberate error in any oracle helper (swapped shift/scale, a dropped (1+.), sigma
instead of 1000 sigma, swapped grid axes, a swapped [o | GELU(u)] concat, swapped final
chunks) must turn these comparisons red: `test_mutations_are_caught` injects each one.
"""
import math

import numpy as np
import pytest

import oracle
import oracle.instgenie as oi
import synth

EPS = 1e-6


# ---------------------------------------------------------------- scalar building blocks
def _mat(W, name):
    return W[name].tolist()


def _vecmat(x, M, b):
    """y[o] = sum_k x[k] M[o][k] + b[o] for M stored [out][in]."""
    return [sum(x[k] * M[o][k] for k in range(len(x))) + (b[o] if b is not None else 0.0)
            for o in range(len(M))]


def _silu1(v):
    return v / (1.0 + math.exp(-v))


def _gelu1(v):
    return 0.5 * v * (1.0 + math.tanh(math.sqrt(2.0 / math.pi) * (v + 0.044715 * v * v * v)))


def _ln_mod(row, shift, scale):
    n = len(row)
    mu = sum(row) / n
    var = sum((v - mu) * (v - mu) for v in row) / n
    r = 1.0 / math.sqrt(var + EPS)
    return [(row[c] - mu) * r * (1.0 + scale[c]) + shift[c] for c in range(n)]


def _rms_heads(row, g, heads):
    dh = len(row) // heads
    out = []
    for h in range(heads):
        seg = row[h * dh:(h + 1) * dh]
        ms = sum(v * v for v in seg) / dh
        r = 1.0 / math.sqrt(ms + EPS)
        out += [seg[t] * r * g[t] for t in range(dh)]
    return out


def _rope_row(row, pos3, heads, axes, theta):
    dh = len(row) // heads
    out = list(row)
    for h in range(heads):
        base = h * dh
        off = 0
        for a in range(3):
            da = axes[a]
            for j in range(da // 2):
                phi = pos3[a] * theta ** (-2.0 * j / da)
                c, s = math.cos(phi), math.sin(phi)
                i0, i1 = base + off + 2 * j, base + off + 2 * j + 1
                x0, x1 = row[i0], row[i1]
                out[i0] = x0 * c - x1 * s
                out[i1] = x0 * s + x1 * c
            off += da
    return out


def _attend(qrows, K, V, heads):
    H = len(qrows[0]) if qrows else 0
    dh = H // heads
    out = []
    for q in qrows:
        row = [0.0] * H
        for h in range(heads):
            c0 = h * dh
            s = [sum(q[c0 + t] * k[c0 + t] for t in range(dh)) / math.sqrt(dh) for k in K]
            mx = max(s)
            e = [math.exp(v - mx) for v in s]
            z = sum(e)
            for j in range(len(V)):
                for t in range(dh):
                    row[c0 + t] += e[j] / z * V[j][c0 + t]
        out.append(row)
    return out


def _chunks(v, k):
    n = len(v) // k
    return [v[i * n:(i + 1) * n] for i in range(k)]


# ---------------------------------------------------------------- the brute-force step
class Brute:
    def __init__(self, d, W):
        self.d, self.W = d, W

    def vec(self, sigma, cond):
        W = self.W
        t = 1000.0 * float(sigma)
        e = [math.cos(t * math.exp(-math.log(10000.0) * k / 128)) for k in range(128)] + \
            [math.sin(t * math.exp(-math.log(10000.0) * k / 128)) for k in range(128)]
        h = [_silu1(v) for v in _vecmat(e, _mat(W, "t_mlp1.w"), W["t_mlp1.b"].tolist())]
        o = _vecmat(h, _mat(W, "t_mlp2.w"), W["t_mlp2.b"].tolist())
        return [o[c] + float(cond[c]) for c in range(len(o))]

    def mod(self, prefix, vec, k):
        sv = [_silu1(v) for v in vec]
        return _chunks(_vecmat(sv, _mat(self.W, prefix + ".mod.w"), self.W[prefix + ".mod.b"].tolist()), k)

    def pos(self, tok):
        """tok = -1 for a text token, else the image token index."""
        if tok < 0:
            return (0, 0, 0)
        return (0, tok // self.d.grid_w, tok % self.d.grid_w)

    def qk(self, prefix, row, tok, is_q):
        d = self.d
        if d.qk_norm:
            row = _rms_heads(row, self.W[prefix + (".q_norm_g" if is_q else ".k_norm_g")].tolist(), d.heads)
        if d.rope:
            row = _rope_row(row, self.pos(tok), d.heads, d.rope_axes, d.rope_theta)
        return row

    def keys(self, fresh_k, fresh_v, toks, kv_cache_blk):
        """Positional merged K/V over all L tokens: text rows, then image 0..L_img-1."""
        d = self.d
        Lt = d.txt_len
        K, V = [None] * d.L, [None] * d.L
        for r, tok in enumerate(toks):
            p = Lt + tok if tok >= 0 else r
            K[p], V[p] = fresh_k[r], fresh_v[r]
        for i in range(d.L_img):
            if K[Lt + i] is None:
                K[Lt + i] = [float(v) for v in kv_cache_blk[0][i]]
                V[Lt + i] = [float(v) for v in kv_cache_blk[1][i]]
        return K, V

    def double(self, i, x_txt, x_img, img_toks, vec, kv_cache_blk):
        d, W = self.d, self.W
        H = d.hidden
        pre_only = bool(d.context_pre_only_last) and i == d.n_double - 1
        streams = [("txt", x_txt, [-1] * len(x_txt)), ("img", x_img, list(img_toks))]
        qs, ks, vs, mods = [], [], [], {}
        for s, X, toks in streams:
            p = f"double.{i}.{s}"
            if s == "txt" and pre_only:
                sc, sh = self.mod(p, vec, 2)
                m = [sh, sc]
            else:
                m = self.mod(p, vec, 6)
            mods[s] = m
            for r, row in enumerate(X):
                h = _ln_mod(row, m[0], m[1])
                qkv = _vecmat(h, _mat(W, p + ".qkv.w"), W[p + ".qkv.b"].tolist())
                qs.append(self.qk(p, qkv[:H], toks[r], True))
                ks.append(self.qk(p, qkv[H:2 * H], toks[r], False))
                vs.append(qkv[2 * H:])
        toks_all = [-1] * len(x_txt) + list(img_toks)
        K, V = self.keys(ks, vs, toks_all, kv_cache_blk)
        o = _attend(qs, K, V, d.heads)
        out = {}
        for s, X, _ in streams:
            p = f"double.{i}.{s}"
            o_s = o[:len(x_txt)] if s == "txt" else o[len(x_txt):]
            if s == "txt" and pre_only:
                out[s] = X
                continue
            m = mods[s]
            new = []
            for r, row in enumerate(X):
                a = _vecmat(o_s[r], _mat(W, p + ".proj.w"), W[p + ".proj.b"].tolist())
                row = [row[c] + m[2][c] * a[c] for c in range(H)]
                z = _ln_mod(row, m[3], m[4])
                u = [_gelu1(v) for v in _vecmat(z, _mat(W, p + ".fc1.w"), W[p + ".fc1.b"].tolist())]
                f = _vecmat(u, _mat(W, p + ".fc2.w"), W[p + ".fc2.b"].tolist())
                new.append([row[c] + m[5][c] * f[c] for c in range(H)])
            out[s] = new
        return out["txt"], out["img"]

    def single(self, i, x, toks, vec, kv_cache_blk):
        d, W = self.d, self.W
        H = d.hidden
        p = f"single.{i}"
        sh, sc, g = self.mod(p, vec, 3)
        qs, ks, vs, us = [], [], [], []
        for r, row in enumerate(x):
            h = _ln_mod(row, sh, sc)
            y = _vecmat(h, _mat(W, p + ".lin1.w"), W[p + ".lin1.b"].tolist())
            qs.append(self.qk(p, y[:H], toks[r], True))
            ks.append(self.qk(p, y[H:2 * H], toks[r], False))
            vs.append(y[2 * H:3 * H])
            us.append(y[3 * H:])
        K, V = self.keys(ks, vs, toks, kv_cache_blk)
        o = _attend(qs, K, V, d.heads)
        out = []
        for r, row in enumerate(x):
            cat = o[r] + [_gelu1(v) for v in us[r]]
            y = _vecmat(cat, _mat(W, p + ".lin2.w"), W[p + ".lin2.b"].tolist())
            out.append([row[c] + g[c] * y[c] for c in range(H)])
        return out

    def step(self, latent, mask, kv_cache_step, sigma, sigma_next, txt, cond):
        """One step on the masked rows (all rows when the mask is all ones)."""
        d, W = self.d, self.W
        toks = [i for i in range(d.L_img) if mask[i]]
        vec = self.vec(sigma, cond)
        x_img = []
        for i in toks:
            row = _vecmat([float(v) for v in latent[i]], _mat(W, "img_in.w"), W["img_in.b"].tolist())
            if d.pos_embed_2d:
                row = [row[c] + float(W["pos_embed"][i][c]) for c in range(d.hidden)]
            x_img.append(row)
        x_txt = [[float(v) for v in r] for r in txt]
        for b in range(d.n_double):
            kvb = kv_cache_step[b] if kv_cache_step is not None else None
            x_txt, x_img = self.double(b, x_txt, x_img, toks, vec, kvb)
        x = x_txt + x_img
        rtoks = [-1] * d.txt_len + toks
        for i in range(d.n_single):
            b = d.n_double + i
            kvb = kv_cache_step[b] if kv_cache_step is not None else None
            x = self.single(i, x, rtoks, vec, kvb)
        sv = [_silu1(v) for v in vec]
        sc, sh = _chunks(_vecmat(sv, _mat(W, "final_mod.w"), W["final_mod.b"].tolist()), 2)
        out = np.array(latent, dtype=np.float64).copy()
        for r, tok in enumerate(toks):
            z = _ln_mod(x[d.txt_len + r], sh, sc)
            v = _vecmat(z, _mat(W, "proj_out.w"), W["proj_out.b"].tolist())
            for c in range(d.lat_ch):
                out[tok][c] = float(latent[tok][c]) + (float(sigma_next) - float(sigma)) * v[c]
        return out


# ---------------------------------------------------------------- models and inputs
FLUXB = synth.ModelDesc("brute_flux", 1, 1, 16, 2, 8, 32, 4, 4, 4, 3, rope_axes=(2, 2, 4))
SD3B = synth.ModelDesc("brute_sd3", 2, 0, 16, 2, 8, 32, 4, 3, 4, 3, qk_norm=0, rope=0,
                       rope_axes=(0, 0, 0), pos_embed_2d=1, context_pre_only_last=1)


def _setup(d, seed=0, rid=5):
    W = {k: v.double().numpy() for k, v in synth.make_weights(d, seed).items()}
    # make modulation (and so the gates, shifts, scales) large enough that a swapped or
    # dropped chunk moves the output far above rounding (the table's x0.1 keeps them small)
    for k in W:
        if k.endswith(".mod.w") or k.startswith("final_mod"):
            W[k] = W[k] * 10.0
    lat = synth.make_latent(d, rid).double().numpy()
    txt = synth.make_txt(d, rid).double().numpy()
    cond = synth.make_cond(d, rid).double().numpy()
    return W, lat, txt, cond


def _close(a, b, tol=1e-11):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b)) <= tol * max(1.0, np.abs(b).max())


@pytest.mark.parametrize("d", [FLUXB, SD3B], ids=["flux", "sd3"])
def test_dense_step_matches_brute_force(d):
    W, lat, txt, cond = _setup(d)
    ref = Brute(d, W).step(lat, np.ones(d.L_img, np.uint8), None, 0.9, 0.55, txt, cond)
    got, _ = oracle.dense_step(d, W, lat, 0.9, 0.55, txt, cond)
    assert _close(got, ref)
    # the step must actually move the latent (not a no-op agreement)
    assert np.max(np.abs(ref - lat)) > 1e-3


@pytest.mark.parametrize("d", [FLUXB, SD3B], ids=["flux", "sd3"])
def test_edit_step_with_foreign_cache_matches_brute_force(d):
    # a cache from OTHER inputs: the merge, positions of masked rows and the text-first key
    # order are all exercised, not only the same-input special case
    W, lat, txt, cond = _setup(d, rid=6)
    kv = synth.make_cache_kv(d, 3, 1).double().numpy()[0]
    mask = np.zeros(d.L_img, np.uint8)
    mask[[1, 4, 5, 9, d.L_img - 1]] = 1
    ref = Brute(d, W).step(lat, mask, kv, 0.7, 0.4, txt, cond)
    got = oracle.edit_step(d, W, lat, mask, kv, 0.7, 0.4, txt, cond)
    assert _close(got, ref)
    assert np.array_equal(got[mask == 0], lat[mask == 0])


def test_masked_blocks_match_brute_force():
    d = FLUXB
    W, lat, txt, cond = _setup(d, rid=7)
    kv = synth.make_cache_kv(d, 4, 1).double().numpy()[0]
    idx_m = np.array([0, 3, 6, 7, 12])
    idx_u = np.setdiff1d(np.arange(d.L_img), idx_m)
    rng = np.random.default_rng(0)
    x_txt = rng.standard_normal((d.txt_len, d.hidden))
    x_img = rng.standard_normal((len(idx_m), d.hidden))
    br = Brute(d, W)
    vec = oracle.conditioning(W, 0.6, cond)
    assert _close(vec, br.vec(0.6, cond))
    t1, i1 = oracle.double_block_masked(d, W, 0, x_txt, x_img, vec, idx_m, idx_u, kv[0])
    t2, i2 = br.double(0, x_txt.tolist(), x_img.tolist(), list(idx_m), vec.tolist(), kv[0])
    assert _close(t1, t2) and _close(i1, i2)
    x = np.concatenate([x_txt, x_img])
    s1 = oracle.single_block_masked(d, W, 0, x, vec, idx_m, idx_u, kv[1])
    s2 = br.single(0, x.tolist(), [-1] * d.txt_len + list(idx_m), vec.tolist(), kv[1])
    assert _close(s1, s2)


def test_recorded_cache_matches_brute_force_keys():
    # cache_template records K/V post-norm, post-RoPE (C-AMB 2): recompute block 0's image
    # keys by the brute-force path and compare
    d = FLUXB
    W, lat, txt, cond = _setup(d, rid=8)
    _, cache, _ = oracle.cache_template(d, W, lat, txt, cond, [0.8, 0.5])
    br = Brute(d, W)
    vec = br.vec(0.8, cond)
    m = br.mod("double.0.img", vec, 6)
    H = d.hidden
    for i in range(d.L_img):
        row = _vecmat(lat[i].tolist(), _mat(W, "img_in.w"), W["img_in.b"].tolist())
        h = _ln_mod(row, m[0], m[1])
        qkv = _vecmat(h, _mat(W, "double.0.img.qkv.w"), W["double.0.img.qkv.b"].tolist())
        assert _close(cache[0, 0, 0, i], br.qk("double.0.img", qkv[H:2 * H], i, False))
        assert _close(cache[0, 0, 1, i], qkv[2 * H:])


# ---------------------------------------------------------------- mutation kill test
def _mut_swap_shift_scale(mp):
    orig = oi.modulation
    mp.setattr(oi, "modulation", lambda W, p, vec, k: (lambda c: [c[1], c[0]] + c[2:])(orig(W, p, vec, k)))


def _mut_sigma_not_1000(mp):
    orig = oi.sinusoid
    mp.setattr(oi, "sinusoid", lambda t, dim=256: orig(t / 1000.0, dim))


def _mut_grid_axes(mp):
    mp.setattr(oi, "image_positions",
               lambda d, idx: np.stack([np.zeros_like(idx), idx % d.grid_w, idx // d.grid_w], axis=1))


def _mut_final_chunks(mp):
    orig = oi._final_mod
    mp.setattr(oi, "_final_mod", lambda W, vec: orig(W, vec)[::-1])


def _mut_no_one_plus_scale(mp):
    # h = LN(x) scale + shift instead of LN(x)(1 + scale) + shift
    orig = oi._qkv_stream
    mp.setattr(oi, "_qkv_stream", lambda d, W, p, x, mods, pos, flags:
               orig(d, W, p, x, [mods[0], mods[1] - 1.0] + list(mods[2:]), pos, flags))


def _mut_concat_order(mp):
    # [GELU(u) | o] W_2 instead of [o | GELU(u)] W_2
    def bad(d, W, p, x, o, u, mods):
        y = oi.linear(np.concatenate([oi.gelu_tanh(u), o], axis=1), W[p + ".lin2.w"], W[p + ".lin2.b"])
        return x + mods[2] * y
    mp.setattr(oi, "_single_out", bad)


def _mut_gate_before_bias(mp):
    # x += g (o W_o) + b instead of x += g (o W_o + b): shift the bias out of the gate
    orig = oi._double_out

    def bad(d, W, p, x, o, mods, flags):
        Wb = dict(W)
        Wb[p + ".proj.b"] = np.zeros_like(W[p + ".proj.b"])
        return orig(d, Wb, p, x + W[p + ".proj.b"], o, mods, flags)
    mp.setattr(oi, "_double_out", bad)


MUTATIONS = {
    "swap_shift_scale": _mut_swap_shift_scale,
    "sigma_not_1000sigma": _mut_sigma_not_1000,
    "swapped_grid_axes": _mut_grid_axes,
    "swapped_final_chunks": _mut_final_chunks,
    "dropped_one_plus_scale": _mut_no_one_plus_scale,
    "gelu_o_concat_order": _mut_concat_order,
    "gate_before_bias": _mut_gate_before_bias,
}


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_mutations_are_caught(name, monkeypatch):
    d = FLUXB
    W, lat, txt, cond = _setup(d, rid=9)
    ref = Brute(d, W).step(lat, np.ones(d.L_img, np.uint8), None, 0.9, 0.55, txt, cond)
    MUTATIONS[name](monkeypatch)
    got, _ = oracle.dense_step(d, W, lat, 0.9, 0.55, txt, cond)
    assert not _close(got, ref), f"mutation {name} not detected by the brute-force pin"
