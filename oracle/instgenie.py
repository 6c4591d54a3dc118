"""ORACLE (test infrastructure only) — float64 NumPy reference of the mask-aware step.

What it computes, and where the paper says so
---------------------------------------------
* Token mask -> ascending masked/unmasked index lists ("mask ... encoded into
  latent space"; "extract the matrix of masked tokens").               index_build
* Token-wise ops (projections, feed-forward, LayerNorm, GELU) run on masked rows only
  ("for these token-wise operations, we can precisely differentiate the
  computations of the masked tokens and the unmasked tokens").       linear, layernorm, ...
* K/V-caching variant (fig:transformer_alter): masked tokens get fresh K,V;
  unmasked tokens' K,V come from the template cache; masked Q attends to all tokens
  ("Q ... of only the newly generated token along with the K and V
  matrices of all present tokens").                                 merge_kv, attention
* Scaled dot-product attention softmax(Q K^T / sqrt(d)) V (C-AMB 4: d is
  the head dimension).                                                          attention
* Table 1 cost model: every projection / FF MAC scales with the number of
  query rows, attention with query rows x L.                       MACS counter, macs_*
* Dense step (no cache, all L tokens; fig:transformer-Top P:387-402) with K/V recording
  = the template cache ("pre-computed activations from previous requests").
                                                                     dense_step(record=)
* Y-caching variant (fig:transformer-Bottom): the cache holds the
  template's block outputs Y of the image tokens; unmasked rows of each block's input are
  replenished from it and only feed K/V.        kv_from_y, edit_step_y, cache_template_y
  A hybrid cache keeps K/V for some blocks and Y for the others.     edit_step_y(y_blocks=)
* Algorithm 1 dense prefix (C-AMB 23).            edit_step_planned, edit_step_y(k=)
Readings where the paper is silent (Flux-shaped blocks, adaLN, QK-RMSNorm, RoPE,
GELU-tanh, flow-matching Euler, row order) are the numbered C-AMB readings in DESIGN.md
(SURVEY §8(c)).  Everything is float64; inputs are the exact fp32/bf16 values.

Pins: tests/test_oracle.py (closed forms, the worked example in tests/golden/, textbook
library routines, brute force, exactness invariants).  Parity-unpinned: none of the
functions below; the *approximation quality* of a cache from other inputs is unpinned
(the paper pins it only with trained-model image metrics) and is not claimed.
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np

# Multiply-accumulate counter for the Table 1 pin.  Reset by the caller.
MACS = {"linear": 0, "attn": 0}


def reset_macs():
    MACS["linear"] = 0
    MACS["attn"] = 0


# --------------------------------------------------------------------------------------
# a1. Index build (C-AMB 13-16)
# --------------------------------------------------------------------------------------
def index_build(mask) -> Tuple[np.ndarray, np.ndarray, int]:
    """idx_m = ascending token indices with mask != 0, idx_u = the complement, n_m."""
    mask = np.asarray(mask).reshape(-1)
    idx_m, idx_u = [], []
    for i in range(mask.shape[0]):
        if mask[i] != 0:
            idx_m.append(i)
        else:
            idx_u.append(i)
    return (np.array(idx_m, dtype=np.int64), np.array(idx_u, dtype=np.int64), len(idx_m))


# --------------------------------------------------------------------------------------
# Token-wise primitives
# --------------------------------------------------------------------------------------
def linear(x: np.ndarray, W: np.ndarray, b: Optional[np.ndarray]) -> np.ndarray:
    """y = x W^T + b with W stored [out, in] (weight-table convention)."""
    MACS["linear"] += x.shape[0] * W.shape[0] * W.shape[1]
    y = x @ W.T
    return y + b if b is not None else y


def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    """C-AMB 6: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))."""
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def layernorm(x, eps):
    """LayerNorm without affine (C-AMB 6): (x - mean) / sqrt(var + eps), biased var."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


def rmsnorm_heads(x, g, heads, eps):
    """Per-head RMSNorm with learned gain g[d] (C-AMB 6)."""
    n, H = x.shape
    xh = x.reshape(n, heads, H // heads)
    r = np.sqrt((xh ** 2).mean(axis=-1, keepdims=True) + eps)
    return (xh / r * g).reshape(n, H)


def rope(x, pos, heads, axes, theta):
    """3-axis rotary embedding (C-AMB 7).  pos: [n, 3] integer positions.

    Head dim split into consecutive axis chunks of widths axes[a]; in chunk a, pair j =
    dims (2j, 2j+1) rotates by phi = pos_a * theta^(-2j/axes[a])."""
    n, H = x.shape
    dh = H // heads
    xh = x.reshape(n, heads, dh).copy()
    off = 0
    for a, da in enumerate(axes):
        for j in range(da // 2):
            w = theta ** (-2.0 * j / da)
            phi = pos[:, a].astype(np.float64) * w
            c, s = np.cos(phi)[:, None], np.sin(phi)[:, None]
            x0 = xh[:, :, off + 2 * j].copy()
            x1 = xh[:, :, off + 2 * j + 1].copy()
            xh[:, :, off + 2 * j] = x0 * c - x1 * s
            xh[:, :, off + 2 * j + 1] = x0 * s + x1 * c
        off += da
    return xh.reshape(n, H)


def attention(q, K, V, heads):
    """Per head j: O = softmax(q_j K_j^T / sqrt(d)) V_j (C-AMB 4, 19).

    q: [n, H] query rows; K, V: [L, H] all tokens; softmax subtracts the row max."""
    n, H = q.shape
    L = K.shape[0]
    dh = H // heads
    MACS["attn"] += 2 * n * L * H
    out = np.empty((n, H))
    for j in range(heads):
        sl = slice(j * dh, (j + 1) * dh)
        S = q[:, sl] @ K[:, sl].T / math.sqrt(dh)
        S = S - S.max(axis=1, keepdims=True)
        P = np.exp(S)
        P = P / P.sum(axis=1, keepdims=True)
        out[:, sl] = P @ V[:, sl]
    return out


# --------------------------------------------------------------------------------------
# a3. Conditioning (C-ALG 2; C-AMB readings, Flux convention)
# --------------------------------------------------------------------------------------
def sinusoid(t: float, dim: int = 256) -> np.ndarray:
    """[cos(t f_k) | sin(t f_k)], f_k = exp(-ln(10000) k / (dim/2)) — cos first."""
    half = dim // 2
    k = np.arange(half, dtype=np.float64)
    f = np.exp(-math.log(10000.0) * k / half)
    return np.concatenate([np.cos(t * f), np.sin(t * f)])


def conditioning(W, sigma: float, cond_vec: np.ndarray) -> np.ndarray:
    """vec = MLP_t(sinusoid(1000 sigma)) + cond_vec (C-AMB 12: t = 1000 sigma)."""
    e = sinusoid(1000.0 * float(sigma))[None, :]
    h = silu(linear(e, W["t_mlp1.w"], W["t_mlp1.b"]))
    return (linear(h, W["t_mlp2.w"], W["t_mlp2.b"]) + cond_vec[None, :])[0]


def modulation(W, prefix: str, vec: np.ndarray, k: int):
    """k chunks of SiLU(vec) W_mod^T + b, each [H]."""
    m = linear(silu(vec)[None, :], W[prefix + ".mod.w"], W[prefix + ".mod.b"])[0]
    return np.split(m, k)


def image_positions(d, idx: np.ndarray) -> np.ndarray:
    """RoPE positions of image tokens: (0, i div W, i mod W) (C-AMB 7)."""
    return np.stack([np.zeros_like(idx), idx // d.grid_w, idx % d.grid_w], axis=1)


# --------------------------------------------------------------------------------------
# Blocks.  `flags` switch the Flux-shaped token-wise extras off for the SPEC reduction
# (C-AMB 5): adaln (LN + modulate), residual (+ gates), gelu, norm (QK-RMSNorm), rope.
# --------------------------------------------------------------------------------------
FLUX_FLAGS = dict(adaln=True, residual=True, gelu=True)


def _qkv_stream(d, W, p, x, mods, pos, flags):
    """h = LN(x)(1+scale)+shift; [q|k|v] = h W_qkv^T + b; QK-RMSNorm; RoPE."""
    H = d.hidden
    if flags["adaln"]:
        shift, scale = mods[0], mods[1]
        h = layernorm(x, d.ln_eps) * (1.0 + scale) + shift
    else:
        h = x
    qkv = linear(h, W[p + ".qkv.w"], W.get(p + ".qkv.b"))
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]
    if d.qk_norm:
        q = rmsnorm_heads(q, W[p + ".q_norm_g"], d.heads, 1e-6)
        k = rmsnorm_heads(k, W[p + ".k_norm_g"], d.heads, 1e-6)
    if d.rope:
        q = rope(q, pos, d.heads, d.rope_axes, d.rope_theta)
        k = rope(k, pos, d.heads, d.rope_axes, d.rope_theta)
    return q, k, v


def _double_out(d, W, p, x, o, mods, flags):
    """x += g1 (o W_o^T + b); x += g2 MLP(LN(x)(1+sc2)+sh2) (Flux double-stream block)."""
    y = linear(o, W[p + ".proj.w"], W.get(p + ".proj.b"))
    if flags["residual"]:
        x = x + mods[2] * y
    else:
        x = y
    if flags["adaln"]:
        z = layernorm(x, d.ln_eps) * (1.0 + mods[4]) + mods[3]
    else:
        z = x
    u = linear(z, W[p + ".fc1.w"], W.get(p + ".fc1.b"))
    if flags["gelu"]:
        u = gelu_tanh(u)
    f = linear(u, W[p + ".fc2.w"], W.get(p + ".fc2.b"))
    return x + mods[5] * f if flags["residual"] else f


def _single_pre(d, W, p, x, mods, pos):
    H = d.hidden
    h = layernorm(x, d.ln_eps) * (1.0 + mods[1]) + mods[0]
    y = linear(h, W[p + ".lin1.w"], W[p + ".lin1.b"])
    q, k, v, u = y[:, :H], y[:, H:2 * H], y[:, 2 * H:3 * H], y[:, 3 * H:]
    if d.qk_norm:
        q = rmsnorm_heads(q, W[p + ".q_norm_g"], d.heads, 1e-6)
        k = rmsnorm_heads(k, W[p + ".k_norm_g"], d.heads, 1e-6)
    if d.rope:
        q = rope(q, pos, d.heads, d.rope_axes, d.rope_theta)
        k = rope(k, pos, d.heads, d.rope_axes, d.rope_theta)
    return q, k, v, u


def _single_out(d, W, p, x, o, u, mods):
    """x += g ([o | GELU(u)] W_2^T + b)."""
    y = linear(np.concatenate([o, gelu_tanh(u)], axis=1), W[p + ".lin2.w"], W[p + ".lin2.b"])
    return x + mods[2] * y


def merge_kv(d, k_txt, k_img_fresh, idx_m, idx_u, k_cache_img):
    """Positional merge by mask index (C-ALG 4 'Merge'; C-AMB 8):
    rows [0, L_txt) <- fresh text K; row L_txt+i <- fresh K for i in idx_m, cached K for
    i in idx_u."""
    L_txt = d.txt_len
    K = np.zeros((d.L, k_img_fresh.shape[1]))
    K[:L_txt] = k_txt
    K[L_txt + idx_m] = k_img_fresh
    if len(idx_u):
        K[L_txt + idx_u] = k_cache_img[idx_u]
    return K


def _is_pre_only(d, i, stream):
    return bool(d.context_pre_only_last) and stream == "txt" and i == d.n_double - 1


# --------------------------------------------------------------------------------------
# The masked step (C-ALG 1-6), one request.
# --------------------------------------------------------------------------------------
def double_block_masked(d, W, i, x_txt, x_img, vec, idx_m, idx_u, kv_cache_blk, flags=FLUX_FLAGS):
    """One double-stream block on [txt | masked img] rows with K/V merge.

    kv_cache_blk: [2, L_img, H] cached (K, V) of this (step, block); may be None when
    idx_u is empty.  Returns (x_txt, x_img)."""
    pi, pt = f"double.{i}.img", f"double.{i}.txt"
    pos_img = image_positions(d, idx_m)
    pos_txt = np.zeros((d.txt_len, 3), np.int64)
    mi = modulation(W, pi, vec, 6) if flags["adaln"] else None
    qi, ki, vi = _qkv_stream(d, W, pi, x_img, mi, pos_img, flags)
    pre_only = _is_pre_only(d, i, "txt")
    if d.txt_len:
        mt = modulation(W, pt, vec, 2 if pre_only else 6) if flags["adaln"] else None
        if pre_only:  # AdaLayerNormContinuous order (scale, shift)
            mt = [mt[1], mt[0]]
        qt, kt, vt = _qkv_stream(d, W, pt, x_txt, mt, pos_txt, flags)
    else:
        qt = kt = vt = np.zeros((0, d.hidden))
    kc = kv_cache_blk[0] if kv_cache_blk is not None else None
    vc = kv_cache_blk[1] if kv_cache_blk is not None else None
    K = merge_kv(d, kt, ki, idx_m, idx_u, kc)
    V = merge_kv(d, vt, vi, idx_m, idx_u, vc)
    o = attention(np.concatenate([qt, qi]), K, V, d.heads)
    ot, oi = o[:d.txt_len], o[d.txt_len:]
    x_img = _double_out(d, W, pi, x_img, oi, mi, flags)
    if d.txt_len and not pre_only:
        x_txt = _double_out(d, W, pt, x_txt, ot, mt, flags)
    return x_txt, x_img


def single_block_masked(d, W, i, x, vec, idx_m, idx_u, kv_cache_blk):
    """One single-stream block on rows [txt | masked img] (C-ALG 5)."""
    p = f"single.{i}"
    pos = np.concatenate([np.zeros((d.txt_len, 3), np.int64), image_positions(d, idx_m)])
    m = modulation(W, p, vec, 3)
    q, k, v, u = _single_pre(d, W, p, x, m, pos)
    Lt = d.txt_len
    kc = kv_cache_blk[0] if kv_cache_blk is not None else None
    vc = kv_cache_blk[1] if kv_cache_blk is not None else None
    K = merge_kv(d, k[:Lt], k[Lt:], idx_m, idx_u, kc)
    V = merge_kv(d, v[:Lt], v[Lt:], idx_m, idx_u, vc)
    o = attention(q, K, V, d.heads)
    return _single_out(d, W, p, x, o, u, m)


def img_in(d, W, latent, idx):
    x = linear(latent[idx], W["img_in.w"], W["img_in.b"])
    if d.pos_embed_2d:
        x = x + W["pos_embed"][idx]
    return x


def final_velocity(d, W, x_img, vec):
    """v = (LN(x)(1+scale)+shift) W_out^T + b (final adaLN: chunk order (scale, shift))."""
    sc, sh = _final_mod(W, vec)
    return linear(layernorm(x_img, d.ln_eps) * (1.0 + sc) + sh, W["proj_out.w"], W["proj_out.b"])


def _final_mod(W, vec):
    m = linear(silu(vec)[None, :], W["final_mod.w"], W["final_mod.b"])[0]
    return np.split(m, 2)


def edit_step(d, W, latent, mask, kv_cache_step, sigma, sigma_next, txt, cond_vec):
    """One mask-aware denoising step for one request (C-ALG 1-6).

    latent: [L_img, C]; mask: [L_img] uint8; kv_cache_step: [blocks, 2, L_img, H] cached
    K/V of this step (None allowed only if the mask is all ones).  Returns the new latent:
    masked rows get latent += (sigma_next - sigma) v (C-AMB 12); all other rows are the
    input rows unchanged (C-AMB 11)."""
    latent = np.asarray(latent, np.float64)
    idx_m, idx_u, n_m = index_build(mask)
    if n_m == 0:
        return latent.copy()
    if len(idx_u) and kv_cache_step is None:
        raise KeyError("cache-miss: 0 < n_m < L_img needs a cache entry (S:134)")
    vec = conditioning(W, sigma, np.asarray(cond_vec, np.float64))
    x_img = img_in(d, W, latent, idx_m)
    x_txt = np.asarray(txt, np.float64).copy()
    for i in range(d.n_double):
        kv = kv_cache_step[i] if len(idx_u) else None
        x_txt, x_img = double_block_masked(d, W, i, x_txt, x_img, vec, idx_m, idx_u, kv)
    x = np.concatenate([x_txt, x_img])
    for i in range(d.n_single):
        kv = kv_cache_step[d.n_double + i] if len(idx_u) else None
        x = single_block_masked(d, W, i, x, vec, idx_m, idx_u, kv)
    v = final_velocity(d, W, x[d.txt_len:], vec)
    out = latent.copy()
    out[idx_m] = latent[idx_m] + (float(sigma_next) - float(sigma)) * v
    return out


def edit_step_planned(d, W, latent, mask, kv_cache_step, tlatent, k, sigma, sigma_next, txt, cond_vec):
    """Algorithm 1 plan under the K/V variant (C-AMB 23): blocks [0, k) use no
    cached activations ("computes all tokens — both masked and unmasked — without
    distinguishing between them"), blocks [k, N) use the cache.  Under K/V caching
    the dense blocks must form a prefix (a cached block does not produce the unmasked rows'
    hidden states), and the unmasked image tokens enter the prefix from the TEMPLATE's input
    latent at this step (`tlatent`), the trajectory the cache was recorded on.  After block
    k-1 the unmasked rows are dropped; their K/V come from the cache from block k on."""
    latent = np.asarray(latent, np.float64)
    idx_m, idx_u, n_m = index_build(mask)
    if n_m == 0:
        return latent.copy()
    if k <= 0 or len(idx_u) == 0:
        return edit_step(d, W, latent, mask, kv_cache_step, sigma, sigma_next, txt, cond_vec)
    k = min(k, d.n_blocks)
    vec = conditioning(W, sigma, np.asarray(cond_vec, np.float64))
    full = latent.copy()
    full[idx_u] = np.asarray(tlatent, np.float64)[idx_u]
    all_idx = np.arange(d.L_img)
    none = np.zeros(0, np.int64)
    x_img = img_in(d, W, full, all_idx)
    x_txt = np.asarray(txt, np.float64).copy()
    x = None
    for b in range(d.n_blocks):
        dense = b < k
        if dense:  # the all-tokens block = the masked block with every token masked
            if b < d.n_double:
                x_txt, x_img = double_block_masked(d, W, b, x_txt, x_img, vec, all_idx, none, None)
            else:
                if x is None:
                    x = np.concatenate([x_txt, x_img])
                x = single_block_masked(d, W, b - d.n_double, x, vec, all_idx, none, None)
            if b == k - 1:  # switch: keep only the masked image rows
                if x is None:
                    x_img = x_img[idx_m]
                else:
                    x = np.concatenate([x[:d.txt_len], x[d.txt_len:][idx_m]])
        else:
            if b < d.n_double:
                x_txt, x_img = double_block_masked(d, W, b, x_txt, x_img, vec, idx_m, idx_u, kv_cache_step[b])
            else:
                if x is None:
                    x = np.concatenate([x_txt, x_img])
                x = single_block_masked(d, W, b - d.n_double, x, vec, idx_m, idx_u, kv_cache_step[b])
    if x is None:
        x = np.concatenate([x_txt, x_img])
    v = final_velocity(d, W, x[d.txt_len:], vec)
    out = latent.copy()
    out[idx_m] = latent[idx_m] + (float(sigma_next) - float(sigma)) * v
    return out


# --------------------------------------------------------------------------------------
# Y-caching variant (fig:transformer-Bottom; SPEC forward_masked_ycache S:113-121;
# SURVEY N2).  The cache holds Y_b = the template's block-b OUTPUT rows of the image tokens.
# Block b's input X holds every token: the masked rows computed by this request, the unmasked
# rows "replenished" from the cache (Y_{b-1}; for b = 0 the template's block input
# img_in(template latent) — C-AMB 23's reading of the unmasked tokens' trajectory).  K and V
# come from the full X ("K and V computed from full x"); Q, the attention output and
# every later token-wise op only from the masked rows ("project it into Q, and compute an Y
# matrix exclusively for the masked tokens").
# --------------------------------------------------------------------------------------
def kv_from_y(d, W, b, x_u, vec, idx_u):
    """K, V of the unmasked tokens recomputed from their block input rows x_u [n_u, H] with
    THIS request's modulation and block-b weights; returned positionally as a [2, L_img, H]
    array (rows idx_u filled), i.e. the K/V variant's cache slice that the Y variant implies."""
    kv = np.zeros((2, d.L_img, d.hidden))
    if len(idx_u) == 0:
        return kv
    pos = image_positions(d, idx_u)
    if b < d.n_double:
        p = f"double.{b}.img"
        _, k, v = _qkv_stream(d, W, p, x_u, modulation(W, p, vec, 6), pos, FLUX_FLAGS)
    else:
        p = f"single.{b - d.n_double}"
        _, k, v, _ = _single_pre(d, W, p, x_u, modulation(W, p, vec, 3), pos)
    kv[0][idx_u], kv[1][idx_u] = k, v
    return kv


def edit_step_y(d, W, latent, mask, y_cache_step, tlatent, sigma, sigma_next, txt, cond_vec, k=0,
                y_blocks=None, kv_cache_step=None):
    """One mask-aware step under the Y variant, with an optional Algorithm-1 dense prefix of k
    blocks.  y_cache_step: [blocks, L_img, H] = Y_b of the template at this step;
    tlatent: the template's input latent of this step [L_img, C].  A block whose predecessor
    ran densely takes its unmasked input rows from that computation; otherwise from Y_{b-1}
    (block 0: img_in(tlatent)).  Latent update and untouched rows as in edit_step.
    Hybrid cache (DESIGN reading 30): only the blocks in y_blocks (None = all) are Y-variant
    blocks; the others are K/V-variant blocks on kv_cache_step[b]."""
    latent = np.asarray(latent, np.float64)
    idx_m, idx_u, n_m = index_build(mask)
    if n_m == 0:
        return latent.copy()
    if len(idx_u) == 0:
        return edit_step(d, W, latent, mask, None, sigma, sigma_next, txt, cond_vec)
    if y_cache_step is None:
        raise KeyError("cache-miss: 0 < n_m < L_img needs a cache entry (S:134)")
    k = max(0, min(k, d.n_blocks))
    vec = conditioning(W, sigma, np.asarray(cond_vec, np.float64))
    full = latent.copy()
    full[idx_u] = np.asarray(tlatent, np.float64)[idx_u]
    all_idx = np.arange(d.L_img)
    none = np.zeros(0, np.int64)
    Lt = d.txt_len
    x_txt = np.asarray(txt, np.float64).copy()
    x = None  # single-stream rows [txt | img]
    if k > 0:
        x_img = img_in(d, W, full, all_idx)
    else:
        x_img = img_in(d, W, latent, idx_m)
    x_u = img_in(d, W, full, idx_u)  # block-0 input of the unmasked tokens
    for b in range(d.n_blocks):
        if b < k:  # dense block: every token, no cache
            if b < d.n_double:
                x_txt, x_img = double_block_masked(d, W, b, x_txt, x_img, vec, all_idx, none, None)
            else:
                if x is None:
                    x = np.concatenate([x_txt, x_img])
                x = single_block_masked(d, W, b - d.n_double, x, vec, all_idx, none, None)
            if b == k - 1:  # unmasked rows leave the row set; their output feeds block k
                rows = x_img if x is None else x[Lt:]
                x_u = rows[idx_u]
                if x is None:
                    x_img = x_img[idx_m]
                else:
                    x = np.concatenate([x[:Lt], x[Lt:][idx_m]])
            continue
        if y_blocks is not None and b not in y_blocks:  # K/V-variant block of a hybrid cache
            kv = kv_cache_step[b]
        else:
            if b > k:  # predecessor used the cache: replenish from Y_{b-1}
                x_u = np.asarray(y_cache_step[b - 1], np.float64)[idx_u]
            kv = kv_from_y(d, W, b, x_u, vec, idx_u)
        if b < d.n_double:
            x_txt, x_img = double_block_masked(d, W, b, x_txt, x_img, vec, idx_m, idx_u, kv)
        else:
            if x is None:
                x = np.concatenate([x_txt, x_img])
            x = single_block_masked(d, W, b - d.n_double, x, vec, idx_m, idx_u, kv)
    if x is None:
        x = np.concatenate([x_txt, x_img])
    v = final_velocity(d, W, x[Lt:], vec)
    out = latent.copy()
    out[idx_m] = latent[idx_m] + (float(sigma_next) - float(sigma)) * v
    return out


# --------------------------------------------------------------------------------------
# Dense step (independent code path: all L tokens, no index lists, no cache) + recording
# --------------------------------------------------------------------------------------
def dense_step(d, W, latent, sigma, sigma_next, txt, cond_vec, record: bool = False,
               record_y: bool = False):
    """Textbook full-token step (fig:transformer-Top).  Returns (new_latent, kv) where
    kv[b] = (K_img, V_img) [2, L_img, H] exactly as consumed by attention (post-norm,
    post-RoPE; C-AMB 2) when record=True.  With record_y, returns (new_latent, kv, y) where
    y[b] = the image tokens' rows of block b's output (the Y matrix of fig:transformer)."""
    latent = np.asarray(latent, np.float64)
    L_img, Lt, H = d.L_img, d.txt_len, d.hidden
    vec = conditioning(W, sigma, np.asarray(cond_vec, np.float64))
    x_img = linear(latent, W["img_in.w"], W["img_in.b"])
    if d.pos_embed_2d:
        x_img = x_img + W["pos_embed"]
    x_txt = np.asarray(txt, np.float64).copy()
    all_idx = np.arange(L_img)
    pos_img = image_positions(d, all_idx)
    pos_all = np.concatenate([np.zeros((Lt, 3), np.int64), pos_img])
    kv = np.zeros((d.n_blocks, 2, L_img, H)) if record else None
    y = np.zeros((d.n_blocks, L_img, H)) if record_y else None
    for i in range(d.n_double):
        pi, pt = f"double.{i}.img", f"double.{i}.txt"
        mi = modulation(W, pi, vec, 6)
        qi, ki, vi = _qkv_stream(d, W, pi, x_img, mi, pos_img, FLUX_FLAGS)
        pre_only = _is_pre_only(d, i, "txt")
        if Lt:
            mt = modulation(W, pt, vec, 2 if pre_only else 6)
            if pre_only:
                mt = [mt[1], mt[0]]
            qt, kt, vt = _qkv_stream(d, W, pt, x_txt, mt, pos_all[:Lt], FLUX_FLAGS)
        else:
            qt = kt = vt = np.zeros((0, H))
        K = np.concatenate([kt, ki])
        V = np.concatenate([vt, vi])
        if record:
            kv[i, 0], kv[i, 1] = ki, vi
        o = attention(np.concatenate([qt, qi]), K, V, d.heads)
        x_img = _double_out(d, W, pi, x_img, o[Lt:], mi, FLUX_FLAGS)
        if Lt and not pre_only:
            x_txt = _double_out(d, W, pt, x_txt, o[:Lt], mt, FLUX_FLAGS)
        if record_y:
            y[i] = x_img
    x = np.concatenate([x_txt, x_img])
    for i in range(d.n_single):
        p = f"single.{i}"
        m = modulation(W, p, vec, 3)
        q, k, v, u = _single_pre(d, W, p, x, m, pos_all)
        if record:
            kv[d.n_double + i, 0], kv[d.n_double + i, 1] = k[Lt:], v[Lt:]
        o = attention(q, k, v, d.heads)
        x = _single_out(d, W, p, x, o, u, m)
        if record_y:
            y[d.n_double + i] = x[Lt:]
    vel = final_velocity(d, W, x[Lt:], vec)
    if record_y:
        return latent + (float(sigma_next) - float(sigma)) * vel, kv, y
    return latent + (float(sigma_next) - float(sigma)) * vel, kv


def cache_template(d, W, latent, txt, cond_vec, sigmas):
    """Dense sampler over the template's own schedule, recording every (step, block) K/V
    (C-AMB 10).  Returns (final_latent, cache[steps, blocks, 2, L_img, H], trajectory)."""
    n = len(sigmas) - 1
    cache = np.zeros((n, d.n_blocks, 2, d.L_img, d.hidden))
    traj = [np.asarray(latent, np.float64).copy()]
    x = traj[0]
    for s in range(n):
        x, kv = dense_step(d, W, x, sigmas[s], sigmas[s + 1], txt, cond_vec, record=True)
        cache[s] = kv
        traj.append(x.copy())
    return x, cache, traj


def cache_template_y(d, W, latent, txt, cond_vec, sigmas):
    """Y-variant recording over the template's own schedule: returns (final_latent,
    ycache[steps, blocks, L_img, H], trajectory)."""
    n = len(sigmas) - 1
    cache = np.zeros((n, d.n_blocks, d.L_img, d.hidden))
    traj = [np.asarray(latent, np.float64).copy()]
    x = traj[0]
    for s in range(n):
        x, _, y = dense_step(d, W, x, sigmas[s], sigmas[s + 1], txt, cond_vec, record_y=True)
        cache[s] = y
        traj.append(x.copy())
    return x, cache, traj


# --------------------------------------------------------------------------------------
# SPEC reduced block, single head, row-vector convention x W
# --------------------------------------------------------------------------------------
def reduced_forward_full(x, Wq, Wk, Wv, Wo, W1, W2):
    """y = FF(Attn(x)): Attn = softmax(Q K^T / sqrt(H)) V W_o, FF = (. W1) W2."""
    Q, K, V = x @ Wq, x @ Wk, x @ Wv
    y = attention(Q, K, V, 1) @ Wo
    return (y @ W1) @ W2, K, V


def reduced_forward_masked_kvcache(x, mask, K_cache, V_cache, Wq, Wk, Wv, Wo, W1, W2):
    """masked rows computed with fresh K/V for masked tokens and cached K/V for
    unmasked ones; returns the masked rows [n_m, H] in ascending token order."""
    idx_m, idx_u, _ = index_build(mask)
    xm = x[idx_m]
    K = np.zeros_like(K_cache)
    V = np.zeros_like(V_cache)
    K[idx_m], V[idx_m] = xm @ Wk, xm @ Wv
    K[idx_u], V[idx_u] = K_cache[idx_u], V_cache[idx_u]
    y = attention(xm @ Wq, K, V, 1) @ Wo
    return (y @ W1) @ W2


# --------------------------------------------------------------------------------------
# FP8 (e4m3) K/V cache, SURVEY N4 (a byte reducer for the cache, not in the paper): the
# quantize-dequantize round trip the attention then consumes, mirrored in float32 exactly:
# per (token, head) scale = amax / 448, q = e4m3 round-to-nearest-even of x / scale
# (saturating at 448; subnormal quantum 2^-9), x' = bf16(q * scale).
# --------------------------------------------------------------------------------------
def e4m3_round(y: np.ndarray) -> np.ndarray:
    """Nearest e4m3 (fn) value, ties to even, saturating at +-448 (float32 in/out)."""
    y = np.asarray(y, np.float32)
    a = np.minimum(np.abs(y).astype(np.float64), 448.0)
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.clip(e, -6, 8)                     # normal exponents; below 2^-6 the quantum is 2^-9
    quantum = 2.0 ** (e - 3)                  # 3 mantissa bits
    q = a / quantum
    r = np.floor(q + 0.5)
    tie = (q + 0.5) == r                      # exact .5 -> round to even
    r = np.where(tie & (r % 2 == 1), r - 1, r)
    out = np.minimum(r * quantum, 448.0)
    return (np.sign(y) * out).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 (round to nearest even) -> float32."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def fp8_kv_roundtrip(kv: np.ndarray, heads: int) -> np.ndarray:
    """kv [..., L, H] (bf16 values) -> the bf16 values attention reads from an FP8 cache."""
    x = np.asarray(kv, np.float32)
    shp = x.shape
    xh = x.reshape(shp[:-1] + (heads, shp[-1] // heads))
    amax = np.abs(xh).max(axis=-1, keepdims=True).astype(np.float32)
    scale = np.where(amax > 0, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)
    q = e4m3_round((xh / scale).astype(np.float32))
    deq = (q * scale).astype(np.float32)
    return bf16_round(deq).reshape(shp).astype(np.float64)


# --------------------------------------------------------------------------------------
# Table 1 closed forms for the Flux-shaped model, per query row per step
# --------------------------------------------------------------------------------------
def macs_per_row_linear(d) -> int:
    """Per query row per step: projections + FF of every block (double blocks per stream
    row, single blocks), excluding img_in/final/modulation (per-request terms)."""
    H, F = d.hidden, d.mlp_hidden
    dbl = H * (3 * H) + H * H + H * F + F * H
    sgl = H * (3 * H + F) + (H + F) * H
    return d.n_double * dbl + d.n_single * sgl


def macs_per_row_attn(d) -> int:
    """QK^T and AV per query row per step: 2 L H per block (Table 1 row QK^T)."""
    return d.n_blocks * 2 * d.L * d.hidden
