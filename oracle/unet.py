"""ORACLE (test infrastructure only) — float64 NumPy reference of the mask-aware step on the
SDXL-UNet attention stack (BASELINE config 5).

What it computes, and where the paper says so
---------------------------------------------
* A UNet's transformer part: "a latent of shape (B, C, H, W) is reshaped to (B, H x W, C)
  to pass through transformer blocks"; these blocks are 82% of SDXL's compute
  (P:213 footnote).  The block internals (LayerNorm with affine, self-attention, cross-
  attention to the text context, GEGLU feed-forward) are SDXL's public architecture, not
  the paper's: readings C-AMB 31-33 in DESIGN.md.                      unet_block_masked
* Token-wise ops on masked rows only, K/V-caching variant for self-attention
  (fig:transformer_alter): masked rows get fresh K/V, unmasked rows' K/V come
  from the template cache, masked Q attends to all L_img tokens.  Cross-attention
  keys/values come from the request's text context and are computed fresh (nothing about
  them depends on the image tokens).                              unet_block_masked
* The dense block (fig:transformer-Top) with K/V recording = the template
  cache.                                                   unet_dense_step(record=)
* Y-caching variant and hybrid per-block choice (fig:transformer-Bottom): Y_{b-1}
  of the unmasked tokens replenishes their block input, which only feeds K/V.
                                                    unet_kv_from_y, unet_edit_step_y
* Per-level masks: a 2x2 any-pool of the finer level's token mask (C-AMB 13, SURVEY
  §8(d) config 5).                                                                any_pool2
* One synthetic step applies the level's stack to its hidden state and feeds the output
  back as the next step's input (C-AMB 31: the dense ResBlocks / resampling around the
  stack are outside this path).                            unet_edit_step, unet_dense_step

Everything is float64; inputs are the exact fp32/bf16 values.  Pins: tests/test_oracle_unet.py
(math.erf values, closed forms with zeroed sub-blocks, a pure-Python brute-force block,
exactness invariants).  Parity-unpinned: none of the functions below.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import numpy as np
from scipy.special import erf

from .instgenie import attention, index_build, layernorm, linear


def _w(W, name) -> np.ndarray:
    return np.asarray(W[name], dtype=np.float64)


def gelu_erf(x: np.ndarray) -> np.ndarray:
    """Exact GELU x * Phi(x) = 0.5 x (1 + erf(x / sqrt 2)) (GEGLU's gate; C-AMB 32)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def layernorm_affine(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float) -> np.ndarray:
    """LN(x) * g + b over the hidden dim (biased variance)."""
    return layernorm(x, eps) * g + b


def geglu_ff(d, W, p: str, h: np.ndarray) -> np.ndarray:
    """GEGLU feed-forward: [a | g] = h W1^T + b1, out = (a * gelu(g)) W2^T + b2 (C-AMB 32)."""
    F = d.mlp_hidden
    u = linear(h, _w(W, p + ".ff.geglu.w"), _w(W, p + ".ff.geglu.b"))
    return linear(u[:, :F] * gelu_erf(u[:, F:]), _w(W, p + ".ff.out.w"), _w(W, p + ".ff.out.b"))


def cross_kv(d, W, i: int, ctx: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Cross-attention keys / values of the text context [ctx_len, ctx_dim] (fresh each step)."""
    H = d.hidden
    kv = linear(np.asarray(ctx, np.float64), _w(W, f"unet.{i}.attn2.kv.w"), None)
    return kv[:, :H], kv[:, H:]


def unet_block_masked(d, W, i: int, x_m: np.ndarray, idx_m: np.ndarray, idx_u: np.ndarray,
                      kv_cache_blk: Optional[np.ndarray], ctx: np.ndarray):
    """One BasicTransformerBlock on the masked rows x_m [n_m, H] (ascending token order).

    Self-attention: q, k, v of the masked rows; K/V of all L_img tokens merged by mask
    index (fresh at idx_m, kv_cache_blk[0/1] at idx_u); masked queries attend to all.
    Returns (x_out [n_m, H], fresh k [n_m, H], fresh v [n_m, H])."""
    H, eps, p = d.hidden, d.ln_eps, f"unet.{i}"
    x = np.asarray(x_m, np.float64)
    h = layernorm_affine(x, _w(W, p + ".ln1.g"), _w(W, p + ".ln1.b"), eps)
    qkv = linear(h, _w(W, p + ".attn1.qkv.w"), None)
    q, k, v = qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:]
    K = np.zeros((d.L_img, H))
    V = np.zeros((d.L_img, H))
    K[idx_m], V[idx_m] = k, v
    if len(idx_u):
        K[idx_u] = np.asarray(kv_cache_blk[0], np.float64)[idx_u]
        V[idx_u] = np.asarray(kv_cache_blk[1], np.float64)[idx_u]
    x = x + linear(attention(q, K, V, d.heads), _w(W, p + ".attn1.out.w"), _w(W, p + ".attn1.out.b"))
    h = layernorm_affine(x, _w(W, p + ".ln2.g"), _w(W, p + ".ln2.b"), eps)
    q2 = linear(h, _w(W, p + ".attn2.q.w"), None)
    K2, V2 = cross_kv(d, W, i, ctx)
    x = x + linear(attention(q2, K2, V2, d.heads), _w(W, p + ".attn2.out.w"), _w(W, p + ".attn2.out.b"))
    h = layernorm_affine(x, _w(W, p + ".ln3.g"), _w(W, p + ".ln3.b"), eps)
    x = x + geglu_ff(d, W, p, h)
    return x, k, v


def unet_edit_step(d, W, state: np.ndarray, mask, kv_cache_step: Optional[np.ndarray],
                   ctx: np.ndarray) -> np.ndarray:
    """Mask-aware step of the level's stack: the masked rows of `state` [L_img, H] go
    through every block (K/V cache per block, kv_cache_step [n_blocks][2][L_img][H]); the
    unmasked rows are returned untouched (their pixels stay the template's)."""
    idx_m, idx_u, n_m = index_build(mask)
    out = np.array(state, dtype=np.float64, copy=True)
    if n_m == 0:
        return out
    x = out[idx_m]
    for b in range(d.n_unet):
        x, _, _ = unet_block_masked(d, W, b, x, idx_m, idx_u,
                                    None if kv_cache_step is None else kv_cache_step[b], ctx)
    out[idx_m] = x
    return out


def unet_dense_step(d, W, state: np.ndarray, ctx: np.ndarray, record: bool = False, record_y: bool = False):
    """Dense step (all L_img tokens, no cache); record=True also returns the K/V of every
    block [n_blocks][2][L_img][H] (the template cache of this step), record_y=True also the
    block outputs Y [n_blocks][L_img][H] (the Y variant's cache, fig:transformer-Bottom)."""
    all_idx = np.arange(d.L_img)
    none = np.zeros(0, dtype=np.int64)
    x = np.array(state, dtype=np.float64, copy=True)
    kv = np.zeros((d.n_unet, 2, d.L_img, d.hidden)) if record else None
    y = np.zeros((d.n_unet, d.L_img, d.hidden)) if record_y else None
    for b in range(d.n_unet):
        x, k, v = unet_block_masked(d, W, b, x, all_idx, none, None, ctx)
        if record:
            kv[b, 0], kv[b, 1] = k, v
        if record_y:
            y[b] = x
    out = (x,) + ((kv,) if record else ()) + ((y,) if record_y else ())
    return out if len(out) > 1 else x


def unet_cache_template(d, W, state0: np.ndarray, ctx: np.ndarray, n_steps: int, record_y: bool = False):
    """Template pass: n_steps dense steps from state0; returns (inputs [n_steps+1][L_img][H],
    K/V cache [n_steps][n_blocks][2][L_img][H]) (+ Y cache [n_steps][n_blocks][L_img][H])."""
    states = [np.array(state0, np.float64)]
    cache, ys = [], []
    for _ in range(n_steps):
        r = unet_dense_step(d, W, states[-1], ctx, record=True, record_y=True)
        states.append(r[0])
        cache.append(r[1])
        ys.append(r[2])
    return (np.stack(states), np.stack(cache)) + ((np.stack(ys),) if record_y else ())


def unet_kv_from_y(d, W, b: int, u: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Y variant: K/V of unmasked rows from their block input u (LN1 + the K/V projections,
    P:423-426 "replenishing cached activations for the unmasked tokens")."""
    H, p = d.hidden, f"unet.{b}"
    h = layernorm_affine(np.asarray(u, np.float64), _w(W, p + ".ln1.g"), _w(W, p + ".ln1.b"), d.ln_eps)
    kv = linear(h, _w(W, p + ".attn1.qkv.w")[H:], None)
    return kv[:, :H], kv[:, H:]


def unet_edit_step_y(d, W, state: np.ndarray, mask, y_cache_step: np.ndarray, tstate: np.ndarray,
                     ctx: np.ndarray, y_blocks=None, kv_cache_step: Optional[np.ndarray] = None) -> np.ndarray:
    """Y-variant (and hybrid) mask-aware step of the level's stack.  For a Y block b the
    unmasked tokens' block input is the template's Y_{b-1} (block 0: the template's input
    state tstate of this step); it only feeds their K/V (unet_kv_from_y).  Blocks outside
    y_blocks (default: all are Y blocks) read K/V from kv_cache_step.  Unmasked rows of the
    result are untouched."""
    idx_m, idx_u, n_m = index_build(mask)
    out = np.array(state, dtype=np.float64, copy=True)
    if n_m == 0:
        return out
    yb = set(range(d.n_unet)) if y_blocks is None else set(y_blocks)
    x = out[idx_m]
    for b in range(d.n_unet):
        if b in yb:
            u = (np.asarray(tstate, np.float64) if b == 0 else np.asarray(y_cache_step[b - 1], np.float64))[idx_u]
            ku, vu = unet_kv_from_y(d, W, b, u)
            blk = np.zeros((2, d.L_img, d.hidden))
            blk[0][idx_u], blk[1][idx_u] = ku, vu
        else:
            blk = kv_cache_step[b]
        x, _, _ = unet_block_masked(d, W, b, x, idx_m, idx_u, blk, ctx)
    out[idx_m] = x
    return out


def any_pool2(mask, grid_h: int, grid_w: int) -> np.ndarray:
    """Next-coarser UNet level's token mask: a coarse token is masked if any of its 2x2
    fine tokens is (C-AMB 13: no edited pixel is lost)."""
    m = np.asarray(mask).reshape(grid_h, grid_w) != 0
    out = np.zeros((grid_h // 2, grid_w // 2), np.uint8)
    for r in range(grid_h // 2):
        for c in range(grid_w // 2):
            out[r, c] = 1 if m[2 * r:2 * r + 2, 2 * c:2 * c + 2].any() else 0
    return out.reshape(-1)


def unet_macs_per_row(d) -> Dict[str, int]:
    """Multiply-accumulates per masked query row and block (Table 1's per-row terms,
    P:461-482, for this block type): projections + FF, and the two attentions."""
    H, F, L, Lc = d.hidden, d.mlp_hidden, d.L_img, d.ctx_len
    return {"linear": 3 * H * H + H * H + H * H + H * H + 2 * F * H + F * H,
            "attn": 2 * L * H + 2 * Lc * H}


def unet_edit_step_planned(d, W, state: np.ndarray, mask, tstate: np.ndarray, ctx: np.ndarray, k: int,
                           kv_cache_step: Optional[np.ndarray] = None, y_cache_step: Optional[np.ndarray] = None,
                           y_blocks=()) -> np.ndarray:
    """Algorithm 1 (C-AMB 23) on the UNet stack: the first k blocks run dense — all
    L_img tokens, the unmasked ones entering from the template's input state tstate of this
    step, fresh K/V, no cache — and blocks >= k run mask-aware: K/V blocks read kv_cache_step,
    Y blocks (y_blocks) recompute the unmasked tokens' K/V from their block input (the rows
    computed by the prefix for block k, else the template's Y_{b-1}).  Unmasked rows of the
    result are untouched."""
    idx_m, idx_u, n_m = index_build(mask)
    out = np.array(state, dtype=np.float64, copy=True)
    if n_m == 0:
        return out
    all_idx = np.arange(d.L_img)
    none = np.zeros(0, dtype=np.int64)
    X = np.array(tstate, dtype=np.float64, copy=True)
    X[idx_m] = out[idx_m]
    yb = set(y_blocks)
    for b in range(min(k, d.n_unet)):
        X, _, _ = unet_block_masked(d, W, b, X, all_idx, none, None, ctx)
    x = X[idx_m]
    for b in range(min(k, d.n_unet), d.n_unet):
        if b in yb:
            u = X[idx_u] if b == k else np.asarray(y_cache_step[b - 1], np.float64)[idx_u]
            ku, vu = unet_kv_from_y(d, W, b, u)
            blk = np.zeros((2, d.L_img, d.hidden))
            blk[0][idx_u], blk[1][idx_u] = ku, vu
        else:
            blk = kv_cache_step[b]
        x, _, _ = unet_block_masked(d, W, b, x, idx_m, idx_u, blk, ctx)
    out[idx_m] = x
    return out
