"""ORACLE (test infrastructure only) — float64 NumPy reference of the mask-aware step on a whole
SDXL-shaped UNet (BASELINE config 5, "SDXL-UNet config (5) ... ResBlocks dense").

What it computes, and where the paper says so
---------------------------------------------
* A UNet reshapes its latent (B, C, H, W) to (B, H x W, C) tokens for its transformer blocks
  (P:212-214); those blocks are 82% of SDXL's compute (P:213 footnote) and are the part the
  method makes mask-aware.  Everything else (ResBlocks, resamplers, GroupNorms, the in/out
  convolutions) mixes neighbouring pixels and runs DENSE on the full latent.
* Each Transformer2D (GroupNorm -> proj_in -> BasicTransformerBlocks -> proj_out -> residual)
  is computed for the MASKED tokens of its level only (P:384-386 token-wise ops; the blocks use
  the K/V cache, fig:transformer_alter P:435-446, through oracle.unet.unet_block_masked); its
  output rows of the UNMASKED tokens are the template's (the Y matrix of fig:transformer-Bottom,
  P:423-426, cached at Transformer2D granularity), so the dense ResBlocks downstream see a full
  hidden state.  GroupNorm statistics are taken over the full input (available: the ResBlock
  before it is dense).                                                  t2d_masked, t2d_dense
* Per-level masks by 2x2 any-pool of the latent mask (C-AMB 13).       oracle.unet.any_pool2
* The denoising update is the Euler step x += (sigma' - sigma) * eps_hat on the masked latent
  rows (unmasked rows untouched, C-AMB 11), with the UNet input scaled by 1/sqrt(sigma^2 + 1)
  and timestep t = 1000 sigma (C-AMB 34, an EDM-style epsilon-prediction reading).
* The dense step (all tokens, no cache) with recording of every block's K/V and every
  Transformer2D output = the template cache.          unet_full_dense_step(record=)

Architecture readings (C-AMB 34, public SDXL / diffusers layout, not the paper): ResBlock
h = conv3x3(SiLU(GN(x))) + Linear(SiLU(temb)); h = conv3x3(SiLU(GN(h))); out = skip(x) + h with
a 1x1 (linear) skip when channels change; GroupNorm 32 groups (eps 1e-5; 1e-6 in Transformer2D);
downsample = conv3x3 stride 2 pad 1; upsample = nearest x2 then conv3x3; up-path ResBlocks take
[h | skip] channel concatenations; timestep embedding = Linear(SiLU(Linear(sinusoid_c0(t)))),
sinusoid cos-first.  Convolution weights are [C_out][ky][kx][C_in].

Everything is float64.  Pins: tests/test_oracle_unet_full.py (torch float64 conv2d / group_norm
/ interpolate, a pure-Python brute-force ResBlock, the same-input exactness and degenerate-mask
invariants of the whole step).  Parity-unpinned: none of the functions below.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Tuple

import numpy as np

from .instgenie import index_build, linear, silu
from .unet import any_pool2, unet_block_masked


def _w(W, name) -> np.ndarray:
    return np.asarray(W[name], dtype=np.float64)


# ------------------------------------------------------------------------------- primitives
def conv3x3(x: np.ndarray, w: np.ndarray, b: np.ndarray, stride: int = 1) -> np.ndarray:
    """x [N, H, W, Ci]; w [Co, 9*Ci] as [Co][ky][kx][Ci]; zero padding 1.
    out[n, y, x, o] = b[o] + sum_{ky, kx, c} xpad[n, s*y + ky, s*x + kx, c] w[o, ky, kx, c]."""
    N, H, W_, Ci = x.shape
    Co = w.shape[0]
    wk = np.asarray(w, np.float64).reshape(Co, 3, 3, Ci)
    xp = np.zeros((N, H + 2, W_ + 2, Ci))
    xp[:, 1:H + 1, 1:W_ + 1] = x
    Ho, Wo = (H - 1) // stride + 1, (W_ - 1) // stride + 1
    out = np.zeros((N, Ho, Wo, Co)) + np.asarray(b, np.float64)
    for ky in range(3):
        for kx in range(3):
            patch = xp[:, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride, :]
            out += patch @ wk[:, ky, kx, :].T
    return out


def group_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, groups: int, eps: float) -> np.ndarray:
    """x [N, P, C] (P pixels): per image and group of C/groups channels, normalise over the
    pixels and the group's channels (biased variance), then the per-channel affine."""
    N, P, C = x.shape
    xg = x.reshape(N, P, groups, C // groups)
    mu = xg.mean(axis=(1, 3), keepdims=True)
    var = ((xg - mu) ** 2).mean(axis=(1, 3), keepdims=True)
    return ((xg - mu) / np.sqrt(var + eps)).reshape(N, P, C) * g + b


def upsample2(x: np.ndarray) -> np.ndarray:
    """Nearest-neighbour x2 on [N, H, W, C]."""
    return x.repeat(2, axis=1).repeat(2, axis=2)


def timestep_embedding(u, W, t: float) -> np.ndarray:
    """temb = Linear2(SiLU(Linear1(sinusoid_{c0}(t)))), sinusoid cos-first,
    f_k = exp(-ln(10000) k / (c0 / 2))."""
    half = u.ch[0] // 2
    f = np.exp(-math.log(10000.0) * np.arange(half) / half)
    e = np.concatenate([np.cos(t * f), np.sin(t * f)])[None, :]
    h = silu(linear(e, _w(W, "time.lin1.w"), _w(W, "time.lin1.b")))
    return linear(h, _w(W, "time.lin2.w"), _w(W, "time.lin2.b"))[0]


def resblock(u, W, p: str, x: np.ndarray, temb: np.ndarray) -> np.ndarray:
    """x [N, H, W, Ci] -> [N, H, W, Co]; temb [N, E] (per image)."""
    N, H, W_, Ci = x.shape
    P = H * W_
    h = silu(group_norm(x.reshape(N, P, Ci), _w(W, p + ".gn1.g"), _w(W, p + ".gn1.b"), u.gn_groups, u.gn_eps))
    h = conv3x3(h.reshape(N, H, W_, Ci), _w(W, p + ".conv1.w"), _w(W, p + ".conv1.b"))
    Co = h.shape[-1]
    h = h + linear(silu(temb), _w(W, p + ".temb.w"), _w(W, p + ".temb.b"))[:, None, None, :]
    h = silu(group_norm(h.reshape(N, P, Co), _w(W, p + ".gn2.g"), _w(W, p + ".gn2.b"), u.gn_groups, u.gn_eps))
    h = conv3x3(h.reshape(N, H, W_, Co), _w(W, p + ".conv2.w"), _w(W, p + ".conv2.b"))
    skip = x if Ci == Co else linear(x.reshape(N * P, Ci), _w(W, p + ".skip.w"), _w(W, p + ".skip.b")).reshape(N, H, W_, Co)
    return skip + h


# ------------------------------------------------------------------------------- Transformer2D
def t2d_block_desc(u, lvl: int, depth: int, c: int):
    """The ModelDesc of a Transformer2D's block stack (oracle.unet's block functions)."""
    import synth
    return synth._unet(f"t2d_l{lvl}", depth, c, c // u.head_dim, u.level_grid(lvl), u.ctx_len, u.ctx_dim)


def _t2d_weights(W, p: str, depth: int) -> Dict[str, np.ndarray]:
    """Rename a Transformer2D's block weights to oracle.unet's 'unet.{i}.*' names."""
    out = {}
    for i in range(depth):
        pre = f"{p}.blk.{i}."
        for k, v in W.items():
            if k.startswith(pre):
                out[f"unet.{i}." + k[len(pre):]] = v
    return out


def _t2d_in(u, W, p, x2d):
    """GroupNorm (full statistics) + proj_in over all rows of x2d [P, C] of ONE image."""
    h = group_norm(x2d[None], _w(W, p + ".gn.g"), _w(W, p + ".gn.b"), u.gn_groups, u.t2d_gn_eps)[0]
    return linear(h, _w(W, p + ".proj_in.w"), _w(W, p + ".proj_in.b"))


def t2d_dense(u, W, p: str, lvl: int, depth: int, x: np.ndarray, ctx: np.ndarray, record: bool = False):
    """Dense Transformer2D on one image x [P, C]; returns out [P, C] (and, with record, the
    blocks' K/V [depth][2][P][C] and the output rows = this Transformer2D's Y cache)."""
    c = x.shape[1]
    d = t2d_block_desc(u, lvl, depth, c)
    Wt = _t2d_weights(W, p, depth)
    all_idx = np.arange(x.shape[0])
    none = np.zeros(0, np.int64)
    h = _t2d_in(u, W, p, x)
    kv = np.zeros((depth, 2, x.shape[0], c)) if record else None
    for i in range(depth):
        h, k, v = unet_block_masked(d, Wt, i, h, all_idx, none, None, ctx)
        if record:
            kv[i, 0], kv[i, 1] = k, v
    out = x + linear(h, _w(W, p + ".proj_out.w"), _w(W, p + ".proj_out.b"))
    return (out, kv) if record else out


def t2d_masked(u, W, p: str, lvl: int, depth: int, x: np.ndarray, mask_lvl, kv_cache: Optional[np.ndarray],
               y_cache: Optional[np.ndarray], ctx: np.ndarray) -> np.ndarray:
    """Mask-aware Transformer2D on one image x [P, C] (full input, GroupNorm statistics over all
    rows): the masked rows go through proj_in, the blocks (K/V cache kv_cache [depth][2][P][C]
    for the unmasked keys) and proj_out; the unmasked rows of the output are y_cache [P, C]."""
    idx_m, idx_u, n_m = index_build(mask_lvl)
    if n_m == x.shape[0]:
        return t2d_dense(u, W, p, lvl, depth, x, ctx)
    out = np.array(y_cache, dtype=np.float64, copy=True)
    if n_m == 0:
        return out
    c = x.shape[1]
    d = t2d_block_desc(u, lvl, depth, c)
    Wt = _t2d_weights(W, p, depth)
    h = _t2d_in(u, W, p, x)[idx_m]  # token-wise after the (full) statistics
    for i in range(depth):
        h, _, _ = unet_block_masked(d, Wt, i, h, idx_m, idx_u, kv_cache[i], ctx)
    out[idx_m] = x[idx_m] + linear(h, _w(W, p + ".proj_out.w"), _w(W, p + ".proj_out.b"))
    return out


# ------------------------------------------------------------------------------- the UNet
def level_masks(u, mask) -> List[np.ndarray]:
    """Latent-level token mask -> the three levels' masks (2x2 any-pool, C-AMB 13)."""
    m0 = (np.asarray(mask).reshape(-1) != 0).astype(np.uint8)
    m1 = any_pool2(m0, u.grid, u.grid)
    m2 = any_pool2(m1, u.grid // 2, u.grid // 2)
    return [m0, m1, m2]


def unet_forward(u, W, x_lat: np.ndarray, t: float, cond: Optional[np.ndarray], ctx: np.ndarray,
                 masks: Optional[List[np.ndarray]] = None, cache: Optional[dict] = None,
                 record: bool = False):
    """One UNet evaluation for ONE request.  x_lat [grid*grid, lat_ch] (already scaled).
    Dense when masks is None (record=True returns the template cache of this evaluation:
    {t2d prefix: (K/V [depth][2][P][C], Y [P][C])}); mask-aware with masks (level_masks) and
    the template cache of this step.  Returns eps_hat [grid*grid, lat_ch] (+ cache)."""
    import synth
    g = u.grid
    temb = timestep_embedding(u, W, t)
    if cond is not None:
        temb = temb + np.asarray(cond, np.float64)
    temb = temb[None, :]
    rec = {} if record else None

    def t2d(p, lvl, dep, h):
        N, H, W_, C = h.shape
        x2 = h.reshape(H * W_, C)
        if masks is None:
            if record:
                out, kv = t2d_dense(u, W, p, lvl, dep, x2, ctx, record=True)
                rec[p] = (kv, out.copy())
            else:
                out = t2d_dense(u, W, p, lvl, dep, x2, ctx)
        else:
            kv, y = cache[p]
            out = t2d_masked(u, W, p, lvl, dep, x2, masks[lvl], kv, y, ctx)
        return out.reshape(1, H, W_, C)

    h = conv3x3(np.asarray(x_lat, np.float64).reshape(1, g, g, u.lat_ch), _w(W, "conv_in.w"), _w(W, "conv_in.b"))
    skips = [h]
    for lvl in range(3):
        for r in range(u.n_res):
            h = resblock(u, W, f"down.{lvl}.res.{r}", h, temb)
            if u.depth[lvl]:
                h = t2d(f"down.{lvl}.attn.{r}", lvl, u.depth[lvl], h)
            skips.append(h)
        if lvl < 2:
            h = conv3x3(h, _w(W, f"down.{lvl}.downsample.conv.w"), _w(W, f"down.{lvl}.downsample.conv.b"), stride=2)
            skips.append(h)
    h = resblock(u, W, "mid.res.0", h, temb)
    h = t2d("mid.attn.0", 2, u.depth[2], h)
    h = resblock(u, W, "mid.res.1", h, temb)
    for j, lvl in enumerate((2, 1, 0)):
        for r in range(u.n_res + 1):
            h = np.concatenate([h, skips.pop()], axis=-1)
            h = resblock(u, W, f"up.{j}.res.{r}", h, temb)
            if u.depth[lvl]:
                h = t2d(f"up.{j}.attn.{r}", lvl, u.depth[lvl], h)
        if lvl > 0:
            h = conv3x3(upsample2(h), _w(W, f"up.{j}.upsample.conv.w"), _w(W, f"up.{j}.upsample.conv.b"))
    N, H, W_, C = h.shape
    h = silu(group_norm(h.reshape(N, H * W_, C), _w(W, "out.gn.g"), _w(W, "out.gn.b"), u.gn_groups, u.gn_eps))
    eps = conv3x3(h.reshape(N, H, W_, C), _w(W, "conv_out.w"), _w(W, "conv_out.b")).reshape(g * g, u.lat_ch)
    return (eps, rec) if record else eps


def c_in(sigma: float) -> float:
    return 1.0 / math.sqrt(float(sigma) ** 2 + 1.0)


def unet_full_dense_step(u, W, latent, sigma, sigma_next, cond, ctx, record: bool = False):
    """Dense denoising step: eps = UNet(latent * c_in(sigma), t = 1000 sigma);
    latent' = latent + (sigma' - sigma) eps (every row)."""
    x = np.asarray(latent, np.float64)
    r = unet_forward(u, W, x * c_in(sigma), 1000.0 * float(sigma), cond, ctx, record=record)
    eps = r[0] if record else r
    out = x + (float(sigma_next) - float(sigma)) * eps
    return (out, r[1]) if record else out


def unet_full_edit_step(u, W, latent, mask, cache, sigma, sigma_next, cond, ctx):
    """Mask-aware step: Transformer2Ds on masked tokens with the template cache of this step,
    everything else dense; only the masked latent rows are updated."""
    x = np.asarray(latent, np.float64)
    idx_m, _, n_m = index_build(mask)
    if n_m == 0:
        return x.copy()
    if n_m == x.shape[0]:
        return unet_full_dense_step(u, W, x, sigma, sigma_next, cond, ctx)
    eps = unet_forward(u, W, x * c_in(sigma), 1000.0 * float(sigma), cond, ctx, masks=level_masks(u, mask),
                       cache=cache)
    out = x.copy()
    out[idx_m] = x[idx_m] + (float(sigma_next) - float(sigma)) * eps[idx_m]
    return out


def unet_full_cache_template(u, W, latent, cond, ctx, sigmas):
    """Template pass along its own trajectory: per step the dense step with recording.
    Returns (trajectory [steps+1][L][C], [per-step cache dict])."""
    traj = [np.asarray(latent, np.float64).copy()]
    caches = []
    for s in range(len(sigmas) - 1):
        x, rec = unet_full_dense_step(u, W, traj[-1], sigmas[s], sigmas[s + 1], cond, ctx, record=True)
        traj.append(x)
        caches.append(rec)
    return np.stack(traj), caches


def unet_full_macs(u) -> Dict[str, float]:
    """Dense multiply-accumulates of one UNet evaluation by part (convolutions / resamplers /
    skips vs Transformer2Ds), for the FLOP model of the sweep (P:213's 82% share)."""
    g = u.grid
    conv = 0.0
    t2d = 0.0
    conv += (g * g) * 9 * u.lat_ch * u.ch[0]
    for p, lvl, ci, co, _ in __import__("synth").unet_resblocks(u):
        P = (g >> lvl) ** 2
        conv += P * 9 * (ci * co + co * co) + (P * ci * co if ci != co else 0)
    for lvl in (0, 1):
        conv += ((g >> (lvl + 1)) ** 2) * 9 * u.ch[lvl] ** 2                       # downsample
    for j, lvl in enumerate((2, 1)):
        conv += ((g >> (lvl - 1)) ** 2) * 9 * u.ch[lvl] ** 2                       # upsample
    conv += (g * g) * 9 * u.ch[0] * u.lat_ch
    for p, lvl, c, dep in __import__("synth").unet_t2ds(u):
        P = (g >> lvl) ** 2
        F = 4 * c
        per_row = 6 * c * c + 3 * F * c + 2 * P * c + 2 * u.ctx_len * c
        t2d += 2 * P * c * c + dep * (P * per_row + u.ctx_len * 2 * c * u.ctx_dim)
    return {"conv": conv, "t2d": t2d}
