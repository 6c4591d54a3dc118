"""Seeded synthetic inputs for the InstGenIE mask-aware step (test/bench input generators).

This module is shared by the oracle (`oracle/`), the tests and `bench.py`.  It holds NONE
of the method's arithmetic: it only draws numbers (weights, latents, text tokens, masks,
sigma schedules, synthetic caches) and describes the model shapes and the weight-table
layout as data.  See DESIGN.md "Input recipe".

Random numbers come from a counter-based generator (SplitMix64 finaliser applied to
key+index, key = SplitMix64(seed ^ FNV1a(name))) written with torch int64 ops, so CPU
and CUDA produce bit-identical values.  Uniforms are odd multiples of 2^-24 in (-1, 1),
exact in fp32; approximate normals are Irwin-Hall(4) sums rescaled to unit variance,
computed in float64 and rounded once to fp32 (then to bf16 when asked).  No
transcendental function touches a value that both sides consume.

Masks are drawn on the host with numpy (rectangles and smooth "blobs") and
passed as uint8 token bitmaps (nonzero = masked), so both sides see the same bytes.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Tuple

import numpy as np
import torch

_M64 = (1 << 64) - 1


def _s64(c: int) -> int:
    """uint64 constant -> the int64 with the same bit pattern."""
    c &= _M64
    return c - (1 << 64) if c >= (1 << 63) else c


_GAMMA = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor (torch's >> is arithmetic)."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def _mix_int(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fnv1a(name: str) -> int:
    h = 0xCBF29CE484222325
    for b in name.encode():
        h = ((h ^ b) * 0x100000001B3) & _M64
    return h


def stream_key(seed: int, name: str) -> int:
    return _mix_int((seed ^ _fnv1a(name)) + 0x9E3779B97F4A7C15)


def _raw(key: int, n: int, offset: int, device) -> torch.Tensor:
    idx = torch.arange(offset, offset + n, dtype=torch.int64, device=device)
    z = idx * _GAMMA + _s64(key)
    return _mix(z)


def uniform(seed: int, name: str, shape, device="cpu", offset: int = 0) -> torch.Tensor:
    """float64 tensor of odd multiples of 2^-24 in (-1, 1); identical on every device."""
    n = int(np.prod(shape)) if len(shape) else 1
    z = _raw(stream_key(seed, name), n, offset, device)
    u24 = _lsr(z, 40)  # 24 high bits
    v = (2 * u24 - (1 << 24) + 1).to(torch.float64) * (2.0 ** -24)
    return v.reshape(shape)


def normal(seed: int, name: str, shape, device="cpu") -> torch.Tensor:
    """Irwin-Hall(4) approximate N(0,1), float64 (exact sums of 2^-24 multiples)."""
    n = int(np.prod(shape)) if len(shape) else 1
    s = torch.zeros(n, dtype=torch.float64, device=device)
    for j in range(4):
        s += uniform(seed, f"{name}#ih{j}", (n,), device)
    # Var(U(-1,1)) = 1/3, four of them: 4/3 -> scale by sqrt(3/4)
    return (s * math.sqrt(0.75)).reshape(shape)


# --------------------------------------------------------------------------------------
# Model shapes.  Data only.
# --------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class ModelDesc:
    name: str
    n_double: int
    n_single: int
    hidden: int
    heads: int
    head_dim: int
    mlp_hidden: int
    lat_ch: int
    grid_h: int
    grid_w: int
    txt_len: int
    qk_norm: int = 1
    rope: int = 1
    rope_axes: Tuple[int, int, int] = (16, 56, 56)
    rope_theta: float = 10000.0
    ln_eps: float = 1e-6
    pos_embed_2d: int = 0
    context_pre_only_last: int = 0
    # SDXL-UNet attention stack (config 5): n_unet BasicTransformerBlocks
    # (LN -> self-attn -> LN -> cross-attn to a [ctx_len, ctx_dim] context -> LN -> GEGLU FF);
    # no conditioning, no text rows, lat_ch = hidden (the level's hidden state is the latent)
    n_unet: int = 0
    ctx_len: int = 0
    ctx_dim: int = 0

    @property
    def L_img(self) -> int:
        return self.grid_h * self.grid_w

    @property
    def L(self) -> int:
        return self.L_img + self.txt_len

    @property
    def n_blocks(self) -> int:
        return self.n_double + self.n_single + self.n_unet


TINY = ModelDesc("tiny", 0, 1, 64, 4, 16, 256, 16, 16, 16, 0, rope_axes=(4, 6, 6))
TINY_DOUBLE = ModelDesc("tiny_double", 1, 1, 64, 4, 16, 256, 16, 16, 16, 8, rope_axes=(4, 6, 6))
SD3 = ModelDesc("sd3_medium", 24, 0, 1536, 24, 64, 6144, 64, 32, 32, 333, qk_norm=0, rope=0,
                rope_axes=(0, 0, 0), pos_embed_2d=1, context_pre_only_last=1)
FLUX = ModelDesc("flux1_dev", 19, 38, 3072, 24, 128, 12288, 64, 64, 64, 512)
# Small Flux-structured model for multi-block / multi-step parity (tiles span >1 CTA tile)
FLUX_SMALL = ModelDesc("flux_small", 2, 2, 256, 2, 128, 1024, 64, 16, 16, 32)
# Small SD3-structured model (joint blocks, d=64, no RoPE / QK-norm, 2-D pos-embed, ragged
# text length, context-pre-only last block)
SD3_SMALL = ModelDesc("sd3_small", 2, 0, 128, 2, 64, 512, 64, 8, 8, 13, qk_norm=0, rope=0,
                      rope_axes=(0, 0, 0), pos_embed_2d=1, context_pre_only_last=1)



def _unet(name, n, H, heads, grid, ctx_len, ctx_dim):
    return ModelDesc(name, 0, 0, H, heads, H // heads, 4 * H, H, grid, grid, 0, qk_norm=0, rope=0,
                     rope_axes=(0, 0, 0), ln_eps=1e-5, n_unet=n, ctx_len=ctx_len, ctx_dim=ctx_dim)


# SDXL-UNet attention stacks (config 5): the 64x64 level (10 blocks, C=640, h=10) and the
# 32x32 level (60 blocks, C=1280, h=20), d = 64, cross-attention to 77 x 2048 text tokens
UNET_TINY = _unet("unet_tiny", 2, 64, 4, 16, 7, 32)
UNET_SMALL = _unet("unet_small", 3, 128, 2, 16, 13, 64)
SDXL_L64 = _unet("sdxl_attn64", 10, 640, 10, 64, 77, 2048)
SDXL_L32 = _unet("sdxl_attn32", 60, 1280, 20, 32, 77, 2048)
MODELS = {m.name: m for m in (TINY, TINY_DOUBLE, SD3, FLUX, FLUX_SMALL, SD3_SMALL,
                              UNET_TINY, UNET_SMALL, SDXL_L64, SDXL_L32)}


def weight_table(d: ModelDesc) -> List[Tuple[str, Tuple[int, ...], int]]:
    """(name, shape, fan_in) in the fixed C-ABI table order (include/ig.h).

    Matrices are [out, in] row-major, each followed by its bias [out]."""
    H, C, Fm, dh = d.hidden, d.lat_ch, d.mlp_hidden, d.head_dim
    t: List[Tuple[str, Tuple[int, ...], int]] = []

    def lin(name, out, inp):
        t.append((name + ".w", (out, inp), inp))
        t.append((name + ".b", (out,), inp))

    if d.n_unet:
        for i in range(d.n_unet):
            p = f"unet.{i}"
            t += [(p + ".ln1.g", (H,), 0), (p + ".ln1.b", (H,), 0)]
            t.append((p + ".attn1.qkv.w", (3 * H, H), H))      # to_q|to_k|to_v, no bias
            lin(p + ".attn1.out", H, H)
            t += [(p + ".ln2.g", (H,), 0), (p + ".ln2.b", (H,), 0)]
            t.append((p + ".attn2.q.w", (H, H), H))             # no bias
            t.append((p + ".attn2.kv.w", (2 * H, d.ctx_dim), d.ctx_dim))  # to_k|to_v, no bias
            lin(p + ".attn2.out", H, H)
            t += [(p + ".ln3.g", (H,), 0), (p + ".ln3.b", (H,), 0)]
            lin(p + ".ff.geglu", 2 * Fm, H)                     # [hidden | gate]
            lin(p + ".ff.out", H, Fm)
        return t

    lin("img_in", H, C)
    lin("t_mlp1", H, 256)
    lin("t_mlp2", H, H)
    lin("final_mod", 2 * H, H)
    lin("proj_out", C, H)
    if d.pos_embed_2d:
        t.append(("pos_embed", (d.L_img, H), 0))
    for i in range(d.n_double):
        for s in ("img", "txt"):
            p = f"double.{i}.{s}"
            pre_only = d.context_pre_only_last and s == "txt" and i == d.n_double - 1
            lin(p + ".mod", (2 if pre_only else 6) * H, H)
            lin(p + ".qkv", 3 * H, H)
            if d.qk_norm:
                t.append((p + ".q_norm_g", (dh,), 0))
                t.append((p + ".k_norm_g", (dh,), 0))
            if not pre_only:
                lin(p + ".proj", H, H)
                lin(p + ".fc1", Fm, H)
                lin(p + ".fc2", H, Fm)
    for i in range(d.n_single):
        p = f"single.{i}"
        lin(p + ".mod", 3 * H, H)
        lin(p + ".lin1", 3 * H + Fm, H)
        if d.qk_norm:
            t.append((p + ".q_norm_g", (dh,), 0))
            t.append((p + ".k_norm_g", (dh,), 0))
        lin(p + ".lin2", H, H + Fm)
    return t


def make_weight(d: ModelDesc, name: str, shape, fan_in: int, seed: int = 0, device="cpu",
                dtype=torch.float32) -> torch.Tensor:
    """One table tensor.  uniform(+-1/sqrt(fan_in)); modulation weights x0.1; norm gains 1."""
    if name.endswith("_norm_g"):
        return torch.ones(shape, dtype=dtype, device=device)
    if ".ln" in name:  # UNet LayerNorm affine: gain 1 + 0.1 u, bias 0.1 u
        v = uniform(seed, name, shape, device) * 0.1 + (1.0 if name.endswith(".g") else 0.0)
        return v.to(torch.float32).to(dtype)
    if name == "pos_embed":
        v = uniform(seed, name, shape, device) * 0.5
    else:
        a = 1.0 / math.sqrt(fan_in)
        if ".mod." in name or name.startswith("final_mod"):
            a *= 0.1
        v = uniform(seed, name, shape, device) * a
    return v.to(torch.float32).to(dtype)


def make_weights(d: ModelDesc, seed: int = 0, device="cpu", dtype=torch.float32,
                 names=None) -> Dict[str, torch.Tensor]:
    out = {}
    for name, shape, fan_in in weight_table(d):
        if names is not None and name not in names:
            continue
        out[name] = make_weight(d, name, shape, fan_in, seed, device, dtype)
    return out


# --------------------------------------------------------------------------------------
# Per-request inputs
# --------------------------------------------------------------------------------------
def make_latent(d: ModelDesc, rid: int, device="cpu") -> torch.Tensor:
    return normal(rid, "latent", (d.L_img, d.lat_ch), device).to(torch.float32)


def make_txt(d: ModelDesc, rid: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    return normal(rid, "txt", (d.txt_len, d.hidden), device).to(torch.float32).to(dtype)


def make_ctx(d: ModelDesc, rid: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    """UNet cross-attention context (encoder hidden states) [ctx_len, ctx_dim]."""
    return normal(rid, "ctx", (d.ctx_len, d.ctx_dim), device).to(torch.float32).to(dtype)


def make_cond(d: ModelDesc, rid: int, device="cpu") -> torch.Tensor:
    return normal(rid, "cond_vec", (d.hidden,), device).to(torch.float32)


def make_cache_kv(d: ModelDesc, template: int, n_steps: int, dtype=torch.float32, device="cpu"):
    """A synthetic template cache K,V [steps][blocks][2][L_img][H] (cache 'from other
    inputs'; used to test the edit step independently of cache recording)."""
    shape = (n_steps, d.n_blocks, 2, d.L_img, d.hidden)
    return normal(1000 + template, "cache_kv", shape, device).to(torch.float32).to(dtype)


def make_cache_y(d: ModelDesc, template: int, n_steps: int, dtype=torch.float32, device="cpu"):
    """A synthetic Y-variant template cache [steps][blocks][L_img][H] (block outputs of the
    image tokens), for testing the edit step independently of cache recording."""
    shape = (n_steps, d.n_blocks, d.L_img, d.hidden)
    return normal(2000 + template, "cache_y", shape, device).to(torch.float32).to(dtype)


def flow_sigmas(n_steps: int, shift: float = 3.0) -> np.ndarray:
    """Shift-3 flow schedule on linspace(1, 0, n+1) [proposal, SURVEY §8(d) config 3]."""
    s = np.linspace(1.0, 0.0, n_steps + 1)
    return (shift * s / (1.0 + (shift - 1.0) * s)).astype(np.float32)


# --------------------------------------------------------------------------------------
# Masks: uint8 token bitmaps, nonzero = masked (C-AMB 13-15)
# --------------------------------------------------------------------------------------
def rect_mask(d: ModelDesc, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    m = np.zeros((d.grid_h, d.grid_w), np.uint8)
    m[r0:r1, c0:c1] = 1
    return m.reshape(-1)


def rect_mask_count(d: ModelDesc, n: int, rng: np.random.Generator) -> np.ndarray:
    """Near-square rectangle holding exactly n tokens (last row ragged)."""
    m = np.zeros(d.L_img, np.uint8)
    if n <= 0:
        return m
    if n >= d.L_img:
        m[:] = 1
        return m
    aspect = math.exp(rng.uniform(-0.5, 0.5))
    w = int(min(d.grid_w, max(1, round(math.sqrt(n * aspect)))))
    h = int(min(d.grid_h, math.ceil(n / w)))
    while h * w < n:
        w = min(d.grid_w, w + 1)
        h = min(d.grid_h, math.ceil(n / w))
    r0 = int(rng.integers(0, d.grid_h - h + 1))
    c0 = int(rng.integers(0, d.grid_w - w + 1))
    cnt = 0
    for r in range(r0, r0 + h):
        for c in range(c0, c0 + w):
            if cnt < n:
                m[r * d.grid_w + c] = 1
                cnt += 1
    return m


def blob_mask_count(d: ModelDesc, n: int, rng: np.random.Generator) -> np.ndarray:
    """Top-n tokens of a smooth field (3 Gaussian bumps + 0.1 noise); ties -> lower index."""
    m = np.zeros(d.L_img, np.uint8)
    if n <= 0:
        return m
    yy, xx = np.meshgrid(np.arange(d.grid_h), np.arange(d.grid_w), indexing="ij")
    f = np.zeros((d.grid_h, d.grid_w))
    for _ in range(3):
        cy, cx = rng.uniform(0, d.grid_h), rng.uniform(0, d.grid_w)
        s = rng.uniform(0.1, 0.3) * max(d.grid_h, d.grid_w)
        f += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
    f = f.reshape(-1) + 0.1 * rng.standard_normal(d.L_img)
    order = np.argsort(-f, kind="stable")
    m[order[:min(n, d.L_img)]] = 1
    return m


def mixed_mask(d: ModelDesc, rid: int, lo: float = 0.05, hi: float = 0.60) -> np.ndarray:
    """Headline mix: m ~ U[lo, hi], n_m = round(m L_img); even ids rectangles, odd blobs."""
    rng = np.random.default_rng(7919 * rid + 17)
    m = rng.uniform(lo, hi)
    n = int(round(m * d.L_img))
    return rect_mask_count(d, n, rng) if rid % 2 == 0 else blob_mask_count(d, n, rng)


def tiny_rect_mask() -> np.ndarray:
    """Config 1: rectangle rows 4-11 x cols 4-11 on the 16x16 grid (64 tokens, 25%)."""
    return rect_mask(TINY, 4, 12, 4, 12)


# --------------------------------------------------------------------------------------
# Whole SDXL-shaped UNet (BASELINE config 5): conv_in -> 3 down levels (ResBlocks,
# Transformer2Ds at levels 1 and 2, stride-2 downsamplers) -> mid (ResBlock, Transformer2D,
# ResBlock) -> 3 up levels (ResBlocks on [h | skip] concatenations, Transformer2Ds, nearest x2
# upsamplers + conv) -> GroupNorm, SiLU, conv_out.  Data only: shapes and the weight table.
# --------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class UNetDesc:
    name: str
    lat_ch: int             # latent channels (4)
    grid: int               # latent H = W (128 for 1024^2)
    ch: Tuple[int, int, int]       # channels per level (320, 640, 1280)
    depth: Tuple[int, int, int]    # transformer blocks per Transformer2D per level (0, 2, 10)
    head_dim: int = 64
    ctx_len: int = 77
    ctx_dim: int = 2048
    n_res: int = 2          # ResBlocks per down level (up levels: n_res + 1)
    gn_groups: int = 32
    gn_eps: float = 1e-5    # ResBlock / output GroupNorm
    t2d_gn_eps: float = 1e-6
    ln_eps: float = 1e-5    # LayerNorms inside the transformer blocks

    @property
    def temb_dim(self) -> int:
        return 4 * self.ch[0]

    def level_grid(self, lvl: int) -> int:
        return self.grid >> lvl


def unet_resblocks(u: UNetDesc):
    """(prefix, level, c_in, c_out, has_t2d) of every ResBlock in execution order, with the
    channel bookkeeping of the skip concatenations on the up path (SDXL / diffusers layout)."""
    out = []
    skips = [u.ch[0]]  # conv_in output
    c = u.ch[0]
    for lvl in range(3):
        for r in range(u.n_res):
            out.append((f"down.{lvl}.res.{r}", lvl, c, u.ch[lvl], u.depth[lvl] > 0))
            c = u.ch[lvl]
            skips.append(c)
        if lvl < 2:
            skips.append(c)  # downsampler output
    out.append(("mid.res.0", 2, c, c, True))
    out.append(("mid.res.1", 2, c, c, False))
    for j, lvl in enumerate((2, 1, 0)):
        for r in range(u.n_res + 1):
            cs = skips.pop()
            out.append((f"up.{j}.res.{r}", lvl, c + cs, u.ch[lvl], u.depth[lvl] > 0))
            c = u.ch[lvl]
    return out


def unet_t2ds(u: UNetDesc):
    """(prefix, level, channels, depth) of every Transformer2D in execution order."""
    out = []
    for lvl in range(3):
        if u.depth[lvl]:
            for r in range(u.n_res):
                out.append((f"down.{lvl}.attn.{r}", lvl, u.ch[lvl], u.depth[lvl]))
    out.append(("mid.attn.0", 2, u.ch[2], u.depth[2]))
    for j, lvl in enumerate((2, 1, 0)):
        if u.depth[lvl]:
            for r in range(u.n_res + 1):
                out.append((f"up.{j}.attn.{r}", lvl, u.ch[lvl], u.depth[lvl]))
    return out


def unet_full_weight_table(u: UNetDesc) -> List[Tuple[str, Tuple[int, ...], int]]:
    """(name, shape, fan_in) in the fixed C-ABI order (include/ig_unet.h).  Convolutions are
    [C_out, 3 * 3 * C_in] with k = (ky * 3 + kx) * C_in + c (K-major, the implicit-GEMM B
    operand); linears [out, in] + bias; GroupNorm / LayerNorm gains and shifts [C]."""
    t: List[Tuple[str, Tuple[int, ...], int]] = []

    def lin(name, out_, in_, bias=True):
        t.append((name + ".w", (out_, in_), in_))
        if bias:
            t.append((name + ".b", (out_,), in_))

    def conv(name, cin, cout):
        t.append((name + ".w", (cout, 9 * cin), 9 * cin))
        t.append((name + ".b", (cout,), 9 * cin))

    def gn(name, c):
        t.append((name + ".g", (c,), 0))
        t.append((name + ".b", (c,), 0))

    E = u.temb_dim
    lin("time.lin1", E, u.ch[0])
    lin("time.lin2", E, E)
    conv("conv_in", u.lat_ch, u.ch[0])
    res = {p: (ci, co) for p, _, ci, co, _ in unet_resblocks(u)}
    t2d = {p: (c, dep) for p, _, c, dep in unet_t2ds(u)}
    order = []
    for lvl in range(3):
        for r in range(u.n_res):
            order.append(f"down.{lvl}.res.{r}")
            if u.depth[lvl]:
                order.append(f"down.{lvl}.attn.{r}")
        if lvl < 2:
            order.append(f"down.{lvl}.downsample")
    order += ["mid.res.0", "mid.attn.0", "mid.res.1"]
    for j, lvl in enumerate((2, 1, 0)):
        for r in range(u.n_res + 1):
            order.append(f"up.{j}.res.{r}")
            if u.depth[lvl]:
                order.append(f"up.{j}.attn.{r}")
        if lvl > 0:
            order.append(f"up.{j}.upsample")
    for p in order:
        if p in res:
            ci, co = res[p]
            gn(p + ".gn1", ci)
            conv(p + ".conv1", ci, co)
            lin(p + ".temb", co, E)
            gn(p + ".gn2", co)
            conv(p + ".conv2", co, co)
            if ci != co:
                lin(p + ".skip", co, ci)
        elif p in t2d:
            c, dep = t2d[p]
            gn(p + ".gn", c)
            lin(p + ".proj_in", c, c)
            F = 4 * c
            for i in range(dep):
                q = f"{p}.blk.{i}"
                t += [(q + ".ln1.g", (c,), 0), (q + ".ln1.b", (c,), 0)]
                t.append((q + ".attn1.qkv.w", (3 * c, c), c))
                lin(q + ".attn1.out", c, c)
                t += [(q + ".ln2.g", (c,), 0), (q + ".ln2.b", (c,), 0)]
                t.append((q + ".attn2.q.w", (c, c), c))
                t.append((q + ".attn2.kv.w", (2 * c, u.ctx_dim), u.ctx_dim))
                lin(q + ".attn2.out", c, c)
                t += [(q + ".ln3.g", (c,), 0), (q + ".ln3.b", (c,), 0)]
                lin(q + ".ff.geglu", 2 * F, c)
                lin(q + ".ff.out", c, F)
            lin(p + ".proj_out", c, c)
        else:  # resampler conv
            lvl = int(p.split(".")[1])
            c = u.ch[lvl] if p.startswith("down") else u.ch[(2, 1, 0)[lvl]]
            conv(p + ".conv", c, c)
    gn("out.gn", u.ch[0])
    conv("conv_out", u.ch[0], u.lat_ch)
    return t


def make_unet_full_weights(u: UNetDesc, seed: int = 0, device="cpu", dtype=torch.float32, names=None):
    """uniform(+-1/sqrt(fan_in)) matrices and biases; GroupNorm / LayerNorm gains 1 + 0.1 u and
    shifts 0.1 u (the same recipe as the attention stack, C-AMB 20)."""
    out = {}
    for name, shape, fan_in in unet_full_weight_table(u):
        if names is not None and name not in names:
            continue
        if fan_in == 0:  # norm gain / shift
            v = uniform(seed, "unetfull." + name, shape, device) * 0.1 + (1.0 if name.endswith(".g") else 0.0)
        else:
            v = uniform(seed, "unetfull." + name, shape, device) * (1.0 / math.sqrt(fan_in))
        out[name] = v.to(torch.float32).to(dtype)
    return out


def make_unet_latent(u: UNetDesc, rid: int, device="cpu") -> torch.Tensor:
    """Request latent [grid * grid, lat_ch] fp32 (tokens = latent pixels, row-major)."""
    return normal(rid, "unet_latent", (u.grid * u.grid, u.lat_ch), device).to(torch.float32)


UNET_FULL_TINY = UNetDesc("unet_full_tiny", 4, 16, (64, 64, 128), (0, 1, 1), head_dim=64, ctx_len=7, ctx_dim=64)
UNET_FULL_SMALL = UNetDesc("unet_full_small", 4, 32, (64, 128, 128), (0, 2, 2), head_dim=64, ctx_len=13, ctx_dim=64)
SDXL_UNET = UNetDesc("sdxl_unet", 4, 128, (320, 640, 1280), (0, 2, 10))
UNET_FULL = {u.name: u for u in (UNET_FULL_TINY, UNET_FULL_SMALL, SDXL_UNET)}
