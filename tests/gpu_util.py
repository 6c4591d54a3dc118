"""Helpers for the -m gpu parity tests: build a context from synth weights, run steps
through the C ABI, and compare with the oracle using C-TOL."""
import numpy as np
import torch

import synth
from paper_2505_20600_b200 import ig

TDT = {ig.IG_F32: torch.float32, ig.IG_BF16: torch.bfloat16}


def ctol(g, o, rtol, atol_mult=1.0):
    """C-TOL (DESIGN.md C-AMB 22): |g - o| <= rtol |o| + atol_mult rtol RMS(o), elementwise."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    atol = atol_mult * rtol * np.sqrt(np.mean(o * o)) if o.size else 0.0
    err = np.abs(g - o)
    ok = err <= rtol * np.abs(o) + atol
    worst = float(np.max(err / (rtol * np.abs(o) + atol + 1e-300))) if o.size else 0.0
    return bool(ok.all()), worst


def bf16_rounding_bound(parts, n_elems, stages=4, p_fail=1e-3):
    """Elementwise bound on the bf16 rounding error of a gated block update (DESIGN.md C-AMB 22,
    C-TOL-full), from a probabilistic model of the arithmetic, not from measurement.

    The update is a sum of gated GEMMs u_ij = sum_parts g_j sum_k a_ik w_jk (+ bias), whose A
    operand a_ik reaches the tensor core rounded to bf16: a_ik (1 + d_ik), |d_ik| <= u = 2^-9
    (round to nearest, 8 significant bits), independent, zero mean, variance u^2/3.  The error
    e_ij = g_j sum_k a_ik w_jk d_ik is a sum of independent bounded terms, so by Hoeffding
    P(|e_ij| > t) <= 2 exp(-t^2 / (2 sigma^2 ...)); with a family-wise failure probability
    p_fail over n_elems elements, |e_ij| <= z * sigma_ij, z = sqrt(2 ln(2 n / p_fail)),
    sigma_ij^2 = (u^2/3) sum_parts g_j^2 sum_k a_ik^2 w_jk^2.  The operand a itself carries the
    errors of the upstream bf16 roundings on its path (h, q/k/v, P, O: `stages` of them, each of
    the same form and magnitude to first order), which multiplies sigma by sqrt(1 + stages).
    parts: [(A [n, K] exact float64 operand rows, W [N, K], g [N])].  Returns [n, N]."""
    u = 2.0 ** -9
    z = np.sqrt(2.0 * np.log(2.0 * n_elems / p_fail))
    var = None
    for A, W, g in parts:
        v = (A * A) @ (W * W).T * (g * g)[None, :]
        var = v if var is None else var + v
    return z * np.sqrt(1.0 + stages) * u / np.sqrt(3.0) * np.sqrt(var)


def ctol_or_bound(g, o, rtol, bound):
    """C-TOL-full: an element passes if it meets C-TOL (|g-o| <= rtol |o| + rtol RMS(o)) or lies
    within its own bf16 rounding bound (bf16_rounding_bound).  Returns (ok, worst ratio against
    the larger of the two allowances)."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    err = np.abs(g - o)
    allow = np.maximum(rtol * np.abs(o) + rtol * np.sqrt(np.mean(o * o)), bound) + 1e-300
    return bool((err <= allow).all()), float(np.max(err / allow))


class Model:
    """Synthetic weights on the device + an ig context."""

    def __init__(self, d, dtype, seed=0, opts=None, device="cuda"):
        self.d, self.dtype = d, dtype
        tdt = TDT[dtype]
        self.W = {}
        ptrs = []
        for name, shape, fan_in in synth.weight_table(d):
            t = synth.make_weight(d, name, shape, fan_in, seed, device, tdt).contiguous()
            self.W[name] = t
            ptrs.append(t.data_ptr())
        self.desc = ig.make_desc(d, dtype)
        self.ctx = ig.ig_ctx_create(self.desc, ptrs, 0, opts)

    def host_weights(self):
        return {k: v.double().cpu().numpy() for k, v in self.W.items()}

    def close(self):
        if self.ctx:
            ig.ig_ctx_destroy(self.ctx)
            self.ctx = None


class Request:
    def __init__(self, m, rid, mask_np, device="cuda"):
        d = m.d
        self.latent = synth.make_latent(d, rid, device).contiguous()
        self.latent0 = self.latent.clone()
        if d.n_unet:  # UNet: the txt slot carries the cross-attention context
            self.txt = synth.make_ctx(d, rid, device, TDT[m.dtype]).contiguous()
        else:
            self.txt = synth.make_txt(d, rid, device, TDT[m.dtype]).contiguous()
        self.cond = synth.make_cond(d, rid, device).contiguous()
        self.mask_np = mask_np.astype(np.uint8)
        self.mask_dev = torch.from_numpy(self.mask_np).to(device)
        self.mask, self.n_m = ig.ig_mask_build(m.ctx, self.mask_dev.data_ptr(), 0)

    def req(self, slot, cache, step, sigma, sigma_next):
        return ig.make_req(slot, self.latent.data_ptr(), self.mask, cache, step, sigma, sigma_next,
                           self.txt.data_ptr() if self.txt.numel() else None, self.cond.data_ptr())

    def host_inputs(self):
        return (self.latent0.double().cpu().numpy(), self.txt.double().cpu().numpy(),
                self.cond.double().cpu().numpy())

    def free(self):
        ig.ig_mask_free(self.mask)


def cache_to_numpy(cache, d, n_steps, dtype, y=False):
    """Host-tier cache readback: K/V [steps, blocks, 2, L_img, H] (or Y [steps, blocks, L_img, H])."""
    ptr, nbytes, tier = ig.ig_cache_storage(cache)
    shape = (n_steps, d.n_blocks) + (() if y else (2,)) + (d.L_img, d.hidden)
    nbytes = int(np.prod(shape)) * (4 if dtype == ig.IG_F32 else 2)  # K/V (Y) region
    assert tier == ig.IG_CACHE_HOST, 'host-tier readback only'
    import ctypes
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    raw = np.frombuffer(buf, dtype=np.uint8).copy()
    if dtype == ig.IG_F32:
        return raw.view(np.float32).reshape(shape).astype(np.float64)
    u16 = raw.view(np.uint16).astype(np.uint32) << 16
    return u16.view(np.float32).reshape(shape).astype(np.float64)


def fill_cache(m, cache, kv: torch.Tensor, latents: torch.Tensor = None):
    """Write a synthetic cache [steps, blocks, 2, L_img, H] (+ optional template latents
    [steps, L_img, C]) through ig_cache_write."""
    src = kv.contiguous().cuda()
    lat = latents.contiguous().cuda().float() if latents is not None else None
    ig.ig_cache_write(m.ctx, cache, src.data_ptr(), lat.data_ptr() if lat is not None else 0)


def hybrid_planes(kv, y, ymodes):
    """Storage order of a hybrid cache step by step (ig.h cache_kv_blocks): block b contributes
    [K_b, V_b] if it is a K/V block, then [Y_b] if block b or b + 1 is a Y block.
    kv: [steps, blocks, 2, L_img, H], y: [steps, blocks, L_img, H], ymodes: set of Y blocks
    -> [steps, planes, L_img, H]."""
    import torch as _t
    steps, nb = kv.shape[0], kv.shape[1]
    out = []
    for s in range(steps):
        pl = []
        for b in range(nb):
            if b not in ymodes:
                pl += [kv[s, b, 0], kv[s, b, 1]]
            if b in ymodes or (b + 1) in ymodes:
                pl.append(y[s, b])
        out.append(_t.stack(pl))
    return _t.stack(out)


def split_hybrid(raw, nb, ymodes):
    """Inverse of hybrid_planes on a numpy [steps, planes, L_img, H] array -> (kv, y) with
    zeros where a block stores nothing."""
    steps = raw.shape[0]
    kv = np.zeros((steps, nb, 2) + raw.shape[2:])
    y = np.zeros((steps, nb) + raw.shape[2:])
    for s in range(steps):
        i = 0
        for b in range(nb):
            if b not in ymodes:
                kv[s, b, 0], kv[s, b, 1] = raw[s, i], raw[s, i + 1]
                i += 2
            if b in ymodes or (b + 1) in ymodes:
                y[s, b] = raw[s, i]
                i += 1
    return kv, y


def n_planes(nb, ymodes):
    return sum((0 if b in ymodes else 2) + (1 if (b in ymodes or (b + 1) in ymodes) else 0) for b in range(nb))


def cache_raw_numpy(cache, d, n_steps, n_planes, dtype):
    """Host-tier cache readback of the plane region [steps, planes, L_img, H]."""
    import ctypes
    ptr, nbytes, tier = ig.ig_cache_storage(cache)
    assert tier == ig.IG_CACHE_HOST
    shape = (n_steps, n_planes, d.L_img, d.hidden)
    nbytes = int(np.prod(shape)) * (4 if dtype == ig.IG_F32 else 2)
    raw = np.frombuffer((ctypes.c_char * nbytes).from_address(ptr), dtype=np.uint8).copy()
    if dtype == ig.IG_F32:
        return raw.view(np.float32).reshape(shape).astype(np.float64)
    return (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).reshape(shape).astype(np.float64)
