"""Thin ctypes binding of libig (include/ig.h, include/ig_ops.h) — argument marshalling only.

Every function has the C name and forwards to libig.so; every step of the hot path runs in
the library's CUDA kernels.  There is no fallback: if libig.so is missing or fails to load,
`lib()` raises.  Pointers are plain integers (e.g. torch `tensor.data_ptr()`), streams are
`torch.cuda.Stream.cuda_stream` integers (0 = legacy default stream).
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IG_LIB_OVERRIDE") or os.path.join(_HERE, "lib", "libig.so")  # override: A/B benchmarking only
_lib = None

IG_F32, IG_BF16 = 0, 1
IG_CACHE_HOST, IG_CACHE_DEVICE = 0, 1
STATUS = {0: "IG_OK", 1: "IG_EINVAL", 2: "IG_ECACHE_INCOMPAT", 3: "IG_ECACHE_MISS",
          4: "IG_ENUMERIC", 5: "IG_ENOMEM", 6: "IG_ECUDA", 7: "IG_EUNSUPPORTED"}

EXPORTS = ["ig_weight_count", "ig_ctx_create", "ig_ctx_destroy", "ig_cache_create",
           "ig_cache_template", "ig_cache_storage", "ig_cache_free", "ig_mask_build",
           "ig_mask_indices", "ig_mask_free", "ig_edit_step", "ig_prefetch_layer",
           "ig_last_error", "ig_last_stats", "ig_op_gemm", "ig_op_gemm_gated", "ig_op_attention", "ig_copy",
           "ig_profile_enable", "ig_profile_read", "ig_debug_block", "ig_cache_clone", "ig_cache_write",
           "ig_set_plan", "ig_last_plan", "ig_debug_set", "ig_debug_dump_kv",
           "ig_mask_build_host", "ig_stage_input", "ig_cache_template_into", "ig_cache_bytes",
           "ig_cache_attach", "ig_cache_export", "ig_cache_import", "ig_record_step",
           "ig_tuning_get", "ig_tuning_set",
           "ig_unet_weight_count", "ig_unet_create", "ig_unet_destroy", "ig_unet_mask_build",
           "ig_unet_mask_free", "ig_unet_template", "ig_unet_cache_free", "ig_unet_step", "ig_unet_last_stats",
           "ig_op_conv3x3", "ig_plan_copy_groups"]
IG_CACHE_HANDLE_BYTES = 128
IG_DBG_SPIN_COPY_NS, IG_DBG_SPIN_COMPUTE_NS, IG_DBG_DROP_RAW, IG_DBG_DROP_WAR = 1, 2, 3, 4
IG_DBG_CORRUPT_ROW, IG_DBG_POISON_RING, IG_DBG_SEQUENTIAL = 5, 6, 7
KCLASS = ["gemm", "attn", "lnmod", "qkvpost", "cond", "rows", "copy"]


class IgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class ig_model_desc(ctypes.Structure):
    _fields_ = [("n_double", ctypes.c_int), ("n_single", ctypes.c_int),
                ("hidden", ctypes.c_int), ("heads", ctypes.c_int), ("head_dim", ctypes.c_int),
                ("mlp_hidden", ctypes.c_int), ("lat_ch", ctypes.c_int), ("grid_h", ctypes.c_int),
                ("grid_w", ctypes.c_int), ("txt_len", ctypes.c_int), ("qk_norm", ctypes.c_int),
                ("rope", ctypes.c_int), ("rope_axes", ctypes.c_int * 3),
                ("rope_theta", ctypes.c_float), ("ln_eps", ctypes.c_float),
                ("pos_embed_2d", ctypes.c_int), ("context_pre_only_last", ctypes.c_int),
                ("dtype", ctypes.c_int), ("n_unet", ctypes.c_int), ("ctx_len", ctypes.c_int),
                ("ctx_dim", ctypes.c_int)]


class ig_ctx_opts(ctypes.Structure):
    _fields_ = [("max_batch", ctypes.c_int), ("max_rows", ctypes.c_int),
                ("prefetch_depth", ctypes.c_int), ("copy_mode", ctypes.c_int),
                ("debug_checks", ctypes.c_int), ("cache_fp8", ctypes.c_int), ("cache_y", ctypes.c_int),
                ("cache_kv_blocks", ctypes.c_int), ("use_graphs", ctypes.c_int)]


class ig_edit_req(ctypes.Structure):
    _fields_ = [("slot", ctypes.c_int), ("latent", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("cache", ctypes.c_void_p), ("step", ctypes.c_int), ("sigma", ctypes.c_float),
                ("sigma_next", ctypes.c_float), ("txt", ctypes.c_void_p),
                ("cond_vec", ctypes.c_void_p)]


class ig_unet_desc(ctypes.Structure):
    _fields_ = [("lat_ch", ctypes.c_int), ("grid", ctypes.c_int), ("ch", ctypes.c_int * 3),
                ("depth", ctypes.c_int * 3), ("head_dim", ctypes.c_int), ("ctx_len", ctypes.c_int),
                ("ctx_dim", ctypes.c_int), ("n_res", ctypes.c_int), ("gn_groups", ctypes.c_int),
                ("gn_eps", ctypes.c_float), ("t2d_gn_eps", ctypes.c_float), ("ln_eps", ctypes.c_float)]


class ig_unet_req(ctypes.Structure):
    _fields_ = [("latent", ctypes.c_void_p), ("mask", ctypes.c_void_p), ("cache", ctypes.c_void_p),
                ("step", ctypes.c_int), ("sigma", ctypes.c_float), ("sigma_next", ctypes.c_float),
                ("ctx", ctypes.c_void_p), ("cond", ctypes.c_void_p)]


class ig_stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_longlong), ("h2d_bytes", ctypes.c_longlong),
                ("d2d_bytes", ctypes.c_longlong), ("d2h_bytes", ctypes.c_longlong),
                ("rows", ctypes.c_longlong), ("host_ns", ctypes.c_longlong),
                ("dma_calls", ctypes.c_longlong)]


class ig_prof_entry(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_longlong), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]



class ig_tuning(ctypes.Structure):
    """include/ig_ops.h ig_tuning: process-wide libig knobs (see the header for each field)."""
    _fields_ = [(n, ctypes.c_int) for n in ("pdl", "copy_thread", "load_dedupe", "cross_kv_overlap",
                                            "gemm_two_cta", "gemm_small_tiles", "gemm_bn64", "conv_two_cta",
                                            "precise_gelu", "op_repeat", "txt_overlap")]


def lib():
    """Load libig.so (in-tree).  Raises if it is missing: there is no other path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libig.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
        P = ctypes.POINTER
        L.ig_weight_count.argtypes = [P(ig_model_desc)]
        L.ig_weight_count.restype = i
        L.ig_ctx_create.argtypes = [P(ig_model_desc), P(vp), i, i, P(ig_ctx_opts), P(vp)]
        L.ig_ctx_destroy.argtypes = [vp]
        L.ig_ctx_destroy.restype = None
        L.ig_cache_create.argtypes = [vp, i, i, P(vp)]
        L.ig_cache_template.argtypes = [vp, vp, vp, vp, P(ctypes.c_float), i, i, vp, P(vp)]
        L.ig_cache_storage.argtypes = [vp, P(vp), P(ctypes.c_size_t), P(i)]
        L.ig_cache_free.argtypes = [vp]
        L.ig_cache_free.restype = None
        L.ig_mask_build.argtypes = [vp, vp, vp, P(vp), P(i)]
        L.ig_mask_indices.argtypes = [vp, P(vp), P(vp), P(i)]
        L.ig_mask_free.argtypes = [vp]
        L.ig_mask_free.restype = None
        L.ig_edit_step.argtypes = [vp, P(ig_edit_req), i, vp]
        L.ig_prefetch_layer.argtypes = [vp, P(ig_edit_req), i]
        L.ig_last_error.restype = ctypes.c_char_p
        L.ig_last_plan.restype = ctypes.c_int
        L.ig_last_stats.argtypes = [vp, P(ig_stats)]
        L.ig_plan_copy_groups.argtypes = [vp, i, i, i, P(ctypes.c_int), i, P(i)]
        L.ig_op_gemm.argtypes = [i, vp, ll, vp, ll, vp, vp, ll, i, i, i, i, i, vp]
        L.ig_op_attention.argtypes = [i, vp, ll, vp, ll, vp, P(ctypes.c_int32), i, i, i, i, vp]
        L.ig_copy.argtypes = [vp, vp, ctypes.c_size_t, vp]
        L.ig_op_gemm_gated.argtypes = [i, vp, ll, vp, ll, vp, vp, ll, vp, i, i, i, vp]
        L.ig_profile_enable.argtypes = [vp, i]
        L.ig_cache_clone.argtypes = [vp, vp, i, P(vp)]
        L.ig_cache_write.argtypes = [vp, vp, vp, vp, vp]
        d_ = ctypes.c_double
        L.ig_set_plan.argtypes = [vp, i, i, d_, d_, d_, d_]
        L.ig_last_plan.argtypes = [vp]
        L.ig_debug_block.argtypes = [vp, P(ig_edit_req), i, vp, vp, vp]
        L.ig_profile_read.argtypes = [vp, P(ig_prof_entry)]
        L.ig_debug_set.argtypes = [vp, i, ll]
        L.ig_mask_build_host.argtypes = [vp, vp, vp, P(vp), P(i)]
        L.ig_stage_input.argtypes = [vp, vp, ctypes.c_size_t, vp]
        L.ig_tuning_get.argtypes = [P(ig_tuning)]
        L.ig_tuning_set.argtypes = [P(ig_tuning)]
        L.ig_cache_template_into.argtypes = [vp, vp, vp, vp, P(ctypes.c_float), i, vp, vp]
        L.ig_cache_bytes.argtypes = [vp, i, P(ctypes.c_size_t)]
        L.ig_cache_attach.argtypes = [vp, i, vp, ctypes.c_size_t, P(vp)]
        L.ig_cache_export.argtypes = [vp, vp, ctypes.c_size_t]
        L.ig_record_step.argtypes = [vp, P(ig_edit_req), vp, i, vp]
        L.ig_op_conv3x3.argtypes = [vp, i, i, i, i, vp, vp, i, vp, vp]
        L.ig_unet_weight_count.argtypes = [P(ig_unet_desc)]
        L.ig_unet_weight_count.restype = i
        L.ig_unet_create.argtypes = [P(ig_unet_desc), P(vp), i, i, i, i, P(vp)]
        L.ig_unet_destroy.argtypes = [vp]
        L.ig_unet_destroy.restype = None
        L.ig_unet_mask_build.argtypes = [vp, vp, vp, P(vp), P(i)]
        L.ig_unet_mask_free.argtypes = [vp]
        L.ig_unet_mask_free.restype = None
        L.ig_unet_template.argtypes = [vp, vp, vp, vp, P(ctypes.c_float), i, i, vp, P(vp)]
        L.ig_unet_cache_free.argtypes = [vp]
        L.ig_unet_cache_free.restype = None
        L.ig_unet_step.argtypes = [vp, P(ig_unet_req), i, vp]
        L.ig_unet_last_stats.argtypes = [vp, P(ig_stats)]
        L.ig_cache_import.argtypes = [vp, vp, P(vp)]
        L.ig_debug_dump_kv.argtypes = [vp, i, i, vp, vp, vp]
        for name in EXPORTS:
            if name not in ("ig_ctx_destroy", "ig_cache_free", "ig_mask_free", "ig_last_error",
                            "ig_weight_count", "ig_last_plan", "ig_unet_weight_count", "ig_unet_destroy",
                            "ig_unet_mask_free", "ig_unet_cache_free"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise IgError(status, lib().ig_last_error().decode())


def make_desc(m, dtype: int) -> ig_model_desc:
    """Fill ig_model_desc from any object with the ig.h field names as attributes."""
    d = ig_model_desc()
    for f, _ in ig_model_desc._fields_:
        if f == "rope_axes":
            d.rope_axes = (ctypes.c_int * 3)(*m.rope_axes)
        elif f == "dtype":
            d.dtype = dtype
        else:
            setattr(d, f, getattr(m, f))
    return d


def ig_weight_count(desc: ig_model_desc) -> int:
    return lib().ig_weight_count(ctypes.byref(desc))


def ig_ctx_create(desc: ig_model_desc, weight_ptrs: Sequence[int], device: int = 0,
                  opts: Optional[ig_ctx_opts] = None) -> int:
    arr = (ctypes.c_void_p * len(weight_ptrs))(*weight_ptrs)
    out = ctypes.c_void_p()
    _check(lib().ig_ctx_create(ctypes.byref(desc), arr, len(weight_ptrs), device,
                               ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def ig_ctx_destroy(ctx: int):
    lib().ig_ctx_destroy(ctx)


def ig_mask_build(ctx: int, mask_ptr: int, stream: int = 0):
    out, n = ctypes.c_void_p(), ctypes.c_int()
    _check(lib().ig_mask_build(ctx, mask_ptr, stream, ctypes.byref(out), ctypes.byref(n)))
    return out.value, n.value


def ig_mask_build_host(ctx: int, mask_u8, stream: int = 0):
    """mask_u8: a host buffer of L_img bytes (numpy uint8 array or ctypes address)."""
    if hasattr(mask_u8, "ctypes"):
        import numpy as _np
        mask_u8 = _np.ascontiguousarray(mask_u8, dtype=_np.uint8)
        ptr = mask_u8.ctypes.data
    else:
        ptr = int(mask_u8)
    out, n = ctypes.c_void_p(), ctypes.c_int()
    _check(lib().ig_mask_build_host(ctx, ptr, stream, ctypes.byref(out), ctypes.byref(n)))
    return out.value, n.value


def ig_stage_input(dst: int, src: int, nbytes: int, stream: int = 0):
    _check(lib().ig_stage_input(dst, src, nbytes, stream))


def ig_mask_indices(mask: int):
    pm, pu, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int()
    _check(lib().ig_mask_indices(mask, ctypes.byref(pm), ctypes.byref(pu), ctypes.byref(n)))
    return pm.value, pu.value, n.value


def ig_mask_free(mask: int):
    lib().ig_mask_free(mask)


def ig_cache_create(ctx: int, n_steps: int, tier: int = IG_CACHE_HOST) -> int:
    out = ctypes.c_void_p()
    _check(lib().ig_cache_create(ctx, n_steps, tier, ctypes.byref(out)))
    return out.value


def ig_cache_template(ctx: int, latent_ptr: int, txt_ptr: int, cond_ptr: int,
                      sigmas: Sequence[float], tier: int = IG_CACHE_HOST, stream: int = 0) -> int:
    s = (ctypes.c_float * len(sigmas))(*[float(x) for x in sigmas])
    out = ctypes.c_void_p()
    _check(lib().ig_cache_template(ctx, latent_ptr, txt_ptr, cond_ptr, s, len(sigmas) - 1, tier,
                                   stream, ctypes.byref(out)))
    return out.value


def ig_cache_template_into(ctx: int, latent_ptr: int, txt_ptr: int, cond_ptr: int,
                           sigmas: Sequence[float], cache: int, stream: int = 0):
    s = (ctypes.c_float * len(sigmas))(*[float(x) for x in sigmas])
    _check(lib().ig_cache_template_into(ctx, latent_ptr, txt_ptr, cond_ptr, s, len(sigmas) - 1, cache, stream))


def ig_cache_bytes(ctx: int, n_steps: int) -> int:
    b = ctypes.c_size_t()
    _check(lib().ig_cache_bytes(ctx, n_steps, ctypes.byref(b)))
    return b.value


def ig_cache_attach(ctx: int, n_steps: int, host_ptr: int, nbytes: int) -> int:
    out = ctypes.c_void_p()
    _check(lib().ig_cache_attach(ctx, n_steps, host_ptr, nbytes, ctypes.byref(out)))
    return out.value


def ig_cache_export(cache: int) -> bytes:
    buf = ctypes.create_string_buffer(IG_CACHE_HANDLE_BYTES)
    _check(lib().ig_cache_export(cache, buf, IG_CACHE_HANDLE_BYTES))
    return buf.raw


def ig_cache_import(ctx: int, handle: bytes) -> int:
    buf = ctypes.create_string_buffer(bytes(handle), IG_CACHE_HANDLE_BYTES)
    out = ctypes.c_void_p()
    _check(lib().ig_cache_import(ctx, buf, ctypes.byref(out)))
    return out.value


def ig_cache_storage(cache: int):
    p, b, t = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_int()
    _check(lib().ig_cache_storage(cache, ctypes.byref(p), ctypes.byref(b), ctypes.byref(t)))
    return p.value, b.value, t.value


def ig_cache_free(cache: int):
    lib().ig_cache_free(cache)


def make_req(slot, latent, mask, cache, step, sigma, sigma_next, txt, cond) -> ig_edit_req:
    return ig_edit_req(slot, latent, mask, cache or None, step, sigma, sigma_next, txt or None, cond)


def ig_edit_step(ctx: int, reqs: List[ig_edit_req], stream: int = 0):
    arr = (ig_edit_req * max(1, len(reqs)))(*reqs)
    _check(lib().ig_edit_step(ctx, arr, len(reqs), stream))


def ig_prefetch_layer(ctx: int, req: ig_edit_req, layer: int):
    _check(lib().ig_prefetch_layer(ctx, ctypes.byref(req), layer))


def ig_last_error() -> str:
    return lib().ig_last_error().decode()


def ig_plan_copy_groups(mask_u8, W: int = 0, row_bytes: int = 6144) -> list:
    """Host-only: the copy lane's DMA groups [(start, len, stride, count)] for a mask."""
    import numpy as _np
    m = _np.ascontiguousarray(mask_u8, dtype=_np.uint8).reshape(-1)
    cap = m.size + 1
    buf = (ctypes.c_int * (4 * cap))()
    n = ctypes.c_int()
    _check(lib().ig_plan_copy_groups(m.ctypes.data, int(m.size), int(W), int(row_bytes), buf, cap, ctypes.byref(n)))
    return [tuple(buf[4 * k:4 * k + 4]) for k in range(n.value)]


def ig_last_stats(ctx: int) -> dict:
    s = ig_stats()
    _check(lib().ig_last_stats(ctx, ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in ig_stats._fields_}


def ig_op_gemm(dtype, A, lda, B, ldb, bias, C, ldc, M, N, K, epi=0, out_f32=0, stream=0):
    _check(lib().ig_op_gemm(dtype, A, lda, B, ldb, bias or None, C, ldc, M, N, K, epi, out_f32,
                            stream))


def ig_op_gemm_gated(dtype, A, lda, B, ldb, bias, X, ldx, gate, M, N, K, stream=0):
    _check(lib().ig_op_gemm_gated(dtype, A, lda, B, ldb, bias or None, X, ldx, gate, M, N, K, stream))


def ig_op_attention(dtype, Q, ldq, O, ldo, kv, segs, L, heads, head_dim, stream=0):
    flat = [int(x) for s in segs for x in s]
    arr = (ctypes.c_int32 * len(flat))(*flat)
    _check(lib().ig_op_attention(dtype, Q, ldq, O, ldo, kv, arr, len(segs), L, heads, head_dim,
                                 stream))


def ig_copy(dst: int, src: int, nbytes: int, stream: int = 0):
    _check(lib().ig_copy(dst, src, nbytes, stream))


def ig_profile_enable(ctx: int, enable: bool = True):
    _check(lib().ig_profile_enable(ctx, int(enable)))


def ig_profile_read(ctx: int) -> dict:
    arr = (ig_prof_entry * len(KCLASS))()
    _check(lib().ig_profile_read(ctx, arr))
    return {k: {f: getattr(arr[i], f) for f, _ in ig_prof_entry._fields_} for i, k in enumerate(KCLASS)}


def ig_debug_block(ctx: int, req: ig_edit_req, block: int, X_in: int, X_out: int, stream: int = 0):
    _check(lib().ig_debug_block(ctx, ctypes.byref(req), block, X_in, X_out, stream))


def ig_debug_set(ctx: int, key: int, value: int = 0):
    _check(lib().ig_debug_set(ctx, key, value))


def ig_debug_dump_kv(ctx: int, slot: int, block: int, k_out: int, v_out: int, stream: int = 0):
    _check(lib().ig_debug_dump_kv(ctx, slot, block, k_out, v_out, stream))


def ig_cache_clone(ctx: int, cache: int, tier: int) -> int:
    out = ctypes.c_void_p()
    _check(lib().ig_cache_clone(ctx, cache, tier, ctypes.byref(out)))
    return out.value


def ig_cache_write(ctx: int, cache: int, kv_ptr: int, latents_ptr: int = 0, stream: int = 0):
    _check(lib().ig_cache_write(ctx, cache, kv_ptr, latents_ptr or None, stream))


def ig_set_plan(ctx: int, mode: int, k: int = 0, comp_s_per_flop: float = 0.0, comp_s: float = 0.0,
                load_s_per_byte: float = 0.0, load_s: float = 0.0):
    _check(lib().ig_set_plan(ctx, mode, k, comp_s_per_flop, comp_s, load_s_per_byte, load_s))


def ig_last_plan(ctx: int) -> int:
    return lib().ig_last_plan(ctx)


def y_block_modes(n_blocks: int, kv_blocks: int):
    """The Y blocks of a hybrid cache (ig.h cache_kv_blocks): the first n_blocks - kv_blocks
    entries of the bit-reversal order over the next power of two >= n_blocks."""
    bits = max(0, (n_blocks - 1).bit_length())
    ny = n_blocks - max(0, min(kv_blocks, n_blocks))
    out, k = [], 0
    while len(out) < ny:
        v = int(format(k, f"0{bits}b")[::-1], 2) if bits else 0
        if v < n_blocks:
            out.append(v)
        k += 1
    return sorted(out)


# ---------------------------------------------------------------------------- whole UNet
def ig_record_step(ctx: int, req: ig_edit_req, cache: int, step: int, stream: int = 0):
    _check(lib().ig_record_step(ctx, ctypes.byref(req), cache, step, stream))


def make_unet_desc(u) -> ig_unet_desc:
    d = ig_unet_desc()
    d.lat_ch, d.grid = u.lat_ch, u.grid
    d.ch = (ctypes.c_int * 3)(*u.ch)
    d.depth = (ctypes.c_int * 3)(*u.depth)
    d.head_dim, d.ctx_len, d.ctx_dim, d.n_res, d.gn_groups = u.head_dim, u.ctx_len, u.ctx_dim, u.n_res, u.gn_groups
    d.gn_eps, d.t2d_gn_eps, d.ln_eps = u.gn_eps, u.t2d_gn_eps, u.ln_eps
    return d


def ig_unet_weight_count(desc: ig_unet_desc) -> int:
    return lib().ig_unet_weight_count(ctypes.byref(desc))


def ig_unet_create(desc: ig_unet_desc, weight_ptrs, device: int = 0, max_batch: int = 8, prefetch_depth: int = 2) -> int:
    arr = (ctypes.c_void_p * len(weight_ptrs))(*weight_ptrs)
    out = ctypes.c_void_p()
    _check(lib().ig_unet_create(ctypes.byref(desc), arr, len(weight_ptrs), device, max_batch, prefetch_depth,
                                ctypes.byref(out)))
    return out.value


def ig_unet_destroy(u: int):
    lib().ig_unet_destroy(u)


def ig_unet_mask_build(u: int, mask_u8, stream: int = 0):
    import numpy as _np
    m = _np.ascontiguousarray(mask_u8, dtype=_np.uint8)
    out, n = ctypes.c_void_p(), ctypes.c_int()
    _check(lib().ig_unet_mask_build(u, m.ctypes.data, stream, ctypes.byref(out), ctypes.byref(n)))
    return out.value, n.value


def ig_unet_mask_free(m: int):
    lib().ig_unet_mask_free(m)


def ig_unet_template(u: int, latent_ptr: int, ctx_ptr: int, cond_ptr: int, sigmas, tier: int = IG_CACHE_DEVICE,
                     stream: int = 0) -> int:
    s = (ctypes.c_float * len(sigmas))(*[float(x) for x in sigmas])
    out = ctypes.c_void_p()
    _check(lib().ig_unet_template(u, latent_ptr, ctx_ptr, cond_ptr or None, s, len(sigmas) - 1, tier, stream,
                                  ctypes.byref(out)))
    return out.value


def ig_unet_cache_free(c: int):
    lib().ig_unet_cache_free(c)


def make_unet_req(latent, mask, cache, step, sigma, sigma_next, ctx, cond=None) -> ig_unet_req:
    return ig_unet_req(latent, mask, cache or None, step, sigma, sigma_next, ctx, cond or None)


def ig_unet_step(u: int, reqs, stream: int = 0):
    arr = (ig_unet_req * max(1, len(reqs)))(*reqs)
    _check(lib().ig_unet_step(u, arr, len(reqs), stream))


def ig_unet_last_stats(u: int) -> dict:
    s = ig_stats()
    _check(lib().ig_unet_last_stats(u, ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in ig_stats._fields_}


def ig_op_conv3x3(x_padded: int, n_img: int, H: int, W: int, cin: int, w: int, bias: int, cout: int, y: int,
                  stream: int = 0):
    _check(lib().ig_op_conv3x3(x_padded, n_img, H, W, cin, w, bias or None, cout, y, stream))


def ig_tuning_get() -> "ig_tuning":
    t = ig_tuning()
    _check(lib().ig_tuning_get(ctypes.byref(t)))
    return t


def ig_tuning_set(t: "ig_tuning"):
    _check(lib().ig_tuning_set(ctypes.byref(t)))
