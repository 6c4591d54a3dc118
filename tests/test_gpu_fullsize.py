"""Full-size (Flux.1-dev-shaped, BASELINE configs[2]) GPU checks in the launch configuration
bench.py times (bf16, tcgen05 kernels, max_batch 8 context):

* teacher-forced blocks: one double and one single block at full width
  (H = 3072, L = 4608) through ig_debug_block vs the oracle's block functions on the same
  inputs, m in {0.05, 0.2, 0.6}; compared on the block's update (X_out - X_in) with C-TOL 2e-2;
* exactness invariants at full scale: with a cache recorded from the same
  trajectory, the edited masked rows equal the dense step's rows bitwise; unmasked rows are
  untouched; a request alone equals the same request inside a batch, bitwise.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_20600_b200 import ig
import oracle.instgenie as oi
from gpu_util import Model, Request, bf16_rounding_bound, ctol, ctol_or_bound

pytestmark = pytest.mark.gpu

D = synth.FLUX


@pytest.fixture(scope="module")
def flux():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    m = Model(D, ig.IG_BF16, opts=ig.ig_ctx_opts(8, 8 * D.L, 2, 1, 0))
    yield m
    m.close()


def _update_bound(d, W, block, Xh, vec, idx_m, idx_u, kvh):
    """bf16 rounding bound of a block's update rows (gpu_util.bf16_rounding_bound): the exact
    operands of the block's final gated GEMMs, recomputed with the oracle's own functions."""
    Lt = d.txt_len
    n = Xh.shape[0]
    N = n * d.hidden
    if block >= d.n_double:
        p = f"single.{block - d.n_double}"
        m = oi.modulation(W, p, vec, 3)
        pos = np.concatenate([np.zeros((Lt, 3), np.int64), oi.image_positions(d, idx_m)])
        q, k, v, u = oi._single_pre(d, W, p, Xh, m, pos)
        K = oi.merge_kv(d, k[:Lt], k[Lt:], idx_m, idx_u, kvh[0])
        V = oi.merge_kv(d, v[:Lt], v[Lt:], idx_m, idx_u, kvh[1])
        o = oi.attention(q, K, V, d.heads)
        A = np.concatenate([o, oi.gelu_tanh(u)], axis=1)
        return bf16_rounding_bound([(A, W[p + ".lin2.w"], m[2])], N)
    pi, pt = f"double.{block}.img", f"double.{block}.txt"
    pre_only = bool(d.context_pre_only_last) and block == d.n_double - 1
    mi = oi.modulation(W, pi, vec, 6)
    mt = oi.modulation(W, pt, vec, 2 if pre_only else 6)
    if pre_only:
        mt = [mt[1], mt[0]]
    qi, ki, vi = oi._qkv_stream(d, W, pi, Xh[Lt:], mi, oi.image_positions(d, idx_m), oi.FLUX_FLAGS)
    qt, kt, vt = oi._qkv_stream(d, W, pt, Xh[:Lt], mt, np.zeros((Lt, 3), np.int64), oi.FLUX_FLAGS)
    K = oi.merge_kv(d, kt, ki, idx_m, idx_u, kvh[0])
    V = oi.merge_kv(d, vt, vi, idx_m, idx_u, kvh[1])
    o = oi.attention(np.concatenate([qt, qi]), K, V, d.heads)
    out = np.zeros((n, d.hidden))
    for rows, pfx, m, streams in ((slice(0, Lt), pt, mt, not pre_only), (slice(Lt, n), pi, mi, True)):
        if not streams:
            continue
        x = Xh[rows]
        a1 = o[rows]
        x1 = x + m[2] * oi.linear(a1, W[pfx + ".proj.w"], W[pfx + ".proj.b"])
        z = oi.layernorm(x1, d.ln_eps) * (1.0 + m[4]) + m[3]
        a2 = oi.gelu_tanh(oi.linear(z, W[pfx + ".fc1.w"], W[pfx + ".fc1.b"]))
        out[rows] = bf16_rounding_bound([(a1, W[pfx + ".proj.w"], m[2]), (a2, W[pfx + ".fc2.w"], m[5])], N)
    return out


def _host_block_weights(names):
    return {k: v.double().numpy() for k, v in synth.make_weights(D, 0, "cpu", torch.bfloat16, names=names).items()}


def _fill_cache_block(cache, block, step_count, kv):
    """Write kv [2, L_img, H] (bf16) into (step 0, block) of a device-tier cache."""
    ptr, nbytes, tier = ig.ig_cache_storage(cache)
    plane = D.L_img * D.hidden * 2
    off = (0 * D.n_blocks + block) * 2 * plane
    src = kv.contiguous()
    ig.ig_copy(ptr + off, src.data_ptr(), 2 * plane)


@pytest.mark.parametrize("block,m_ratio,kind", [(3, 0.05, "rect"), (3, 0.6, "blob"), (19 + 7, 0.2, "rect")])
def test_flux_teacher_forced_block(flux, block, m_ratio, kind):
    rng = np.random.default_rng(block)
    n = int(round(m_ratio * D.L_img))
    mask = synth.rect_mask_count(D, n, rng) if kind == "rect" else synth.blob_mask_count(D, n, rng)
    rq = Request(flux, 77 + block, mask)
    cache = ig.ig_cache_create(flux.ctx, 1, ig.IG_CACHE_DEVICE)
    kv = synth.normal(500 + block, "kv_blk", (2, D.L_img, D.hidden), "cuda").float().bfloat16()
    _fill_cache_block(cache, block, 1, kv)
    rows = D.txt_len + rq.n_m
    X_in = synth.normal(900 + block, "X_in", (rows, D.hidden), "cuda").float()
    X_out = torch.full_like(X_in, float("nan"))
    sigma, sigma_next = 0.7, 0.65
    ig.ig_debug_block(flux.ctx, rq.req(0, cache, 0, sigma, sigma_next), block, X_in.data_ptr(), X_out.data_ptr())
    # oracle on the same inputs
    if block < D.n_double:
        names = {nm for nm, _, _ in synth.weight_table(D) if nm.startswith(f"double.{block}.")}
    else:
        names = {nm for nm, _, _ in synth.weight_table(D) if nm.startswith(f"single.{block - D.n_double}.")}
    names |= {"t_mlp1.w", "t_mlp1.b", "t_mlp2.w", "t_mlp2.b"}
    W = _host_block_weights(names)
    _, _, cond = rq.host_inputs()
    vec = oracle.conditioning(W, sigma, cond)
    idx_m, idx_u, _ = oracle.index_build(mask)
    Xh = X_in.double().cpu().numpy()
    kvh = kv.double().cpu().numpy()
    if block < D.n_double:
        xt, xi = oracle.double_block_masked(D, W, block, Xh[:D.txt_len], Xh[D.txt_len:], vec, idx_m, idx_u, kvh)
        ref = np.concatenate([xt, xi])
    else:
        ref = oracle.single_block_masked(D, W, block - D.n_double, Xh, vec, idx_m, idx_u, kvh)
    got = X_out.double().cpu().numpy()
    assert np.isfinite(got).all()
    dg, do = got - Xh, ref - Xh
    # C-TOL for a gated update (DESIGN.md C-AMB 22): normwise ||g-o||/||o|| <= rtol and the
    # elementwise bound with atol per output channel (the gate scales each channel's error)
    normwise = np.linalg.norm(dg - do) / np.linalg.norm(do)
    assert normwise <= 2e-2, normwise
    bound = _update_bound(D, W, block, Xh, vec, idx_m, idx_u, kvh)
    ok, worst = ctol_or_bound(dg, do, 2e-2, bound)
    ok1, worst1 = ctol(dg, do, 2e-2)
    print(f"\nC-TOL-full worst {worst:.3f}; plain C-TOL worst {worst1:.3f}; "
          f"elements outside C-TOL {int((np.abs(dg - do) > 2e-2 * np.abs(do) + 2e-2 * np.sqrt(np.mean(do * do))).sum())}")
    err = np.abs(dg - do)
    rms = np.sqrt(np.mean(do * do))
    i, j = np.unravel_index(np.argmax(err), err.shape)
    print(f"\nblock {block} m {m_ratio}: worst {worst:.3f} rel_rms_err {np.sqrt(np.mean(err**2))/rms:.4e} "
          f"max_err/rms {err.max()/rms:.4e} at row {i} (txt={i < D.txt_len}) col {j} head {j // 128} "
          f"txt-rows rel {np.sqrt(np.mean(err[:D.txt_len]**2))/rms:.3e} img-rows rel {np.sqrt(np.mean(err[D.txt_len:]**2))/rms:.3e}")
    q = np.quantile(err / rms, [0.5, 0.99, 0.999, 0.9999])
    top = np.argsort(err.ravel())[-6:]
    print("quantiles err/rms", q, "top", [(int(t // D.hidden), int(t % D.hidden), float(err.ravel()[t] / rms),
                                             float(do.ravel()[t] / rms)) for t in top])
    assert ok, ("update", worst)
    ig.ig_cache_free(cache)
    rq.free()


@pytest.mark.parametrize("block", [5, 19 + 9])
def test_flux_teacher_forced_y_block(flux, block):
    """Full-width Y block through ig_debug_block: the unmasked rows' block input is
    the staged Y_{b-1}, their K/V recomputed with this request's modulation; vs the oracle's
    kv_from_y + masked block on the same inputs (C-TOL-full)."""
    ptrs = [flux.W[n].data_ptr() for n, _, _ in synth.weight_table(D)]
    ctx = ig.ig_ctx_create(flux.desc, ptrs, 0, ig.ig_ctx_opts(8, 8 * D.L, 2, 1, 0, 0, 1, 0))
    rng = np.random.default_rng(block + 100)
    mask = synth.blob_mask_count(D, int(round(0.2 * D.L_img)), rng)
    rq = Request(flux, 88 + block, mask)
    cache = ig.ig_cache_create(ctx, 1, ig.IG_CACHE_DEVICE)
    y = synth.normal(600 + block, "y_blk", (D.L_img, D.hidden), "cuda").float().bfloat16()
    ptr, _, _ = ig.ig_cache_storage(cache)
    plane = D.L_img * D.hidden * 2
    ig.ig_copy(ptr + (block - 1) * plane, y.data_ptr(), plane)  # pure Y: plane b holds Y_b
    rows = D.txt_len + rq.n_m
    X_in = synth.normal(950 + block, "X_in_y", (rows, D.hidden), "cuda").float()
    X_out = torch.full_like(X_in, float("nan"))
    sigma, sigma_next = 0.6, 0.55
    ig.ig_debug_block(ctx, rq.req(0, cache, 0, sigma, sigma_next), block, X_in.data_ptr(), X_out.data_ptr())
    pre = f"double.{block}." if block < D.n_double else f"single.{block - D.n_double}."
    names = {nm for nm, _, _ in synth.weight_table(D) if nm.startswith(pre)} | {"t_mlp1.w", "t_mlp1.b", "t_mlp2.w", "t_mlp2.b"}
    W = _host_block_weights(names)
    _, _, cond = rq.host_inputs()
    vec = oracle.conditioning(W, sigma, cond)
    idx_m, idx_u, _ = oracle.index_build(mask)
    kv = oracle.kv_from_y(D, W, block, y.double().cpu().numpy()[idx_u], vec, idx_u)
    Xh = X_in.double().cpu().numpy()
    if block < D.n_double:
        xt, xi = oracle.double_block_masked(D, W, block, Xh[:D.txt_len], Xh[D.txt_len:], vec, idx_m, idx_u, kv)
        ref = np.concatenate([xt, xi])
    else:
        ref = oracle.single_block_masked(D, W, block - D.n_double, Xh, vec, idx_m, idx_u, kv)
    got = X_out.double().cpu().numpy()
    dg, do = got - Xh, ref - Xh
    normwise = np.linalg.norm(dg - do) / np.linalg.norm(do)
    assert normwise <= 2e-2, normwise
    ok, worst = ctol_or_bound(dg, do, 2e-2, _update_bound(D, W, block, Xh, vec, idx_m, idx_u, kv))
    print(f"\nY block {block}: C-TOL-full worst {worst:.3f}; plain C-TOL worst {ctol(dg, do, 2e-2)[1]:.3f}")
    assert ok, ("update", worst)
    ig.ig_cache_free(cache)
    rq.free()
    ig.ig_ctx_destroy(ctx)


def test_flux_same_trajectory_bitwise_and_batch_invariance(flux):
    sig = (1.0, 0.96)
    rng = np.random.default_rng(5)
    mask = synth.blob_mask_count(D, 1400, rng)
    a = Request(flux, 31, mask)
    # dense step of the same request = the template's own first step, recording its K/V
    lat_dense = a.latent.clone()
    cache = ig.ig_cache_template(flux.ctx, lat_dense.data_ptr(), a.txt.data_ptr(), a.cond.data_ptr(), sig,
                                 ig.IG_CACHE_DEVICE, 0)
    # edit alone
    ig.ig_edit_step(flux.ctx, [a.req(0, cache, 0, *sig)], 0)
    torch.cuda.synchronize()
    idx = torch.from_numpy(np.flatnonzero(mask)).cuda()
    un = torch.from_numpy(np.flatnonzero(mask == 0)).cuda()
    assert torch.equal(a.latent[idx], lat_dense[idx]), \
        float((a.latent[idx] - lat_dense[idx]).abs().max())
    assert torch.equal(a.latent[un], a.latent0[un])
    alone = a.latent.clone()
    # the same request inside a batch of three (other masks, other slots, other order)
    a.latent.copy_(a.latent0)
    b = Request(flux, 32, synth.rect_mask_count(D, 700, rng))
    c = Request(flux, 33, np.ones(D.L_img, np.uint8))
    ig.ig_edit_step(flux.ctx, [b.req(0, cache, 0, *sig), c.req(1, None, 0, *sig), a.req(5, cache, 0, *sig)], 0)
    torch.cuda.synchronize()
    assert torch.equal(a.latent, alone)
    ig.ig_cache_free(cache)
    for r in (a, b, c):
        r.free()



def test_flux_hybrid_cache_same_trajectory_and_batch_invariance(flux):
    """Full Flux shape, the bench's hybrid cache (37 K/V blocks, 20 interleaved Y blocks,
    DESIGN reading 30) recorded by ig_cache_template from the request's own inputs: the edited
    masked rows match the dense step (C-TOL: Y blocks recompute K/V from the bf16 Y cache, so
    not bitwise), unmasked rows are untouched, and the request alone equals the request inside
    a mixed batch (hybrid + K/V + all-ones) bitwise."""
    ptrs = [flux.W[n].data_ptr() for n, _, _ in synth.weight_table(D)]
    ctx = ig.ig_ctx_create(flux.desc, ptrs, 0, ig.ig_ctx_opts(8, 8 * D.L, 2, 1, 0, 0, 1, 37))
    sig = (1.0, 0.96)
    rng = np.random.default_rng(6)
    mask = synth.blob_mask_count(D, 1100, rng)
    a = Request(flux, 34, mask)
    lat_dense = a.latent.clone()
    cache = ig.ig_cache_template(ctx, lat_dense.data_ptr(), a.txt.data_ptr(), a.cond.data_ptr(), sig,
                                 ig.IG_CACHE_DEVICE, 0)
    ig.ig_edit_step(ctx, [a.req(0, cache, 0, *sig)], 0)
    torch.cuda.synchronize()
    idx = np.flatnonzero(mask)
    ok, worst = ctol(a.latent.double().cpu().numpy()[idx], lat_dense.double().cpu().numpy()[idx], 2e-2)
    assert ok, worst
    un = torch.from_numpy(np.flatnonzero(mask == 0)).cuda()
    assert torch.equal(a.latent[un], a.latent0[un])
    alone = a.latent.clone()
    kvcache = ig.ig_cache_template(flux.ctx, a.latent0.clone().data_ptr(), a.txt.data_ptr(), a.cond.data_ptr(), sig,
                                   ig.IG_CACHE_DEVICE, 0)
    a.latent.copy_(a.latent0)
    b = Request(flux, 35, synth.rect_mask_count(D, 900, rng))
    c = Request(flux, 36, np.ones(D.L_img, np.uint8))
    ig.ig_edit_step(ctx, [b.req(0, kvcache, 0, *sig), c.req(1, None, 0, *sig), a.req(6, cache, 0, *sig)], 0)
    torch.cuda.synchronize()
    assert torch.equal(a.latent, alone)
    ig.ig_cache_free(cache)
    ig.ig_cache_free(kvcache)
    for r in (a, b, c):
        r.free()
    ig.ig_ctx_destroy(ctx)


def test_sd3_teacher_forced_blocks():
    """SD3-medium-shaped (BASELINE configs[1]) joint blocks at full width (H=1536, d=64,
    333 text tokens, context-pre-only last block) through ig_debug_block vs the oracle,
    random-blob mask m=0.3."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = synth.SD3
    m = Model(d, ig.IG_BF16)
    rng = np.random.default_rng(3)
    mask = synth.blob_mask_count(d, int(round(0.3 * d.L_img)), rng)
    rq = Request(m, 91, mask)
    cache = ig.ig_cache_create(m.ctx, 1, ig.IG_CACHE_DEVICE)
    ptr, _, _ = ig.ig_cache_storage(cache)
    plane = d.L_img * d.hidden * 2
    for block in (5, d.n_blocks - 1):
        kv = synth.normal(700 + block, "kv_sd3", (2, d.L_img, d.hidden), "cuda").float().bfloat16()
        ig.ig_copy(ptr + block * 2 * plane, kv.data_ptr(), 2 * plane)
        rows = d.txt_len + rq.n_m
        X_in = synth.normal(800 + block, "X_sd3", (rows, d.hidden), "cuda").float()
        X_out = torch.full_like(X_in, float("nan"))
        ig.ig_debug_block(m.ctx, rq.req(0, cache, 0, 0.5, 0.45), block, X_in.data_ptr(), X_out.data_ptr())
        names = {nm for nm, _, _ in synth.weight_table(d) if nm.startswith(f"double.{block}.")}
        names |= {"t_mlp1.w", "t_mlp1.b", "t_mlp2.w", "t_mlp2.b"}
        W = {k: v.double().numpy() for k, v in synth.make_weights(d, 0, "cpu", torch.bfloat16, names=names).items()}
        _, _, cond = rq.host_inputs()
        vec = oracle.conditioning(W, 0.5, cond)
        idx_m, idx_u, _ = oracle.index_build(mask)
        Xh = X_in.double().cpu().numpy()
        xt, xi = oracle.double_block_masked(d, W, block, Xh[:d.txt_len], Xh[d.txt_len:], vec, idx_m, idx_u,
                                            kv.double().cpu().numpy())
        ref = np.concatenate([xt, xi])
        got = X_out.double().cpu().numpy()
        dg, do = got - Xh, ref - Xh
        if block == d.n_blocks - 1:  # context-pre-only: text rows pass through unchanged
            assert np.array_equal(got[:d.txt_len], Xh[:d.txt_len])
            dg, do = dg[d.txt_len:], do[d.txt_len:]
        normwise = np.linalg.norm(dg - do) / np.linalg.norm(do)
        assert normwise <= 2e-2, (block, normwise)
        bound = _update_bound(d, W, block, Xh, vec, idx_m, idx_u, kv.double().cpu().numpy())
        if block == d.n_blocks - 1:
            bound = bound[d.txt_len:]
        ok, worst = ctol_or_bound(dg, do, 2e-2, bound)
        print(f"\nSD3 block {block}: C-TOL-full worst {worst:.3f}; plain C-TOL worst {ctol(dg, do, 2e-2)[1]:.3f}")
        assert ok, (block, worst)
    ig.ig_cache_free(cache)
    rq.free()
    m.close()
