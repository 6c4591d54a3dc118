"""GPU parity tests (B200): the CUDA path through the C ABI vs the float64 oracle on the
same seeded inputs.  Tolerances: bit-exact for indices/copies; C-TOL rtol 1e-4 (fp32 parity
mode) and 2e-2 (bf16) (BASELINE.json north_star; DESIGN.md C-TOL)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_20600_b200 import ig
from gpu_util import Model, Request, cache_to_numpy, ctol, fill_cache

pytestmark = pytest.mark.gpu

RTOL = {ig.IG_F32: 1e-4, ig.IG_BF16: 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ig.lib()


# ------------------------------------------------------------------ a1 index build
@pytest.mark.parametrize("L", [256, 1024, 4096, 9000])
def test_mask_index_bit_exact(L):
    d = synth.ModelDesc("m", 0, 1, 64, 4, 16, 256, 16, 1, L, 0, rope_axes=(4, 6, 6))
    m = Model(d, ig.IG_F32)
    rng = np.random.default_rng(L)
    masks = [np.zeros(L, np.uint8), np.ones(L, np.uint8)]
    one = np.zeros(L, np.uint8); one[0] = 1; masks.append(one)
    last = np.zeros(L, np.uint8); last[-1] = 7; masks.append(last)
    for _ in range(6):
        masks.append((rng.random(L) < rng.random()).astype(np.uint8) * rng.integers(1, 256, L).astype(np.uint8))
    for mk in masks:
        dev = torch.from_numpy(mk).cuda()
        h, n = ig.ig_mask_build(m.ctx, dev.data_ptr(), 0)
        pm, pu, n2 = ig.ig_mask_indices(h)
        ref_m, ref_u, ref_n = oracle.index_build(mk)
        assert n == n2 == ref_n
        got = torch.empty(2 * L, dtype=torch.int32, device="cuda")
        ig.ig_copy(got.data_ptr(), pm, 2 * L * 4)
        g = got.cpu().numpy()
        assert np.array_equal(g[:n], ref_m) and np.array_equal(g[L:L + L - n], ref_u)
        ig.ig_mask_free(h)
    m.close()


# ------------------------------------------------------------------ kernel (c) GEMM
@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (127, 128, 128), (129, 256, 192), (300, 576, 320),
                                   (1331, 384, 256)])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_vs_oracle(dtype, M, N, K, epi):
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    A = (synth.uniform(1, "A", (M, K), "cuda")).float().to(tdt)
    B = (synth.uniform(2, "B", (N, K), "cuda") / K ** 0.5).float().to(tdt)
    bias = synth.uniform(3, "b", (N,), "cuda").float().to(tdt)
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    ig.ig_op_gemm(dtype, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), C.data_ptr(), N,
                  M, N, K, epi, 1, 0)
    torch.cuda.synchronize()
    ref = oracle.linear(A.double().cpu().numpy(), B.double().cpu().numpy(), bias.double().cpu().numpy())
    if epi == 1:
        ref = oracle.gelu_tanh(ref)
    ok, worst = ctol(C.cpu().numpy(), ref, 1e-4 if dtype == ig.IG_F32 else 2e-3)
    assert ok, worst


# ------------------------------------------------------------------ kernel (d) attention
@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("heads,dh,L,qlens", [(4, 16, 256, [64]), (2, 128, 300, [0, 1, 127, 128, 129]),
                                              (3, 64, 1357, [333, 200]), (2, 128, 4608, [512, 819])])
def test_attention_vs_oracle(dtype, heads, dh, L, qlens):
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    H = heads * dh
    nseg = len(qlens)
    M = sum(qlens)
    Q = synth.normal(5, "Q", (max(M, 1), H), "cuda").float().to(tdt)
    kv = synth.normal(6, "KV", (nseg, 2, L, H), "cuda").float().to(tdt)
    O = torch.full((max(M, 1), H), float("nan"), dtype=tdt, device="cuda")
    segs, s = [], 0
    for i, q in enumerate(qlens):
        segs.append((s, q, i))
        s += q
    ig.ig_op_attention(dtype, Q.data_ptr(), H, O.data_ptr(), H, kv.data_ptr(), segs, L, heads, dh, 0)
    torch.cuda.synchronize()
    Qh, KVh, Oh = Q.double().cpu().numpy(), kv.double().cpu().numpy(), O.double().cpu().numpy()
    for (q0, ql, i) in segs:
        if ql == 0:
            continue
        ref = oracle.attention(Qh[q0:q0 + ql], KVh[i, 0], KVh[i, 1], heads)
        ok, worst = ctol(Oh[q0:q0 + ql], ref, 1e-4 if dtype == ig.IG_F32 else 2e-2)
        assert ok, (i, worst)


# ------------------------------------------------------------------ end to end
def _run_edit(m, reqs_objs, masks_cache, n_steps, sig):
    for s in range(n_steps):
        rr = [r.req(i, masks_cache, s, sig[s], sig[s + 1]) for i, r in enumerate(reqs_objs)]
        ig.ig_edit_step(m.ctx, rr, 0)
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
def test_tiny_config_end_to_end(dtype):
    """Config 1: tiny single block, 25% rectangle, 2 steps.  GPU cache_template vs the
    oracle's recorded cache, then the edit steps with a synthetic cache shared by both."""
    d = synth.TINY
    sig = [1.0, 0.5, 0.0]
    m = Model(d, dtype)
    W = m.host_weights()
    rq = Request(m, 0, synth.tiny_rect_mask())
    lat0, txt, cond = rq.host_inputs()
    # cache recording (dense trajectory)
    lat_t = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, lat_t.data_ptr(), 0, rq.cond.data_ptr(), sig)
    _, ocache, traj = oracle.cache_template(d, W, lat0, txt, cond, sig)
    g = cache_to_numpy(cache, d, 2, dtype)
    ok, worst = ctol(g, ocache, RTOL[dtype])
    assert ok, ("cache", worst)
    ok, worst = ctol(lat_t.double().cpu().numpy(), traj[-1], RTOL[dtype])
    assert ok, ("dense trajectory", worst)
    # edit steps with a synthetic cache (same bytes for both sides)
    kv = synth.make_cache_kv(d, 0, 2, dtype=torch.float32 if dtype == ig.IG_F32 else torch.bfloat16)
    syn = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, syn, kv)
    kvh = kv.double().numpy()
    _run_edit(m, [rq], syn, 2, sig)
    x = lat0
    for s in range(2):
        x = oracle.edit_step(d, W, x, rq.mask_np, kvh[s], sig[s], sig[s + 1], txt, cond)
    got = rq.latent.double().cpu().numpy()
    ok, worst = ctol(got, x, RTOL[dtype])
    assert ok, ("edit", worst)
    assert np.array_equal(got[rq.mask_np == 0], lat0[rq.mask_np == 0])  # untouched rows
    ig.ig_cache_free(cache)
    ig.ig_cache_free(syn)
    rq.free()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("copy_mode", [0, 1, 2])
def test_flux_small_batch_end_to_end(dtype, copy_mode):
    """Flux-structured small model (2 double + 2 single blocks, text tokens): a continuous
    batch of 3 requests with different masks (rectangle, blob, all-ones) and a synthetic
    cache, 2 steps, against the oracle request by request."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    opts = ig.ig_ctx_opts(4, 0, 2, copy_mode, 0, 0)
    m = Model(d, dtype, opts=opts)
    W = m.host_weights()
    rng = np.random.default_rng(0)
    masks = [synth.rect_mask_count(d, 50, rng), synth.blob_mask_count(d, 120, rng),
             np.ones(d.L_img, np.uint8)]
    reqs = [Request(m, 10 + i, mk) for i, mk in enumerate(masks)]
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    kv = synth.make_cache_kv(d, 3, 2, dtype=tdt)
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv)
    kvh = kv.double().numpy()
    _run_edit(m, reqs, cache, 2, sig)
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step(d, W, x, r.mask_np, kvh[s], sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, worst
        assert np.array_equal(got[r.mask_np == 0], lat0[r.mask_np == 0])
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def test_degenerate_and_errors():
    d = synth.FLUX_SMALL
    m = Model(d, ig.IG_BF16)
    empty = Request(m, 1, np.zeros(d.L_img, np.uint8))
    ig.ig_edit_step(m.ctx, [empty.req(0, None, 0, 1.0, 0.9)], 0)
    torch.cuda.synchronize()
    assert torch.equal(empty.latent, empty.latent0)
    st = ig.ig_last_stats(m.ctx)
    assert st["h2d_bytes"] == 0 and st["kernel_launches"] == 0
    part = Request(m, 2, synth.rect_mask(d, 0, 4, 0, 4))
    with pytest.raises(ig.IgError) as e:
        ig.ig_edit_step(m.ctx, [part.req(0, None, 0, 1.0, 0.9)], 0)
    assert e.value.name == "IG_ECACHE_MISS"
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    with pytest.raises(ig.IgError) as e:
        ig.ig_edit_step(m.ctx, [part.req(0, cache, 5, 1.0, 0.9)], 0)
    assert e.value.name == "IG_ECACHE_INCOMPAT"
    with pytest.raises(ig.IgError) as e:
        ig.ig_edit_step(m.ctx, [part.req(0, cache, 0, 1.0, 0.9), part.req(0, cache, 0, 1.0, 0.9)], 0)
    assert e.value.name == "IG_EINVAL"
    ig.ig_cache_free(cache)
    empty.free(); part.free()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("M,N,K", [(129, 256, 192), (300, 3072, 320)])
def test_gemm_gated_residual_vs_oracle(dtype, M, N, K):
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    A = synth.uniform(1, "A", (M, K), "cuda").float().to(tdt)
    B = (synth.uniform(2, "B", (N, K), "cuda") / K ** 0.5).float().to(tdt)
    bias = synth.uniform(3, "b", (N,), "cuda").float().to(tdt)
    X0 = synth.normal(4, "X", (M, N), "cuda").float()
    gate = synth.uniform(5, "g", (N,), "cuda").float()
    X = X0.clone()
    ig.ig_op_gemm_gated(dtype, A.data_ptr(), K, B.data_ptr(), K, bias.data_ptr(), X.data_ptr(), N,
                        gate.data_ptr(), M, N, K, 0)
    torch.cuda.synchronize()
    y = oracle.linear(A.double().cpu().numpy(), B.double().cpu().numpy(), bias.double().cpu().numpy())
    ref = X0.double().cpu().numpy() + gate.double().cpu().numpy() * y
    ok, worst = ctol(X.cpu().numpy(), ref, 1e-4 if dtype == ig.IG_F32 else 2e-3)
    assert ok, worst


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("model", ["sd3_small", "tiny_double"])
def test_sd3_and_double_structures_end_to_end(dtype, model):
    """SD3-structured joint blocks (d=64, 2-D pos-embed, ragged text, context-pre-only last
    block) and a tiny double+single model: batch of 2 requests, 2 steps, synthetic cache."""
    d = synth.MODELS[model]
    sig = [0.9, 0.6, 0.3]
    m = Model(d, dtype)
    W = m.host_weights()
    rng = np.random.default_rng(1)
    masks = [synth.blob_mask_count(d, int(0.3 * d.L_img), rng), synth.rect_mask_count(d, int(0.1 * d.L_img) + 1, rng)]
    reqs = [Request(m, 40 + i, mk) for i, mk in enumerate(masks)]
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    kv = synth.make_cache_kv(d, 5, 2, dtype=tdt)
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv)
    kvh = kv.double().numpy()
    _run_edit(m, reqs, cache, 2, sig)
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step(d, W, x, r.mask_np, kvh[s], sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()



@pytest.mark.parametrize("tier", [ig.IG_CACHE_HOST, ig.IG_CACHE_DEVICE])
def test_fp8_cache_end_to_end(tier):
    """FP8 (e4m3) K/V cache: the oracle mirrors the quantize/dequantize round trip
    of the same synthetic bf16 cache; batch of 2 requests, 2 steps, host and HBM tiers."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 1))
    W = m.host_weights()
    rng = np.random.default_rng(2)
    masks = [synth.blob_mask_count(d, 70, rng), synth.rect_mask_count(d, 30, rng)]
    reqs = [Request(m, 60 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 9, 2, dtype=torch.bfloat16, device="cuda")
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    ig.ig_cache_write(m.ctx, cache, kv.data_ptr())
    if tier == ig.IG_CACHE_DEVICE:
        dc = ig.ig_cache_clone(m.ctx, cache, ig.IG_CACHE_DEVICE)
        ig.ig_cache_free(cache)
        cache = dc
    kvh = oracle.fp8_kv_roundtrip(kv.float().cpu().numpy(), d.heads)
    _run_edit(m, reqs, cache, 2, sig)
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step(d, W, x, r.mask_np, kvh[s], sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, 2e-2)
        assert ok, worst
    st = ig.ig_last_stats(m.ctx)
    assert st["h2d_bytes"] + st["d2d_bytes"] > 0
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()



@pytest.mark.parametrize("k", [1, 2, 4])
def test_algorithm1_dense_prefix_end_to_end(k):
    """Algorithm-1 plan (N1) executed: the first k blocks run every token of each request (the
    unmasked ones from the template's input latent of the step), the rest use the cache; vs
    the oracle's planned step (C-AMB 23).  Batch of 3 (one all-ones request), 2 steps."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 4, 1, 0, 0))
    ig.ig_set_plan(m.ctx, 1, k)
    W = m.host_weights()
    rng = np.random.default_rng(4)
    masks = [synth.blob_mask_count(d, 80, rng), synth.rect_mask_count(d, 25, rng), np.ones(d.L_img, np.uint8)]
    reqs = [Request(m, 70 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 4, 2, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(d, 900 + s) for s in range(2)])
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv, tlat)
    kvh, tlh = kv.double().numpy(), tlat.double().numpy()
    _run_edit(m, reqs, cache, 2, sig)
    assert ig.ig_last_plan(m.ctx) == min(k, d.n_blocks)
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step_planned(d, W, x, r.mask_np, kvh[s], tlh[s], k, sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, 2e-2)
        assert ok, worst
        assert np.array_equal(got[r.mask_np == 0], lat0[r.mask_np == 0])
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def test_algorithm1_model_plan_extremes():
    d = synth.FLUX_SMALL
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 4, 1, 0, 0))
    r = Request(m, 80, synth.rect_mask_count(d, 40, np.random.default_rng(0)))
    kv = synth.make_cache_kv(d, 4, 1, dtype=torch.bfloat16)
    cache = ig.ig_cache_create(m.ctx, 1, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv, torch.stack([synth.make_latent(d, 1)]))
    # free loads -> never dense; very slow loads -> every block dense
    for load_s_per_byte, expect in ((0.0, 0), (1.0, d.n_blocks)):
        ig.ig_set_plan(m.ctx, 2, 0, 1e-15, 1e-6, load_s_per_byte, 0.0)
        ig.ig_edit_step(m.ctx, [r.req(0, cache, 0, 1.0, 0.9)], 0)
        torch.cuda.synchronize()
        assert ig.ig_last_plan(m.ctx) == expect
    ig.ig_cache_free(cache)
    r.free()
    m.close()


# ------------------------------------------------------------------ Y variant (N2)
@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("copy_mode,tier", [(0, ig.IG_CACHE_HOST), (1, ig.IG_CACHE_HOST), (2, ig.IG_CACHE_HOST),
                                            (1, ig.IG_CACHE_DEVICE)])
def test_y_cache_mixed_batch_end_to_end(dtype, copy_mode, tier):
    """Y-caching variant (fig:transformer-Bottom): a continuous batch mixing two
    Y-cache requests, one K/V-cache request and an all-ones request, 2 steps, vs the oracle's
    edit_step_y / edit_step request by request (synthetic caches shared by both sides)."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    m = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, copy_mode, 0, 0, 1))
    W = m.host_weights()
    rng = np.random.default_rng(11)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 40, rng),
             synth.blob_mask_count(d, 60, rng), np.ones(d.L_img, np.uint8)]
    reqs = [Request(m, 110 + i, mk) for i, mk in enumerate(masks)]
    yv = synth.make_cache_y(d, 5, 2, dtype=tdt)
    tlat = torch.stack([synth.make_latent(d, 950 + s) for s in range(2)])
    ycache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)  # cache_y ctx -> Y cache
    fill_cache(m, ycache, yv, tlat)
    if tier == ig.IG_CACHE_DEVICE:
        dc = ig.ig_cache_clone(m.ctx, ycache, ig.IG_CACHE_DEVICE)
        ig.ig_cache_free(ycache)
        ycache = dc
    mk = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, copy_mode, 0, 0, 0))  # same weights, K/V caches
    kv = synth.make_cache_kv(d, 6, 2, dtype=tdt)
    kvcache = ig.ig_cache_create(mk.ctx, 2, tier)
    fill_cache(mk, kvcache, kv)
    caches = [ycache, ycache, kvcache, None]
    for s in range(2):
        rr = [r.req(i, caches[i], s, sig[s], sig[s + 1]) for i, r in enumerate(reqs)]
        ig.ig_edit_step(m.ctx, rr, 0)
    torch.cuda.synchronize()
    st = ig.ig_last_stats(m.ctx)
    n_u = [d.L_img - int(mk_.sum()) for mk_ in masks]
    es = 4 if dtype == ig.IG_F32 else 2
    if copy_mode != 0:  # compacted: one plane per Y request (blocks 1..N-1), two per K/V request
        exp = ((d.n_blocks - 1) * (n_u[0] + n_u[1]) + 2 * d.n_blocks * n_u[2]) * d.hidden * es
        assert st["h2d_bytes"] + st["d2d_bytes"] == exp
    yh, kvh, tlh = yv.double().numpy(), kv.double().numpy(), tlat.double().numpy()
    for i, r in enumerate(reqs):
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            if i < 2:
                x = oracle.edit_step_y(d, W, x, r.mask_np, yh[s], tlh[s], sig[s], sig[s + 1], txt, cond)
            else:
                x = oracle.edit_step(d, W, x, r.mask_np, kvh[s] if i == 2 else None, sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, (i, worst)
        assert np.array_equal(got[r.mask_np == 0], lat0[r.mask_np == 0])
    ig.ig_cache_free(ycache)
    ig.ig_cache_free(kvcache)
    for r in reqs:
        r.free()
    mk.close()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("model", ["tiny", "flux_small"])
def test_y_cache_template_recording(dtype, model):
    """ig_cache_template on a cache_y ctx records every (step, block) image-token block output
    (the Y of fig:transformer): vs the oracle's dense pass (cache_template_y), 2 steps; then a
    2-step edit on that recorded cache along the template trajectory stays on it."""
    d = synth.TINY if model == "tiny" else synth.FLUX_SMALL
    sig = [1.0, 0.5, 0.0]
    m = Model(d, dtype, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0, 0, 1))
    W = m.host_weights()
    rq = Request(m, 3, synth.tiny_rect_mask() if model == "tiny" else synth.blob_mask_count(d, 64, np.random.default_rng(3)))
    lat0, txt, cond = rq.host_inputs()
    lat_t = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, lat_t.data_ptr(), rq.txt.data_ptr() if d.txt_len else 0,
                                 rq.cond.data_ptr(), sig)
    _, oy, traj = oracle.cache_template_y(d, W, lat0, txt, cond, sig)
    g = cache_to_numpy(cache, d, 2, dtype, y=True)
    ok, worst = ctol(g, oy, RTOL[dtype])
    assert ok, ("Y cache", worst)
    _run_edit(m, [rq], cache, 2, sig)
    got = rq.latent.double().cpu().numpy()
    idx = rq.mask_np != 0
    ok, worst = ctol(got[idx], traj[-1][idx], RTOL[dtype])
    assert ok, ("edit on the recorded Y cache", worst)
    ig.ig_cache_free(cache)
    rq.free()
    m.close()


@pytest.mark.parametrize("k", [1, 3])
def test_y_cache_dense_prefix_end_to_end(k):
    """Algorithm-1 prefix under the Y variant: block k takes the prefix's computed unmasked
    rows, later blocks replenish from Y_{b-1}; vs oracle edit_step_y(k=)."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 4, 1, 0, 0, 1))
    ig.ig_set_plan(m.ctx, 1, k)
    W = m.host_weights()
    rng = np.random.default_rng(12)
    masks = [synth.blob_mask_count(d, 70, rng), synth.rect_mask_count(d, 35, rng)]
    reqs = [Request(m, 130 + i, mk) for i, mk in enumerate(masks)]
    yv = synth.make_cache_y(d, 7, 2, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(d, 960 + s) for s in range(2)])
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, yv, tlat)
    _run_edit(m, reqs, cache, 2, sig)
    assert ig.ig_last_plan(m.ctx) == k
    yh, tlh = yv.double().numpy(), tlat.double().numpy()
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step_y(d, W, x, r.mask_np, yh[s], tlh[s], sig[s], sig[s + 1], txt, cond, k=k)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, 2e-2)
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def test_host_pinned_latent_bitwise_equals_device_latent():
    """The public API's host-buffer path: a latent in pinned host memory is gathered and
    updated in place by the kernels over the host link; same bits as a device latent."""
    d = synth.FLUX_SMALL
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0, 0))
    r = Request(m, 140, synth.blob_mask_count(d, 77, np.random.default_rng(14)))
    kv = synth.make_cache_kv(d, 8, 2, dtype=torch.bfloat16)
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv)
    host = r.latent0.cpu().pin_memory()
    sig = [1.0, 0.7, 0.4]
    for s in range(2):
        ig.ig_edit_step(m.ctx, [r.req(0, cache, s, sig[s], sig[s + 1])], 0)
        q = ig.make_req(0, host.data_ptr(), r.mask, cache, s, sig[s], sig[s + 1], r.txt.data_ptr(), r.cond.data_ptr())
        ig.ig_edit_step(m.ctx, [q], 0)
    torch.cuda.synchronize()
    assert torch.equal(host, r.latent.cpu())
    assert not torch.equal(host, r.latent0.cpu())
    ig.ig_cache_free(cache)
    r.free()
    m.close()


# ------------------------------------------------------------------ hybrid K/V + Y cache
@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("tier", [ig.IG_CACHE_HOST, ig.IG_CACHE_DEVICE])
def test_hybrid_cache_batch_end_to_end(dtype, tier):
    """Hybrid caches (DESIGN reading 30: kv_blocks blocks keep K/V, the others — interleaved in
    bit-reversal order — are Y blocks) with different splits in one continuous batch, plus a
    pure K/V cache and an all-ones request; 2 steps vs the oracle's edit_step_y(y_blocks=)."""
    from gpu_util import hybrid_planes
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    tdt = torch.float32 if dtype == ig.IG_F32 else torch.bfloat16
    rng = np.random.default_rng(21)
    masks = [synth.blob_mask_count(d, 85, rng), synth.rect_mask_count(d, 45, rng),
             synth.blob_mask_count(d, 66, rng), np.ones(d.L_img, np.uint8)]
    splits = [2, 3, None, None]  # kv_blocks per request (None: pure K/V cache / no cache)
    ms, caches, refs = [], [], []
    base = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 0))
    reqs = [Request(base, 150 + i, mk) for i, mk in enumerate(masks)]
    tlat = torch.stack([synth.make_latent(d, 970 + s) for s in range(2)])
    for i, kvb in enumerate(splits[:3]):
        kv = synth.make_cache_kv(d, 20 + i, 2, dtype=tdt)
        yv = synth.make_cache_y(d, 20 + i, 2, dtype=tdt)
        if kvb is None:
            c = ig.ig_cache_create(base.ctx, 2, tier)
            fill_cache(base, c, kv, tlat)
            refs.append((kv.double().numpy(), None, None))
        else:
            m = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, kvb))
            ms.append(m)
            ym = set(ig.y_block_modes(d.n_blocks, kvb))
            c = ig.ig_cache_create(m.ctx, 2, tier)
            fill_cache(m, c, hybrid_planes(kv, yv, ym), tlat)
            refs.append((kv.double().numpy(), yv.double().numpy(), ym))
        caches.append(c)
    caches.append(None)
    for s in range(2):
        rr = [r.req(i, caches[i], s, sig[s], sig[s + 1]) for i, r in enumerate(reqs)]
        ig.ig_edit_step(base.ctx, rr, 0)
    torch.cuda.synchronize()
    W = base.host_weights()
    tlh = tlat.double().numpy()
    for i, r in enumerate(reqs):
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            if i < 3 and refs[i][2] is not None:
                kvh, yh, ym = refs[i]
                x = oracle.edit_step_y(d, W, x, r.mask_np, yh[s], tlh[s], sig[s], sig[s + 1], txt, cond,
                                       y_blocks=ym, kv_cache_step=kvh[s])
            else:
                x = oracle.edit_step(d, W, x, r.mask_np, refs[i][0][s] if i < 3 else None, sig[s], sig[s + 1], txt, cond)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, (i, worst)
    for c in caches[:3]:
        ig.ig_cache_free(c)
    for r in reqs:
        r.free()
    for m in ms:
        m.close()
    base.close()


@pytest.mark.parametrize("kv_blocks", [1, 3])
def test_hybrid_cache_template_recording_and_plan(kv_blocks):
    """ig_cache_template on a hybrid ctx records K/V for the K/V blocks and Y_b where block b or
    b + 1 is a Y block (vs the oracle's dense pass); then an edit with a dense prefix k = 1 on
    that cache stays on the template trajectory (same inputs)."""
    from gpu_util import cache_raw_numpy, n_planes, split_hybrid
    d = synth.FLUX_SMALL
    sig = [1.0, 0.5, 0.0]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 4, 1, 0, 0, 1, kv_blocks))
    W = m.host_weights()
    ym = set(ig.y_block_modes(d.n_blocks, kv_blocks))
    rq = Request(m, 160, synth.rect_mask_count(d, 70, np.random.default_rng(16)))
    lat0, txt, cond = rq.host_inputs()
    lat_t = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, lat_t.data_ptr(), rq.txt.data_ptr(), rq.cond.data_ptr(), sig)
    _, okv, _ = oracle.cache_template(d, W, lat0, txt, cond, sig)
    _, oy, traj = oracle.cache_template_y(d, W, lat0, txt, cond, sig)
    gkv, gy = split_hybrid(cache_raw_numpy(cache, d, 2, n_planes(d.n_blocks, ym), ig.IG_BF16), d.n_blocks, ym)
    kvb = [b for b in range(d.n_blocks) if b not in ym]
    yb = [b for b in range(d.n_blocks) if b in ym or (b + 1) in ym]
    ok, worst = ctol(gkv[:, kvb], okv[:, kvb], 2e-2)
    assert ok, ("K/V part", worst)
    ok, worst = ctol(gy[:, yb], oy[:, yb], 2e-2)
    assert ok, ("Y part", worst)
    ig.ig_set_plan(m.ctx, 1, 1)
    _run_edit(m, [rq], cache, 2, sig)
    idx = rq.mask_np != 0
    ok, worst = ctol(rq.latent.double().cpu().numpy()[idx], traj[-1][idx], 2e-2)
    assert ok, ("edit on the recorded hybrid cache", worst)
    ig.ig_cache_free(cache)
    rq.free()
    m.close()


@pytest.mark.parametrize("k", [2])
def test_fp8_cache_with_dense_prefix(k):
    """FP8 K/V cache (N4) under the Algorithm-1 dense prefix (N1): the oracle's planned step
    on the fp8-round-tripped cache; batch of 2, 2 steps."""
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 4, 1, 0, 1))
    ig.ig_set_plan(m.ctx, 1, k)
    W = m.host_weights()
    rng = np.random.default_rng(31)
    masks = [synth.blob_mask_count(d, 75, rng), synth.rect_mask_count(d, 33, rng)]
    reqs = [Request(m, 170 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 11, 2, dtype=torch.bfloat16, device="cuda")
    tlat = torch.stack([synth.make_latent(d, 980 + s) for s in range(2)]).cuda()
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    ig.ig_cache_write(m.ctx, cache, kv.data_ptr(), tlat.data_ptr())
    kvh = oracle.fp8_kv_roundtrip(kv.float().cpu().numpy(), d.heads)
    tlh = tlat.double().cpu().numpy()
    _run_edit(m, reqs, cache, 2, sig)
    assert ig.ig_last_plan(m.ctx) == k
    for r in reqs:
        lat0, txt, cond = r.host_inputs()
        x = lat0
        for s in range(2):
            x = oracle.edit_step_planned(d, W, x, r.mask_np, kvh[s], tlh[s], k, sig[s], sig[s + 1], txt, cond)
        ok, worst = ctol(r.latent.double().cpu().numpy(), x, 2e-2)
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def test_cuda_graph_steps_bitwise_equal_eager():
    """ig_ctx_opts.use_graphs: steps on an HBM-resident cache are captured as CUDA graphs per
    step shape and replayed; 8 steps (a request leaves after step 4 -> a new shape) must equal
    the eager path bitwise, including a hybrid cache and an all-ones request."""
    from gpu_util import hybrid_planes
    d = synth.FLUX_SMALL
    sig = synth.flow_sigmas(8)
    eager = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    ptrs = [eager.W[n].data_ptr() for n, _, _ in synth.weight_table(d)]
    gctx = ig.ig_ctx_create(eager.desc, ptrs, 0, ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 0, 0, 1))
    rng = np.random.default_rng(41)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 40, rng), np.ones(d.L_img, np.uint8)]
    ra = [Request(eager, 180 + i, mk) for i, mk in enumerate(masks)]
    rb = [Request(eager, 180 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 12, 8, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(d, 990 + s) for s in range(8)])
    kvc = ig.ig_cache_create(eager.ctx, 8, ig.IG_CACHE_DEVICE)
    fill_cache(eager, kvc, kv, tlat)
    m2 = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, 2))
    hyc = ig.ig_cache_create(m2.ctx, 8, ig.IG_CACHE_DEVICE)
    ym = set(ig.y_block_modes(d.n_blocks, 2))
    fill_cache(m2, hyc, hybrid_planes(kv, synth.make_cache_y(d, 12, 8, dtype=torch.bfloat16), ym), tlat)
    caches = [kvc, hyc, None]
    stream = torch.cuda.Stream()  # graphs need a capturable (non-default) stream
    for s in range(8):
        live = range(3) if s < 4 else (0, 2)
        for ctx, rs in ((eager.ctx, ra), (gctx, rb)):
            ig.ig_edit_step(ctx, [rs[i].req(i, caches[i], s, float(sig[s]), float(sig[s + 1])) for i in live],
                            stream.cuda_stream)
    torch.cuda.synchronize()
    for a, b in zip(ra, rb):
        assert torch.equal(a.latent, b.latent)
        assert not torch.equal(a.latent, a.latent0)
    st = ig.ig_last_stats(gctx)
    assert st["kernel_launches"] > 0
    ig.ig_cache_free(kvc)
    ig.ig_cache_free(hyc)
    for r in ra + rb:
        r.free()
    ig.ig_ctx_destroy(gctx)
    m2.close()
    eager.close()


def test_cuda_graph_update_on_new_shapes_bitwise_equal_eager():
    """A new step shape updates a stale graph of the same topology in place (cudaGraphExecUpdate)
    instead of instantiating: three phases of 5 steps, each with two fresh requests (new masks, so
    new row counts / keys; same cache kinds, so the same kernel sequence) — phases 2 and 3 find
    phase 1's / 2's graphs stale — and every latent equals the eager path bitwise."""
    d = synth.FLUX_SMALL
    sig = synth.flow_sigmas(8)
    eager = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    ptrs = [eager.W[n].data_ptr() for n, _, _ in synth.weight_table(d)]
    gctx = ig.ig_ctx_create(eager.desc, ptrs, 0, ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 0, 0, 1))
    kv = synth.make_cache_kv(d, 13, 8, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(d, 970 + s) for s in range(8)])
    kvc = ig.ig_cache_create(eager.ctx, 8, ig.IG_CACHE_DEVICE)
    fill_cache(eager, kvc, kv, tlat)
    stream = torch.cuda.Stream()
    rng = np.random.default_rng(43)
    for phase in range(3):
        masks = [synth.blob_mask_count(d, int(rng.integers(30, 110)), rng), synth.rect_mask_count(d, int(rng.integers(20, 60)), rng)]
        ra = [Request(eager, 300 + 10 * phase + i, mk) for i, mk in enumerate(masks)]
        rb = [Request(eager, 300 + 10 * phase + i, mk) for i, mk in enumerate(masks)]
        for s in range(5):
            for ctx, rs in ((eager.ctx, ra), (gctx, rb)):
                ig.ig_edit_step(ctx, [rs[i].req(i, kvc, s, float(sig[s]), float(sig[s + 1])) for i in range(2)],
                                stream.cuda_stream)
        torch.cuda.synchronize()
        for a, b in zip(ra, rb):
            assert torch.equal(a.latent, b.latent), phase
            assert not torch.equal(a.latent, a.latent0)
        for r in ra + rb:
            r.free()
    ig.ig_cache_free(kvc)
    ig.ig_ctx_destroy(gctx)
    eager.close()


@pytest.mark.parametrize("kind", ["kv", "hybrid"])
def test_load_dedupe_same_template_and_step(kind):
    """Requests on the same (host-tier cache, step) share their staged rows (SURVEY N4 load
    deduplication): a lockstep batch equals each request run alone bit for bit, and moves
    fewer host-link bytes than the requests alone."""
    from gpu_util import hybrid_planes
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    opts = ig.ig_ctx_opts(4, 0, 2, 1, 0, 0) if kind == "kv" else ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, 2)
    m = Model(d, ig.IG_BF16, opts=opts)
    rng = np.random.default_rng(51)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 40, rng), synth.blob_mask_count(d, 130, rng)]
    alone = [Request(m, 190 + i, mk) for i, mk in enumerate(masks)]
    batch = [Request(m, 190 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 13, 2, dtype=torch.bfloat16)
    tlat = torch.stack([synth.make_latent(d, 995 + s) for s in range(2)])
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    if kind == "kv":
        fill_cache(m, cache, kv, tlat)
    else:
        ym = set(ig.y_block_modes(d.n_blocks, 2))
        fill_cache(m, cache, hybrid_planes(kv, synth.make_cache_y(d, 13, 2, dtype=torch.bfloat16), ym), tlat)
    h2d_alone = 0
    for s in range(2):
        for i, r in enumerate(alone):
            ig.ig_edit_step(m.ctx, [r.req(i, cache, s, sig[s], sig[s + 1])], 0)
            h2d_alone += ig.ig_last_stats(m.ctx)["h2d_bytes"]
    h2d_batch = 0
    for s in range(2):
        ig.ig_edit_step(m.ctx, [r.req(i, cache, s, sig[s], sig[s + 1]) for i, r in enumerate(batch)], 0)
        st = ig.ig_last_stats(m.ctx)
        h2d_batch += st["h2d_bytes"]
        assert st["d2d_bytes"] > 0
    torch.cuda.synchronize()
    for a, b in zip(alone, batch):
        assert torch.equal(a.latent, b.latent)
    assert h2d_batch < h2d_alone
    ig.ig_cache_free(cache)
    for r in alone + batch:
        r.free()
    m.close()


def test_load_dedupe_mixed_cache_kinds():
    """Two dedupe groups in one batch, one on a hybrid host cache and one on a pure K/V host
    cache (the skip / V-only decision is per group, from the group's own cache).
    Order [hyb, kv, hyb, kv] puts the hybrid group first, so a batch-wide decision taken from it
    would skip the K plane of the K/V group's shared rows at every Y block.  Each request must
    equal itself run alone, bit for bit."""
    from gpu_util import hybrid_planes
    d = synth.FLUX_SMALL
    sig = [1.0, 0.7, 0.4]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    mh = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, 2))
    rng = np.random.default_rng(53)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 40, rng),
             synth.blob_mask_count(d, 130, rng), synth.rect_mask_count(d, 70, rng)]
    alone = [Request(m, 200 + i, mk) for i, mk in enumerate(masks)]
    batch = [Request(m, 200 + i, mk) for i, mk in enumerate(masks)]
    tlat = torch.stack([synth.make_latent(d, 996 + s) for s in range(2)])
    kvc = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, kvc, synth.make_cache_kv(d, 14, 2, dtype=torch.bfloat16), tlat)
    ym = set(ig.y_block_modes(d.n_blocks, 2))
    hyc = ig.ig_cache_create(mh.ctx, 2, ig.IG_CACHE_HOST)
    kv2 = synth.make_cache_kv(d, 15, 2, dtype=torch.bfloat16)
    fill_cache(mh, hyc, hybrid_planes(kv2, synth.make_cache_y(d, 15, 2, dtype=torch.bfloat16), ym), tlat)
    caches = [hyc, kvc, hyc, kvc]
    for s in range(2):
        for i, r in enumerate(alone):
            ig.ig_edit_step(m.ctx, [r.req(i, caches[i], s, sig[s], sig[s + 1])], 0)
    for s in range(2):
        ig.ig_edit_step(m.ctx, [r.req(i, caches[i], s, sig[s], sig[s + 1]) for i, r in enumerate(batch)], 0)
        assert ig.ig_last_stats(m.ctx)["d2d_bytes"] > 0  # both groups deduplicated
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(zip(alone, batch)):
        assert torch.equal(a.latent, b.latent), i
    ig.ig_cache_free(kvc)
    ig.ig_cache_free(hyc)
    for r in alone + batch:
        r.free()
    mh.close()
    m.close()
