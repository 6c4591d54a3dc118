"""GPU parity of the SDXL-UNet attention stack (BASELINE config 5) through the C ABI
against oracle/unet.py on the same seeded inputs: C-TOL rtol 1e-4 (fp32 parity mode) and
2e-2 (bf16); unmasked rows bit-identical."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_20600_b200 import ig
from gpu_util import Model, Request, cache_to_numpy, ctol, fill_cache

pytestmark = pytest.mark.gpu

RTOL = {ig.IG_F32: 1e-4, ig.IG_BF16: 2e-2}
TDT = {ig.IG_F32: torch.float32, ig.IG_BF16: torch.bfloat16}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ig.lib()


def _steps(m, reqs, cache, n_steps, stream=0):
    for s in range(n_steps):
        rr = [r.req(i, cache, s, 0.0, 0.0) for i, r in enumerate(reqs)]
        ig.ig_edit_step(m.ctx, rr, stream)
    torch.cuda.synchronize()


def _oracle_steps(d, W, r, kvh, n_steps):
    x, ctx = r.latent0.double().cpu().numpy(), r.txt.double().cpu().numpy()
    for s in range(n_steps):
        x = oracle.unet_edit_step(d, W, x, r.mask_np, kvh[s], ctx)
    return x


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
def test_unet_tiny_template_and_edit(dtype):
    """Template recording (dense stack, K/V of every block and step) vs the oracle's cache and
    trajectory; then two edit steps with a synthetic cache shared by both sides."""
    d = synth.UNET_TINY
    m = Model(d, dtype)
    W = m.host_weights()
    rq = Request(m, 0, synth.rect_mask(d, 4, 12, 4, 12))
    x0, ctx = rq.latent0.double().cpu().numpy(), rq.txt.double().cpu().numpy()
    st = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, st.data_ptr(), rq.txt.data_ptr(), 0, [1.0, 0.5, 0.0])
    states, ocache = oracle.unet_cache_template(d, W, x0, ctx, 2)
    ok, worst = ctol(cache_to_numpy(cache, d, 2, dtype), ocache, RTOL[dtype])
    assert ok, ("cache", worst)
    ok, worst = ctol(st.double().cpu().numpy(), states[-1], RTOL[dtype])
    assert ok, ("dense trajectory", worst)
    kv = synth.make_cache_kv(d, 0, 2, dtype=TDT[dtype])
    syn = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, syn, kv)
    _steps(m, [rq], syn, 2)
    want = _oracle_steps(d, W, rq, kv.double().numpy(), 2)
    got = rq.latent.double().cpu().numpy()
    ok, worst = ctol(got, want, RTOL[dtype])
    assert ok, ("edit", worst)
    assert np.array_equal(got[rq.mask_np == 0], x0[rq.mask_np == 0])
    ig.ig_cache_free(cache)
    ig.ig_cache_free(syn)
    rq.free()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("copy_mode,tier", [(0, ig.IG_CACHE_HOST), (1, ig.IG_CACHE_HOST), (1, ig.IG_CACHE_DEVICE)])
def test_unet_small_batch(dtype, copy_mode, tier):
    """d = 64 (tcgen05 attention, fused K/V-merge epilogue, fused GEGLU epilogue in bf16): a
    batch of 3 requests (rectangle, blob, all-ones) over 2 steps of a synthetic cache."""
    d = synth.UNET_SMALL
    opts = ig.ig_ctx_opts(4, 0, 2, copy_mode, 0, 0)
    m = Model(d, dtype, opts=opts)
    W = m.host_weights()
    rng = np.random.default_rng(1)
    masks = [synth.rect_mask_count(d, 40, rng), synth.blob_mask_count(d, 150, rng), np.ones(d.L_img, np.uint8)]
    reqs = [Request(m, 20 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 4, 2, dtype=TDT[dtype])
    cache = ig.ig_cache_create(m.ctx, 2, tier)
    fill_cache(m, cache, kv)
    _steps(m, reqs, cache, 2)
    kvh = kv.double().numpy()
    for r in reqs:
        want = _oracle_steps(d, W, r, kvh, 2)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, want, RTOL[dtype])
        assert ok, worst
        assert np.array_equal(got[r.mask_np == 0], r.latent0.cpu().numpy()[r.mask_np == 0])
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def test_unet_same_inputs_cache_matches_dense_on_gpu():
    """bf16: a cache recorded on the GPU along the dense trajectory, then an edit step from the
    template's own state reproduces the GPU dense step on the masked rows (same arithmetic per
    row: K/V of the unmasked rows are the recorded ones), and is alone == in-batch bitwise."""
    d = synth.UNET_SMALL
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    mask = synth.blob_mask_count(d, 70, np.random.default_rng(2))
    rq = Request(m, 5, mask)
    st = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, st.data_ptr(), rq.txt.data_ptr(), 0, [1.0, 0.5])
    _steps(m, [rq], cache, 1)
    got = rq.latent.double().cpu().numpy()
    dense = st.double().cpu().numpy()
    ok, worst = ctol(got[mask != 0], dense[mask != 0], 2e-2)
    assert ok, worst
    # alone == together with another request (batch invariance of the fixed-tile kernels)
    other = Request(m, 6, synth.rect_mask_count(d, 90, np.random.default_rng(3)))
    rq2 = Request(m, 5, mask)
    rr = [rq2.req(0, cache, 0, 0.0, 0.0), other.req(1, cache, 0, 0.0, 0.0)]
    ig.ig_edit_step(m.ctx, rr, 0)
    torch.cuda.synchronize()
    assert torch.equal(rq2.latent, rq.latent)
    ig.ig_cache_free(cache)
    for r in (rq, rq2, other):
        r.free()
    m.close()


def test_unet_cuda_graph_bitwise_equals_eager():
    d = synth.UNET_SMALL
    res = []
    for graphs in (0, 1):
        m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 0, 0, graphs))
        rng = np.random.default_rng(4)
        reqs = [Request(m, 30 + i, synth.blob_mask_count(d, 60 + 40 * i, rng)) for i in range(2)]
        kv = synth.make_cache_kv(d, 5, 3, dtype=torch.bfloat16)
        cache = ig.ig_cache_create(m.ctx, 3, ig.IG_CACHE_DEVICE)
        fill_cache(m, cache, kv)
        s = torch.cuda.Stream()
        _steps(m, reqs, cache, 2, s.cuda_stream)
        # a third step eagerly (profiling forces eager launches) after the graph replays:
        # the ring events recorded inside captures must not be waited on
        ig.ig_profile_enable(m.ctx, 1)
        ig.ig_edit_step(m.ctx, [r.req(i, cache, 2, 0.0, 0.0) for i, r in enumerate(reqs)], s.cuda_stream)
        torch.cuda.synchronize()
        ig.ig_profile_read(m.ctx)
        ig.ig_profile_enable(m.ctx, 0)
        res.append([r.latent.clone() for r in reqs])
        ig.ig_cache_free(cache)
        for r in reqs:
            r.free()
        m.close()
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("which", ["sdxl_attn64", "sdxl_attn32_2blocks"])
def test_sdxl_level_full_width(which):
    """Full SDXL level widths (64x64 level: all 10 blocks, C=640, 4096 tokens; 32x32 level:
    C=1280, 1024 tokens, 2 of its 60 blocks), 77 x 2048 context, bf16, a batch of 2 requests
    (m = 0.1 rectangle, 0.3 blob) over one step of a synthetic cache vs the oracle."""
    d = synth.SDXL_L64 if which == "sdxl_attn64" else synth._unet("sdxl32_2", 2, 1280, 20, 32, 77, 2048)
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0, 0))
    W = m.host_weights()
    rng = np.random.default_rng(6)
    masks = [synth.rect_mask_count(d, round(0.1 * d.L_img), rng), synth.blob_mask_count(d, round(0.3 * d.L_img), rng)]
    reqs = [Request(m, 40 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 6, 1, dtype=torch.bfloat16)
    cache = ig.ig_cache_create(m.ctx, 1, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv)
    _steps(m, reqs, cache, 1)
    kvh = kv.double().numpy()
    for r in reqs:
        want = _oracle_steps(d, W, r, kvh, 1)
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got[r.mask_np != 0], want[r.mask_np != 0], 2e-2)
        assert ok, worst
        assert np.array_equal(got[r.mask_np == 0], r.latent0.cpu().numpy()[r.mask_np == 0])
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("tier", [ig.IG_CACHE_HOST, ig.IG_CACHE_DEVICE])
def test_unet_y_and_hybrid_caches(dtype, tier):
    """Y (kv_blocks = 0) and hybrid (kv_blocks = 1: blocks {0, 2} Y, block 1 K/V) caches next to
    a plain K/V cache in one batch, 2 steps, vs the oracle's unet_edit_step_y(y_blocks=)."""
    from gpu_util import hybrid_planes
    d = synth.UNET_SMALL
    rng = np.random.default_rng(31)
    masks = [synth.blob_mask_count(d, 85, rng), synth.rect_mask_count(d, 45, rng), synth.blob_mask_count(d, 66, rng)]
    splits = [0, 1, None]
    base = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    reqs = [Request(base, 60 + i, mk) for i, mk in enumerate(masks)]
    tst = torch.stack([synth.make_latent(d, 990 + s) for s in range(2)])  # template input states
    ms, caches, refs = [], [], []
    for i, kvb in enumerate(splits):
        kv = synth.make_cache_kv(d, 30 + i, 2, dtype=TDT[dtype])
        yv = synth.make_cache_y(d, 30 + i, 2, dtype=TDT[dtype])
        if kvb is None:
            c = ig.ig_cache_create(base.ctx, 2, tier)
            fill_cache(base, c, kv, tst)
            refs.append((kv.double().numpy(), None, None))
        else:
            m = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, kvb))
            ms.append(m)
            ym = set(ig.y_block_modes(d.n_blocks, kvb))
            c = ig.ig_cache_create(m.ctx, 2, tier)
            fill_cache(m, c, hybrid_planes(kv, yv, ym), tst)
            refs.append((kv.double().numpy(), yv.double().numpy(), ym))
        caches.append(c)
    for s in range(2):
        ig.ig_edit_step(base.ctx, [r.req(i, caches[i], s, 0.0, 0.0) for i, r in enumerate(reqs)], 0)
    torch.cuda.synchronize()
    W = base.host_weights()
    tsh = tst.double().numpy()
    for i, r in enumerate(reqs):
        x, ctx = r.latent0.double().cpu().numpy(), r.txt.double().cpu().numpy()
        kvh, yh, ym = refs[i]
        for s in range(2):
            if ym is None:
                x = oracle.unet_edit_step(d, W, x, r.mask_np, kvh[s], ctx)
            else:
                x = oracle.unet_edit_step_y(d, W, x, r.mask_np, yh[s], tsh[s], ctx, y_blocks=ym, kv_cache_step=kvh[s])
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, (i, worst)
        assert np.array_equal(got[r.mask_np == 0], r.latent0.cpu().numpy()[r.mask_np == 0])
    for c in caches:
        ig.ig_cache_free(c)
    for r in reqs:
        r.free()
    for m in ms:
        m.close()
    base.close()


@pytest.mark.parametrize("kv_blocks", [0, 1])
def test_unet_hybrid_template_recording(kv_blocks):
    """fp32: ig_cache_template on a cache_y ctx records K/V for the K/V blocks and Y_b where
    block b or b + 1 is a Y block, against the oracle's dense pass; an edit from the template's
    own state then stays on the dense trajectory for the masked rows."""
    from gpu_util import cache_raw_numpy, n_planes, split_hybrid
    d = synth.UNET_SMALL
    m = Model(d, ig.IG_F32, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0, 0, 1, kv_blocks))
    W = m.host_weights()
    mask = synth.blob_mask_count(d, 77, np.random.default_rng(12))
    rq = Request(m, 70, mask)
    st = rq.latent.clone()
    cache = ig.ig_cache_template(m.ctx, st.data_ptr(), rq.txt.data_ptr(), 0, [1.0, 0.5, 0.0])
    ym = set(ig.y_block_modes(d.n_blocks, kv_blocks))
    states, okv, oy = oracle.unet_cache_template(d, W, rq.latent0.double().cpu().numpy(), rq.txt.double().cpu().numpy(),
                                                 2, record_y=True)
    raw = cache_raw_numpy(cache, d, 2, n_planes(d.n_blocks, ym), ig.IG_F32)
    gkv, gy = split_hybrid(raw, d.n_blocks, ym)
    for b in range(d.n_blocks):
        if b not in ym:
            ok, worst = ctol(gkv[:, b], okv[:, b], 1e-4)
            assert ok, ("kv", b, worst)
        if b in ym or (b + 1) in ym:
            ok, worst = ctol(gy[:, b], oy[:, b], 1e-4)
            assert ok, ("y", b, worst)
    ok, worst = ctol(st.double().cpu().numpy(), states[-1], 1e-4)
    assert ok, ("trajectory", worst)
    for s in range(2):  # edit from the template's own input state at step s
        x = torch.from_numpy(states[s]).float().cuda().contiguous()
        rr = ig.make_req(0, x.data_ptr(), rq.mask, cache, s, 0.0, 0.0, rq.txt.data_ptr(), None)
        ig.ig_edit_step(m.ctx, [rr], 0)
        torch.cuda.synchronize()
        got = x.double().cpu().numpy()
        ok, worst = ctol(got[mask != 0], states[s + 1][mask != 0], 1e-4)
        assert ok, ("same trajectory", s, worst)
    ig.ig_cache_free(cache)
    rq.free()
    m.close()


@pytest.mark.parametrize("tier", [ig.IG_CACHE_HOST, ig.IG_CACHE_DEVICE])
def test_unet_fp8_cache(tier):
    """FP8 (e4m3, per (token, head) scale) K/V cache on a UNet context: the oracle
    mirrors the quantize/dequantize round trip of the same bf16 cache; 2 requests, 2 steps."""
    d = synth.UNET_SMALL
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 1))
    W = m.host_weights()
    rng = np.random.default_rng(41)
    reqs = [Request(m, 80 + i, mk) for i, mk in
            enumerate([synth.blob_mask_count(d, 70, rng), synth.rect_mask_count(d, 30, rng)])]
    kv = synth.make_cache_kv(d, 11, 2, dtype=torch.bfloat16, device="cuda")
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    ig.ig_cache_write(m.ctx, cache, kv.data_ptr())
    if tier == ig.IG_CACHE_DEVICE:
        dc = ig.ig_cache_clone(m.ctx, cache, ig.IG_CACHE_DEVICE)
        ig.ig_cache_free(cache)
        cache = dc
    kvh = oracle.fp8_kv_roundtrip(kv.float().cpu().numpy(), d.heads)
    _steps(m, reqs, cache, 2)
    for r in reqs:
        want = _oracle_steps(d, W, r, kvh, 2)
        ok, worst = ctol(r.latent.double().cpu().numpy(), want, 2e-2)
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


@pytest.mark.parametrize("dtype", [ig.IG_F32, ig.IG_BF16])
@pytest.mark.parametrize("k", [1, 3])
def test_unet_dense_prefix(dtype, k):
    """Algorithm-1 dense prefix (ig_set_plan mode 1, k blocks) on the UNet stack: a K/V-cache
    request and a hybrid-cache request (blocks {0, 2} Y) in one batch, 2 steps, vs the oracle's
    unet_edit_step_planned (unmasked rows of the prefix from the template's input state)."""
    from gpu_util import hybrid_planes
    d = synth.UNET_SMALL
    rng = np.random.default_rng(51)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 52, rng)]
    base = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0))
    hyb = Model(d, dtype, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, 1))
    reqs = [Request(base, 90 + i, mk) for i, mk in enumerate(masks)]
    tst = torch.stack([synth.make_latent(d, 995 + s) for s in range(2)])
    kv = synth.make_cache_kv(d, 40, 2, dtype=TDT[dtype])
    yv = synth.make_cache_y(d, 40, 2, dtype=TDT[dtype])
    ym = set(ig.y_block_modes(d.n_blocks, 1))
    c_kv = ig.ig_cache_create(base.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(base, c_kv, kv, tst)
    c_hy = ig.ig_cache_create(hyb.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(hyb, c_hy, hybrid_planes(kv, yv, ym), tst)
    ig.ig_set_plan(base.ctx, 1, k)
    caches = [c_kv, c_hy]
    for s in range(2):
        ig.ig_edit_step(base.ctx, [r.req(i, caches[i], s, 0.0, 0.0) for i, r in enumerate(reqs)], 0)
        assert ig.ig_last_plan(base.ctx) == k
    torch.cuda.synchronize()
    W = base.host_weights()
    kvh, yh, tsh = kv.double().numpy(), yv.double().numpy(), tst.double().numpy()
    for i, r in enumerate(reqs):
        x, ctx = r.latent0.double().cpu().numpy(), r.txt.double().cpu().numpy()
        for s in range(2):
            x = oracle.unet_edit_step_planned(d, W, x, r.mask_np, tsh[s], ctx, k, kv_cache_step=kvh[s],
                                              y_cache_step=yh[s], y_blocks=ym if i == 1 else ())
        got = r.latent.double().cpu().numpy()
        ok, worst = ctol(got, x, RTOL[dtype])
        assert ok, (i, worst)
        assert np.array_equal(got[r.mask_np == 0], r.latent0.cpu().numpy()[r.mask_np == 0])
    ig.ig_cache_free(c_kv)
    ig.ig_cache_free(c_hy)
    for r in reqs:
        r.free()
    hyb.close()
    base.close()


@pytest.mark.parametrize("kind", ["kv", "hybrid"])
def test_unet_load_dedupe_bitwise(kind):
    """Lockstep UNet requests on one (host-tier cache, step) share staged rows (load
    deduplication): the batch equals each request alone bit for bit with fewer link bytes."""
    from gpu_util import hybrid_planes
    d = synth.UNET_SMALL
    opts = ig.ig_ctx_opts(4, 0, 2, 1, 0, 0) if kind == "kv" else ig.ig_ctx_opts(4, 0, 2, 1, 0, 0, 1, 1)
    m = Model(d, ig.IG_BF16, opts=opts)
    rng = np.random.default_rng(61)
    masks = [synth.blob_mask_count(d, 90, rng), synth.rect_mask_count(d, 40, rng), synth.blob_mask_count(d, 130, rng)]
    alone = [Request(m, 290 + i, mk) for i, mk in enumerate(masks)]
    batch = [Request(m, 290 + i, mk) for i, mk in enumerate(masks)]
    kv = synth.make_cache_kv(d, 14, 2, dtype=torch.bfloat16)
    tst = torch.stack([synth.make_latent(d, 996 + s) for s in range(2)])
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    if kind == "kv":
        fill_cache(m, cache, kv, tst)
    else:
        ym = set(ig.y_block_modes(d.n_blocks, 1))
        fill_cache(m, cache, hybrid_planes(kv, synth.make_cache_y(d, 14, 2, dtype=torch.bfloat16), ym), tst)
    h2d_alone = h2d_batch = 0
    for s in range(2):
        for i, r in enumerate(alone):
            ig.ig_edit_step(m.ctx, [r.req(i, cache, s, 0.0, 0.0)], 0)
            h2d_alone += ig.ig_last_stats(m.ctx)["h2d_bytes"]
    for s in range(2):
        ig.ig_edit_step(m.ctx, [r.req(i, cache, s, 0.0, 0.0) for i, r in enumerate(batch)], 0)
        h2d_batch += ig.ig_last_stats(m.ctx)["h2d_bytes"]
    torch.cuda.synchronize()
    for a, b in zip(alone, batch):
        assert torch.equal(a.latent, b.latent)
    assert h2d_batch < h2d_alone
    ig.ig_cache_free(cache)
    for r in alone + batch:
        r.free()
    m.close()


def test_unet_zero_copy_gather_mode():
    """copy_mode 2 (SM gather straight from pinned host memory) on a UNet context vs the oracle."""
    d = synth.UNET_SMALL
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 2, 0, 0))
    W = m.host_weights()
    rng = np.random.default_rng(71)
    reqs = [Request(m, 300 + i, mk) for i, mk in enumerate([synth.blob_mask_count(d, 77, rng), synth.rect_mask_count(d, 33, rng)])]
    kv = synth.make_cache_kv(d, 15, 2, dtype=torch.bfloat16)
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, kv)
    _steps(m, reqs, cache, 2)
    for r in reqs:
        want = _oracle_steps(d, W, r, kv.double().numpy(), 2)
        ok, worst = ctol(r.latent.double().cpu().numpy(), want, 2e-2)
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


@pytest.mark.parametrize("model,kv_blocks", [("unet_small", 0), ("unet_small", 1), ("flux_small", 2)])
@pytest.mark.parametrize("tier", [ig.IG_CACHE_HOST, ig.IG_CACHE_DEVICE])
def test_fp8_y_and_hybrid_caches(model, kv_blocks, tier):
    """FP8 Y / hybrid caches (SURVEY N4 x N2): every plane (K, V and Y) stored as e4m3 with a
    per (token, head) scale; the oracle mirrors the round trip of the same bf16 planes and runs
    the Y-variant step (UNet and Flux-structured models), 2 requests, 2 steps."""
    from gpu_util import hybrid_planes
    d = synth.MODELS[model]
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(4, 0, 2, 1, 0, 1, 1, kv_blocks))
    W = m.host_weights()
    rng = np.random.default_rng(81)
    reqs = [Request(m, 310 + i, mk) for i, mk in enumerate([synth.blob_mask_count(d, 80, rng), synth.rect_mask_count(d, 36, rng)])]
    kv = synth.make_cache_kv(d, 16, 2, dtype=torch.bfloat16)
    yv = synth.make_cache_y(d, 16, 2, dtype=torch.bfloat16)
    tst = torch.stack([synth.make_latent(d, 997 + s) for s in range(2)])
    ym = set(ig.y_block_modes(d.n_blocks, kv_blocks))
    cache = ig.ig_cache_create(m.ctx, 2, ig.IG_CACHE_HOST)
    fill_cache(m, cache, hybrid_planes(kv, yv, ym), tst)
    if tier == ig.IG_CACHE_DEVICE:
        dc = ig.ig_cache_clone(m.ctx, cache, ig.IG_CACHE_DEVICE)
        ig.ig_cache_free(cache)
        cache = dc
    kvq = oracle.fp8_kv_roundtrip(kv.float().numpy(), d.heads)
    yq = oracle.fp8_kv_roundtrip(yv.float().numpy(), d.heads)
    tsh = tst.double().numpy()
    sig = [1.0, 0.7, 0.4]
    for s in range(2):
        ig.ig_edit_step(m.ctx, [r.req(i, cache, s, sig[s], sig[s + 1]) for i, r in enumerate(reqs)], 0)
    torch.cuda.synchronize()
    for r in reqs:
        x = r.latent0.double().cpu().numpy()
        for s in range(2):
            if d.n_unet:
                x = oracle.unet_edit_step_y(d, W, x, r.mask_np, yq[s], tsh[s], r.txt.double().cpu().numpy(),
                                            y_blocks=ym, kv_cache_step=kvq[s])
            else:
                _, txt, cond = r.host_inputs()
                x = oracle.edit_step_y(d, W, x, r.mask_np, yq[s], tsh[s], sig[s], sig[s + 1], txt, cond,
                                       y_blocks=ym, kv_cache_step=kvq[s])
        ok, worst = ctol(r.latent.double().cpu().numpy(), x, 2e-2)
        assert ok, worst
    ig.ig_cache_free(cache)
    for r in reqs:
        r.free()
    m.close()


def _e4m3_to_f32(b: np.ndarray) -> np.ndarray:
    """OCP e4m3 (bias 7, no infinities; 0x7f / 0xff NaN) -> float32, written from the format."""
    b = b.astype(np.int32)
    sgn = np.where(b & 0x80, -1.0, 1.0)
    e, m = (b >> 3) & 0xF, b & 0x7
    val = np.where(e == 0, m / 8.0 * 2.0 ** -6, (1.0 + m / 8.0) * 2.0 ** (e.astype(np.float64) - 7))
    val = np.where((b & 0x7F) == 0x7F, np.nan, val)
    return (sgn * val).astype(np.float32)


def _bf16_rne(x: np.ndarray) -> np.ndarray:
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def test_fp8_hybrid_template_recording_vs_oracle():
    """ig_cache_template on an FP8 hybrid ctx (include/ig.h cache_fp8 + cache_y + cache_kv_blocks):
    the recorded planes, read back and dequantized as the header defines (e4m3 data planes, then
    fp32 scales per (token, head) in plane order; x' = bf16(q * scale)), (1) match the oracle's
    dense template (unet_cache_template) within e4m3 rounding, and (2) drive the GPU edit step to
    the oracle's Y-variant step (unet_edit_step_y) on those same planes within the bf16 bar."""
    from gpu_util import n_planes, split_hybrid
    import ctypes
    d = synth.UNET_SMALL
    kv_blocks = 1
    m = Model(d, ig.IG_BF16, opts=ig.ig_ctx_opts(2, 0, 2, 1, 0, 1, 1, kv_blocks))
    W = m.host_weights()
    mask = synth.blob_mask_count(d, 70, np.random.default_rng(91))
    rq = Request(m, 320, mask)
    st = rq.latent.clone()
    x0 = rq.latent.clone()
    state0 = x0.double().cpu().numpy()
    ctx_np = rq.txt.double().cpu().numpy()
    cache = ig.ig_cache_template(m.ctx, st.data_ptr(), rq.txt.data_ptr(), 0, [1.0, 0.5])
    torch.cuda.synchronize()
    ym = set(ig.y_block_modes(d.n_blocks, kv_blocks))
    P, L, H = n_planes(d.n_blocks, ym), d.L_img, d.hidden
    ptr, _, tier = ig.ig_cache_storage(cache)
    assert tier == ig.IG_CACHE_HOST
    nq = P * L * H
    q = np.frombuffer((ctypes.c_char * nq).from_address(ptr), dtype=np.uint8).copy().reshape(1, P, L, H)
    scl = np.frombuffer((ctypes.c_char * (P * L * d.heads * 4)).from_address(ptr + nq), dtype=np.float32)
    scl = scl.copy().reshape(1, P, L, d.heads)
    deq = _bf16_rne(_e4m3_to_f32(q) * np.repeat(scl, H // d.heads, axis=3)).astype(np.float64)
    assert np.isfinite(deq).all()
    kv_g, y_g = split_hybrid(deq, d.n_blocks, ym)
    # (1) recording vs the oracle's dense template, within e4m3 rounding (3 mantissa bits: a
    # relative step of 2^-3, so ~2^-4 max rounding error; 2^-3 per element leaves room for one
    # flipped rounding of a bf16-vs-fp64 input) plus the per-(token, head) scale's subnormal floor
    _, kv_o, y_o = oracle.unet_cache_template(d, W, state0, ctx_np, 1, record_y=True)
    for b in range(d.n_blocks):
        pairs = ([(y_g[0, b], y_o[0, b])] if (b in ym or b + 1 in ym) else []) + \
                ([(kv_g[0, b, 0], kv_o[0, b, 0]), (kv_g[0, b, 1], kv_o[0, b, 1])] if b not in ym else [])
        for g, o in pairs:
            amax = np.abs(o).reshape(L, d.heads, -1).max(axis=2).repeat(H // d.heads, axis=1)
            assert (np.abs(g - o) <= 0.125 * np.abs(o) + amax / 448.0 * 2.0 ** -6 + 2e-2 * amax).all(), b
            assert np.linalg.norm(g - o) <= 0.06 * np.linalg.norm(o), b
    # (2) the GPU edit on its recorded FP8 template vs the oracle on the same (dequantized) planes
    rr = ig.make_req(0, x0.data_ptr(), rq.mask, cache, 0, 0.0, 0.0, rq.txt.data_ptr(), None)
    ig.ig_edit_step(m.ctx, [rr], 0)
    torch.cuda.synchronize()
    want = oracle.unet_edit_step_y(d, W, state0, mask, y_g[0], state0, ctx_np, y_blocks=ym, kv_cache_step=kv_g[0])
    ok, worst = ctol(x0.double().cpu().numpy(), want, 2e-2)
    assert ok, worst
    ig.ig_cache_free(cache)
    rq.free()
    m.close()


@pytest.fixture(scope="module")
def sdxl32():
    """The full 32x32 SDXL level (60 blocks, C = 1280; 2.1 B bf16 parameters) in the launch
    configuration tools/unet_sweep.py times (max_batch 8, prefetch depth 4, compacted copies)."""
    m = Model(synth.SDXL_L32, ig.IG_BF16, opts=ig.ig_ctx_opts(8, 0, 4, 1, 0, 0))
    yield m
    m.close()


@pytest.mark.parametrize("block,m_ratio", [(0, 0.05), (37, 0.2), (59, 0.6)])
def test_sdxl32_teacher_forced_block(sdxl32, block, m_ratio):
    """Full-size SDXL 32x32 blocks through ig_debug_block (teacher-forced input rows, K/V of the
    unmasked rows from the cache) vs the oracle's unet_block_masked on the same inputs, compared
    on the block's update (X_out - X_in) with C-TOL 2e-2."""
    d = synth.SDXL_L32
    mask = synth.blob_mask_count(d, round(m_ratio * d.L_img), np.random.default_rng(100 + block))
    rq = Request(sdxl32, 400 + block, mask)
    kv = synth.make_cache_kv(d, 17, 1, dtype=torch.bfloat16, device="cuda")
    cache = ig.ig_cache_create(sdxl32.ctx, 1, ig.IG_CACHE_HOST)
    fill_cache(sdxl32, cache, kv)
    rows = rq.n_m
    X_in = synth.normal(960 + block, "X_in_unet", (rows, d.hidden), "cuda").float()
    X_out = torch.full_like(X_in, float("nan"))
    ig.ig_debug_block(sdxl32.ctx, rq.req(0, cache, 0, 0.0, 0.0), block, X_in.data_ptr(), X_out.data_ptr())
    torch.cuda.synchronize()
    names = {nm for nm, _, _ in synth.weight_table(d) if nm.startswith(f"unet.{block}.")}
    W = {k: sdxl32.W[k].double().cpu().numpy() for k in names}
    idx_m, idx_u, _ = oracle.index_build(mask)
    want, _, _ = oracle.unet_block_masked(d, W, block, X_in.double().cpu().numpy(), idx_m, idx_u,
                                          kv[0, block].double().cpu().numpy(), rq.txt.double().cpu().numpy())
    xin = X_in.double().cpu().numpy()
    ok, worst = ctol(X_out.double().cpu().numpy() - xin, want - xin, 2e-2)
    assert ok, worst
    ig.ig_cache_free(cache)
    rq.free()


@pytest.mark.parametrize("M,F,K", [(1, 128, 64), (300, 256, 128), (1992, 640, 320)])
def test_op_gemm_geglu_epilogue(M, F, K):
    """The fused GEGLU epilogue alone (ig_op_gemm epi 5, tile-interleaved weights) vs the oracle's
    hidden * GELU_erf(gate) on the same bf16 inputs (C-TOL rtol 4e-3: the bf16 output rounding
    alone is up to 2^-9 relative, the north_star bf16 bar is 2e-2)."""
    A = synth.uniform(1, "A", (M, K), "cuda").float().to(torch.bfloat16)
    W = (synth.uniform(2, "W", (2 * F, K), "cuda") / K ** 0.5).float().to(torch.bfloat16)
    b = synth.uniform(3, "b", (2 * F,), "cuda").float().to(torch.bfloat16)
    perm = np.array([(128 * (r // 256) + r % 256) if r % 256 < 128 else (F + 128 * (r // 256) + r % 256 - 128)
                     for r in range(2 * F)])
    Wi, bi = W[perm].contiguous(), b[perm].contiguous()
    C = torch.full((M, F), float("nan"), dtype=torch.bfloat16, device="cuda")
    ig.ig_op_gemm(ig.IG_BF16, A.data_ptr(), K, Wi.data_ptr(), K, bi.data_ptr(), C.data_ptr(), F, M, 2 * F, K, 5, 0, 0)
    torch.cuda.synchronize()
    u = oracle.linear(A.double().cpu().numpy(), W.double().cpu().numpy(), b.double().cpu().numpy())
    want = u[:, :F] * oracle.gelu_erf(u[:, F:])
    ok, worst = ctol(C.double().cpu().numpy(), want, 4e-3)
    assert ok, worst
