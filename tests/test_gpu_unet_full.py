"""Whole-UNet mask-aware step (include/ig_unet.h; BASELINE config 5) on the GPU vs
the float64 oracle (oracle/unet_full.py): dense ResBlocks / resamplers / GroupNorms as implicit-
GEMM and im2col tcgen05 convolutions, mask-aware Transformer2Ds with K/V + output caches.

* template recording (2 dense steps) follows the oracle's trajectory (C-TOL 2e-2);
* an edit step on a template cache from OTHER inputs matches the oracle's edit step on the
  oracle's cache of the same template (C-TOL 2e-2), for a batch of two requests at different
  steps plus an all-ones request;
* with the cache recorded from the request's own inputs, the edited masked rows equal the GPU's
  dense step bit for bit (same kernels, per-row batch-invariant GEMMs / attention, fp32 cached
  Transformer2D outputs); an empty mask leaves the latent bit-identical.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2505_20600_b200 import ig
from gpu_util import ctol

pytestmark = pytest.mark.gpu

U = synth.UNET_FULL_SMALL


@pytest.fixture(scope="module")
def unet():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    W = {}
    ptrs = []
    for name, shape, fan_in in synth.unet_full_weight_table(U):
        pass
    Wt = synth.make_unet_full_weights(U, dtype=torch.bfloat16)
    for name, _, _ in synth.unet_full_weight_table(U):
        t = Wt[name].contiguous().cuda()
        W[name] = t
        ptrs.append(t.data_ptr())
    h = ig.ig_unet_create(ig.make_unet_desc(U), ptrs, 0, 4, 2)
    Wh = {k: v.double().cpu().numpy() for k, v in W.items()}
    yield h, Wh
    ig.ig_unet_destroy(h)


def _inputs(rid):
    lat = synth.make_unet_latent(U, rid)
    ctx = synth.normal(rid, "unet_full_ctx", (U.ctx_len, U.ctx_dim)).float().bfloat16()
    cond = (synth.normal(rid, "unet_full_cond", (U.temb_dim,)) * 0.1).float()
    return lat, ctx, cond


def _mask(kind, rid=0):
    g = U.grid
    m = np.zeros((g, g), np.uint8)
    if kind == "rect":
        m[5:17, 9:25] = 1
    else:
        rng = np.random.default_rng(rid)
        m = (rng.random((g, g)) < 0.15).astype(np.uint8)
    return m.reshape(-1)


def _dev(t):
    return t.contiguous().cuda()


def test_template_follows_oracle(unet):
    h, Wh = unet
    lat, ctx, cond = _inputs(1)
    sig = [0.9, 0.6, 0.3]
    lat_d, ctx_d, cond_d = _dev(lat), _dev(ctx), _dev(cond)
    cache = ig.ig_unet_template(h, lat_d.data_ptr(), ctx_d.data_ptr(), cond_d.data_ptr(), sig)
    traj, _ = oracle.unet_full_cache_template(U, Wh, lat.double().numpy(), cond.double().numpy(),
                                              ctx.double().numpy(), sig)
    ok, worst = ctol(lat_d.double().cpu().numpy(), traj[-1], 2e-2)
    assert ok, worst
    ig.ig_unet_cache_free(cache)


def test_edit_batch_vs_oracle_on_foreign_template(unet):
    h, Wh = unet
    sig = [0.9, 0.6, 0.3]
    tl, tctx, tcond = _inputs(2)
    tl_d, tctx_d, tcond_d = _dev(tl), _dev(tctx), _dev(tcond)
    cache = ig.ig_unet_template(h, tl_d.data_ptr(), tctx_d.data_ptr(), tcond_d.data_ptr(), sig)
    _, ocache = oracle.unet_full_cache_template(U, Wh, tl.double().numpy(), tcond.double().numpy(),
                                                tctx.double().numpy(), sig)
    reqs, masks, hs, steps = [], [], [], [0, 1, 0]
    kinds = ["rect", "blob", "ones"]
    objs = []
    for i, kind in enumerate(kinds):
        lat, ctx, cond = _inputs(10 + i)
        mk = np.ones(U.grid * U.grid, np.uint8) if kind == "ones" else _mask(kind, i)
        mh, n = ig.ig_unet_mask_build(h, mk)
        objs.append((lat, _dev(lat), _dev(ctx), _dev(cond), mk, mh, ctx, cond))
        s = steps[i]
        reqs.append(ig.make_unet_req(objs[-1][1].data_ptr(), mh, cache, s, sig[s], sig[s + 1], objs[-1][2].data_ptr(),
                                     objs[-1][3].data_ptr()))
    ig.ig_unet_step(h, reqs)
    torch.cuda.synchronize()
    for i, (lat, lat_d, ctx_d, cond_d, mk, mh, ctx, cond) in enumerate(objs):
        s = steps[i]
        ref = oracle.unet_full_edit_step(U, Wh, lat.double().numpy(), mk, ocache[s], sig[s], sig[s + 1],
                                         cond.double().numpy(), ctx.double().numpy())
        got = lat_d.double().cpu().numpy()
        ok, worst = ctol(got, ref, 2e-2)
        assert ok, (kinds[i], worst)
        assert np.array_equal(got[mk == 0], lat.double().numpy()[mk == 0])
        ig.ig_unet_mask_free(mh)
    ig.ig_unet_cache_free(cache)


def test_same_input_cache_is_bitwise_dense_and_empty_mask_untouched(unet):
    h, _ = unet
    sig = [0.8, 0.5]
    lat, ctx, cond = _inputs(3)
    ctx_d, cond_d = _dev(ctx), _dev(cond)
    t_lat = _dev(lat)
    cache = ig.ig_unet_template(h, t_lat.data_ptr(), ctx_d.data_ptr(), cond_d.data_ptr(), sig)  # t_lat -> dense step
    mk = _mask("blob", 5)
    mh, _ = ig.ig_unet_mask_build(h, mk)
    e_lat = _dev(lat)
    ig.ig_unet_step(h, [ig.make_unet_req(e_lat.data_ptr(), mh, cache, 0, sig[0], sig[1], ctx_d.data_ptr(), cond_d.data_ptr())])
    torch.cuda.synchronize()
    idx = torch.from_numpy(np.flatnonzero(mk)).cuda()
    assert torch.equal(e_lat[idx], t_lat[idx])
    un = torch.from_numpy(np.flatnonzero(mk == 0)).cuda()
    assert torch.equal(e_lat[un], _dev(lat)[un])
    zero = np.zeros(U.grid * U.grid, np.uint8)
    zh, _ = ig.ig_unet_mask_build(h, zero)
    z_lat = _dev(lat)
    ig.ig_unet_step(h, [ig.make_unet_req(z_lat.data_ptr(), zh, cache, 0, sig[0], sig[1], ctx_d.data_ptr(), cond_d.data_ptr())])
    torch.cuda.synchronize()
    assert torch.equal(z_lat, _dev(lat))
    ig.ig_unet_mask_free(mh)
    ig.ig_unet_mask_free(zh)
    ig.ig_unet_cache_free(cache)


@pytest.mark.parametrize("n,H,W,cin,cout", [(2, 32, 32, 128, 256), (1, 64, 64, 64, 320), (1, 128, 128, 64, 128),
                                            (3, 16, 8, 64, 64), (2, 8, 8, 64, 128), (1, 32, 32, 1280, 1280),
                                            (1, 4, 4, 64, 64), (4, 32, 32, 1280, 1280), (2, 64, 64, 640, 640),
                                            (2, 128, 128, 320, 320)])
def test_conv3x3_vs_torch(n, H, W, cin, cout):
    """ig_op_conv3x3 (implicit-GEMM tcgen05 conv: 1-CTA, 2-CTA 256x256 and 256x160 tiles, every run
    width; im2col fallback for (H*W) % 128 != 0) against torch conv2d in fp32 on the same bf16
    inputs."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.backends.cudnn.allow_tf32 = False  # a true fp32 reference
    g = torch.Generator(device="cuda").manual_seed(H * W + cin + cout)
    x = torch.randn(n, H, W, cin, device="cuda", generator=g).bfloat16()
    w = (torch.randn(cout, 3, 3, cin, device="cuda", generator=g) / (9 * cin) ** 0.5).bfloat16()
    b = torch.randn(cout, device="cuda", generator=g).bfloat16()
    xp = torch.nn.functional.pad(x, (0, 0, 1, 1, 1, 1)).contiguous()
    y = torch.empty(n * H * W, cout, device="cuda", dtype=torch.float32)
    ig.ig_op_conv3x3(xp.data_ptr(), n, H, W, cin, w.data_ptr(), b.data_ptr(), cout, y.data_ptr())
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), b.float(),
                                     padding=1).permute(0, 2, 3, 1).reshape(n * H * W, cout)
    ok, worst = ctol(y.cpu().numpy(), ref.cpu().numpy(), 1e-3)
    assert ok, worst
