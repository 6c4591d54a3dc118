"""Config 5 on the WHOLE SDXL-shaped UNet (BASELINE configs[4]): mask-ratio sweep of
the mask-aware step (Transformer2Ds on masked tokens with K/V + output caches, dense ResBlocks /
resamplers / convolutions) against the dense step, batch of 8 requests at distinct steps of one
template, template cache in HBM or pinned host memory.

    python tools/unet_full_sweep.py [--model sdxl_unet] [--batch 8] [--steps 6] [--tier device|host]
                                    [--ms 0.01,0.05,...] [--out profiles/r02_unet_full_sweep.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_20600_b200 import ig, levels  # noqa: E402

N_SCHED = 8


def dense_conv_macs(u):
    """Multiply-accumulates of every convolution / resampler / linear skip of one UNet pass."""
    g = u.grid
    macs = (g * g) * 9 * u.lat_ch * u.ch[0] * 2  # conv_in + conv_out
    for _, lvl, ci, co, _ in synth.unet_resblocks(u):
        P = (g >> lvl) ** 2
        macs += P * 9 * (ci * co + co * co) + (P * ci * co if ci != co else 0)
    macs += sum(((g >> (l + 1)) ** 2) * 9 * u.ch[l] ** 2 for l in (0, 1))   # downsamplers
    macs += sum(((g >> (l - 1)) ** 2) * 9 * u.ch[l] ** 2 for l in (2, 1))   # upsamplers
    return macs


def flops(u, mask):
    """Algorithmic FLOPs of one request-step: every convolution / resampler / skip dense, each
    Transformer2D's proj_in/out, token-wise block ops and attention rows scaled by its level's
    masked rows (Table 1 scaling; the cross-attention context K/V does not depend on
    the mask)."""
    g = u.grid
    lv = [np.asarray(mask) != 0]
    lv.append(levels.any_pool2(lv[0], g, g) != 0)
    lv.append(levels.any_pool2(lv[1], g // 2, g // 2) != 0)
    frac = [float(x.mean()) for x in lv]
    macs = dense_conv_macs(u)
    for _, lvl, c, dep in synth.unet_t2ds(u):
        P = (g >> lvl) ** 2
        F = 4 * c
        per_row = 6 * c * c + 3 * F * c + 2 * P * c + 2 * u.ctx_len * c
        macs += frac[lvl] * (2 * P * c * c + dep * P * per_row) + dep * u.ctx_len * 2 * c * u.ctx_dim
    return 2.0 * macs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="sdxl_unet")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--tier", default="device", choices=["device", "host"])
    ap.add_argument("--ms", default="0.01,0.05,0.1,0.2,0.3,0.5,0.8,1.0")
    ap.add_argument("--out", default=None)
    ap.add_argument("--depth", type=int, default=2, help="copy-lane ring depth of each Transformer2D")
    ap.add_argument("--profile", action="store_true",
                    help="bracket the timed steps with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    u = synth.UNET_FULL[args.model]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    W = [synth.make_unet_full_weights(u, device=dev, dtype=torch.bfloat16, names={n})[n].contiguous()
         for n, _, _ in synth.unet_full_weight_table(u)]  # drawn on the device (2.6 B parameters)
    h = ig.ig_unet_create(ig.make_unet_desc(u), [t.data_ptr() for t in W], 0, args.batch, args.depth)
    sig = synth.flow_sigmas(N_SCHED)
    stream = torch.cuda.Stream()
    tl = synth.make_unet_latent(u, 10 ** 6).to(dev)
    tctx = synth.normal(10 ** 6, "unet_full_ctx", (u.ctx_len, u.ctx_dim)).float().bfloat16().to(dev)
    tcond = (synth.normal(10 ** 6, "unet_full_cond", (u.temb_dim,)) * 0.1).float().to(dev)
    t0 = time.time()
    cache = ig.ig_unet_template(h, tl.data_ptr(), tctx.data_ptr(), tcond.data_ptr(), sig,
                                ig.IG_CACHE_DEVICE if args.tier == "device" else ig.IG_CACHE_HOST, stream.cuda_stream)
    t_tpl = time.time() - t0
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1400.0
    g = u.grid
    res = []
    ctxs = [synth.normal(r, "unet_full_ctx", (u.ctx_len, u.ctx_dim)).float().bfloat16().to(dev) for r in range(args.batch)]
    conds = [(synth.normal(r, "unet_full_cond", (u.temb_dim,)) * 0.1).float().to(dev) for r in range(args.batch)]
    for m in [float(x) for x in args.ms.split(",")]:
        lats, masks, mh = [], [], []
        for r in range(args.batch):
            rng = np.random.default_rng(1000 * r + int(m * 1000))
            n = int(round(m * g * g))
            d2 = synth.ModelDesc("g", 0, 1, 64, 1, 64, 64, 4, g, g, 0)
            mk = synth.rect_mask_count(d2, n, rng) if r % 2 == 0 else synth.blob_mask_count(d2, n, rng)
            masks.append(mk)
            mh.append(ig.ig_unet_mask_build(h, mk, stream.cuda_stream)[0])
            lats.append(synth.make_unet_latent(u, r).to(dev))
        reqs = lambda t: [ig.make_unet_req(lats[r].data_ptr(), mh[r], cache, (r + t) % N_SCHED, float(sig[(r + t) % N_SCHED]),
                                           float(sig[(r + t) % N_SCHED + 1]), ctxs[r].data_ptr(), conds[r].data_ptr())
                          for r in range(args.batch)]
        for t in range(args.warmup):
            ig.ig_unet_step(h, reqs(t), stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        if args.profile:
            torch.cuda.profiler.start()
        e0.record(stream)
        for t in range(args.steps):
            ig.ig_unet_step(h, reqs(t), stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        if args.profile:
            torch.cuda.profiler.stop()
        ms = e0.elapsed_time(e1) / args.steps
        st = ig.ig_unet_last_stats(h)
        fl = sum(flops(u, mk) for mk in masks)
        res.append({"m": m, "ms_per_step": round(ms, 3), "tflops_alg": round(fl / (ms * 1e-3) / 1e12, 1),
                    "frac_of_sustained": round(fl / (ms * 1e-3) / 1e12 / pk, 4),
                    "launches": st["kernel_launches"], "h2d_GB": round(st["h2d_bytes"] / 1e9, 3)})
        print(json.dumps(res[-1]), flush=True)
        for x in mh:
            ig.ig_unet_mask_free(x)
    dense = [r for r in res if r["m"] == 1.0]
    if dense:
        for r in res:
            r["speedup_vs_dense"] = round(dense[0]["ms_per_step"] / r["ms_per_step"], 3)
    out = {"model": u.name, "grid": u.grid, "batch": args.batch, "tier": args.tier, "depth": args.depth,
           "template_s": round(t_tpl, 1),
           "note": "whole SDXL-shaped UNet at 1024^2 (latent 128x128x4): Transformer2Ds mask-aware on the "
                   "level's masked tokens (K/V + output caches), ResBlocks / resamplers / convs dense; "
                   "requests at distinct steps of one template; m=1.0 is the dense step", "sweep": res}
    print(json.dumps(out))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    ig.ig_unet_cache_free(cache)
    ig.ig_unet_destroy(h)


if __name__ == "__main__":
    main()
