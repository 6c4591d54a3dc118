"""Config 5 (BASELINE.json): mask-ratio sweep of the mask-aware step on the
SDXL-UNet attention stack vs the dense step, on one B200.

Both attention levels of SDXL at 1024²: the 64x64 level (10 BasicTransformerBlocks, C=640,
10 heads) and the 32x32 level (60 blocks, C=1280, 20 heads), d = 64, cross-attention to a
77 x 2048 context, GEGLU FF; bf16; random-init weights, synthetic K/V caches.  A batch of
--batch requests, each with a 64-level mask of n = round(m * 4096) tokens (even ids
rectangles, odd blobs) and its 32-level mask by 2x2 any-pool (paper_2505_20600_b200.levels).
One "step" = one ig_edit_step on each level's context (the dense ResBlocks between them are
outside this path, C-AMB 31).  The cache holds --cache-steps (default 8) distinct steps, and
the batch's requests sit at staggered steps of it (no two on one step: no load deduplication,
as under continuous batching; ~0.4 GB of K/V per request-step across both levels, far larger
than L2), in HBM (--tier device, default, replayed as CUDA graphs) or pinned host memory
(--tier host); --cache kv | y | fp8 | fp8y picks the cache form.

    python tools/unet_sweep.py [--ratios 0.01,0.02,...] [--tier device|host] [--batch 8]

Prints one JSON line per (m) and a summary line; FLOPs are the algorithmic per-row counts of
DESIGN.md §6 (UNet rows).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_20600_b200 import ig, levels  # noqa: E402

RATIOS = "0.01,0.02,0.05,0.1,0.2,0.3,0.4,0.5,0.6,0.8,1.0"


def step_flops(d, n_rows, n_req):
    """Algorithmic FLOPs of one step of level d over n_rows masked rows of n_req requests."""
    H, F, L, Lc, Dc = d.hidden, d.mlp_hidden, d.L_img, d.ctx_len, d.ctx_dim
    per_row = 2 * (6 * H * H + 3 * F * H) + 4 * L * H + 4 * Lc * H
    per_req = 2 * Lc * 2 * H * Dc
    return d.n_unet * (n_rows * per_row + n_req * per_req)


class Level:
    def __init__(self, d, batch, tier, cache_steps, dev, graphs=0, y=0, kv_blocks=0, fp8=0):
        self.d = d
        self.W = []
        ptrs = []
        for name, shape, fan_in in synth.weight_table(d):
            t = synth.make_weight(d, name, shape, fan_in, 0, dev, torch.bfloat16).contiguous()
            self.W.append(t)
            ptrs.append(t.data_ptr())
        opts = ig.ig_ctx_opts(batch, 0, 4, 1, 0, fp8, y, kv_blocks, graphs)
        self.ctx = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, 0, opts)
        self.cache_steps = cache_steps
        if fp8:  # quantized on the device by ig_cache_write (per (token, head) scales)
            self.cache = ig.ig_cache_create(self.ctx, cache_steps, ig.IG_CACHE_HOST)
            ym = set(ig.y_block_modes(d.n_blocks, kv_blocks)) if y else set()
            planes = sum((0 if b in ym else 2) + (1 if (b in ym or (b + 1) in ym) else 0) for b in range(d.n_blocks))
            kv = torch.empty((cache_steps, planes, d.L_img, d.hidden), dtype=torch.bfloat16, device=dev)
            for s in range(cache_steps):
                kv[s] = synth.normal(7000 + s, "cache_planes", tuple(kv.shape[1:]), dev).to(torch.bfloat16)
            lat = synth.normal(7100, "cache_states", (cache_steps, d.L_img * d.hidden), dev).float()
            ig.ig_cache_write(self.ctx, self.cache, kv.data_ptr(), lat.data_ptr())
            del kv
            if tier == ig.IG_CACHE_DEVICE:
                dc = ig.ig_cache_clone(self.ctx, self.cache, tier)
                ig.ig_cache_free(self.cache)
                self.cache = dc
            self._inputs(batch, dev)
            return
        self.cache = ig.ig_cache_create(self.ctx, cache_steps, tier)
        ym = set(ig.y_block_modes(d.n_blocks, kv_blocks)) if y else set()
        planes = sum((0 if b in ym else 2) + (1 if (b in ym or (b + 1) in ym) else 0) for b in range(d.n_blocks))
        ptr, nbytes, t = ig.ig_cache_storage(self.cache)
        plane = d.L_img * d.hidden
        for s in range(cache_steps):  # fill step by step (bounded staging memory)
            pl = synth.normal(7000 + s, "cache_planes", (planes, plane), dev).to(torch.bfloat16)
            ig.ig_copy(ptr + s * planes * plane * 2, pl.data_ptr(), planes * plane * 2)
            torch.cuda.synchronize()
        lat = synth.normal(7100, "cache_states", (cache_steps, plane), dev).float()  # template input states
        ig.ig_copy(ptr + cache_steps * planes * plane * 2, lat.data_ptr(), lat.numel() * 4)
        torch.cuda.synchronize()
        torch.cuda.synchronize()
        self._inputs(batch, dev)

    def _inputs(self, batch, dev):
        d = self.d
        self.state = [synth.make_latent(d, 100 + i, dev).contiguous() for i in range(batch)]
        self.ctxemb = [synth.make_ctx(d, 100 + i, dev, torch.bfloat16).contiguous() for i in range(batch)]
        self.masks = []

    def set_masks(self, masks_np, dev):
        for mk, mdev in self.masks:
            ig.ig_mask_free(mk)
        self.masks = []
        for m in masks_np:
            mdev = torch.from_numpy(m.astype(np.uint8)).to(dev)
            h, n = ig.ig_mask_build(self.ctx, mdev.data_ptr(), 0)
            self.masks.append((h, mdev))
        self.n_rows = int(sum(int(m.astype(bool).sum()) for m in masks_np))

    def step(self, s, stream):
        # requests at staggered schedule positions (no two on one cache step when cache_steps >=
        # batch: no load deduplication, as under continuous batching)
        rr = [ig.make_req(i, self.state[i].data_ptr(), self.masks[i][0], self.cache, (s + i) % self.cache_steps,
                          0.0, 0.0, self.ctxemb[i].data_ptr(), None) for i in range(len(self.state))]
        ig.ig_edit_step(self.ctx, rr, stream)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratios", default=RATIOS)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=6)  # > NSTAGE: every staging slot's graph captured
    ap.add_argument("--tier", default="device", choices=["device", "host"])
    ap.add_argument("--cache-steps", type=int, default=8)
    ap.add_argument("--cache", default="kv", choices=["kv", "y", "fp8", "fp8y"],
                    help="K/V, Y (the paper's SDXL form), FP8 K/V or FP8 Y cache")
    ap.add_argument("--graphs", type=int, default=-1,
                    help="CUDA graphs of whole steps (default: on for the HBM tier; host-tier DMA sources change per step)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ig.lib()
    tier = ig.IG_CACHE_DEVICE if args.tier == "device" else ig.IG_CACHE_HOST
    graphs = (1 if args.tier == "device" else 0) if args.graphs < 0 else args.graphs
    yc = 1 if args.cache in ("y", "fp8y") else 0
    f8 = 1 if args.cache in ("fp8", "fp8y") else 0
    lv = [Level(synth.SDXL_L64, args.batch, tier, args.cache_steps, dev, graphs, yc, 0, f8),
          Level(synth.SDXL_L32, args.batch, tier, args.cache_steps, dev, graphs, yc, 0, f8)]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1384.7
    stream = torch.cuda.Stream(device=dev)
    pts = []
    d64 = synth.SDXL_L64
    for m in [float(x) for x in args.ratios.split(",")]:
        n = int(round(m * d64.L_img))
        m64 = []
        for i in range(args.batch):
            rng = np.random.default_rng(4242 + 17 * i)
            m64.append(synth.rect_mask_count(d64, n, rng) if i % 2 == 0 else synth.blob_mask_count(d64, n, rng))
        m32 = [levels.any_pool2(x, 64, 64) for x in m64]
        lv[0].set_masks(m64, dev)
        lv[1].set_masks(m32, dev)
        res = {"m": m}
        tot_ms, tot_f = 0.0, 0.0
        for L, name in zip(lv, ("l64", "l32")):
            with torch.cuda.stream(stream):
                for s in range(args.warmup):
                    L.step(s, stream.cuda_stream)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for s in range(args.steps):
                    L.step(s, stream.cuda_stream)
                b.record(stream)
                torch.cuda.synchronize()
                ig.ig_profile_enable(L.ctx, 1)  # per-class kernel times: separate eager pass
                for s in range(2):
                    L.step(s, stream.cuda_stream)
            torch.cuda.synchronize()
            prof = ig.ig_profile_read(L.ctx)
            ig.ig_profile_enable(L.ctx, 0)
            ms = a.elapsed_time(b) / args.steps
            f = step_flops(L.d, L.n_rows, args.batch)
            g, at = prof["gemm"], prof["attn"]
            res[name] = {"ms_per_step": round(ms, 3), "rows": L.n_rows, "alg_tflops": round(f / ms / 1e9, 1),
                         "gemm_tflops": round(g["flops"] / g["ms"] / 1e9, 1) if g["ms"] else None,
                         "attn_tflops": round(at["flops"] / at["ms"] / 1e9, 1) if at["ms"] else None}
            tot_ms += ms
            tot_f += f
        res["ms_per_step"] = round(tot_ms, 3)
        res["frac_of_sustained"] = round(tot_f / tot_ms / 1e9 / peak, 4)
        pts.append(res)
        print(json.dumps(res), flush=True)
    dense = [p["ms_per_step"] for p in pts if p["m"] >= 1.0]
    if dense:
        for p in pts:
            p["speedup_vs_dense"] = round(dense[0] / p["ms_per_step"], 3)
            f_m = sum(step_flops(L.d, r, args.batch) for L, r in zip(lv, (p["l64"]["rows"], p["l32"]["rows"])))
            f_1 = sum(step_flops(L.d, args.batch * L.d.L_img, args.batch) for L in lv)
            p["flop_ratio_dense_over_masked"] = round(f_1 / f_m, 3)
    print(json.dumps({"config": "sdxl_unet_attention_stack", "batch": args.batch, "tier": args.tier, "graphs": graphs,
                      "cache": args.cache,
                      "cache_steps": args.cache_steps, "points": pts}))


if __name__ == "__main__":
    main()
