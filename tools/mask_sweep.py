"""Mask-ratio sweep (the shape of the paper's fig:micro_kernel_image; SURVEY §8(d)
config 5's sweep applied to the Flux shape): batch-step time and images/s of the mask-aware
step at fixed mask ratios m (every request of the batch at n_m = round(m L_img)) against the
dense step, with the K/V cache resident in HBM (compute only) and, optionally, streamed from
host memory.  Also prints the Table 1 prediction (time ~ F(m) / F(1)).

    python tools/mask_sweep.py [--ratios 0.01,0.05,...] [--host]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2505_20600_b200 import ig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ratios", default="0.01,0.05,0.1,0.2,0.3,0.4,0.6,0.8,1.0")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-batch", type=int, default=8)
    ap.add_argument("--host", action="store_true", help="also stream the cache from pinned host memory")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    ig.lib()
    d = synth.FLUX
    W, ptrs = bench.build_model(d, dev)
    opts = ig.ig_ctx_opts(args.max_batch, args.max_batch * d.L, 8, 1, 0, 0)
    ctx = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, 0, opts)
    sig = synth.flow_sigmas(bench.N_STEPS)
    tl = synth.make_latent(d, 10 ** 6, dev)
    tt = synth.make_txt(d, 10 ** 6, dev, torch.bfloat16)
    tc = synth.make_cond(d, 10 ** 6, dev)
    tiers = [("hbm", ig.IG_CACHE_DEVICE)] + ([("host", ig.IG_CACHE_HOST)] if args.host else [])
    stream = torch.cuda.Stream(device=dev)
    out = {"model": d.name, "batch": args.max_batch, "points": []}
    pool = args.max_batch + 4
    for tname, tier in tiers:
        cache = ig.ig_cache_template(ctx, tl.data_ptr(), tt.data_ptr(), tc.data_ptr(), sig, tier, 0)
        for m in [float(x) for x in args.ratios.split(",")]:
            bench.MASKS.update(lo=m, hi=m, kind="mixed")
            dense = m >= 1.0
            bt = bench.Batch(ig, ctx, d, dev, args.max_batch, pool, rid0=7000, stream=stream, dense=dense)
            bench.run_loop(ig, ctx, bt, None if dense else cache, sig, args.warmup, stream)
            lg = bench.run_loop(ig, ctx, bt, None if dense else cache, sig, args.steps, stream, profile=True)
            ms = lg.ms / args.steps
            f = sum(bench.request_step_flops(d, r.n_m) for r in bt.slots) / len(bt.slots)
            out["points"].append({"tier": tname, "m": m, "ms_per_batch_step": round(ms, 3),
                                  "images_per_s": round(lg.rsteps / bench.N_STEPS / (lg.ms / 1e3), 4),
                                  "alg_tflop_per_request_step": round(f / 1e12, 3),
                                  "host_link_GBps": round(lg.h2d / (lg.ms * 1e-3) / 1e9, 2),
                                  "gemm_tflops": round(lg.tflops("gemm"), 1), "attn_tflops": round(lg.tflops("attn"), 1)})
            torch.cuda.synchronize()
            bt.close()
            print(json.dumps(out["points"][-1]), flush=True)
            if dense:
                break
        ig.ig_cache_free(cache)
    dense_ms = [p["ms_per_batch_step"] for p in out["points"] if p["m"] >= 1.0]
    if dense_ms:
        for p in out["points"]:
            p["speedup_vs_dense"] = round(dense_ms[0] / p["ms_per_batch_step"], 3)
            p["table1_speedup"] = round(bench.request_step_flops(d, d.L_img) / 1e12 / p["alg_tflop_per_request_step"], 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
