"""Open-loop serving run (BASELINE config 4): Poisson arrivals with per-request
masks m ~ U[0.05, 0.60] (or a skewed preset) on the Flux-shaped model, step-level continuous
(or static) batching on every GPU, requests routed across GPUs by Algorithm 2 (or a
baseline policy).  Prints one JSON line: throughput, mean / P95 latency and queueing time
(nearest rank), next to the latency model's own prediction for the same trace.

    python tools/serve_bench.py [--load 0.7] [--requests 48] [--policy mask_aware]
                                [--batching continuous|static] [--skew public|own]
    torchrun --nproc-per-node N tools/serve_bench.py ...   (one worker process per GPU)
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

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2505_20600_b200 import ig  # noqa: E402
from paper_2505_20600_b200 import serve as S  # noqa: E402
from paper_2505_20600_b200.placement import LatencyModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--load", type=float, default=0.7, help="offered load / predicted capacity")
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--policy", default="mask_aware", choices=list(S.POLICIES))
    ap.add_argument("--batching", default="continuous", choices=["continuous", "static"])
    ap.add_argument("--skew", default=None, choices=[None, "public", "own"])
    ap.add_argument("--max-batch", type=int, default=8)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--tier", default=None, choices=["host", "device"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cache", default="hybrid", choices=["kv", "hybrid"])
    ap.add_argument("--simulate-gpus", type=int, default=0,
                    help="also print the latency model's prediction of every policy on this many GPUs")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control plane only (dispatch + metrics)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ig.lib()
    d = synth.FLUX
    tier = args.tier or ("host" if world == 1 else "device")
    link = bench.measure_h2d(dev)
    W, ptrs = bench.build_model(d, dev)
    opts = ig.ig_ctx_opts(max(args.max_batch, 4), max(args.max_batch, 4) * d.L, args.depth, 1, 0, 0)
    ctx_kv = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, local, opts)
    sig = synth.flow_sigmas(bench.N_STEPS)
    tl = synth.make_latent(d, 10 ** 6, dev)
    tt = synth.make_txt(d, 10 ** 6, dev, torch.bfloat16)
    tc = synth.make_cond(d, 10 ** 6, dev)
    stream = torch.cuda.Stream(device=dev)
    a_c, b_c, a_l, b_l = bench.fit_latency(ig, ctx_kv, d, dev, stream, link if tier == "host" else 1e6)
    kv_blocks = None
    ctx = ctx_kv
    if args.cache == "hybrid" and tier == "host":  # the bench's hybrid K/V + Y cache (DESIGN reading 30)
        kv_blocks = bench.choose_kv_blocks(d, a_c, b_c, a_l, args.max_batch, 0.325)
        ctx = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, local,
                               ig.ig_ctx_opts(args.max_batch, args.max_batch * d.L, args.depth, 1, 0, 0, 1, kv_blocks))
    cache = ig.ig_cache_template(ctx, tl.data_ptr(), tt.data_ptr(), tc.data_ptr(), sig,
                                 ig.IG_CACHE_HOST if tier == "host" else ig.IG_CACHE_DEVICE, 0)
    y_frac = 0.0 if kv_blocks is None else (d.n_blocks - kv_blocks) / d.n_blocks
    sm = S.StepModel(d, LatencyModel(a_c, b_c, a_l, b_l), y_frac=y_frac)
    # predicted per-GPU capacity at a full batch of the mean mask, and the offered rate
    n_mean = int(round(0.325 * d.L_img)) if args.skew is None else int(round((0.05 + 0.55 * (0.25 if args.skew == "public" else 1 / 9)) * d.L_img))
    cap = args.max_batch / (bench.N_STEPS * sm.step([n_mean] * args.max_batch))
    rate = args.load * cap * world
    trace = S.poisson_trace(rate, args.requests, d.L_img, seed=args.seed, skew=args.skew)
    if world > 1:
        mine = S.dispatch_trace(trace, sm, args.policy, args.max_batch, bench.N_STEPS)
    else:
        mine = trace
    _, pred = S.simulate_cluster(trace, world, args.policy, sm, args.max_batch, bench.N_STEPS, args.batching)

    def make_request(a):
        rng = np.random.default_rng(a.rid)
        mk = synth.rect_mask_count(d, a.n_m, rng) if a.rid % 2 == 0 else synth.blob_mask_count(d, a.n_m, rng)
        md = torch.from_numpy(mk).to(dev)
        mh, _ = ig.ig_mask_build(ctx, md.data_ptr(), 0)
        return {"latent": synth.make_latent(d, a.rid, dev), "txt": synth.make_txt(d, a.rid, dev, torch.bfloat16),
                "cond": synth.make_cond(d, a.rid, dev), "mask": mh, "free": lambda: ig.ig_mask_free(mh)}

    eng = S.Engine(ig, ctx, d, cache, sig, args.max_batch, stream, make_request)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    rec, steps, wall = eng.run(mine, args.batching)
    local_rows = [(rid, r[0], r[1], r[2]) for rid, r in rec.items()]
    rows = local_rows
    if world > 1:
        allr = [None] * world
        torch.distributed.all_gather_object(allr, (local_rows, steps, wall))
        rows = [x for part in allr for x in part[0]]
        steps = sum(p[1] for p in allr)
        wall = max(p[2] for p in allr)
    if rank == 0:
        lat = [r[3] - r[1] for r in rows]
        que = [r[2] - r[1] for r in rows]
        plat = [v[2] - v[0] for v in pred.values()]
        pque = [v[1] - v[0] for v in pred.values()]
        makespan = max(r[3] for r in rows) - min(r[1] for r in rows)
        out = {"metric": "serving latency (Flux-shape 1024^2, Poisson arrivals, mixed masks)", "n_gpus": world,
               "policy": args.policy, "batching": args.batching, "skew": args.skew, "tier": tier,
               "offered_rate_rps": round(rate, 4), "predicted_capacity_per_gpu": round(cap, 4),
               "requests": len(rows), "denoise_steps_run": steps,
               "throughput_images_per_s": round(len(rows) / makespan, 4),
               "measured": S.summarize(lat, que), "predicted_by_latency_model": S.summarize(plat, pque),
               "cache": args.cache if kv_blocks is not None else "kv", "kv_blocks": kv_blocks,
               "latency_model": {"comp_s_per_tflop": a_c * 1e12, "comp_s": b_c, "load_s_per_GB": a_l * 1e9},
               "data": "synthetic", "dtype": "bf16"}
        if args.simulate_gpus:  # the model's view of the routing policies at cluster scale
            big = S.poisson_trace(args.load * cap * args.simulate_gpus, 8 * args.requests, d.L_img,
                                  seed=args.seed + 1, skew=args.skew)
            sim = {}
            for pol in S.POLICIES:
                _, rec_p = S.simulate_cluster(big, args.simulate_gpus, pol, sm, args.max_batch, bench.N_STEPS)
                sim[pol] = S.summarize([v[2] - v[0] for v in rec_p.values()], [v[1] - v[0] for v in rec_p.values()])
            out["simulated_policies"] = {"n_gpus": args.simulate_gpus, "requests": len(big),
                                         "note": "latency-model simulation (not measured)", **sim}
        print(json.dumps(out))
    if world > 1:
        torch.distributed.barrier()


if __name__ == "__main__":
    main()
