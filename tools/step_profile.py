"""One representative Flux batch step for ncu: 8 requests (masks m~U[.05,.6]) against a 2-step
template cache in pinned host memory; the profiled step is wrapped in an NVTX range
'profile_step' (use: ncu --nvtx --nvtx-include 'profile_step/' ...).
Env: COPY_MODE (1), KV_BLOCKS (-1 = K/V cache; else hybrid K/V blocks), PLAN_K (0), DEPTH (8).
(bench.py's IG_BENCH_PROFILE_STEP=1 brackets a steady-state step of the real headline loop instead.)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2505_20600_b200 import ig
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model, Batch
d = synth.FLUX
dev = torch.device("cuda", 0)
W, ptrs = build_model(d, dev)
copy_mode = int(os.environ.get("COPY_MODE", "1"))
kv_blocks = int(os.environ.get("KV_BLOCKS", "-1"))
depth = int(os.environ.get("DEPTH", "8"))
opts = ig.ig_ctx_opts(8, 8 * d.L, depth, copy_mode, 0, 0, 1 if kv_blocks >= 0 else 0, max(kv_blocks, 0))
ctx = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, 0, opts)
if int(os.environ.get("PLAN_K", "0")) > 0:
    ig.ig_set_plan(ctx, 1, int(os.environ["PLAN_K"]))
sig = synth.flow_sigmas(28)
tl = synth.make_latent(d, 10 ** 6, dev); tt = synth.make_txt(d, 10 ** 6, dev, torch.bfloat16); tc = synth.make_cond(d, 10 ** 6, dev)
cache = ig.ig_cache_template(ctx, tl.data_ptr(), tt.data_ptr(), tc.data_ptr(), sig[:3], ig.IG_CACHE_HOST, 0)
stream = torch.cuda.Stream()
b = Batch(ig, ctx, d, dev, 8, 12, 0, stream)
def step():
    reqs = b.reqs(cache, sig)
    for r in reqs:
        r.step = r.step % 2
    ig.ig_edit_step(ctx, reqs, stream.cuda_stream)
    b.advance()
for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profile_step")
step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
