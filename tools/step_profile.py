"""One representative Flux batch step for ncu: 8 requests (masks m~U[.05,.6]) against a 2-step
template cache in pinned host memory; the profiled step is wrapped in an NVTX range
'profile_step' (use: ncu --nvtx --nvtx-include 'profile_step/' ...)."""
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
ctx = ig.ig_ctx_create(ig.make_desc(d, ig.IG_BF16), ptrs, 0, ig.ig_ctx_opts(8, 8 * d.L, 2, copy_mode, 0))
sig = synth.flow_sigmas(28)
tl = synth.make_latent(d, 10 ** 6, dev); tt = synth.make_txt(d, 10 ** 6, dev, torch.bfloat16); tc = synth.make_cond(d, 10 ** 6, dev)
cache = ig.ig_cache_template(ctx, tl.data_ptr(), tt.data_ptr(), tc.data_ptr(), sig[:3], ig.IG_CACHE_HOST, 0)
b = Batch(ig, ctx, d, dev, 8, 12, 0)
stream = torch.cuda.Stream()
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
