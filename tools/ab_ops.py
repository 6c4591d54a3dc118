"""Interleaved A/B of libig builds in ONE process (same clocks / power state for every variant):
each variant .so is loaded with ctypes and its ig_op_attention / ig_op_gemm_gated timed in turn,
rounds repeated, median per (variant, shape) printed as JSON.

    python tools/ab_ops.py --libs ablibs/lib_a.so,ablibs/lib_b.so --op attn \
        --shapes "64,20,1024,1024,8;64,10,4096,4096,8" [--rounds 7]
  attn shape = dh,heads,L,qlen,nreq      gated shape = M,N,K
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--op", default="attn", choices=["attn", "gated"])
ap.add_argument("--shapes", required=True)
ap.add_argument("--rounds", type=int, default=7)
ap.add_argument("--calls", type=int, default=20)
args = ap.parse_args()
torch.cuda.set_device(0)
vp, ll, i = ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int
libs = {}
for p in args.libs.split(","):
    L = ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL)
    L.ig_op_attention.argtypes = [i, vp, ll, vp, ll, vp, ctypes.POINTER(ctypes.c_int32), i, i, i, i, vp]
    L.ig_op_gemm_gated.argtypes = [i, vp, ll, vp, ll, vp, vp, ll, vp, i, i, i, vp]
    libs[os.path.basename(p)] = L
REP = 20 if args.op == "attn" else 1  # ig_op_attention repeats the launch REP times per call (one sync)
os.environ["IG_OP_REPEAT"] = str(REP)
IG_BF16 = 1
work = []
for sh in args.shapes.split(";"):
    v = [int(x) for x in sh.split(",")]
    if args.op == "attn":
        dh, heads, L_, q, nreq = v
        H = heads * dh
        M = q * nreq
        Q = torch.randn(M, H, device="cuda", dtype=torch.bfloat16)
        kv = torch.randn(nreq, 2, L_, H, device="cuda", dtype=torch.bfloat16)
        O = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
        flat = []
        for r in range(nreq):
            flat += [r * q, q, r]
        arr = (ctypes.c_int32 * len(flat))(*flat)
        fl = 4.0 * M * L_ * H
        def call(Lb, Q=Q, O=O, kv=kv, arr=arr, H=H, L_=L_, heads=heads, dh=dh, nreq=nreq):
            rc = Lb.ig_op_attention(IG_BF16, Q.data_ptr(), H, O.data_ptr(), H, kv.data_ptr(), arr, nreq, L_, heads, dh, None)
            assert rc == 0
        work.append((sh, call, fl))
    else:
        M, N, K = v
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
        X = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        gate = torch.rand(N, device="cuda", dtype=torch.float32)
        fl = 2.0 * M * N * K
        def call(Lb, A=A, B=B, X=X, gate=gate, M=M, N=N, K=K):
            rc = Lb.ig_op_gemm_gated(IG_BF16, A.data_ptr(), K, B.data_ptr(), K, None, X.data_ptr(), N, gate.data_ptr(), M, N, K, None)
            assert rc == 0
        work.append((sh, call, fl))
# warm the clocks
t0 = time.time()
while time.time() - t0 < 2.0:
    for _, call, _ in work:
        for Lb in libs.values():
            call(Lb)
    torch.cuda.synchronize()
res = {(n, sh): [] for n in libs for sh, _, _ in work}
for _ in range(args.rounds):
    for sh, call, fl in work:
        for n, Lb in libs.items():
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(args.calls):
                call(Lb)
            e1.record()
            torch.cuda.synchronize()
            res[(n, sh)].append(e0.elapsed_time(e1) / args.calls / REP)
out = {}
for (n, sh), v in res.items():
    ms = statistics.median(v)
    fl = next(f for s, _, f in work if s == sh)
    out.setdefault(sh, {})[n] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "min_ms": round(min(v), 4)}
print(json.dumps(out, indent=1))
