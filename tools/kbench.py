"""Kernel micro-bench for the two tensor-core kernels at Flux step shapes (through ig_ops)."""
import sys, os, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2505_20600_b200 import ig

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="gemm,attn")
ap.add_argument("--M", type=int, default=14720)
ap.add_argument("--N", type=int, default=3072)
ap.add_argument("--K", type=int, default=3072)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--epi", type=int, default=0, help="0 store, 1 bias+GELU (fc1), 5 GEGLU (N/2 outputs)")
ap.add_argument("--bias", action="store_true")
ap.add_argument("--dh", type=int, default=128, help="attention head dim (64: SD3 / UNet)")
ap.add_argument("--heads", type=int, default=24)
ap.add_argument("--L", type=int, default=4608, help="attention keys per request")
ap.add_argument("--qlens", default="512,1843", help="query segments per request (comma list)")
ap.add_argument("--nreq", type=int, default=8)
args = ap.parse_args()
res = {}
def timeit(fn, iters):
    import time
    t0 = time.time()
    while time.time() - t0 < float(os.environ.get("KB_WARM", "1.0")):  # ramp the SM clock up from idle
        fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
if "gemm" in args.which:
    M, N, K = args.M, args.N, args.K
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.randn(N, device="cuda", dtype=torch.bfloat16)
    bp = bias.data_ptr() if args.bias else 0
    ms = timeit(lambda: ig.ig_op_gemm(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, bp, C.data_ptr(), N, M, N, K, args.epi, 0, 0), args.iters)
    ref = timeit(lambda: torch.matmul(A, B.t(), out=C), args.iters)
    X = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    gate = torch.rand(N, device="cuda", dtype=torch.float32)
    msg = timeit(lambda: ig.ig_op_gemm_gated(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, 0, X.data_ptr(), N, gate.data_ptr(), M, N, K, 0), args.iters)
    res["gemm_gated_tflops"] = 2 * M * N * K / msg / 1e9
    res["gemm"] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9, "cublas_tflops": 2 * M * N * K / ref / 1e9}
if "gated" in args.which:  # out-projection shape: fp32 residual += gate * (A B^T + bias)
    M, N, K = args.M, args.N, args.K
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
    X = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    gate = torch.rand(N, device="cuda", dtype=torch.float32)
    ms = timeit(lambda: ig.ig_op_gemm_gated(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, 0, X.data_ptr(), N,
                                            gate.data_ptr(), M, N, K, 0), args.iters)
    res["gated"] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9}
if "attn" in args.which:
    heads, dh, L = args.heads, args.dh, args.L
    qlens = [int(x) for x in args.qlens.split(",")] * args.nreq
    H = heads * dh
    M = sum(qlens)
    Q = torch.randn(M, H, device="cuda", dtype=torch.bfloat16)
    kv = torch.randn(args.nreq, 2, L, H, device="cuda", dtype=torch.bfloat16)
    O = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    segs, s = [], 0
    per = len(args.qlens.split(","))
    for i, q in enumerate(qlens):
        segs.append((s, q, i // per)); s += q
    rep = int(os.environ.get("IG_OP_REPEAT", "20"))
    os.environ["IG_OP_REPEAT"] = str(rep)
    ms = timeit(lambda: ig.ig_op_attention(ig.IG_BF16, Q.data_ptr(), H, O.data_ptr(), H, kv.data_ptr(), segs, L, heads, dh, 0), args.iters) / rep
    res["attn"] = {"M": M, "ms": ms, "tflops": 4 * M * L * H / ms / 1e9}
print(json.dumps(res))
