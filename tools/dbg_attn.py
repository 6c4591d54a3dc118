import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
from paper_2505_20600_b200 import ig
heads, dh, L = int(os.environ.get("HEADS", "2")), 128, int(sys.argv[1]) if len(sys.argv) > 1 else 128
qlens = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [128]
H = heads * dh
M = sum(qlens)
Q = synth.normal(5, "Q", (M, H), "cuda").float().bfloat16()
kv = synth.normal(6, "KV", (len(qlens), 2, L, H), "cuda").float().bfloat16()
O = torch.zeros((M, H), dtype=torch.bfloat16, device="cuda")
segs, s = [], 0
for i, q in enumerate(qlens):
    segs.append((s, q, i)); s += q
ig.ig_op_attention(ig.IG_BF16, Q.data_ptr(), H, O.data_ptr(), H, kv.data_ptr(), segs, L, heads, dh, 0)
torch.cuda.synchronize()
Qh, KVh, Oh = Q.double().cpu().numpy(), kv.double().cpu().numpy(), O.double().cpu().numpy()
if os.environ.get("NOCHECK"):
    sys.exit(0)
for (q0, ql, i) in segs:
    ref = oracle.attention(Qh[q0:q0 + ql], KVh[i, 0], KVh[i, 1], heads)
    err = np.abs(Oh[q0:q0+ql] - ref)
    print("seg", i, "max err", err.max(), "ref rms", np.sqrt((ref**2).mean()), "row0", Oh[q0,:4], ref[0,:4])
