import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_20600_b200 import ig
M, N, K = 14720, 3072, int(sys.argv[1]) if len(sys.argv) > 1 else 3072
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) / K ** 0.5
X = torch.zeros(M, N, device="cuda", dtype=torch.float32)
gate = torch.rand(N, device="cuda", dtype=torch.float32)
for _ in range(3):
    ig.ig_op_gemm_gated(ig.IG_BF16, A.data_ptr(), K, B.data_ptr(), K, 0, X.data_ptr(), N, gate.data_ptr(), M, N, K, 0)
torch.cuda.synchronize()
