"""Tail-stage timing vs input distribution (fallback diagnostics)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402
from tools.fused_probe import graph_time  # noqa: E402

m = k = n = 4096
torch.manual_seed(0)
B = torch.randn(k, n, device="cuda").bfloat16()
for name, A in [("randn", torch.randn(m, k, device="cuda").bfloat16()),
                ("uniform12", (torch.rand(m, k, device="cuda") + 1).bfloat16())]:
    g = FusedAbftGemm(B)
    counts = torch.zeros(5, dtype=torch.int64, device="cuda")
    g(A, counts=counts)
    torch.cuda.synchronize()
    print(name, "counts", counts.tolist(), flush=True)
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    t_tail = graph_time(lambda: g(A, out=C, counts=counts, stages=4))
    t_all = graph_time(lambda: g(A, out=C, counts=counts))
    print(f"{name}: tail {t_tail:.1f} us all {t_all:.1f} us", flush=True)
