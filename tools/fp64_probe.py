"""FP64 fused V-ABFT GEMM (SIMT DFMA) throughput vs the plain kernel and cuBLAS
(DMMA) at 2048-8192^3; the overhead of the A-side pass + verify tail."""
import torch, time, json, sys
sys.path.insert(0, '.')
from paper_2602_08043_b200.fused import plain_gemm, FusedAbftGemm
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)/it
for n in (2048, 4096, 8192):
    a=torch.randn(n,n,device='cuda',dtype=torch.float64); b=torch.randn(n,n,device='cuda',dtype=torch.float64)
    fl=2*n**3
    tp=t(lambda: plain_gemm(a,b)); tt=t(lambda: a@b)
    g=FusedAbftGemm(b, mode="online")
    tf=t(lambda: g(a))
    print(json.dumps({"n":n,"dfma_plain_tf":fl/tp/1e9,"cublas_tf":fl/tt/1e9,"fused_tf":fl/tf/1e9,"overhead_pct":100*(tf/tp-1)}))
