import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2602_08043_b200.fused import plain_gemm, FusedAbftGemm
torch.manual_seed(0)
for (m,n,k) in [(128,256,16),(128,256,64),(256,512,256)]:
    a=torch.randn(m,k,device='cuda'); b=torch.randn(k,n,device='cuda')
    ref=(a.double()@b.double())
    c=plain_gemm(a,b); torch.cuda.synchronize()
    print("plain3", m,n,k, c.abs().max().item(), ((c.double()-ref).abs().max()/ref.abs().max()).item())
    for p in (1,3):
        r=FusedAbftGemm(b, tf32_passes=p, e_max=1e-2)(a); torch.cuda.synchronize()
        c=r.C
        print("fused",p, c.abs().max().item(), ((c.double()-ref).abs().max()/ref.abs().max()).item())
        # pattern check: where are the nonzeros / errors
        err=(c.double()-ref).abs()
        bad=(err>1e-2*ref.abs().max())
        if bad.any():
            idx=bad.nonzero()
            print("  bad count", bad.sum().item(), "first", idx[:5].tolist(), "rows bad", bad.any(1).sum().item(), "cols bad", bad.any(0).sum().item())
            print("  c[0,:8]", c[0,:8].tolist()); print("  ref[0,:8]", ref[0,:8].tolist())
