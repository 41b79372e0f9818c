import numpy as np, torch, sys
sys.path.insert(0,'.')
import oracle
from paper_2306_08960_b200 import data, _lib, device
orc=oracle.Oracle(); lib=_lib.load()
T=lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()
for (m,n,k,pad) in [(300,385,513,7),(300,385,513,3),(300,385,1024,7),(300,384,513,8),(64,385,256,7),(300,193,513,7)]:
    rng=np.random.default_rng(1)
    a,wpr=data.random_words(rng,m,k); b,_=data.random_words(rng,n,k)
    ldc=n+pad
    bu=torch.full((m+3,ldc),-7,dtype=torch.int32,device='cuda')
    s=torch.cuda.current_stream().cuda_stream
    da,db=T(a),T(b)
    rc=lib.bitmm_gemm_1x1_dev(da.data_ptr(),m,db.data_ptr(),n,k,wpr,1.0,1.0,bu.data_ptr(),None,ldc,s)
    torch.cuda.synchronize()
    g=bu.cpu().numpy()
    bad=np.argwhere(g[:m,n:]!=-7)
    badr=np.argwhere(g[m:]!=-7)
    ok=np.array_equal(g[:m,:n],orc.gemm_1x1(a,b,k,wpr)[0])
    print((m,n,k,pad),"ldc",ldc,"tma" if (ldc*4)%16==0 else "lsu","inside ok",ok,"bad right cols",np.unique(bad[:,1]+n)[:10] if len(bad) else None, "rows",np.unique(bad[:,0])[:5] if len(bad) else None,"bad below",len(badr))
