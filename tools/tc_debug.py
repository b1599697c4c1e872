import sys, numpy as np
sys.path.insert(0,'/root/repo')
import torch, oracle
from paper_2311_03906_b200 import circuits as CI, Sampler
from paper_2311_03906_b200.sampler import pack_bits
port=oracle.Port()
for (m,v,n) in [(128,256,256),(256,128,256),(128,128,512),(129,131,257),(128,131,256),(128,128,257)]:
    model=CI.random_msym_model(m,v,0.5,1e-3,seed=m+v)
    rng=np.random.default_rng(n)
    S=pack_bits(rng.integers(0,2,size=(model.n_sym,n),dtype=np.uint8))
    want=port.sample(model.row_ptr,model.sym_idx,S,n)
    s=Sampler(None,device=0); s.load_csr(model.row_ptr,model.sym_idx,model.n_sym); s.set_product("tensor")
    got=s.sample_given(torch.from_numpy(S.view(np.int64)).cuda(),n).cpu().numpy().view(np.uint64)
    d=np.argwhere(got!=want)
    print((m,v,n), "n_sym", model.n_sym, "bad words", len(d), d[:8].tolist())
