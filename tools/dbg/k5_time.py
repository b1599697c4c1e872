import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2311_03906_b200 import Sampler, circuits as CI
n = 1 << 20
for dens, p in [(0.5, 1e-3), (0.5, 1e-2), (0.01, 1e-3)]:
    model = CI.random_msym_model(10**4, 10**5, dens, p, seed=7)
    s = Sampler(model)
    out = s.empty_bits(10**4, n)
    s.sample(n, 1, out=out); torch.cuda.synchronize()
    ts = []
    for i in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); s.sample(n, 2 + i, out=out); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(os.environ.get("SP_LIB", "cur"), dens, p, s.plan_info()["fused_ok"], round(min(ts), 2), flush=True)
    del s, out; torch.cuda.empty_cache()
