"""Times sp_sample on a cfg5 model (random M_sym 10^4 x 10^5, Bernoulli(p)),
N = 2^20 shots: prints the sampler the planner picked and ms (CUDA events,
L2 flushed between launches)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits as CI  # noqa: E402

dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
p = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
n = 1 << 20
model = CI.random_msym_model(10**4, 10**5, dens, p, seed=7)
s = Sampler(model)
out = s.empty_bits(model.n_meas, n)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s.sample(n, 1, out=out)
ts = []
for i in range(5):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.sample(n, 10 + i, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(json.dumps({"dens": dens, "p": p, "sampler": s.plan_info()["fused_ok"], "ms": ts[len(ts) // 2]}))
