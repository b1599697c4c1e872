"""sparse_cnot n=1000 sampling time and plan under planner switches (one
setting per process: python tools/dbg/fig3a_probe.py [ENV=VAL ...])."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    os.environ[k] = v
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits, run_initialization  # noqa: E402

init = run_initialization(circuits.bench_family("a", 1000, 0))
s = Sampler(init)
s.sample(4096, 0)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    s.sample(1_000_000, 0)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(sys.argv[1:], "nnz", init.nnz, "n_sym", init.n_sym, "ms", [round(t * 1e3, 2) for t in ts],
      s.plan_info(), flush=True)
