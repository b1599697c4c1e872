import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2311_03906_b200 import Sampler, circuits, run_initialization
init = run_initialization(circuits.CONFIGS["cfg3"]["text"]())
s = Sampler(init)
T = s.shot_tile
n = (10_000_000 + T - 1) // T * T
mm = s.empty_bits(init.n_meas, n)
til = torch.empty(s.tiled_words(n), dtype=torch.int64, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)
print("mm", t(lambda: s.sample(n, 1, out=mm)))
print("tiled", t(lambda: s.sample_tiled(n, 1, out=til)))
print("untile", t(lambda: s.untile(til, n, out=mm)))
s.sample_tiled(n, 1, out=til); ref = s.sample(n, 1, out=torch.empty_like(mm)); s.untile(til, n, out=mm)
print("equal", torch.equal(ref, mm))
