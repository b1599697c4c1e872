"""Breaks the e2e step into its parts: plan build (load), sample_to_host, raw
D2H bandwidth to pinned memory. Usage: python tools/e2e_probe.py [cfg]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits, run_initialization  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
init = run_initialization(circuits.CONFIGS[cfg]["text"]())
n = circuits.CONFIGS[cfg]["shots"] if cfg != "cfg3" else 10**7
s = Sampler(init)
T = s.shot_tile
n = (n + T - 1) // T * T
host = torch.empty(s.encoded_size(n, "b8"), dtype=torch.uint8, pin_memory=True)
dev = torch.empty_like(host, device="cuda")
for _ in range(2):
    s.sample_to_host(n, 1, "b8", out=host)
torch.cuda.synchronize()


def tm(f, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


print(f"{cfg}: shots {n}, bytes {host.numel()/1e6:.1f} MB")
print(f"  d2h copy (torch, pinned)      {tm(lambda: host.copy_(dev, non_blocking=True)):.3f} ms")
print(f"  sample_to_host                {tm(lambda: s.sample_to_host(n, 2, 'b8', out=host)):.3f} ms")
print(f"  load (host copy of model)     {tm(lambda: s.load(init)):.3f} ms")
print(f"  load + shot_tile (plan build) {tm(lambda: (s.load(init), s.shot_tile)):.3f} ms")
print(f"  load + sample_to_host         {tm(lambda: (s.load(init), s.sample_to_host(n, 3, 'b8', out=host))):.3f} ms")
out = s.empty_bits(init.n_meas, n)
print(f"  sample (device only)          {tm(lambda: s.sample(n, 4, out=out)):.3f} ms")
