import os, sys, ctypes
ctypes.CDLL(os.path.join(os.path.dirname(__file__), "segv_bt.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2311_03906_b200 import Sampler, run_initialization
p = float(sys.argv[1])
n_q, shots = 100, 1_000_000
text = f"X_ERROR({p!r}) " + " ".join(map(str, range(n_q))) + "\nM " + " ".join(map(str, range(n_q))) + "\n"
init = run_initialization(text)
s = Sampler(init, device=0)
print("plan", s.plan_info(), flush=True)
counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
s.sample(shots, 3, counts=counts)
print("total", int(counts.sum().item()), flush=True)
