"""Times the dense explicit-S product variants at the cfg5 shape (m = 10^4,
v = 10^5, N shots): Four-Russians (dense) vs the tensor-core GEMM (tensor),
and checks they agree. Prints JSON lines."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler  # noqa: E402
from paper_2311_03906_b200 import circuits as CI  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
m = int(sys.argv[3]) if len(sys.argv) > 3 else 10**4
v = int(sys.argv[4]) if len(sys.argv) > 4 else 10**5
model = CI.random_msym_model(m, v, dens, 1e-3, seed=7)
g = torch.Generator(device="cuda").manual_seed(42)
S = torch.randint(-(2**63), 2**63 - 1, (model.n_sym, n // 64), dtype=torch.int64, device="cuda",
                  generator=g)
s = Sampler(None, device=0)
s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
outs = {}
for variant in ("tensor", "dense"):
    s.set_product(variant)
    out = s.sample_given(S, n)  # warm-up (+ operand layout for tensor)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.sample_given(S, n, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    outs[variant] = out
    ops = 2.0 * model.n_meas * model.n_sym * n
    print(json.dumps({"variant": variant, "m": m, "v": v, "n_shots": n, "density": dens, "ms": min(ts),
                      "int8_tops": ops / (min(ts) / 1e3) / 1e12}), flush=True)
print(json.dumps({"equal": bool(torch.equal(outs["tensor"], outs["dense"]))}))
