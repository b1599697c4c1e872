"""Small driver for ncu captures: one warm-up launch, then one profiled launch
of the chosen kernel path on one workload.

    python tools/profile_kernel.py --config cfg2 --what sample
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits, run_initialization  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--what", default="sample", choices=["sample", "counts", "draw", "given",
                                                         "encode", "compat"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tiled", action="store_true", help="tiled record layout (sample/counts)")
    a = ap.parse_args()
    init = run_initialization(circuits.CONFIGS[a.config]["text"]())
    n = a.shots or circuits.CONFIGS[a.config]["shots"]
    s = Sampler(init, rng="compat" if a.what == "compat" else "philox")
    T = s.shot_tile
    n = (n + T - 1) // T * T
    out = (torch.empty(s.tiled_words(n), dtype=torch.int64, device="cuda") if a.tiled
           else s.empty_bits(init.n_meas, n))
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda")
    S = s.draw_assignments(n, 1) if a.what == "given" else None
    for i in range(a.reps):
        if a.what in ("sample", "compat"):
            (s.sample_tiled if a.tiled else s.sample)(n, 10 + i, out=out)
        elif a.what == "counts":
            (s.sample_tiled if a.tiled else s.sample)(n, 10 + i, out=out, counts=counts)
        elif a.what == "draw":
            s.draw_assignments(n, 10 + i)
        elif a.what == "given":
            s.sample_given(S, n, out=out)
        elif a.what == "encode":
            s.encode(out, n, "b8")
    torch.cuda.synchronize()
    print(f"ok {a.config} {a.what} n={n} T={T} launches={s.launches}")


if __name__ == "__main__":
    main()
