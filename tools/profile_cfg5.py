"""One launch of the cfg5 dense-M_sym kernels for ncu: K5 (sp_sample at
density 0.5, p given) or the Four-Russians K2 (explicit uniform S).

    ncu ... python tools/profile_cfg5.py --what k5 --p 1e-3
    ncu ... python tools/profile_cfg5.py --what m4rm --log2n 16
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits as CI  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", choices=["k5", "m4rm"], default="k5")
    ap.add_argument("--dens", type=float, default=0.5)
    ap.add_argument("--p", type=float, default=1e-3)
    ap.add_argument("--log2n", type=int, default=20)
    a = ap.parse_args()
    m, v, n = 10**4, 10**5, 1 << a.log2n
    model = CI.random_msym_model(m, v, a.dens, a.p, seed=7)
    s = Sampler(model)
    out = s.empty_bits(m, n)
    if a.what == "k5":
        assert s.plan_info()["fused_ok"] == 2
        for i in range(2):
            s.sample(n, 7 + i, out=out)
    else:
        g = torch.Generator(device="cuda").manual_seed(42)
        S = torch.randint(-(2**63), 2**63 - 1, (v + 1, n // 64), dtype=torch.int64, device="cuda",
                          generator=g)
        s.set_product("dense")
        for _ in range(2):
            s.sample_given(S, n, out=out)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
