"""cfg5 sweep (BASELINE.json configs[4]): random M_sym 10^4 x 10^5 at
densities {0.001, 0.01, 0.5}, fault rates {1e-4, 1e-3, 1e-2}, N = 2^20.

Per density:
  * explicit-S product (K2) on a supplied seeded S [v+1][2^20/64]: CSR vs
    dense variants, bits/s and the HBM roofline (S + M_sym + output bytes);
  * per rate (dens < 0.5): the fused sampler (K1, single- or double-buffered
    tile) and the unfused path (draw S on device, then K2).
One JSON line per measurement on stdout. Usage:
    python tools/cfg5_sweep.py [--m 10000] [--v 100000] [--log2n 20] [--dens ...]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2311_03906_b200 import Sampler, circuits as CI  # noqa: E402


def peak_gbs():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 8000.0


def timeit(fn, reps=3):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])  # first is warm-up


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=10**4)
    ap.add_argument("--v", type=int, default=10**5)
    ap.add_argument("--log2n", type=int, default=20)
    ap.add_argument("--dens", type=float, nargs="*", default=list(CI.CFG5_DENSITIES))
    ap.add_argument("--rates", type=float, nargs="*", default=list(CI.CFG5_RATES))
    a = ap.parse_args()
    n = 1 << a.log2n
    peak = peak_gbs()
    g = torch.Generator(device="cuda").manual_seed(42)
    S = torch.randint(-(2**63), 2**63 - 1, (a.v + 1, n // 64), dtype=torch.int64, device="cuda",
                      generator=g)
    out_bytes = a.m * n // 8
    for dens in a.dens:
        t0 = time.perf_counter()
        model = CI.random_msym_model(a.m, a.v, dens, 1e-3, seed=7)
        gen_s = time.perf_counter() - t0
        s = Sampler()
        s.load_csr(model.row_ptr, model.sym_idx, model.n_sym)
        out = s.empty_bits(a.m, n)
        base = {"config": "cfg5", "m": a.m, "v": a.v, "n_shots": n, "dens": dens,
                "nnz": model.nnz, "gen_seconds": round(gen_s, 2)}
        for variant in ("sparse", "dense"):
            s.set_product(variant)
            ms = timeit(lambda: s.sample_given(S, n, out=out))
            m_bytes = (4 * model.nnz + 8 * (a.v + 2)) if variant == "sparse" else \
                a.m * ((a.v + 64) // 64) * 8
            alg = out_bytes + S.numel() * 8 + m_bytes
            print(json.dumps({**base, "path": f"explicit-S K2 {variant}", "ms": ms,
                              "bits_per_s": a.m * n / (ms / 1e3),
                              "alg_bytes": alg, "GBps": alg / (ms / 1e3) / 1e9,
                              "roofline_frac": alg / (ms / 1e3) / 1e9 / peak}), flush=True)
        for p in a.rates:
            s.load_groups(CI.bernoulli_groups(a.v, p))
            info = s.plan_info()
            rec = {**base, "p": p, "plan": info}
            if info["fused_ok"]:
                ms = timeit(lambda: s.sample(n, 7, out=out))
                print(json.dumps({**rec, "path": "fused K1", "ms": ms,
                                  "bits_per_s": a.m * n / (ms / 1e3),
                                  "GBps": out_bytes / (ms / 1e3) / 1e9,
                                  "roofline_frac": out_bytes / (ms / 1e3) / 1e9 / peak}), flush=True)
            s.set_product("auto")  # CSR walk, or Four-Russians above density ~0.17
            ms = timeit(lambda: (s.draw_assignments(n, 7, out=S), s.sample_given(S, n, out=out)))
            print(json.dumps({**rec, "path": "draw + K2 auto", "ms": ms,
                              "bits_per_s": a.m * n / (ms / 1e3)}), flush=True)
            ms = timeit(lambda: s.sample(n, 7, out=out))  # what sp_sample picks
            print(json.dumps({**rec, "path": "sp_sample", "ms": ms,
                              "bits_per_s": a.m * n / (ms / 1e3)}), flush=True)
        del s, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
