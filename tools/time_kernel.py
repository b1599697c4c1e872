"""Times the fused sampler (CUDA events, L2 flushed between launches) for one
workload; env SP_* overrides select the launch shape. Prints one JSON line."""
import argparse
import json
import os
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--counts", action="store_true")
    ap.add_argument("--tiled", action="store_true", help="tiled record layout")
    ap.add_argument("--dets", action="store_true", help="per-detector counts (surface codes)")
    a = ap.parse_args()
    init = run_initialization(circuits.CONFIGS[a.config]["text"]())
    n = a.shots or circuits.CONFIGS[a.config]["shots"]
    s = Sampler(init)
    T = s.shot_tile
    n = (n + T - 1) // T * T
    out = (torch.empty(int(s._L.sp_tiled_words(s._h, n)), dtype=torch.int64, device="cuda")
           if a.tiled else s.empty_bits(init.n_meas, n))
    run = (lambda seed: s.sample_tiled(n, seed, out=out, counts=counts)) if a.tiled else \
          (lambda seed: s.sample(n, seed, out=out, counts=counts))
    counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda") if a.counts else None
    if a.dets:
        dd = {"cfg2": (5, 5), "cfg3": (15, 15)}[a.config]
        dets, obs = circuits.surface_code_detectors(*dd)
        s.set_detectors(dets + obs)
        dc = torch.zeros(len(dets) + 1, dtype=torch.int64, device="cuda")
        run = lambda seed: s.sample_counted(n, seed, out=out, counts=counts, det_counts=dc,  # noqa: E731
                                            tiled=a.tiled)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(3):
        run(i)
    ts = []
    for i in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(100 + i)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    timers = None
    if os.environ.get("SP_PHASE_TIMERS"):
        import ctypes as C
        buf = (C.c_longlong * 8)()
        s._L.sp_debug_timers(s._h, C.cast(buf, C.c_void_p))
        timers = list(buf)
    ms = ts[len(ts) // 2]
    bytes_ = init.n_meas * n / 8
    env = {k: v for k, v in os.environ.items() if k.startswith("SP_")}
    print(json.dumps({"config": a.config, "tiled": a.tiled, "counts": a.counts, "shots": n, "T": T, "env": env,
                      "ms_median": ms,
                      "ms_min": ts[0], "GBps": bytes_ / ms / 1e6,
                      "bits_per_s": init.n_meas * n / ms * 1e3, "timers": timers,
                      "plan": s.plan_info(),
                      "kernel": s.sampler_kernel(a.tiled, a.dets)}))


if __name__ == "__main__":
    main()
