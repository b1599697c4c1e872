"""K7 (queued fused sampler) against K1 on one workload: records and counts
must be bit-identical for the same seed (same slices and streams), then both
are timed (CUDA events, L2 flushed). SP_Q_* env set the K7 shape.
Prints one JSON line."""
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
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tiled", action="store_true")
    ap.add_argument("--dets", action="store_true")
    ap.add_argument("--counts", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    a = ap.parse_args()
    init = run_initialization(circuits.CONFIGS[a.config]["text"]())
    n = a.shots or circuits.CONFIGS[a.config]["shots"]
    res = {}
    outs = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, q in (("k1", "0"), ("k7", "1")):
        os.environ["SP_QUEUED"] = q
        s = Sampler(init)
        T = s.shot_tile
        nn = (n + T - 1) // T * T
        out = (torch.zeros(int(s._L.sp_tiled_words(s._h, nn)), dtype=torch.int64, device="cuda")
               if a.tiled else s.empty_bits(init.n_meas, nn))
        counts = torch.zeros(init.n_meas, dtype=torch.int64, device="cuda") if a.counts else None
        dc = None
        if a.dets:
            dd = {"cfg2": (5, 5), "cfg3": (15, 15)}[a.config]
            dets, obs = circuits.surface_code_detectors(*dd)
            s.set_detectors(dets + obs)
            dc = torch.zeros(len(dets) + 1, dtype=torch.int64, device="cuda")
            run = lambda seed: s.sample_counted(nn, seed, out=out, counts=counts, det_counts=dc,  # noqa: E731
                                                tiled=a.tiled)
        elif a.tiled:
            run = lambda seed: s.sample_tiled(nn, seed, out=out, counts=counts)  # noqa: E731
        else:
            run = lambda seed: s.sample(nn, seed, out=out, counts=counts)  # noqa: E731
        run(7)
        torch.cuda.synchronize()
        if not a.no_check:
            outs[name] = (out.clone(), None if counts is None else counts.clone(),
                          None if dc is None else dc.clone())
        for i in range(2):
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
        res[name] = {"ms_median": ts[len(ts) // 2], "ms_min": ts[0], "plan": s.plan_info()}
        del s, out
    same = None
    if not a.no_check:
        same = all((x is None and y is None) or torch.equal(x, y)
                   for x, y in zip(outs["k1"], outs["k7"]))
        res["nonzero_words"] = int((outs["k1"][0] != 0).sum())
    env = {k: v for k, v in os.environ.items() if k.startswith("SP_")}
    print(json.dumps({"config": a.config, "shots": n, "tiled": a.tiled, "dets": a.dets, "identical": same,
                      "k1_ms": res["k1"]["ms_median"], "k7_ms": res["k7"]["ms_median"],
                      "speedup": res["k1"]["ms_median"] / res["k7"]["ms_median"], "env": env, "res": res}))
    if same is False:
        sys.exit(1)


if __name__ == "__main__":
    main()
