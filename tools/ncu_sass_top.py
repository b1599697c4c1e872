"""Top SASS instructions by stall samples (with their dominant stall reasons).

    python tools/ncu_sass_top.py REPORT.ncu-rep [--top 30]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "(Not" not in h]
    tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
    idx = {d["Address"]: i for i, d in enumerate(data)}
    for d in sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:a.top]:
        st = float(d["Warp Stall Sampling (All Samples)"] or 0)
        reasons = sorted(((float(d[c] or 0), c) for c in stall_cols), reverse=True)[:2]
        rs = " ".join(f"{c[6:]}:{v:.0f}" for v, c in reasons if v)
        print(f"{100 * st / tot:5.1f}% #{idx[d['Address']]:<5} {d['Source'].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
