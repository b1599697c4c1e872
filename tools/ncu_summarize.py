"""Text summary of an ncu report (run here, on the CPU box):

    python tools/ncu_summarize.py gpurun_out/prof.ncu-rep > profiles/<name>.txt

Prints the headline metrics, DRAM traffic, stall-reason totals, the opcode
mix per shot (if --shots is given) and the hottest SASS lines.
"""
import argparse
import collections
import csv
import io
import subprocess

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "No Eligible",
        "SM Frequency"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--shots", type=float, default=0)
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    det = list(csv.reader(io.StringIO(run([a.rep, "--page", "details", "--csv"]))))
    h = det[0]
    print(f"# ncu summary: {a.rep}")
    for row in det[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in WANT:
            print(f'{d["Metric Name"]:40s} {d["Metric Unit"]:14s} {d["Metric Value"]}')
    raw = list(csv.reader(io.StringIO(run([a.rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        rh = raw[0]
        vals = raw[2]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if name in rh:
                print(f"{name:40s} {raw[1][rh.index(name)]:14s} {vals[rh.index(name)]}")
    src = list(csv.reader(io.StringIO(run([a.rep, "--page", "source", "--csv",
                                           "--print-source", "sass"]))))
    sh = src[1]
    data = src[2:]
    ix = {k: i for i, k in enumerate(sh)}
    S = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
    E = [int(r[ix["Instructions Executed"]] or 0) for r in data]
    ts, te = sum(S), sum(E)
    stall_cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    for r in data:
        for c in stall_cols:
            agg[c] += int(r[ix[c]] or 0)
    print(f"\nwarp-level instructions executed: {te}" +
          (f"  ({te / a.shots:.2f} per shot)" if a.shots else ""))
    print("stall reasons (share of samples):")
    for c, v in agg.most_common(10):
        print(f"  {c:32s} {100 * v / max(ts, 1):5.1f}%")
    op = collections.Counter()
    for r, e in zip(data, E):
        t = r[ix["Source"]].strip().split()
        o = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
        op[o.split(".")[0]] += e
    print("opcode mix:")
    for k, v in op.most_common(14):
        per = f"{v / a.shots:8.3f}/shot" if a.shots else ""
        print(f"  {k:10s} {100 * v / max(te, 1):5.1f}% {per}")
    print(f"hottest SASS (stall samples):")
    for r, s_ in sorted(zip(data, S), key=lambda t: -t[1])[:a.top]:
        st = sorted(((int(r[ix[c]] or 0), c) for c in stall_cols), reverse=True)[:1]
        print(f"  {100 * s_ / max(ts, 1):5.1f}%  {r[ix['Source']].strip()[:60]:60s} {st[0][1] if st else ''}")


if __name__ == "__main__":
    main()
