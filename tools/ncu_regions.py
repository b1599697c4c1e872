"""Executed warp instructions and stall samples per SASS region of one
kernel in an ncu report: innermost loops (by backward branch) and the
straight-line code between them.

    python tools/ncu_regions.py REPORT.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    base = int(data[0]["Address"], 16)
    ins = [(int(d["Address"], 16) - base, d["Source"].strip(), int(d["Instructions Executed"] or 0),
            float(d["Warp Stall Sampling (All Samples)"] or 0)) for d in data]
    tot_i = sum(x[2] for x in ins) or 1
    tot_s = sum(x[3] for x in ins) or 1
    # innermost loops: backward branches, smallest span first claims its body
    loops = []
    for i, (adr, src, _, _) in enumerate(ins):
        m = re.search(r"BRA\b.*?0x([0-9a-f]+)", src)
        if m:
            tgt = int(m.group(1), 16) - base if int(m.group(1), 16) >= base else int(m.group(1), 16)
            if tgt < adr:
                loops.append((tgt, adr))
    owner = [None] * len(ins)
    for lo, hi in sorted(loops, key=lambda t: t[1] - t[0]):
        for i, x in enumerate(ins):
            if lo <= x[0] <= hi and owner[i] is None:
                owner[i] = f"loop {lo:#06x}-{hi:#06x}"
    for i in range(len(ins)):
        if owner[i] is None:
            owner[i] = "straight"
    agg = {}
    for (adr, src, n, st), o in zip(ins, owner):
        e = agg.setdefault(o, [0, 0.0, {}, adr])
        e[0] += n
        e[1] += st
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        e[2][op] = e[2].get(op, 0) + n
    print(f"total warp instructions {tot_i}")
    for o, (n, st, ops, adr) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        top = ", ".join(f"{k}:{v * 100 / max(n, 1):.0f}%" for k, v in sorted(ops.items(), key=lambda z: -z[1])[:5])
        print(f"{100 * n / tot_i:5.1f}% inst {100 * st / tot_s:5.1f}% stall  {o:26s} {top}")


if __name__ == "__main__":
    main()
