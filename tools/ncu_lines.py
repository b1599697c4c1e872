"""Per-source-line instruction / stall attribution from an ncu report
(`--page source --print-source cuda,sass`), for the CUDA lines only.

    python tools/ncu_lines.py REPORT.ncu-rep [--top 40] [--shots N]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--shots", type=float, default=0)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = []
    fname = ""
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
            d = dict(zip(hdr, r))
            ie = float(d["Instructions Executed"] or 0)
            st = float(d["Warp Stall Sampling (All Samples)"] or 0)
            if ie or st:
                lines.append((fname, int(r[0]), r[1].strip()[:90], ie, st))
    tot_i = sum(x[3] for x in lines) or 1
    tot_s = sum(x[4] for x in lines) or 1
    print(f"total warp instructions {tot_i:.0f}" +
          (f" ({tot_i / a.shots:.3f}/shot)" if a.shots else "") + f", stall samples {tot_s:.0f}")
    for f, ln, src, ie, st in sorted(lines, key=lambda x: -x[3])[:a.top]:
        per = f" {ie / a.shots:7.3f}/shot" if a.shots else ""
        print(f"{f}:{ln:<5} {100 * ie / tot_i:5.1f}% inst{per} {100 * st / tot_s:5.1f}% stall  {src}")


if __name__ == "__main__":
    main()
