"""Reads dram__bytes_read/write.sum of one profiled launch from an .ncu-rep (ncu --set full)
and records them under profiles/ncu_traffic.json[config] for bench.py's roofline.traffic.

    python tools/ncu_traffic.py REPORT.ncu-rep cfg3 100000000 "note"
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    rep, cfg, shots, note = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    names, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = names.index(name)
        v = float(vals[i].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[units[i]]
        return v * scale

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    kname = vals[names.index("Kernel Name")]
    p = ROOT / "profiles" / "ncu_traffic.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    d[cfg] = {"shots": shots, "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
              "kernel": kname.split("(")[0], "note": note}
    p.write_text(json.dumps(d, indent=1))
    print(cfg, d[cfg])


if __name__ == "__main__":
    main()
