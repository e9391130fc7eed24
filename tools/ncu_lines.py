"""Per-source-line summary of an ncu report (--import-source on, -lineinfo):
stall samples, instructions and shared-memory wavefronts per line, top N.
usage: python tools/ncu_lines.py REPORT.ncu-rep [N] [sort: samples|shared|inst]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "samples"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0] or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))  # skip (Line No, Source); the second "Source" column is SASS
    def f(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    recs.append((fname, int(r[0]), r[1].strip()[:90], f("Warp Stall Sampling (All Samples)"),
                 f("Instructions Executed"), f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Excessive")))
tot = [sum(x[i] for x in recs) for i in (3, 4, 5)]
idx = {"samples": 3, "inst": 4, "shared": 5}[key]
recs.sort(key=lambda x: -x[idx])
print(f"total samples {tot[0]:.0f}, instructions {tot[1]:.3e}, shared wavefronts {tot[2]:.3e}")
for fn, ln, src, s, i, w, we in recs[:top]:
    print(f"{fn}:{ln:5d} samp {100 * s / max(tot[0], 1):5.1f}% inst {100 * i / max(tot[1], 1):5.1f}% "
          f"shw {100 * w / max(tot[2], 1):5.1f}% (excess {we:.2e})  {src}")
