"""Per-source-line warp-stall samples of one ncu capture (the source page,
CUDA lines with their SASS): which lines of a kernel the time goes to.
  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
per_line = {}
cur = None
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:  # a CUDA line row (aggregated over its SASS)
        cur = (fname, int(r[0]), r[1].strip()[:90])
        try:
            s = float(r[si] or 0)
        except ValueError:
            s = 0
        st = {}
        for i, h in stall_cols:
            try:
                v = float(r[i] or 0)
            except ValueError:
                v = 0
            if v:
                st[h[6:]] = v
        per_line[cur] = (s, st)
tot = sum(v[0] for v in per_line.values()) or 1
print(f"total samples {tot:.0f}")
for (f, ln, src), (s, st) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}%  {f}:{ln:<5d} {src:90s} {big}")
