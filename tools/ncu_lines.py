"""Hot CUDA source lines of an ncu report (source page, cuda+sass correlation), split into the
control CTAs' code (few executions per step) and the copy CTAs' code.
Usage: python tools/ncu_lines.py <report.ncu-rep> [top] [exec_threshold]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 20000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, timeout=600).stdout
path = "?"
hdr = None
lines = []
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = {h: i for i, h in enumerate(row)}
        stall_cols = [(h, i) for h, i in hdr.items() if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or not row[0] or row[0] in ("Function Name",):
        continue

    def f(name):
        try:
            return float(row[hdr[name]])
        except (ValueError, KeyError, IndexError):
            return 0.0

    samples = f("# Samples")
    if samples == 0:
        continue
    ex = f("Instructions Executed")
    stalls = {h[6:]: float(row[i]) for h, i in stall_cols if row[i] not in ("", "-") and float(row[i]) > 0}
    lines.append((samples, ex, f"{path}:{row[0]}", row[1].strip()[:70], stalls))

for name, sel in (("control (exec <= %g)" % thr, lambda e: e <= thr), ("copy", lambda e: e > thr)):
    part = [x for x in lines if sel(x[1])]
    tot = sum(x[0] for x in part)
    agg = collections.Counter()
    for x in part:
        agg.update(x[4])
    print(f"== {name}: {tot:.0f} samples; stalls " +
          ", ".join(f"{k} {v:.0f}" for k, v in agg.most_common(8)))
    for s, ex, loc, src, st in sorted(part, reverse=True)[:top]:
        top3 = ", ".join(f"{k} {v:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{s:7.0f} {ex:9.0f} {loc:26s} {src:70s} | {top3}")
