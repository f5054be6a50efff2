"""Per-source-line warp-stall samples of one kernel instance in an ncu
report (ncu --page source --print-source cuda,sass), top lines first.
usage: ncu_lines.py REPORT KERNEL_REGEX [LAUNCH_SKIP] [TOP]
NCU_COLUMN selects another per-line column of the source page (e.g.
"L1 Wavefronts Shared Excessive" for bank conflicts); NCU_COLUMN=? lists them."""
import csv
import os
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, items, tot = "", [], 0.0
idx = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        col = os.environ.get("NCU_COLUMN", "Warp Stall Sampling (All Samples)")
        if col == "?":
            print("\n".join(r))
            sys.exit(0)
        idx = r.index(col)
        continue
    if idx is None or not r[0] or len(r) <= idx:
        continue
    try:
        v = float(r[idx])
    except ValueError:
        continue
    tot += v
    items.append((v, f"{fname}:{r[0]}", r[1].strip()[:110]))
items.sort(reverse=True)
print(f"{kern}: {tot:.0f} samples")
for v, loc, src in items[:top]:
    print(f"{100 * v / tot:5.1f}%  {loc:18s} {src}")
