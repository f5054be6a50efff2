"""SASS opcode mix of one kernel instance in an ncu report (source page,
SASS view): warp-level instructions executed and stall samples per opcode.
usage: ncu_opmix.py REPORT KERNEL_REGEX [LAUNCH_SKIP]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
cnt, st, tot, ie, iss = collections.Counter(), collections.Counter(), 0, None, None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        ie, iss = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie:
        continue
    parts = r[1].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    try:
        n = int(r[ie] or 0)
    except ValueError:
        continue
    cnt[op] += n
    tot += n
    st[op] += int(r[iss] or 0)
stot = sum(st.values()) or 1
print(f"{kern}: {tot} warp instructions")
for op, n in cnt.most_common(24):
    print(f"  {op:10s} {100 * n / tot:5.1f}% of instructions  {100 * st[op] / stot:5.1f}% of stall samples")
