"""Summarise an ncu report: per kernel duration, DRAM bytes/throughput,
occupancy, top stall reasons and top stalled SASS lines."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print("=====", d.get("Kernel Name", "")[:70])
    for k, lab in [("gpu__time_duration.sum", "dur_us"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
                   ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
                   ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
                   ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
                   ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
                   ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "bank_ld"),
                   ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "bank_st"),
                   ("launch__registers_per_thread", "regs")]:
        print(f"   {lab:8s} {d.get(k)}")
    st = []
    for k in d:
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("   stalls", [(n, round(v, 2)) for v, n in st[:7]])
