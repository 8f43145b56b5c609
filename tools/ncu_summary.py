"""Summarise an ncu report (raw page + per-opcode source counts) for profiles/."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
pat = (r"^gpu__time_duration.sum$|^launch__registers_per_thread$|^launch__grid_size$|^launch__block_size$|"
       r"^sm__warps_active.avg.pct_of_peak_sustained_active$|^sm__issue_active.avg.pct_of_peak_sustained_active$|"
       r"^sm__pipe_(fma|alu|fmaheavy|fp64)_cycles_active.avg.pct_of_peak_sustained_(active|elapsed)$|^smsp__issue_active.avg.pct_of_peak_sustained_active$|"
       r"^dram__bytes_(read|write).sum$|^dram__throughput.avg.pct_of_peak_sustained_elapsed$|"
       r"^l1tex__t_sector_hit_rate.pct$|^lts__t_sector_hit_rate.pct$|^smsp__inst_executed.sum$|"
       r"^smsp__sass_inst_executed_op_local_(ld|st).sum$|^sm__cycles_elapsed.avg.per_second$|"
       r"average_warps_issue_stalled_(wait|long_scoreboard|short_scoreboard|math_pipe_throttle|no_instruction|"
       r"dispatch_stall|not_selected|selected|branch_resolving|mio_throttle|lg_throttle)_per_issue_active")
for i, h in enumerate(hdr):
    if re.search(pat, h):
        print(f"{h:90s} {units[i]:16s} {vals[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = srows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter()
tot = 0.0
for r in srows[2:]:
    if len(r) <= ia:
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0]
    try:
        n = float(r[ia] or 0)
    except ValueError:
        continue
    cnt[op] += n
    tot += n
print("executed instruction mix (warp-level):")
for op, n in cnt.most_common(16):
    print(f"  {op:22s} {100 * n / tot:6.2f}%")
