"""Turn the raw outputs of tools/gpu_collect_r01.sh (gpurun_out/) into the committed profile
summaries: profiles/<tag>_ncu_modexp.json (bench-size full capture: DRAM traffic per launch,
stalls, launch share from the launch list), <tag>_ct_evidence.json, <tag>_bench.json,
<tag>_ncu_launches_bench.csv and <tag>_ncu_modexp_full.txt.

  python tools/summarize_collect.py r01_v3
"""
import collections
import csv
import io
import json
import re
import shutil
import subprocess
import sys

tag = sys.argv[1]
G = "gpurun_out"
rep = f"{G}/modexp_bench.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def g(n):
    return float(vals[hdr.index(n)].replace(",", ""))


rd = g("dram__bytes_read.sum") * scale[units[hdr.index("dram__bytes_read.sum")]]
wr = g("dram__bytes_write.sum") * scale[units[hdr.index("dram__bytes_write.sum")]]
st = {k.split("stalled_")[1].split("_per")[0]: round(g(k), 3) for k in hdr
      if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and g(k) > 0.05}
d = {"kernel": "k_modexp<16,1,4,0>",
     "command": "python tools/prof_modexp.py --count 262144  (the bench.py launch: 2048-bit, w=5, truncated, 2^18 operands)",
     "ncu": "ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 (tools/gpu_collect_r01.sh)",
     "gpu_time_ms": g("gpu__time_duration.sum"), "dram_bytes_read": rd, "dram_bytes_write": wr,
     "dram_bytes_per_launch": rd + wr, "operands_per_launch": 262144,
     "registers_per_thread": g("launch__registers_per_thread"),
     "warps_active_pct": round(g("sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
     "l2_hit_pct": round(g("lts__t_sector_hit_rate.pct"), 2), "l1_hit_pct": round(g("l1tex__t_sector_hit_rate.pct"), 2),
     "stalls_per_issue": st, "warp_instructions": g("smsp__inst_executed.sum")}
pipes = {}
for name in ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
             "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum"):
    if name in hdr:
        pipes[name] = g(name)
d["pipes"] = pipes
lines = [l for l in open(f"{G}/launches.csv").read().splitlines() if l.startswith('"') and "gpu__time_duration" in l]
tot = collections.Counter()
for l in csv.reader(lines):
    tot[re.sub(r"\(.*", "", l[4]).split("::")[-1].split("<")[0]] += float(l[-1].replace(",", ""))
T = sum(tot.values())
d["bench_launch_share"] = {k: round(v / T, 4) for k, v in tot.most_common()}
d["bench_launch_share"]["source"] = f"profiles/{tag}_ncu_launches_bench.csv (cold-cache, serialised)"
json.dump(d, open(f"profiles/{tag}_ncu_modexp.json", "w"), indent=1)
ct = {}
for c in ("zero", "ones", "random"):
    m = {}
    for l in csv.reader([x for x in open(f"{G}/ct_{c}.csv").read().splitlines() if x.startswith('"') and "k_modexp" in x]):
        m[l[-3]] = float(l[-1].replace(",", ""))
    ct[c] = m
keys = [k for k in ct["zero"] if k != "gpu__time_duration.sum"]
same = all(ct[c][k] == ct["zero"][k] for c in ct for k in keys)
json.dump({"kernel": "k_modexp<16,1,4,0> (2048-bit, w=5, truncated, 18944 operands, same N and base)",
           "command": "tools/gpu_collect_r01.sh (ncu --metrics ... python tools/ct_check.py --cls {zero,ones,random})",
           "metrics": ct, "identical_across_classes": same,
           "negative_control": "profiles/r01_ct_evidence.json (planted secret-dependent load build differs: 107M vs 182M global loads)"},
          open(f"profiles/{tag}_ct_evidence.json", "w"), indent=1)
shutil.copy(f"{G}/launches.csv", f"profiles/{tag}_ncu_launches_bench.csv")
open(f"profiles/{tag}_bench.json", "w").write(open(f"{G}/bench_final.log").read().strip().splitlines()[-1] + "\n")
full = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
open(f"profiles/{tag}_ncu_modexp_full.txt", "w").write(full)
print(json.dumps(d, indent=1))
print("CT identical:", same)
