"""Round-2 ncu summaries for profiles/: r02_ncu_modexp.json (the bench launch's DRAM traffic, pipes,
stalls -- bench.py's `traffic`), r02_ncu_modexp4096.json (config 4) and r02_ct_evidence.json (SASS
counts per exponent class for four kernels).  Inputs: gpurun_out/ from tools/gpu_collect_r02.sh."""
import csv
import io
import json
import subprocess

G = "gpurun_out"
scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def capture(rep, kernel, command, operands, algorithmic_bytes):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def g(n):
        return float(vals[hdr.index(n)].replace(",", ""))

    def b(n):
        return g(n) * scale[units[hdr.index(n)]]

    st = {k.split("stalled_")[1].split("_per")[0]: round(g(k), 3) for k in hdr
          if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and g(k) > 0.05}
    t = g("gpu__time_duration.sum") * (1000.0 if units[hdr.index("gpu__time_duration.sum")] == "s" else 1.0)
    d = {"kernel": kernel, "command": command,
         "ncu": "ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 (tools/gpu_collect_r02.sh)",
         "gpu_time_ms": t, "dram_bytes_read": b("dram__bytes_read.sum"), "dram_bytes_write": b("dram__bytes_write.sum"),
         "operands_per_launch": operands, "algorithmic_table_scan_bytes": algorithmic_bytes,
         "registers_per_thread": g("launch__registers_per_thread"),
         "warps_active_pct": round(g("sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
         "l2_hit_pct": round(g("lts__t_sector_hit_rate.pct"), 2), "l1_hit_pct": round(g("l1tex__t_sector_hit_rate.pct"), 2),
         "stalls_per_issue": st, "warp_instructions": g("smsp__inst_executed.sum"),
         "pipes": {n: round(g(n), 2) for n in ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                                                "sm__issue_active.avg.pct_of_peak_sustained_elapsed") if n in hdr}}
    d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
    d["traffic_over_algorithmic"] = round(d["dram_bytes_per_launch"] / algorithmic_bytes, 3)
    return d


# algorithmic table-scan bytes: W * 2^w * 4L per modexp
json.dump(capture(f"{G}/r02_modexp2048.ncu-rep", "k_modexp<16,1,4,0>",
                  "python tools/prof_modexp.py --count 262144 (the bench.py launch: 2048-bit, w=5, truncated, 2^18)",
                  262144, 410 * 32 * 4 * 64 * 262144),
          open("profiles/r02_ncu_modexp.json", "w"), indent=1)
json.dump(capture(f"{G}/r02_modexp4096.ncu-rep", "k_modexp<16,1,8,0> (register-Karatsuba blocks)",
                  "python tools/prof_modexp.py --bits 4096 --count 65536 (config 4)", 65536, 820 * 32 * 4 * 128 * 65536),
          open("profiles/r02_ncu_modexp4096.json", "w"), indent=1)
ct = {}
for tag, what in (("k32", "k_modexp<16,1,4,0>, 2048 bits, 18944 operands (the shipped headline kernel)"),
                  ("k4096", "k_modexp<16,1,8,0> with register-Karatsuba blocks, 4096 bits, 18944 operands"),
                  ("coop8", "k_modexp_coop<16,1,8,8>, 8 lanes per operand, 4096 bits, 1024 operands"),
                  ("d52", "k_modexp_d52<8,5,true>, radix-2^52 FP64, 2048 bits, 18944 operands")):
    per = {}
    for c in ("zero", "ones", "random"):
        try:
            lines = [l for l in open(f"{G}/r02_ct_{tag}_{c}.csv").read().splitlines() if l.startswith('"')]
        except FileNotFoundError:
            continue
        r = list(csv.reader(lines))
        h = r[0]
        im, iv = h.index("Metric Name"), h.index("Metric Value")
        per[c] = {x[im]: float(x[iv].replace(",", "")) for x in r[1:]}
    keys = [k for k in (per.get("zero") or {}) if k != "gpu__time_duration.sum"]
    ct[tag] = {"kernel": what, "classes": per,
               "counts_identical_across_classes": bool(per) and all(
                   len({per[c][k] for c in per}) == 1 for k in keys)}
json.dump(ct, open("profiles/r02_ct_evidence.json", "w"), indent=1)
print(json.dumps({k: v["counts_identical_across_classes"] for k, v in ct.items()}))
