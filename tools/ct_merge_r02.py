"""Merge further constant-time captures (gpurun_out/r02_ct_<tag>_<cls>.csv from tools/gpu_r02_ct2.sh)
into profiles/r02_ct_evidence.json: per exponent class (all-zero windows, all-one, random) the
warp-level SASS instruction / branch / load / store counts of the kernel must be identical."""
import csv
import json
import sys

G = "gpurun_out"
P = "profiles/r02_ct_evidence.json"
TAGS = {"reg1024": "k_modexp_reg<32>, register-resident CIOS with squaring rows, 1024 bits, 18944 operands",
        "cios2048": "k_modexp<16,2,4,0>, block-engine CIOS with squaring rows, 2048 bits, 18944 operands",
        "w384": "mpb_w384::k_modexp<16,1,4,0>, one-wave 128-thread-per-SM shape of the 384-thread instance, 2048 bits, "
                "18944 operands",
        "w448": "mpb_w448::k_modexp<16,1,8,0>, one 448-thread CTA per SM (config 4), 4096 bits, 65536 operands"}
TAGS = {t: TAGS[t] for t in (sys.argv[1:] or TAGS)}
ct = json.load(open(P))
for tag, what in TAGS.items():
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
    if not per:
        sys.exit(f"no captures for {tag}")
    keys = [k for k in per["zero"] if k != "gpu__time_duration.sum"]
    ct[tag] = {"kernel": what, "classes": per,
               "counts_identical_across_classes": all(len({per[c][k] for c in per}) == 1 for k in keys)}
json.dump(ct, open(P, "w"), indent=1)
print(json.dumps({k: v.get("counts_identical_across_classes") for k, v in ct.items() if isinstance(v, dict)}))
