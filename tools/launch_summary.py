"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel, launches,
total and mean duration, and share of all kernel time (cold-cache, serialised -- shares, not absolutes)."""
import csv
import re
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) >= 15 and r[0] != "ID"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r[12] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(DevCtx.*$", "", r[4]).replace("void ", "")
    us = float(r[14].replace(",", "")) / (1e3 if r[13] == "ns" else 1.0)
    tot[name] += us
    cnt[name] += 1
allt = sum(tot.values())
with open(dst, "w") as f:
    f.write("kernel,launches,total_us,mean_us,share\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"\"{k}\",{cnt[k]},{tot[k]:.1f},{tot[k] / cnt[k]:.1f},{tot[k] / allt:.4f}\n")
print(open(dst).read())

# per fused-layer call: kernels of the batched schedule-2 path (calls = k_gala_mac2 launches)
STEP = {"k_gala_tc<3>": None, "k_gala_e_can<3>": None, "k_gala_mac2<1, 1>": None, "k_gala_e<3, 4>": None,
        "k_moddown": None, "k_digits_perm": None, "k_digits_intt": None, "k_ntt_inv<0>": None, "k_ks_mac<3>": None,
        "k_sub_plain": None, "k_encode<1>": 1}
calls = cnt.get("k_gala_tc<3>", 0) or cnt.get("k_gala_mac2<1, 1>", 0)
if calls:
    per = {}
    for k, fixed in STEP.items():
        if k not in cnt:
            continue
        n = fixed if fixed is not None else cnt[k] / calls
        per[k] = (n, tot[k] / cnt[k] * n)
    s = sum(v[1] for v in per.values())
    with open(dst.replace(".csv", "_per_call.csv"), "w") as f:
        f.write("kernel,launches_per_call,us_per_call,share_of_call\n")
        for k in sorted(per, key=lambda k: -per[k][1]):
            f.write(f"\"{k}\",{per[k][0]:g},{per[k][1]:.1f},{per[k][1] / s:.4f}\n")
    print(open(dst.replace(".csv", "_per_call.csv")).read())
