"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a bench run
into per-kernel totals and shares of the summed kernel time (dev tool).

  python tools/launch_summary.py launches.csv OUT.txt "header line" [steps]"""
import collections
import csv
import sys

src, out, header = sys.argv[1], sys.argv[2], sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
units = set()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("fsep::", "").replace("(anonymous namespace)::", "")
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    units.add(u)
    tot[name] += v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
    cnt[name] += 1
all_ms = sum(tot.values())
with open(out, "w") as f:
    f.write(f"# {header}\n# kernel | launches | total ms | mean ms | share\n")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{name} | {cnt[name]} | {ms:.3f} | {ms / cnt[name]:.4f} | {ms / all_ms:.3f}\n")
    f.write(f"# total kernel time {all_ms:.3f} ms over {steps} step(s) = {all_ms / steps:.3f} ms per step; units {sorted(units)}\n")
print(open(out).read())
