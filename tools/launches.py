"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
fn = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(fn)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
seq = []
for r in data[skip:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    name = r[ki].split("(")[0].replace("void ", "")[:70]
    tot[name] += v; cnt[name] += 1
    seq.append((name, v))
T = sum(tot.values())
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
for k, v in tot.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{v:11.1f} us {100 * v / T:5.1f}%  n={cnt[k]:6d} avg={v / cnt[k]:9.2f} us  {k}")
