"""Per-kernel device time of one setup from an ncu launch-list CSV, in launch
order, grouped into consecutive runs of the same kernel name."""
import csv, sys, collections
fn = sys.argv[1]
rows = list(csv.reader(open(fn)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.Counter(); cnt = collections.Counter()
for r in data:
    if len(r) <= vi: continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    name = r[ki].split("(")[0].replace("void ", "")[:80]
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"total {T/1e3:.2f} ms over {sum(cnt.values())} launches")
for k, v in tot.most_common(45):
    print(f"{v/1e3:9.3f} ms {100*v/T:5.1f}%  n={cnt[k]:5d}  avg={v/cnt[k]:8.1f} us  {k}")
