"""Summarise an ncu launch list (gpu__time_duration per launch, CSV) of the
bench's timed region: per-kernel launches, total and share."""
import csv, collections, io, re, sys

path = sys.argv[1]
text = open(path).read()
start = text.find('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
per = collections.OrderedDict()
seq = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
    name = re.sub(r"^void ", "", name).replace("vate::", "")
    us = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    if unit in ("nsecond", "ns"):
        us /= 1e3
    elif unit in ("msecond", "ms"):
        us *= 1e3
    seq.append((name, us))
    t = per.setdefault(name, [0, 0.0])
    t[0] += 1
    t[1] += us
total = sum(v[1] for v in per.values())
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
print(f"{'kernel':50s} {'launches':>8s} {'total us':>10s} {'us/launch':>10s} {'share':>6s}")
for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:50]:50s} {n:8d} {us:10.1f} {us / n:10.2f} {100 * us / total:5.1f}%")
print(f"sum {len(seq)} launches, {total:.1f} us -> {total / steps:.1f} us of kernels per slice "
      f"(ncu serialises launches and runs them cold: compare SHARES, not absolutes)")
