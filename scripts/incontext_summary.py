"""Summarise an ncu --cache-control none metric list (scripts/ncu_incontext.sh):
per kernel, mean time, DRAM bytes read / written per launch and the L2 hit
rate, with the L2 as the preceding kernels of the slice left it."""
import collections
import csv
import io
import re
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "%": 1, "sector": 1, "": 1}

text = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
per = collections.OrderedDict()
for r in rows:
    name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
    name = re.sub(r"^void ", "", name).replace("vate::", "")
    v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1)
    per.setdefault(name, collections.defaultdict(list))[r["Metric Name"]].append(v)


def mean(xs):
    return sum(xs) / len(xs) if xs else float("nan")


print(f"{'kernel':48s} {'n':>3s} {'us':>8s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} "
      f"{'L2 hit %':>8s} {'L2 sectors M':>12s}")
for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    print(f"{k[:48]:48s} {len(m['gpu__time_duration.sum']):3d} "
          f"{mean(m['gpu__time_duration.sum']):8.1f} {mean(m['dram__bytes_read.sum']) / 1e6:10.1f} "
          f"{mean(m['dram__bytes_write.sum']) / 1e6:10.1f} {mean(m['lts__t_sector_hit_rate.pct']):8.1f} "
          f"{mean(m['lts__t_sectors.sum']) / 1e6:12.2f}")
print("ncu --cache-control none: the L2 as the slice's earlier kernels left it (launches "
      "serialised by ncu; times are not the overlapped pipeline's)")
