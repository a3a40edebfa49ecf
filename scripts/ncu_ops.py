"""Opcode histogram (instructions executed, stall samples) of one kernel in an
ncu report, from its SASS source page: where a compute-heavy kernel spends
its issue slots.   python scripts/ncu_ops.py report.ncu-rep [top]"""
import collections, csv, io, subprocess, sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[1]
rows = [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]
ops, st = collections.Counter(), collections.Counter()
for d in rows:
    toks = d["Source"].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ops[op] += int(d["Instructions Executed"] or 0)
    st[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
tot, ts = sum(ops.values()) or 1, sum(st.values()) or 1
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {n:11d} {n / tot:6.1%}  stall {st[op] / ts:6.1%}")
print("total warp instructions", tot)
