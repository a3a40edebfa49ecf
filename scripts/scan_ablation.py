"""Where the deferred scan's time goes: the scan's memory skeleton
(vate_bench_scan_ablation: packet stream, one red.or mark and one registry
sector read per packet, on the scan's grid) with the scan's other ingredients
added one at a time, next to the real scan kernel (bench.py's per-launch event
time).  Measurement only.

    python scripts/scan_ablation.py [--c 28] [--hosts 1000000] [--packets 5000000]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {1: "hash64", 2: "stamps", 4: "second_read", 8: "ld256", 16: "as_red_max", 32: "as_touched_bit"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", type=int, default=28)
    ap.add_argument("--k", type=int, default=300)
    ap.add_argument("--hosts", type=int, default=1_000_000)
    ap.add_argument("--packets", type=int, default=5_000_000)
    args = ap.parse_args()
    import paper_1812_00282_b200 as vb
    from paper_1812_00282_b200._lib import check, lib
    pool = vb.AtPool(args.c, args.k, "tail", device=0)
    table = 16 * (1 << max(12, (2 * args.hosts - 1).bit_length()))
    out = {"c": args.c, "registry_table_bytes": table, "packets": args.packets}
    for flags in (0, 1, 2, 4, 8, 15, 18, 31, 34, 47):
        ms = C.c_double()
        check(lib.vate_bench_scan_ablation(pool.handle, args.c, table, args.packets, 10, flags,
                                           C.byref(ms)))
        name = "+".join(v for b, v in NAMES.items() if flags & b) or "skeleton"
        out[name + "_us"] = round(ms.value * 1e3, 1)
    pool.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
