"""Scan micro-benchmark: 5M device-resident packets per launch, registry on/off,
unroll V and L2 persistence variants.  MICRO_CK="24,60" (c,k) selects the pool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200._lib import lib, check

c, k = (int(x) for x in os.environ.get("MICRO_CK", "24,60").split(","))
cfg = vb.EstimatorConfig(1024, c, k)
pool = cfg.build_pool()
pipe = vb.Pipeline(pool, cfg, k)
n = 5_000_000
NB = 12
bufs = torch.empty((NB, n, 2), dtype=torch.int32, device="cuda:0")
zipf = os.environ.get("MICRO_ZIPF") == "1"     # cfg 3 traffic (Zipf hosts + spreaders)
if zipf:
    from paper_1812_00282_b200.synth import ZipfTables
    zt = ZipfTables(0, 1_000_000)
for i in range(NB):
    if zipf:
        zt.packets(pool, i, n, 0x0A000000, 0, bufs[i].data_ptr())
    else:
        check(lib.vate_synth_packets(pool.handle, i, n, 1_000_000, 0x0A000000, 0, bufs[i].data_ptr()))
for t in range(NB):   # fill the registry
    pipe.step_packed(t, bufs[t].data_ptr(), n, True)


T = [1000]


def run(hosts, t0):
    """12 slices x 3 reps, each a NEW slice index with an advance in between,
    as in a real stream (registry stamps and block clocks move); only the scan
    kernels are counted (the sweep is timed under its own kind)."""
    pool.set_timing(False); pool.set_timing(True)
    for rep in range(3):
        for t in range(NB):
            T[0] += 1
            check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                       bufs[t].data_ptr(), n, 1, hosts, T[0]))
            pool.advance_slice()
    ms, kk = pool.kernel_time("scan")
    return ms / (3 * NB)   # per scan call (a call may launch more than one kernel)


tag = f"c={c}{' zipf' if zipf else ''}"
for l2 in [int(x) for x in os.environ.get("MICRO_L2", "0").split(",")]:
    pool.set_option("l2_persist", l2)
    for chk in (0, 1):
        pool.set_option("scan_check", chk)
        for v in (1, 8):
            pool.set_option("scan_v", v)
            ms = run(pipe.hosts.handle, 100)
            print(f"{tag} l2={l2} check={chk} V={v} scan+registry ms/launch {ms:.4f}  "
                  f"({n / ms / 1e6:.1f} Gpps)")
    pool.set_option("scan_v", 1)
    pool.set_option("scan_check", 0)
    print(f"{tag} l2={l2} scan only ms/launch {run(None, 0):.4f}")
