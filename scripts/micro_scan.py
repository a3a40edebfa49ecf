"""Scan micro-benchmark: 5M device-resident packets, with / without registry."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200._lib import lib, check

cfg = vb.EstimatorConfig(1024, 24, 60)
pool = cfg.build_pool()
pipe = vb.Pipeline(pool, cfg, 60)
n = 5_000_000
bufs = torch.empty((12, n, 2), dtype=torch.int32, device="cuda:0")
for i in range(12):
    check(lib.vate_synth_packets(pool.handle, i, n, 1_000_000, 0x0A000000, 0, bufs[i].data_ptr()))
for t in range(12):   # fill the registry
    pipe.step_packed(t, bufs[t].data_ptr(), n, True)
for v in (2, 1, 4, 2, 1):
    pool.set_option("scan_v", v)
    pool.set_timing(False); pool.set_timing(True)
    for rep in range(3):
        for t in range(12):
            check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                       bufs[t].data_ptr(), n, 1, pipe.hosts.handle, 100 + t))
    ms, k = pool.kernel_time("scan")
    print("scan+registry V", v, "ms/launch", ms / k)
pool.set_timing(False); pool.set_timing(True)
for rep in range(3):
    for t in range(12):
        check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                   bufs[t].data_ptr(), n, 1, None, 0))
ms, k = pool.kernel_time("scan")
print("scan only ms/launch", ms / k)
