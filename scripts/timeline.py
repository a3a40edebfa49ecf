"""Device timeline of the slice step (cfg 2 by default; TL_C/TL_K/TL_N/TL_HOSTS/TL_WARM: another
shape; TL_ZIPF=1: cfg 3's Zipf traffic): the host cost of a call, then every launch (CUDA events around each kernel) and the idle
gaps between them, for a few steady-state slices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200._lib import lib, check

C_, K_ = int(os.environ.get("TL_C", 24)), int(os.environ.get("TL_K", 60))
cfg = vb.EstimatorConfig(1024, C_, K_)
pool = cfg.build_pool()
for kv in os.environ.get("TL_OPTS", "").split():
    k_, v_ = kv.split("=")
    pool.set_option(k_, int(v_))
pipe = vb.Pipeline(pool, cfg, K_)
n = int(os.environ.get("TL_N", 5_000_000))
HOSTS = int(os.environ.get("TL_HOSTS", 1_000_000))
NB = 140
bufs = torch.empty((NB, n, 2), dtype=torch.int32, device="cuda:0")
if os.environ.get("TL_ZIPF") == "1":   # cfg 3's traffic (Zipf + super-spreaders)
    from paper_1812_00282_b200.synth import ZipfTables
    zt = ZipfTables(0, HOSTS)
    for i in range(NB):
        zt.packets(pool, i, n, 0x0A000000, 0, bufs[i].data_ptr())
else:
    for i in range(NB):
        check(lib.vate_synth_packets(pool.handle, i, n, HOSTS, 0x0A000000, 0, bufs[i].data_ptr()))
lagged = os.environ.get("TL_LAGGED", "1") == "1"
step = pipe.step_lagged if lagged else pipe.step_fast
import time
WARM = int(os.environ.get("TL_WARM", 130))
for t in range(WARM):
    step(t, bufs[t % NB].data_ptr(), n, "device", None)
pool.synchronize()
import ctypes as C
host_us = []
api0, l0 = C.c_uint64(), pool.launches()
check(lib.vate_api_calls(C.byref(api0)))
for t in range(WARM, WARM + 30):   # untimed: the host cost of a call
    a = time.perf_counter()
    step(t, bufs[t % NB].data_ptr(), n, "device", None)
    host_us.append((time.perf_counter() - a) * 1e6)
pool.synchronize()
api1 = C.c_uint64()
check(lib.vate_api_calls(C.byref(api1)))
print("host us per step call (30 calls, no kernel timing): median %.1f; per call %.1f launches, "
      "%.1f other CUDA calls" % (np.median(host_us), (pool.launches() - l0) / 30,
                                 (api1.value - api0.value) / 30))
pool.set_timing(True)
for t in range(WARM + 30, WARM + 36):
    step(t, bufs[t % NB].data_ptr(), n, "device", None)
if lagged:
    pipe.flush_lagged(None)
pipe.wait_reports()
pool.synchronize()
tl = pool.timeline()
tl.sort(key=lambda x: x[1])
prev_end = None
for kind, s, e in tl:
    gap = (s - prev_end) * 1e3 if prev_end is not None else 0.0
    print(f"{kind:9s} start {s*1e3:9.1f} us  dur {(e-s)*1e3:7.1f} us  gap-before {gap:7.1f} us")
    prev_end = e if prev_end is None else max(prev_end, e)
scans = [s for k, s, e in tl if k == "scan"]
print("slice period us:", np.diff(scans) * 1e3)
