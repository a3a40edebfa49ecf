"""Device timeline of the cfg 2 slice step (TL_C/TL_K/TL_N/TL_HOSTS: another shape): every launch (CUDA events around
each kernel) and the idle gaps between them, for a few steady-state slices."""
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
for i in range(NB):
    check(lib.vate_synth_packets(pool.handle, i, n, HOSTS, 0x0A000000, 0, bufs[i].data_ptr()))
lagged = os.environ.get("TL_LAGGED", "1") == "1"
step = pipe.step_lagged if lagged else pipe.step_fast
for t in range(130):
    step(t, bufs[t].data_ptr(), n, "device", None)
pool.set_timing(True)
for t in range(130, 136):
    step(t, bufs[t].data_ptr(), n, "device", None)
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
