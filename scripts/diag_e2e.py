"""Diagnose the e2e path: per-call host timings of stage / step / wait."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200._lib import lib, check

cfg = vb.EstimatorConfig(1024, 24, 60)
pool = cfg.build_pool()
pipe = vb.Pipeline(pool, cfg, 60)
n = 5_000_000
scratch = torch.empty((n, 2), dtype=torch.int32, device="cuda:0")
hs = torch.empty((int(os.environ.get("NSL", "8")), n, 2), dtype=torch.int32, pin_memory=True)
for i in range(hs.shape[0]):
    check(lib.vate_synth_packets(pool.handle, 500 + i, n, 1_000_000, 0x0A000000, 0, scratch.data_ptr()))
    pool.synchronize()
    hs[i].copy_(scratch)
cap = 1_000_016
outs = [(torch.empty(cap, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
         torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
         torch.empty(cap, dtype=torch.float64, pin_memory=True).numpy(),
         torch.empty(cap, dtype=torch.uint8, pin_memory=True).numpy()) for _ in range(2)]
for t in range(70):
    check(lib.vate_synth_packets(pool.handle, t, n, 1_000_000, 0x0A000000, 0, scratch.data_ptr()))
    pipe.step_packed(t, scratch.data_ptr(), n, True, outs[t % 2], wait=False)
pipe.wait_reports()
t = 70
# raw copy bandwidth
dst = torch.empty((n, 2), dtype=torch.int32, device="cuda:0")
torch.cuda.synchronize(); a = time.perf_counter(); dst.copy_(hs[0], non_blocking=True); torch.cuda.synchronize()
print("torch H2D 40MB ms", (time.perf_counter() - a) * 1e3)
for mode in ("staged", "hostptr", "device"):
    times = []
    staged = [None, None]
    staged[0] = pipe.stage_packed(hs[0].data_ptr(), n)
    pool.synchronize()
    for i in range(8):
        i = i * (hs.shape[0] // 8)
        a = time.perf_counter()
        if mode == "staged":
            if i + 1 < hs.shape[0]:
                staged[(i + 1) % 2] = pipe.stage_packed(hs[i + 1].data_ptr(), n)
            b = time.perf_counter()
            pipe.step_staged(t, staged[i % 2], n, outs[t % 2], wait=False)
        elif mode == "hostptr":
            b = time.perf_counter()
            pipe.step_packed(t, hs[i].data_ptr(), n, False, outs[t % 2], wait=False)
        else:
            b = time.perf_counter()
            pipe.step_packed(t, scratch.data_ptr(), n, True, outs[t % 2], wait=False)
        c = time.perf_counter()
        times.append(((b - a) * 1e3, (c - b) * 1e3))
        t += 1
    a = time.perf_counter(); pipe.wait_reports(); pool.synchronize(); w = (time.perf_counter() - a) * 1e3
    print(mode, [f"{x:.2f}/{y:.2f}" for x, y in times], "final wait ms", round(w, 2))
