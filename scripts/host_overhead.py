"""Host time per pipelined slice call at cfg 1 (100k packets): Python wrapper vs
the library call, to see what bounds small slices."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200 import _lib
from paper_1812_00282_b200._lib import lib, check

cfg = vb.EstimatorConfig(1024, 20, 10)
pool = cfg.build_pool()
pipe = vb.Pipeline(pool, cfg, 10)
n = 100_000
NB = 64
bufs = torch.empty((NB, n, 2), dtype=torch.int32, device="cuda:0")
for i in range(NB):
    check(lib.vate_synth_packets(pool.handle, i, n, 10_000, 0x0A000000, 0, bufs[i].data_ptr()))
for t in range(40):
    pipe.step_lagged(t, bufs[t % NB].data_ptr(), n, "device", None)
orig = lib.vate_slice_step_lagged
acc = [0.0]
def timed(*a):
    t0 = time.perf_counter()
    r = orig(*a)
    acc[0] += time.perf_counter() - t0
    return r
lib.vate_slice_step_lagged = timed
N = 400
t0 = time.perf_counter()
for t in range(40, 40 + N):
    pipe.step_lagged(t, bufs[t % NB].data_ptr(), n, "device", None)
total = time.perf_counter() - t0
print(f"per call: total {total / N * 1e6:.1f} us, in the library {acc[0] / N * 1e6:.1f} us, "
      f"python {(total - acc[0]) / N * 1e6:.1f} us")
