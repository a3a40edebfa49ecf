"""Bitmap-pass micro-benchmark (count_inactive = the estimate's bitmap + P pass)
for words-per-thread 1/2/4 at the cfg 2/3/4 pool shapes, cells populated by
5M-packet slices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1812_00282_b200 as vb
from paper_1812_00282_b200._lib import lib, check

n = 5_000_000
for c, k in ((24, 60), (26, 60), (28, 300)):
    cfg = vb.EstimatorConfig(1024, c, k)
    pool = cfg.build_pool()
    buf = torch.empty((n, 2), dtype=torch.int32, device="cuda:0")
    for t in range(8):
        check(lib.vate_synth_packets(pool.handle, t, n, 1_000_000, 0x0A000000, 0, buf.data_ptr()))
        check(lib.vate_scan_packed(pool.handle, cfg.g, cfg.cell_stream, cfg.group_stream,
                                   buf.data_ptr(), n, 1, None, 0))
        pool.advance_slice()
    ref = pool.count_inactive(k)
    for kw in (4, 2, 1, 0):
        pool.set_option("bitmap_kw", kw)
        assert pool.count_inactive(k) == ref
        pool.set_timing(False); pool.set_timing(True)
        for _ in range(20):
            pool.count_inactive(k)
        ms, kk = pool.kernel_time("bitmap")
        mb = (1 << c) * pool.cell_bytes / 1e6
        print(f"c={c} kw={kw} bitmap ms {ms / kk:.4f}  ({mb / (ms / kk) / 1e3:.2f} TB/s of cells)")
    pool.close()
