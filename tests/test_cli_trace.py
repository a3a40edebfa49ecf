"""Trace ingest and the CLI front-end.

CPU: the host readers' order / truncation errors and the CLI's configuration
exit codes.  GPU: the CLI writes the reference CLI's CSV byte for byte on the
golden traces (tests/golden/cli.npz, made by running `slidecard` itself), the
ATP1 checkpoint is byte-identical, resume continues the stream
(test_cli.py:190-217), and the on-device slice bucketing equals slice_stream
for every chunking.
"""

import os

import numpy as np
import pytest

from _golden import load
from paper_1812_00282_b200 import cli, traceio
from paper_1812_00282_b200.errors import TraceOrderError, TraceParseError


def _grid_trace(lo, hi):
    """Every host in every slice with fresh peers (test_cli.py:175-188)."""
    ts, aips, bips = [], [], []
    for t in range(lo, hi):
        for h in range(3):
            for j in range(5):
                ts.append(t * 1_000_000 + 1000 * j + h)
                aips.append(0x0A000001 + h)
                bips.append(h * 100_000 + t * 5 + j + 1)
    order = np.argsort(np.array(ts), kind="stable")
    return traceio.make_records(np.array(ts, dtype=np.uint64)[order],
                                np.array(aips, dtype=np.uint64)[order],
                                np.array(bips, dtype=np.uint64)[order])


def _write_golden(tmp_path, key, name):
    path = tmp_path / name
    path.write_bytes(load("cli.npz")[key].tobytes())
    return path


# --- CPU -------------------------------------------------------------------------------

def test_binary_reader_errors(tmp_path):
    recs = _grid_trace(0, 3)
    path = tmp_path / "t.bin"
    traceio.write_trace(path, recs, traceio.BINARY)
    assert len(traceio.read_trace(path, traceio.BINARY)) == len(recs)
    path.write_bytes(path.read_bytes()[:-5])
    with pytest.raises(TraceParseError, match="truncated"):
        list(traceio.read_batches(path, traceio.BINARY))
    bad = recs.copy()
    bad["ts"][7] = 0
    traceio.write_trace(path, bad, traceio.BINARY)
    with pytest.raises(TraceOrderError, match=f"byte {7 * 16}"):
        list(traceio.read_batches(path, traceio.BINARY))


def test_text_reader_errors(tmp_path):
    path = tmp_path / "t.csv"
    path.write_text("0,10.0.0.1,0.0.0.1\n5,10.0.0.1\n")
    with pytest.raises(TraceParseError, match="line 2"):
        list(traceio.read_batches(path, traceio.TEXT))
    path.write_text("5,10.0.0.1,0.0.0.1\n3,10.0.0.1,0.0.0.2\n")
    with pytest.raises(TraceOrderError, match="line 2"):
        list(traceio.read_batches(path, traceio.TEXT))
    path.write_text("5,10.0.0.1,300.0.0.2\n")
    with pytest.raises(TraceParseError):
        list(traceio.read_batches(path, traceio.TEXT))


def test_slice_stream_emits_empty_slices():
    recs = traceio.make_records(np.array([2_500_000, 2_600_000, 5_100_000], dtype=np.uint64),
                                np.array([1, 2, 3]), np.array([4, 5, 6]))
    out = [(t, len(a)) for t, a, _ in traceio.slice_stream(iter([recs]), 1_000_000)]
    assert out == [(0, 2), (1, 0), (2, 0), (3, 1)]


def test_golden_traces_read_back(tmp_path):
    b = _write_golden(tmp_path, "trace_bin", "t.bin")
    t = _write_golden(tmp_path, "trace_txt", "t.csv")
    rb = traceio.read_trace(b, traceio.BINARY)
    rt = traceio.read_trace(t, traceio.TEXT)
    assert len(rb) == len(rt) == 5156
    assert np.array_equal(rb["ts"], rt["ts"]) and np.array_equal(rb["aip"], rt["aip"])


@pytest.mark.parametrize("argv,code", [
    (["--k", "4", "--k-prime", "9"], cli.EXIT_CONFIG),
    (["--floor", "-1"], cli.EXIT_CONFIG),
    (["--slice-us", "0"], cli.EXIT_CONFIG),
    (["--counter", "dr", "--resume", "x.atp1"], cli.EXIT_CONFIG),
])
def test_cli_config_errors_without_a_device(tmp_path, capsys, argv, code):
    trace = tmp_path / "t.csv"
    trace.write_text("0,10.0.0.1,0.0.0.1\n")
    assert cli.main(["estimate", "--trace", str(trace)] + argv) == code
    assert "configuration error" in capsys.readouterr().err


# --- GPU -------------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name,argv", [
    ("est_floor0", ["--format", "binary", "--c", "14", "--g", "256", "--k", "6", "--floor", "0"]),
    ("est_default", ["--c", "16", "--g", "256", "--k", "8", "--k-prime", "5"]),
    ("est_lowdev", ["--format", "binary", "--c", "12", "--g", "128", "--k", "6", "--partition",
                    "low-dev", "--floor", "10", "--seed", "9", "--slice-us", "500000"]),
])
def test_cli_estimate_csv_is_byte_identical(tmp_path, name, argv):
    trace = _write_golden(tmp_path, "trace_bin" if "binary" in argv else "trace_txt",
                          "t.bin" if "binary" in argv else "t.csv")
    out = tmp_path / "out.csv"
    assert cli.main(["estimate", "--trace", str(trace), "--out", str(out)] + argv) == 0
    assert out.read_bytes() == load("cli.npz")[name].tobytes()


@pytest.mark.gpu
def test_cli_checkpoint_and_bench_match_reference(tmp_path):
    trace = _write_golden(tmp_path, "trace_bin", "t.bin")
    argv = ["--trace", str(trace), "--format", "binary", "--c", "14", "--g", "256", "--k", "6",
            "--floor", "0"]
    snap = tmp_path / "pool.atp1"
    assert cli.main(["estimate"] + argv + ["--out", str(tmp_path / "x.csv"),
                                           "--checkpoint", str(snap)]) == 0
    assert snap.read_bytes() == load("cli.npz")["checkpoint"].tobytes()
    bench = tmp_path / "bench.csv"
    assert cli.main(["bench"] + argv + ["--out", str(bench)]) == 0
    rows = [line.split(",") for line in bench.read_text().splitlines()[1:]]
    got = np.array([[int(r[0]), int(r[4]), int(r[5])] for r in rows])
    assert np.array_equal(got, load("cli.npz")["bench_cols"])


@pytest.mark.gpu
def test_cli_resume_continues_the_stream(tmp_path):
    """test_cli.py:190-217 against our own CLI."""
    args = ["--c", "12", "--g", "64", "--k", "4", "--floor", "0", "--seed", "3"]
    paths = {}
    for name, (lo, hi) in {"full": (0, 20), "p1": (0, 12), "p2": (12, 20)}.items():
        paths[name] = tmp_path / f"{name}.csv"
        traceio.write_trace(paths[name], _grid_trace(lo, hi), traceio.TEXT)
    snap = tmp_path / "pool.snap"
    assert cli.main(["estimate", "--trace", str(paths["full"]), "--out",
                     str(tmp_path / "full_est.csv")] + args) == 0
    assert cli.main(["estimate", "--trace", str(paths["p1"]), "--out", str(tmp_path / "p1e.csv"),
                     "--checkpoint", str(snap)] + args) == 0
    assert cli.main(["estimate", "--trace", str(paths["p2"]), "--out", str(tmp_path / "p2e.csv"),
                     "--resume", str(snap)] + args) == 0
    full = (tmp_path / "full_est.csv").read_text().splitlines()[1:]
    tail = [r for r in full if int(r.split(",")[0]) >= 12]
    resumed = [f"{int(r.split(',', 1)[0]) + 12},{r.split(',', 1)[1]}"
               for r in (tmp_path / "p2e.csv").read_text().splitlines()[1:]]
    assert resumed == tail
    assert cli.main(["estimate", "--trace", str(paths["p1"]), "--resume", str(snap), "--c", "11",
                     "--g", "64", "--k", "4", "--out", str(tmp_path / "y.csv")]) == cli.EXIT_CONFIG


@pytest.mark.gpu
def test_cli_input_errors(tmp_path):
    assert cli.main(["estimate", "--trace", str(tmp_path / "nope.csv")]) == cli.EXIT_INPUT
    trace = tmp_path / "t.csv"
    trace.write_text("5,10.0.0.1,0.0.0.1\n3,10.0.0.1,0.0.0.2\n")
    assert cli.main(["estimate", "--trace", str(trace), "--floor", "0"]) == cli.EXIT_INPUT
    trace.write_text("0,10.0.0.1,0.0.0.1\n")
    assert cli.main(["estimate", "--trace", str(trace), "--c", "2"]) == cli.EXIT_CONFIG


def _device_items(pool, path, fmt, slice_us, chunk, cudart):
    import ctypes
    from paper_1812_00282_b200 import traceio as tio
    got = []
    for t, dptr, n in tio.DeviceSlices(pool, path, fmt, slice_us, chunk=chunk):
        pool.synchronize()
        buf = np.empty(2 * n, dtype=np.uint32)
        if n:
            assert cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(dptr),
                                     ctypes.c_size_t(8 * n), 2) == 0
        got.append((t, buf[0::2].astype(np.uint64), buf[1::2].astype(np.uint64)))
    return got


def _cudart():
    import ctypes
    import nvidia.cuda_runtime
    return ctypes.CDLL(os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib",
                                    "libcudart.so.12"))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [traceio.BINARY, traceio.TEXT])
@pytest.mark.parametrize("bad_at", [5, 40_000, 70_001])
def test_device_slices_order_errors_like_the_reference(tmp_path, fmt, bad_at):
    """An out-of-order record: DeviceSlices yields exactly the slices the
    reference's reader + slice_stream yield before the error (those completed
    in the 32K-record batches before the failing one, traceio.py:60-145,
    188-230), then raises TraceOrderError at the same position."""
    import paper_1812_00282_b200 as vb
    rng = np.random.default_rng(bad_at)
    n = 90_000
    ts = np.cumsum(rng.integers(0, 40, n)).astype(np.uint64)
    ts[bad_at] = ts[bad_at - 1] - np.uint64(1) if ts[bad_at - 1] else np.uint64(0)
    if ts[bad_at] >= ts[bad_at - 1]:
        ts[bad_at - 1] += np.uint64(5)
    recs = traceio.make_records(ts, (0x0A000000 + rng.integers(0, 50, n)).astype(np.uint32),
                                rng.integers(1, 1 << 32, n, dtype=np.uint64).astype(np.uint32))
    path = tmp_path / ("t.bin" if fmt == traceio.BINARY else "t.csv")
    traceio.write_trace(path, recs, fmt)
    want, want_err = [], None
    try:
        for t, a, b in traceio.slice_stream(traceio.read_batches(path, fmt), 997):
            want.append((t, a, b))
    except traceio.TraceOrderError as e:
        want_err = str(e)
    assert want_err is not None
    pool = vb.AtPool(8, 2)
    cudart = _cudart()
    gen_items, got_err = [], None
    try:
        import ctypes
        for t, dptr, n_ in traceio.DeviceSlices(pool, path, fmt, 997):
            pool.synchronize()
            buf = np.empty(2 * n_, dtype=np.uint32)
            if n_:
                cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(dptr),
                                  ctypes.c_size_t(8 * n_), 2)
            gen_items.append((t, buf[0::2].astype(np.uint64), buf[1::2].astype(np.uint64)))
    except traceio.TraceOrderError as e:
        got_err = str(e)
    assert got_err == want_err
    assert [g[0] for g in gen_items] == [w[0] for w in want]
    for (t, a, b), (_, wa, wb) in zip(gen_items, want):
        assert np.array_equal(a, wa) and np.array_equal(b, wb), t


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [1, 7, 100, 1 << 22])
def test_device_slices_equal_slice_stream(tmp_path, chunk):
    import ctypes
    import nvidia.cuda_runtime
    import paper_1812_00282_b200 as vb
    cudart = ctypes.CDLL(os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib",
                                      "libcudart.so.12"))
    trace = _write_golden(tmp_path, "trace_bin", "t.bin")
    recs = traceio.read_trace(trace, traceio.BINARY)
    gaps = recs.copy()
    gaps["ts"][len(gaps) // 2:] += np.uint64(7_300_000)     # a run of empty slices mid-trace
    traceio.write_trace(tmp_path / "g.bin", gaps, traceio.BINARY)
    pool = vb.AtPool(8, 2)
    for path, records in ((trace, recs), (tmp_path / "g.bin", gaps)):
        want = list(traceio.slice_stream(iter([records]), 700_000))
        got = []
        for t, dptr, n in traceio.DeviceSlices(pool, path, traceio.BINARY, 700_000, chunk=chunk):
            pool.synchronize()
            buf = np.empty(2 * n, dtype=np.uint32)
            if n:
                assert cudart.cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(dptr),
                                         ctypes.c_size_t(8 * n), 2) == 0
            got.append((t, buf[0::2].astype(np.uint64), buf[1::2].astype(np.uint64)))
        assert [g[0] for g in got] == [w[0] for w in want]
        for (t, a, b), (_, wa, wb) in zip(got, want):
            assert np.array_equal(a, wa) and np.array_equal(b, wb), t


@pytest.mark.gpu
@pytest.mark.parametrize("name,argv", [
    ("compare_floor0", ["compare", "--floor", "0"]),
    ("compare_default", ["compare", "--k-prime", "4"]),
    ("est_dr", ["estimate", "--floor", "0", "--counter", "dr"]),
    ("est_ts", ["estimate", "--floor", "20", "--counter", "ts"]),
])
def test_cli_compare_and_comparator_counters_byte_identical(tmp_path, name, argv):
    """`compare` (AT, DR, TS pools all on the device) and `estimate --counter dr|ts`
    write the reference CLI's bytes (tests/golden/cli_compare.npz)."""
    trace = _write_golden(tmp_path, "trace_bin", "t.bin")
    out = tmp_path / "out.csv"
    common = ["--trace", str(trace), "--format", "binary", "--c", "14", "--g", "256", "--k", "6"]
    assert cli.main(argv[:1] + common + argv[1:] + ["--out", str(out)]) == 0
    assert out.read_bytes() == load("cli_compare.npz")[name].tobytes()


def test_cli_checkpoint_requires_the_at_pool(tmp_path, capsys):
    trace = _write_golden(tmp_path, "trace_bin", "t.bin")
    code = cli.main(["estimate", "--trace", str(trace), "--format", "binary", "--counter", "dr",
                     "--checkpoint", str(tmp_path / "p.atp1")])
    assert code == 2
    assert "requires the 'at' counter pool" in capsys.readouterr().err
