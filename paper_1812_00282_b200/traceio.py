"""Trace ingest feeding the device path (reference: traceio.py).

Formats are the reference's: 16-byte little-endian binary records
``{u64 ts_us, u32 aip, u32 bip}`` (traceio.py:24) and text lines
``timestamp_us,aip,bip`` with dotted quads (traceio.py:109-145).  Timestamps
must be non-decreasing; violations raise the reference's TraceOrderError /
TraceParseError with the same messages and positions.

``DeviceSlices`` is the fast path: record chunks go to the GPU, one kernel
(``vate_trace_bucket``) packs them to 8-byte pairs and finds every slice start
(``ts // slice_us - base``, empty slices included, traceio.py:188-230), and
each slice is handed to the pipeline as a device pointer.  ``read_batches`` /
``slice_stream`` keep the reference's host API for callers that want arrays.
"""

from __future__ import annotations

import ctypes as C
import os
from ipaddress import AddressValueError, IPv4Address

import numpy as np

from ._lib import VATE_HOST, check, lib, ptr
from .errors import ConfigError, TraceOrderError, TraceParseError

RECORD_DTYPE = np.dtype([("ts", "<u8"), ("aip", "<u4"), ("bip", "<u4")])
RECORD_BYTES = RECORD_DTYPE.itemsize
TEXT = "text"
BINARY = "binary"
FORMATS = (TEXT, BINARY)
DEFAULT_BATCH = 1 << 15


def parse_ipv4(s: str) -> int:
    """Strict dotted quad (traceio.py:35-40)."""
    try:
        return int(IPv4Address(s))
    except AddressValueError as exc:
        raise ValueError(f"bad IPv4 address {s!r}: {exc}") from None


def format_ipv4(x: int) -> str:
    x = int(x)
    return f"{x >> 24 & 255}.{x >> 16 & 255}.{x >> 8 & 255}.{x & 255}"


def make_records(ts, aips, bips) -> np.ndarray:
    out = np.empty(len(ts), dtype=RECORD_DTYPE)
    out["ts"], out["aip"], out["bip"] = ts, aips, bips
    return out


def write_trace(path, records: np.ndarray, fmt: str) -> None:
    if fmt == BINARY:
        with open(path, "wb") as fh:
            fh.write(np.asarray(records).astype(RECORD_DTYPE, copy=False).tobytes())
    elif fmt == TEXT:
        with open(path, "w", encoding="ascii", newline="\n") as fh:
            for r in records:
                fh.write(f"{int(r['ts'])},{format_ipv4(r['aip'])},{format_ipv4(r['bip'])}\n")
    else:
        raise ConfigError(f"unknown trace format {fmt!r}")


# --- record readers (host) ------------------------------------------------------------

def _binary_chunks(path, chunk: int):
    """(byte offset, record array) chunks; truncation as traceio.py:85-91."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        offset = 0
        while offset < size:
            want = min(chunk * RECORD_BYTES, size - offset)
            data = fh.read(want)
            if len(data) % RECORD_BYTES:
                raise TraceParseError("truncated record at end of file",
                                      byte=offset + len(data) - len(data) % RECORD_BYTES)
            yield offset, np.frombuffer(data, dtype=RECORD_DTYPE)
            offset += len(data)


def _text_chunks(path, chunk: int):
    """(line number of the first record, record array) chunks (traceio.py:109-145)."""
    ts_buf, a_buf, b_buf = [], [], []
    first_line = 1
    with open(path, "r", encoding="ascii", newline=None) as fh:
        for lineno, line in enumerate(fh, 1):
            parts = line.rstrip("\n").split(",")
            if len(parts) != 3:
                raise TraceParseError(
                    f"expected 3 comma-separated fields, got {len(parts)}", line=lineno)
            try:
                ts = int(parts[0])
            except ValueError:
                raise TraceParseError(f"bad timestamp {parts[0]!r}", line=lineno) from None
            if ts < 0:
                raise TraceParseError(f"negative timestamp {ts}", line=lineno)
            try:
                aip, bip = parse_ipv4(parts[1]), parse_ipv4(parts[2])
            except ValueError as exc:
                raise TraceParseError(str(exc), line=lineno) from None
            if not ts_buf:
                first_line = lineno
            ts_buf.append(ts)
            a_buf.append(aip)
            b_buf.append(bip)
            if len(ts_buf) >= chunk:
                yield first_line, make_records(ts_buf, a_buf, b_buf)
                ts_buf, a_buf, b_buf = [], [], []
    if ts_buf:
        yield first_line, make_records(ts_buf, a_buf, b_buf)


def read_batches(path, fmt: str, batch_size: int = DEFAULT_BATCH):
    """Record batches in file order with the order checks (traceio.py:60-66)."""
    if fmt not in FORMATS:
        raise ConfigError(f"unknown trace format {fmt!r}")
    last = None
    chunks = _binary_chunks(path, batch_size) if fmt == BINARY else _text_chunks(path, batch_size)
    for pos, batch in chunks:
        ts = batch["ts"]
        where = (lambda i: dict(byte=pos + i * RECORD_BYTES)) if fmt == BINARY else \
            (lambda i: dict(line=pos + i))
        if last is not None and len(ts) and int(ts[0]) < last:
            raise TraceOrderError(f"timestamp {int(ts[0])} after {last}", **where(0))
        drops = np.nonzero(ts[1:] < ts[:-1])[0]
        if len(drops):
            i = int(drops[0]) + 1
            raise TraceOrderError(f"timestamp {int(ts[i])} after {int(ts[i - 1])}", **where(i))
        if len(ts):
            last = int(ts[-1])
        yield batch


def read_trace(path, fmt: str) -> np.ndarray:
    parts = list(read_batches(path, fmt))
    return np.concatenate(parts) if parts else np.empty(0, dtype=RECORD_DTYPE)


def slice_stream(batches, slice_us: int):
    """(t, aips, bips) host arrays per consecutive slice, empty ones included
    (traceio.py:188-230; first record's slice is 0, floor convention)."""
    if slice_us <= 0:
        raise ConfigError(f"slice duration must be positive, got {slice_us}")
    base, cur = None, 0
    pend_a, pend_b = [], []
    for batch in batches:
        if len(batch) == 0:
            continue
        ts = batch["ts"]
        if base is None:
            base = int(ts[0]) // slice_us
        sl = (ts // np.uint64(slice_us)).astype(np.int64) - base
        edges = np.flatnonzero(np.diff(sl)) + 1
        starts = np.concatenate([[0], edges])
        ends = np.concatenate([edges, [len(sl)]])
        for lo, hi in zip(starts, ends):
            s = int(sl[lo])
            while cur < s:
                yield cur, _cat(pend_a), _cat(pend_b)
                pend_a, pend_b = [], []
                cur += 1
            pend_a.append(batch["aip"][lo:hi].astype(np.uint64))
            pend_b.append(batch["bip"][lo:hi].astype(np.uint64))
    if base is not None:
        yield cur, _cat(pend_a), _cat(pend_b)


def _cat(parts):
    return np.concatenate(parts) if parts else np.empty(0, dtype=np.uint64)


# --- the device path -------------------------------------------------------------------

class DeviceSlices:
    """Iterate a trace as (t, device pointer to packed {u32 aip, u32 bip}, n).

    Each pointer is valid until the next item is requested; consumers that
    enqueue work on the pool's stream (Pipeline.step_fast / step_packed) are
    ordered before the buffer is rewritten.
    """

    def __init__(self, pool, path, fmt: str, slice_us: int, chunk: int = 1 << 22):
        if slice_us <= 0:
            raise ConfigError(f"slice duration must be positive, got {slice_us}")
        if fmt not in FORMATS:
            raise ConfigError(f"unknown trace format {fmt!r}")
        import torch   # device buffers only
        self._torch = torch
        self.pool, self.path, self.fmt = pool, path, fmt
        self.slice_us, self.chunk = int(slice_us), int(chunk)
        self._bufs = [None, None]

    def _buffer(self, which: int, pairs: int):
        b = self._bufs[which]
        if b is None or b.numel() < 2 * pairs:
            self.pool.synchronize()   # the old buffer may still be read by queued scans
            b = self._torch.empty(2 * max(pairs, 1), dtype=self._torch.int32,
                                  device=f"cuda:{self.pool.device}")
            self._bufs[which] = b
        return b

    def __iter__(self):
        h = self.pool.handle
        us = self.slice_us
        base = None
        cur = 0          # slice id of the carried (possibly incomplete) slice
        carry_n = 0      # its packed pairs, at the start of buffer `which`
        which = 0
        prev_ts, has_prev = 0, 0
        chunks = (_binary_chunks(self.path, self.chunk) if self.fmt == BINARY
                  else _text_chunks(self.path, self.chunk))
        for pos, rec in chunks:
            n = len(rec)
            if n == 0:
                continue
            rec = np.ascontiguousarray(rec)
            ts0, ts1 = int(rec["ts"][0]), int(rec["ts"][-1])
            if base is None:
                base = ts0 // us
                cur = 0
            first, last = ts0 // us - base, ts1 // us - base
            buf_old = self._bufs[which]
            if carry_n and first > cur:               # the carried slice is complete
                yield cur, buf_old.data_ptr(), carry_n
                carry_n = 0
                cur += 1
            cont = carry_n > 0 and first == cur
            nxt = which ^ 1 if cont else which
            dst = self._buffer(nxt, (carry_n if cont else 0) + n)
            if cont:
                check(lib.vate_copy_device(h, dst.data_ptr(), buf_old.data_ptr(), carry_n * 8))
            off = carry_n if cont else 0
            if not cont:
                while cur < first:                   # empty slices before this chunk
                    yield cur, dst.data_ptr(), 0
                    cur += 1
            nsl = max(last - first + 1, 1) if last >= first else 1
            starts = np.empty(nsl, dtype=np.uint64)
            viol = C.c_int64()
            check(lib.vate_trace_bucket(h, ptr(rec.view(np.uint8)), n, VATE_HOST, us,
                                        first + base, prev_ts, has_prev, dst.data_ptr(), off,
                                        nsl, ptr(starts), C.byref(viol)))
            if viol.value >= 0 or last < first:
                i = max(viol.value, 0)
                where = (dict(byte=pos + i * RECORD_BYTES) if self.fmt == BINARY
                         else dict(line=pos + i))
                prev = prev_ts if i == 0 else int(rec["ts"][i - 1])
                raise TraceOrderError(f"timestamp {int(rec['ts'][i])} after {prev}", **where)
            total = off + n
            starts[0] = 0 if cont else starts[0]
            for q in range(nsl - 1):                 # every slice but the last is complete
                lo, hi = int(starts[q]), int(starts[q + 1])
                yield first + q, dst.data_ptr() + 8 * lo, hi - lo
            lo = int(starts[nsl - 1])
            if lo:                                   # carry the last slice to the buffer start
                other = self._buffer(nxt ^ 1, total - lo)
                check(lib.vate_copy_device(h, other.data_ptr(), dst.data_ptr() + 8 * lo,
                                           (total - lo) * 8))
                which = nxt ^ 1
            else:
                which = nxt
            carry_n = total - lo
            cur = last
            prev_ts, has_prev = ts1, 1
        if base is not None:
            yield cur, self._bufs[which].data_ptr(), carry_n
