"""Trace ingest feeding the device path (reference: traceio.py).

Formats are the reference's: 16-byte little-endian binary records
``{u64 ts_us, u32 aip, u32 bip}`` (traceio.py:24) and text lines
``timestamp_us,aip,bip`` with dotted quads (traceio.py:109-145).  Timestamps
must be non-decreasing; violations raise the reference's TraceOrderError /
TraceParseError with the same messages and positions.

``DeviceSlices`` is the fast path (the ``vate_tracer_*`` ABI): record chunks
go to the GPU from pinned buffers, one kernel packs them to 8-byte pairs and
emits one run per slice change (``ts // slice_us - base``, empty slices
yielded lazily, traceio.py:188-230), and each slice is handed to the pipeline
as a device pointer.  ``read_batches`` /
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
    """(line number of the first record, record array) chunks (traceio.py:109-145).
    Timestamp order is checked line by line as the reference does, so an
    out-of-order line is reported before any malformed line after it."""
    ts_buf, a_buf, b_buf = [], [], []
    first_line = 1
    last_ts = None
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
            if last_ts is not None and ts < last_ts:
                raise TraceOrderError(f"timestamp {ts} after {last_ts}", line=lineno)
            last_ts = ts
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

_POOL = None


def _reader_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=DeviceSlices.READERS,
                                   thread_name_prefix="vate-trace")
    return _POOL


def _pread_full(fd, mv, offset) -> int:
    """Read len(mv) bytes at offset (fewer only at the end of the file)."""
    got = 0
    while got < len(mv):
        r = os.preadv(fd, [mv[got:]], offset + got)
        if r <= 0:
            break
        got += r
    return got


class DeviceSlices:
    """Iterate a trace as (t, device pointer to packed {u32 aip, u32 bip}, n).

    Line-rate form (csrc/vate_trace.cu, ``vate_tracer_*``): binary chunks are
    read from the file straight into one of two pinned staging buffers while
    the GPU works on the previous chunk; the records go to the device
    asynchronously, where one kernel packs them to 8-byte pairs and emits one
    (slice, offset) run per slice change; the reader turns the runs into
    slices, emitting empty slices lazily (an idle gap costs nothing), and
    carries the last, possibly incomplete slice into the next chunk's buffer
    on the device.  Consumers enqueue their scans on the pool's stream, which
    the tracer orders after each chunk by event; a buffer is rewritten only
    after the scans enqueued for it.  Errors keep the reference's semantics
    (traceio.py:77-145): slices completed before the failing 32K-record batch
    are yielded first, then TraceOrderError / TraceParseError is raised with
    the reference's position.
    """

    REF_BATCH = DEFAULT_BATCH  # the reference reader's batch (error granularity)
    READERS = 4                # file reader threads per chunk

    def __init__(self, pool, path, fmt: str, slice_us: int, chunk: int = 1 << 23):
        if slice_us <= 0:
            raise ConfigError(f"slice duration must be positive, got {slice_us}")
        if fmt not in FORMATS:
            raise ConfigError(f"unknown trace format {fmt!r}")
        self.pool, self.path, self.fmt = pool, path, fmt
        self.slice_us = int(slice_us)
        # text is parsed on the host in the reference's 32K-line batches; binary
        # chunks are whole reference batches (exact error semantics) -- a chunk
        # below one batch is for exercising the carry logic only
        chunk = int(chunk) if fmt == BINARY else self.REF_BATCH
        if chunk >= self.REF_BATCH:
            chunk = chunk // self.REF_BATCH * self.REF_BATCH
        self.chunk = max(1, chunk)
        self._x = None
        self.bytes_read = 0

    def _tracer(self):
        if self._x is None:
            h = C.c_void_p()
            check(lib.vate_tracer_create(C.byref(h), self.pool.handle, self.chunk, self.slice_us))
            self._x = h
            self._host = []
            for slot in range(2):
                ptr_ = C.c_void_p()
                check(lib.vate_tracer_buffer(h, slot, C.byref(ptr_)))
                raw = (C.c_uint8 * (self.chunk * RECORD_BYTES)).from_address(ptr_.value)
                self._host.append(np.frombuffer(raw, dtype=RECORD_DTYPE))
            self._runs = np.empty(2 * self.chunk, dtype=np.uint64)
            self._pairs = [0, 0]
        return self._x

    def close(self):
        if self._x is not None:
            h = self.pool.handle
            if h is not None and h.value:
                self.pool.synchronize()   # scans queued on the pool may still read its buffers
            lib.vate_tracer_destroy(self._x)
            self._x = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _fill(self, slot: int):
        """Generator of (position, n) with the chunk's records in the slot's pinned
        buffer (its previous H2D is waited for first)."""
        x = self._tracer()

        def wait(slot_):
            ptr_ = C.c_void_p()
            check(lib.vate_tracer_buffer(x, slot_, C.byref(ptr_)))   # its last H2D is done
            return self._host[slot_]

        if self.fmt == BINARY:
            size = os.path.getsize(self.path)
            fd = os.open(self.path, os.O_RDONLY)
            pool_ = _reader_pool()
            try:
                offset = 0
                while offset < size:
                    buf = wait(slot)
                    want = min(self.chunk * RECORD_BYTES, size - offset)
                    mv = memoryview(buf.view(np.uint8))[:want]
                    # READERS threads read their parts of the chunk into the pinned
                    # buffer in parallel (os.preadv releases the GIL)
                    part = -(-want // self.READERS // 4096) * 4096
                    jobs = [pool_.submit(_pread_full, fd, mv[lo:min(want, lo + part)], offset + lo)
                            for lo in range(0, want, part)]
                    parts = [j.result() for j in jobs]
                    got = 0
                    for (lo, n_) in zip(range(0, want, part), parts):
                        if n_ < min(want, lo + part) - lo:   # a short read: the file shrank
                            got = lo + n_
                            break
                        got = lo + n_
                    self.bytes_read += got
                    if got % RECORD_BYTES:   # traceio.py:85-91
                        full = got - got % RECORD_BYTES
                        if full:
                            yield offset, full // RECORD_BYTES, slot
                        raise TraceParseError("truncated record at end of file",
                                              byte=offset + full)
                    yield offset, got // RECORD_BYTES, slot
                    offset += got
                    slot ^= 1
            finally:
                os.close(fd)
        else:
            for first_line, rec in _text_chunks(self.path, self.chunk):
                buf = wait(slot)
                buf[:len(rec)] = rec
                yield first_line, len(rec), slot
                slot ^= 1

    def __iter__(self):
        try:
            yield from self._iter()
        finally:                      # the tracer's buffers go with the iteration
            self.close()

    def _iter(self):
        x = self._tracer()
        us = self.slice_us
        base = None
        cur = 0              # the next slice to yield
        carry = None         # (slot, pair offset, pairs) of the carried slice `cur`
        prev_ts, has_prev = 0, 0
        pending = None       # the submitted, not yet collected chunk
        reader = self._fill(0)
        err = None

        def next_chunk():
            nonlocal err
            if err is not None:
                return None
            try:
                return next(reader)
            except StopIteration:
                return None
            except (TraceParseError, TraceOrderError) as e:
                err = e
                return None

        def submit(item):
            nonlocal base, prev_ts, has_prev, carry
            pos, n, slot = item
            rec = self._host[slot]
            ts0, ts1 = int(rec["ts"][0]), int(rec["ts"][n - 1])
            if base is None:
                base = ts0 // us
            first = ts0 // us - base
            c_off, c_n = (carry[1], carry[2]) if carry is not None else (0, 0)
            check(lib.vate_tracer_submit(x, slot, n, first + base, prev_ts, has_prev, c_off, c_n))
            sub = dict(pos=pos, n=n, slot=slot, first=first, carried=c_n, prev_ts=prev_ts)
            prev_ts, has_prev = ts1, 1
            return sub

        item = next_chunk()
        if item is not None:
            pending = submit(item)
        while pending is not None:
            item = next_chunk()          # read the next chunk while the GPU works
            sub = pending
            nr, viol, pairs = C.c_uint64(), C.c_int64(), C.c_void_p()
            check(lib.vate_tracer_collect(x, sub["slot"], ptr(self._runs), self.chunk * 2,
                                          C.byref(nr), C.byref(viol), C.byref(pairs)))
            runs = self._runs[:2 * nr.value].reshape(-1, 2)
            runs = runs[np.argsort(runs[:, 1], kind="stable")]
            base_ptr = self._pairs[sub["slot"]] = pairs.value
            carried, total = sub["carried"], sub["carried"] + sub["n"]
            # an order violation: the reference's reader raises at the 32K-record
            # batch holding it, after slice_stream consumed the batches before
            stop_at = None
            if viol.value >= 0:
                g0 = sub["pos"] // RECORD_BYTES if self.fmt == BINARY else sub["pos"] - 1
                batch = (g0 + viol.value) // self.REF_BATCH * self.REF_BATCH
                stop_at = carried + max(0, batch - g0)
            consumed = (lambda off: stop_at is None or off < stop_at)
            starts = [int(o) for o in runs[:, 1]]
            slices = [sub["first"] + int(s_) for s_ in runs[:, 0]]
            if carry is not None:
                if slices and slices[0] == cur:
                    starts[0] = 0                      # the first run extends the carried slice
                elif consumed(carried):                # its successor's first record completes it
                    yield cur, base_ptr, carry[2]
                    cur += 1
            carry = None
            for r, (s_, lo) in enumerate(zip(slices, starts)):
                first_rec = carried if r == 0 else lo
                if not consumed(first_rec):
                    break
                while cur < s_:                        # empty slices, lazily
                    yield cur, base_ptr, 0
                    cur += 1
                hi = starts[r + 1] if r + 1 < len(starts) else total
                if r + 1 == len(starts):               # may continue in the next chunk
                    carry = (sub["slot"], lo, hi - lo)
                    break
                if not consumed(hi):
                    break
                yield s_, base_ptr + 8 * lo, hi - lo
                cur = s_ + 1
            if stop_at is not None:
                rec = self._host[sub["slot"]]
                i = viol.value
                prev = sub["prev_ts"] if i == 0 else int(rec["ts"][i - 1])
                where = (dict(byte=sub["pos"] + i * RECORD_BYTES) if self.fmt == BINARY
                         else dict(line=sub["pos"] + i))
                raise TraceOrderError(f"timestamp {int(rec['ts'][i])} after {prev}", **where)
            check(lib.vate_tracer_release(x, sub["slot"]))
            pending = submit(item) if item is not None else None
        if err is not None:
            raise err
        if carry is not None:                          # the last slice, where it lies
            yield cur, self._pairs[carry[0]] + 8 * carry[1], carry[2]
