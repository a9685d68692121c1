"""Whole-file compression / decompression (reference pipeline.py:129-167).

``run_stream`` hands the whole newline-framed buffer to libzs in one call
(zs_compress_host / zs_decompress_host): framing, the CR policy, ring
renumbering, the parse, strict/lenient handling and the stats are all
computed on the GPU in the fused tile kernels.  Output bytes are identical
to the reference for any ``workers`` / ``batch_lines`` (both accepted for
API compatibility; the GPU does not batch by lines).

Strict-mode errors: like the reference, the batches before the failing
line's ``batch_lines`` batch are written to ``dst`` before ``LineError``
is raised (pipeline.py:154-161 writes batches in order as they finish).
"""

import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import LineError, from_kind

BATCH_LINES = 4096


@dataclass
class CorpusStats:
    lines: int = 0
    input_bytes: int = 0
    output_bytes: int = 0
    escapes: int = 0
    skipped: int = 0
    flagged: int = 0
    elapsed: float = 0.0

    @property
    def ratio(self) -> float:
        return 1.0 if self.input_bytes == 0 else self.output_bytes / self.input_bytes

    def format_line(self) -> str:
        return (f"lines={self.lines} in_bytes={self.input_bytes} "
                f"out_bytes={self.output_bytes} ratio={self.ratio:.6f} "
                f"escapes={self.escapes} elapsed_ms={int(round(self.elapsed * 1000))}")


def compute_ratio(stats: CorpusStats) -> float:
    """Output over input bytes (newlines included); 1.0 for empty input."""
    return stats.ratio


def run_buffer(buf, d, direction="compress", *, preprocess=False, lenient=False, device=None, out=None):
    """One newline-framed buffer through the GPU.  Returns (output bytes,
    zs_result).  `buf` may be bytes or a uint8 numpy array (pinned memory
    gives full PCIe rate); `out`, if given, is a uint8 array used as the
    output buffer when it is large enough (the result is a view of it)."""
    if direction not in ("compress", "decompress"):
        raise ValueError(f"bad direction {direction!r}")
    arr = buf if isinstance(buf, np.ndarray) else np.frombuffer(buf, np.uint8)
    ctx = _lib.context(device)
    flags = (_lib.F_PREPROCESS if preprocess else 0) | (_lib.F_LENIENT if lenient else 0)
    res = _lib.Result()
    n = arr.size
    with ctx.lock:
        ctx.set_dictionary(d)
        if direction == "compress":
            cap = ctx.lib.zs_compress_bound(n)
            fn = ctx.lib.zs_compress_host
        else:
            cap = max(4 * n + 64, 1024)
            fn = ctx.lib.zs_decompress_host
        given = out
        for _ in range(3):
            if given is not None and given.size >= cap:
                out, cap = given, given.size
            else:
                out = np.empty(cap, np.uint8)
            rc = fn(ctx.h, _lib.ptr(arr), n, _lib.ptr(out), cap, flags, res)
            if rc == _lib.ZS_E_CAPACITY:
                cap = res.out_bytes + 64
                continue
            ctx.check(rc, "zs_compress_host" if direction == "compress" else "zs_decompress_host")
            break
        else:
            raise _lib.ZsCudaError(f"{direction}: output buffer still too small after 3 attempts "
                                   f"({res.out_bytes} bytes needed)")
    return out[:res.out_bytes], res


SEGMENT_BYTES = 256 << 20


def _host_buffer(slot, nbytes, device):
    """Page-locked staging for run_stream (cached per context and slot)."""
    return _lib.context(device).pinned(slot, nbytes)


def _read_into(src, buf, at, n):
    """Read up to n bytes of src into buf[at:at + n]; returns the count."""
    readinto = getattr(src, "readinto", None)
    got = 0
    mv = memoryview(buf)
    while got < n:
        if readinto is not None:
            k = readinto(mv[at + got:at + n])
            if not k:
                break
        else:
            chunk = src.read(n - got)
            if not chunk:
                break
            k = len(chunk)
            buf[at + got:at + got + k] = np.frombuffer(chunk, np.uint8)
        got += k
    return got


def _last_nl(arr, lo, hi):
    """Index of the last '\\n' in arr[lo:hi], or -1 (scans back in blocks)."""
    end = hi
    while end > lo:
        beg = max(lo, end - (1 << 20))
        nz = np.flatnonzero(arr[beg:end] == 10)
        if nz.size:
            return beg + int(nz[-1])
        end = beg
    return -1


def _cut_keeping_last(arr, n, m):
    """Offset in arr[:n] ('\\n'-terminated records) after which exactly the
    last m records remain (0 if there are only m)."""
    need, end = m + 1, n
    while end > 0:
        beg = max(0, end - (1 << 20))
        nz = np.flatnonzero(arr[beg:end] == 10)
        if nz.size >= need:
            return beg + int(nz[nz.size - need]) + 1
        need -= nz.size
        end = beg
    return 0


def run_stream(src, dst, d, direction="compress", *, preprocess=False, lenient=False, workers=1,
               batch_lines=BATCH_LINES, device=None, segment_bytes=SEGMENT_BYTES) -> CorpusStats:
    """Stream src to dst through the GPU codec; returns exact corpus totals.

    The input is read (``readinto``, no intermediate copies) into page-locked
    staging in `segment_bytes` pieces cut at newlines, so files larger than
    host or device memory stream through at PCIe rate (each segment is one
    zs_*_host call, itself pipelined in chunks on three streams); output is
    written from page-locked staging without copies.  Output bytes equal the
    reference's `b"\\n".join(kept records) + ("\\n" if kept and trailing)`
    (pipeline.py:148-166) for any segment size: a segment's final '\\n' is
    held back until the next kept record or the end of the input.

    Strict mode raises LineError (1-based) for the first bad line, after
    writing every complete `batch_lines` batch before it like the reference
    (pipeline.py:154-161); lenient mode drops undecodable / carriage-return
    lines (``skipped``) and keeps unpreprocessable ones raw (``flagged``).

    The page-locked staging belongs to the device's context, so concurrent
    run_stream calls on one device run one after the other (the context
    lock is held for the whole stream); `dst.write` receives bytes."""
    if direction not in ("compress", "decompress"):
        raise ValueError(f"bad direction {direction!r}")
    # the page-locked staging is per device: one stream at a time per device
    with _stream_lock(device):
        return _run_stream(src, dst, d, direction, preprocess, lenient, batch_lines, device, segment_bytes)


_locks_guard = threading.Lock()
_stream_locks = {}


def _stream_lock(device):
    if device is None:
        device = int(os.environ.get("ZS_DEVICE", "0"))  # _lib.context's default
    key = device if isinstance(device, int) else id(device)
    with _locks_guard:
        return _stream_locks.setdefault(key, threading.Lock())


def _run_stream(src, dst, d, direction, preprocess, lenient, batch_lines, device, segment_bytes):
    t0 = time.perf_counter()
    bl = max(1, batch_lines)
    st = CorpusStats()
    line_base = 0        # input lines before the current segment (strict mode: = output records)
    written = 0          # strict mode: output records written (a multiple of batch_lines)
    pend = bytearray()   # strict mode: records of lines [written, line_base), '\\n'-terminated
    held_nl = False      # the written output's last '\\n', held back until more output follows

    def emit(*parts):
        nonlocal held_nl
        if held_nl:
            dst.write(b"\n")
            st.output_bytes += 1
        for body in parts:
            if len(body):
                dst.write(bytes(body))  # a copy: the staging is reused (the reference writes bytes)
                st.output_bytes += len(body)
        held_nl = False

    seg_bytes = max(1, segment_bytes)
    inbuf = _host_buffer("stream_in", seg_bytes + 4096, device)
    carry = 0            # bytes of a partial last line at the front of inbuf
    last_byte = None
    while True:
        if inbuf.size < carry + seg_bytes:  # a line longer than the staging: grow, keep the carry
            keep = inbuf[:carry].copy()
            inbuf = _host_buffer("stream_in", 2 * (carry + seg_bytes), device)
            inbuf[:carry] = keep
        got = _read_into(src, inbuf, carry, seg_bytes)
        total = carry + got
        final = got == 0
        if not final:
            last_byte = int(inbuf[total - 1])
            nl = _last_nl(inbuf, carry, total)
            if nl < 0:
                carry = total
                continue
            cut = nl + 1
        else:
            cut = total
            if cut == 0:
                break
        seg = inbuf[:cut]
        st.input_bytes += cut
        cap = (2 * cut + 64) if direction == "compress" else max(4 * cut + 64, 1024)
        out, res = run_buffer(seg, d, direction, preprocess=preprocess, lenient=lenient, device=device,
                              out=_host_buffer("stream_out", cap, device))
        if res.err_line:
            gl = line_base + int(res.err_line)
            cause = from_kind(res.err_kind, res.err_offset, tuple(res.err_ids), res.err_code)
            keep = ((gl - 1) // bl) * bl
            blob = bytearray()
            if keep > written:
                nrec = min(keep, line_base) - written
                if nrec > 0:
                    pos = _cut_keeping_last(np.frombuffer(pend, np.uint8), len(pend),
                                            (line_base - written) - nrec)
                    blob += pend[:pos]
                if keep > line_base:
                    nls = np.flatnonzero(seg == 0x0A)
                    end = int(nls[keep - line_base - 1]) + 1
                    part, _ = run_buffer(seg[:end].copy(), d, direction, preprocess=preprocess,
                                         lenient=lenient, device=device)
                    blob += part.tobytes()
            if blob.endswith(b"\n"):
                blob = blob[:-1]
            if blob:
                emit(blob)
            raise LineError(gl, cause)
        st.lines += res.lines
        st.escapes += res.escapes
        st.skipped += res.skipped
        st.flagged += res.flagged
        ob = int(res.out_bytes)
        outv = memoryview(out)[:ob]
        if lenient:
            if ob:
                nl_end = out[ob - 1] == 10
                emit(outv[:ob - 1] if nl_end else outv)
                held_nl = bool(nl_end)
        else:
            line_base += int(res.lines)
            flush_to = (line_base // bl) * bl
            if (not final or last_byte == 10) and flush_to > written:
                # whole batches leave; the rest waits for the next segment
                c = _cut_keeping_last(out, ob, line_base - flush_to)
                if c > 0:
                    emit(pend, outv[:c - 1])
                else:  # (cannot happen: a new batch ends inside this segment)
                    emit(pend[:-1])
                held_nl = True
                pend = bytearray(outv[c:])
                written = flush_to
            else:
                pend += outv
        rem = total - cut
        if rem:
            inbuf[:rem] = inbuf[cut:total].copy()
        carry = rem
        if final:
            break
    tail = bytes(pend)  # strict mode: the records after the last whole batch
    if tail.endswith(b"\n"):
        emit(tail[:-1])
        held_nl = True
    elif tail:
        emit(tail)
    if held_nl and last_byte == 10:
        dst.write(b"\n")
        st.output_bytes += 1
    st.elapsed = time.perf_counter() - t0
    return st
