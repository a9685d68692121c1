"""Line-range sharding across GPUs.

Lines are independent, so a library is split into per-rank
byte ranges whose boundaries sit just past a newline; each rank runs the
whole-buffer codec on its shard with no data-path collective.  The only
exchange is an all-gather of four scalars per shard -- output bytes, records
written, input lines, first strict-error line -- from which every rank gets
its output offset, global 1-based error line numbers and the corpus totals.

Framing across shards: each shard emits ``record + '\\n'`` for every kept
record; if the whole input did not end with a newline, the single final
``'\\n'`` of the last shard that kept a record is dropped.  That reproduces
``b"\\n".join(kept) + (b"\\n" if kept and trailing)`` (pipeline.py:154-164)
for any shard count, including empty shards.
"""

from dataclasses import dataclass

import numpy as np


def shard_bounds(buf, world: int):
    """Byte offsets [b0, b1, ..., b_world]: near-equal ranges, each boundary
    moved forward to just past the next '\\n' (so every shard holds whole
    lines; shards may be empty)."""
    arr = buf if isinstance(buf, np.ndarray) else np.frombuffer(buf, np.uint8)
    n = arr.size
    cuts = [0]
    for r in range(1, world):
        c = max(cuts[-1], (n * r) // world)
        if c >= n:
            cuts.append(n)
            continue
        if c > 0 and arr[c - 1] == 0x0A:
            cuts.append(c)  # already just past a newline
            continue
        nl = np.flatnonzero(arr[c:] == 0x0A)
        cuts.append(c + int(nl[0]) + 1 if nl.size else n)
    cuts.append(n)
    return cuts


@dataclass
class ShardResult:
    """Per-shard scalars exchanged between ranks (4 values)."""
    out_bytes: int      # bytes this shard emitted, every kept record + '\n'
    lines: int          # records kept
    in_lines: int       # input lines in the shard
    err_line: int       # shard-local 1-based first strict error, 0 = none

    def as_list(self):
        return [self.out_bytes, self.lines, self.in_lines, self.err_line]


@dataclass
class GlobalView:
    out_offset: int     # where this rank's output starts in the framed stream
    out_bytes: int      # this rank's bytes after the final-newline adjustment
    total_out: int
    total_lines: int
    err_line: int       # global 1-based first error line, 0 = none
    err_rank: int       # rank that holds it, -1 = none


def combine(results, rank: int, trailing: bool) -> GlobalView:
    """Exclusive scan over the gathered per-shard scalars (any rank)."""
    out_off = 0
    line_base = 0
    err_line, err_rank = 0, -1
    last_kept = max((r for r, s in enumerate(results) if s.lines > 0), default=-1)
    sizes = []
    for r, s in enumerate(results):
        size = s.out_bytes
        if not trailing and r == last_kept:
            size -= 1  # the final '\n' is not part of the framed stream
        sizes.append(size)
        if s.err_line and not err_line:
            err_line, err_rank = line_base + s.err_line, r
        line_base += s.in_lines
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    out_off = int(offsets[rank])
    return GlobalView(out_offset=out_off, out_bytes=sizes[rank], total_out=int(offsets[-1]),
                      total_lines=sum(s.lines for s in results), err_line=err_line,
                      err_rank=err_rank)


def exchange(local: ShardResult, group=None):
    """All-gather the 4 scalars of every shard (torch.distributed, any
    backend: gloo on CPU, nccl on GPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    mine = torch.tensor(local.as_list(), dtype=torch.int64, device=dev)
    allv = [torch.zeros(4, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    return [ShardResult(*[int(x) for x in v.cpu().tolist()]) for v in allv]


def count_lines(arr) -> int:
    """Input lines of a newline-framed buffer (pipeline.py:141-146 split)."""
    if arr.size == 0:
        return 0
    return int(np.count_nonzero(arr == 0x0A)) + (0 if arr[-1] == 0x0A else 1)


def normalise(shard, framed_out, lines: int, err_line: int):
    """Turn one shard's framed stream output into (all-newlines output,
    ShardResult): the whole-buffer codec omits the final '\\n' when its input
    does not end with one, the shard protocol always carries it."""
    out = framed_out if isinstance(framed_out, (bytes, bytearray)) else bytes(framed_out)
    if lines and shard.size and shard[-1] != 0x0A:
        out = out + b"\n"
    return out, ShardResult(len(out), int(lines), count_lines(shard), int(err_line))


def gpu_codec(d, direction="compress", *, preprocess=False, lenient=False, device=None):
    """codec_fn running one shard through libzs on this rank's GPU."""
    from .pipeline import run_buffer

    def fn(shard):
        out, res = run_buffer(np.ascontiguousarray(shard), d, direction, preprocess=preprocess,
                              lenient=lenient, device=device)
        return normalise(shard, out.tobytes(), res.lines, res.err_line)
    return fn


def run_sharded(buf, codec_fn, rank: int, world: int, group=None):
    """Run `codec_fn(shard_bytes) -> (out_bytes_with_all_newlines, ShardResult)`
    on this rank's shard and return (my output slice, GlobalView).

    `codec_fn` must emit every kept record followed by '\\n' (the
    whole-buffer codec does, before the host trims the final newline) and
    report shard-local stats."""
    arr = buf if isinstance(buf, np.ndarray) else np.frombuffer(buf, np.uint8)
    cuts = shard_bounds(arr, world)
    shard = arr[cuts[rank]:cuts[rank + 1]]
    out, local = codec_fn(shard)
    results = exchange(local, group) if world > 1 else [local]
    trailing = arr.size == 0 or arr[-1] == 0x0A
    view = combine(results, rank, trailing)
    return bytes(out[:view.out_bytes]), view


def run_library(buf, d, direction="compress", *, preprocess=False, lenient=False, devices=None):
    """One library over several GPUs of this process (the multi-GPU form of
    ``run_buffer``; the reference spreads batches over a thread pool,
    pipeline.py:77-94).  The buffer is cut into one newline-aligned shard
    per device (shard_bounds), the shards run concurrently (one host thread
    per device; the C-ABI calls release the GIL), and the shard protocol
    combines the per-shard scalars (combine).  Returns (output uint8 array,
    GlobalView, per-shard zs_result list); the output equals the
    single-device stream byte for byte.  Strict-mode errors are reported,
    not raised: GlobalView.err_line is the global 1-based first bad line
    (the caller raises, as run_stream does)."""
    import threading

    from . import _lib
    from .pipeline import run_buffer
    arr = buf if isinstance(buf, np.ndarray) else np.frombuffer(buf, np.uint8)
    if devices is None:
        devices = list(range(max(1, _lib.device_count())))
    world = len(devices)
    cuts = shard_bounds(arr, world)
    outs, res, errs = [None] * world, [None] * world, []

    def work(r):
        try:
            sh = np.ascontiguousarray(arr[cuts[r]:cuts[r + 1]])
            o, z = run_buffer(sh, d, direction, preprocess=preprocess, lenient=lenient, device=devices[r])
            outs[r] = o.copy()
            res[r] = z
        except BaseException as e:  # re-raised in the caller's thread
            errs.append(e)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    locals_ = []
    for r in range(world):
        sh = arr[cuts[r]:cuts[r + 1]]
        body, loc = normalise(sh, outs[r].tobytes(), res[r].lines, res[r].err_line)
        outs[r] = body
        locals_.append(loc)
    trailing = arr.size == 0 or arr[-1] == 0x0A
    views = [combine(locals_, r, trailing) for r in range(world)]
    blob = b"".join(o[:v.out_bytes] for o, v in zip(outs, views))
    return np.frombuffer(blob, np.uint8), views[0], res

