"""Random access into a compressed library held in HBM.

ZSMILES keeps one record per line, so a line can be fetched and decoded on
its own (pkg/README.md:106-110: "grab line i, decode line
i").  ``RecordIndex`` uploads a compressed buffer once, builds its record
offsets on the device (zs_index_build) and decodes any set of records in
one launch sequence (zs_decode_records).  Bad records raise the same
exceptions as the reference ``decompress_line`` (codec.py:88-92):
UnknownCode(code, offset) and TruncatedEscape(offset).

Device buffers are torch CUDA tensors (plumbing only; the work is in
libzs.so).  There is no CPU fallback.
"""

import ctypes

import numpy as np

from . import _lib
from .errors import TruncatedEscape, UnknownCode


class RecordIndex:
    def __init__(self, comp, d, device=None):
        import torch
        self._ctx = _lib.context(device)
        self._dev = torch.device("cuda", self._ctx.device)
        self._d = d
        if isinstance(comp, torch.Tensor):
            self._comp = comp.to(self._dev, torch.uint8).contiguous()
        else:
            arr = comp if isinstance(comp, np.ndarray) else np.frombuffer(bytes(comp), np.uint8)
            self._comp = torch.from_numpy(np.array(arr, np.uint8, copy=True)).to(self._dev)
        n = int(self._comp.numel())
        nrec = ctypes.c_int64(0)
        cap = n // 2 + 2
        with self._ctx.lock:
            self._ctx.follow_torch_stream()
            for _ in range(2):
                self._off = torch.empty(cap, dtype=torch.int64, device=self._dev)
                rc = self._ctx.lib.zs_index_build(self._ctx.h, self._comp.data_ptr() if n else None, n,
                                                  self._off.data_ptr(), cap, ctypes.byref(nrec))
                if rc == _lib.ZS_E_CAPACITY:
                    cap = nrec.value + 1
                    continue
                self._ctx.check(rc, "zs_index_build")
                break
            else:
                raise _lib.ZsCudaError(f"zs_index_build: offsets still too small ({nrec.value} records)")
        self._n = int(nrec.value)

    def __len__(self):
        return self._n

    def decode_packed(self, indices):
        """Records `indices` decoded into one buffer: (data uint8[total],
        offsets int64[k + 1]); record j is data[offsets[j]:offsets[j + 1]].
        The bulk form of ``decode`` (no per-record Python objects)."""
        import torch
        idx = np.ascontiguousarray(indices if isinstance(indices, np.ndarray) else list(indices), np.int64)
        k = idx.size
        if k == 0:
            return np.zeros(0, np.uint8), np.zeros(1, np.int64)
        if idx.min() < 0 or idx.max() >= self._n:
            raise IndexError("record index out of range")
        d_idx = torch.from_numpy(idx).to(self._dev)
        d_off = torch.empty(k + 1, dtype=torch.int64, device=self._dev)
        d_st = torch.empty(k, dtype=torch.int8, device=self._dev)
        d_ep = torch.empty(k, dtype=torch.int64, device=self._dev)
        total = ctypes.c_int64(0)
        cap = max(64, 96 * k)  # ~2x the mean record (45 B); a second call sizes it exactly
        with self._ctx.lock:
            self._ctx.set_dictionary(self._d)
            self._ctx.follow_torch_stream()
            for _ in range(2):
                d_out = torch.empty(cap, dtype=torch.uint8, device=self._dev)
                rc = self._ctx.lib.zs_decode_records(self._ctx.h, self._comp.data_ptr(), self._off.data_ptr(),
                                                     self._n, d_idx.data_ptr(), k, d_out.data_ptr(), cap,
                                                     d_off.data_ptr(), d_st.data_ptr(), d_ep.data_ptr(),
                                                     ctypes.byref(total))
                if rc == _lib.ZS_E_CAPACITY:
                    cap = total.value + 64
                    continue
                self._ctx.check(rc, "zs_decode_records")
                break
            else:
                raise _lib.ZsCudaError(f"zs_decode_records: output still too small ({total.value} bytes)")
        st = d_st.cpu().numpy()
        bad = np.flatnonzero(st)
        if bad.size:  # the first bad record in request order, as decompress_line would raise
            j = int(bad[0])
            ep = int(d_ep[j].item())
            if st[j] == 1:
                raise UnknownCode(ep >> 40, ep & ((1 << 40) - 1))
            raise TruncatedEscape(ep)
        return d_out[:total.value].cpu().numpy(), d_off.cpu().numpy()

    def decode(self, indices):
        """Decoded bytes of records `indices` (any order, repeats allowed)."""
        data, off = self.decode_packed(indices)
        raw = data.tobytes()
        return [raw[a:b] for a, b in zip(off[:-1].tolist(), off[1:].tolist())]

    def __getitem__(self, i):
        return self.decode([i])[0]
