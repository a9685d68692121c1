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
            for _ in range(2):
                self._off = torch.empty(cap, dtype=torch.int64, device=self._dev)
                rc = self._ctx.lib.zs_index_build(self._ctx.h, self._comp.data_ptr() if n else None, n,
                                                  self._off.data_ptr(), cap, ctypes.byref(nrec))
                if rc == _lib.ZS_E_CAPACITY:
                    cap = nrec.value + 1
                    continue
                self._ctx.check(rc, "zs_index_build")
                break
        self._n = int(nrec.value)

    def __len__(self):
        return self._n

    def decode(self, indices):
        """Decoded bytes of records `indices` (any order, repeats allowed)."""
        import torch
        idx = np.asarray(list(indices) if not isinstance(indices, np.ndarray) else indices, np.int64)
        k = idx.size
        if k == 0:
            return []
        if idx.min() < 0 or idx.max() >= self._n:
            raise IndexError("record index out of range")
        d_idx = torch.from_numpy(idx).to(self._dev)
        d_off = torch.empty(k + 1, dtype=torch.int64, device=self._dev)
        d_st = torch.empty(k, dtype=torch.int8, device=self._dev)
        d_ep = torch.empty(k, dtype=torch.int64, device=self._dev)
        total = ctypes.c_int64(0)
        cap = max(64, 8 * k)
        with self._ctx.lock:
            self._ctx.set_dictionary(self._d)
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
        out = d_out[:total.value].cpu().numpy().tobytes()
        off = d_off.cpu().numpy()
        st = d_st.cpu().numpy()
        ep = d_ep.cpu().numpy()
        res = []
        for j in range(k):
            if st[j] == 1:
                raise UnknownCode(int(ep[j] >> 40), int(ep[j] & ((1 << 40) - 1)))
            if st[j] == 2:
                raise TruncatedEscape(int(ep[j]))
            res.append(out[off[j]:off[j + 1]])
        return res

    def __getitem__(self, i):
        return self.decode([i])[0]
