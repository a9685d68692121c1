"""ctypes binding of libzs.so (include/zs.h) and per-device contexts.

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2404_19391_b200.build``).  There is no CPU fallback: if
the library is missing, or no CUDA device is present when a compute call is
made, this module raises.
"""

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ZS_LIB: an alternative build of the same library (tools load the
# -DZS_PHASES=1 measurement build, libzs_phases.so, this way)
LIB_PATH = os.environ.get("ZS_LIB") or os.path.join(_HERE, "libzs.so")

ZS_OK, ZS_E_ARG, ZS_E_CUDA, ZS_E_NOMEM, ZS_E_NODICT, ZS_E_CAPACITY = 0, -1, -2, -3, -4, -5
F_PREPROCESS, F_LENIENT = 1, 2

# every symbol include/zs.h declares
EXPORTS = (
    "zs_ctx_create", "zs_ctx_destroy", "zs_last_error", "zs_device_count", "zs_set_dictionary",
    "zs_dictionary_fast", "zs_compress_batch", "zs_decompress_sizes", "zs_decompress_fill",
    "zs_preprocess_batch", "zs_compress_device", "zs_decompress_device", "zs_compress_host",
    "zs_decompress_host", "zs_compress_bound", "zs_decompress_bound", "zs_last_kernel_ms",
    "zs_last_kernel", "zs_stream", "zs_set_stream", "zs_index_build", "zs_decode_records",
    "zs_train_count", "zs_train_rows", "zs_train_load", "zs_train_select", "zs_overlap_batch",
    "zs_host_alloc", "zs_host_free",
)
# measurement / inspection hooks (include/zs_debug.h), not part of the boundary
DEBUG_EXPORTS = ("zs_build_tables_host", "zs_build_t2_host", "zs_set_transducer", "zs_set_phase_timing",
                 "zs_last_phase_cycles", "zs_debug_chunk_cuts")


class Result(ctypes.Structure):
    """zs_result (include/zs.h)"""
    _fields_ = [("lines", ctypes.c_int64), ("in_bytes", ctypes.c_int64),
                ("out_bytes", ctypes.c_int64), ("escapes", ctypes.c_int64),
                ("skipped", ctypes.c_int64), ("flagged", ctypes.c_int64),
                ("err_line", ctypes.c_int64), ("err_kind", ctypes.c_int32),
                ("err_code", ctypes.c_int32), ("err_offset", ctypes.c_int64),
                ("err_ids", ctypes.c_uint64 * 2), ("gpu_launches", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class ZsCudaError(RuntimeError):
    pass


_lib = None
_lib_lock = threading.Lock()


def load():
    """Load libzs.so (raises if it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        sig = {
            "zs_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
            "zs_ctx_destroy": (ctypes.c_int, [P]),
            "zs_last_error": (ctypes.c_char_p, [P]),
            "zs_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
            "zs_set_dictionary": (ctypes.c_int, [P, P, P, I32, P, P, P, P]),
            "zs_dictionary_fast": (ctypes.c_int, [P]),
            "zs_compress_batch": (ctypes.c_int, [P, P, P, I64, P, P, P]),
            "zs_decompress_sizes": (ctypes.c_int, [P, P, P, I64, P, P, P, P, P]),
            "zs_decompress_fill": (ctypes.c_int, [P, P, P, I64, P, P, P]),
            "zs_preprocess_batch": (ctypes.c_int, [P, P, P, I64, P, P, P, P, P]),
            "zs_compress_device": (ctypes.c_int, [P, P, I64, P, I64, ctypes.c_int, ctypes.POINTER(Result)]),
            "zs_decompress_device": (ctypes.c_int, [P, P, I64, P, I64, ctypes.c_int, ctypes.POINTER(Result)]),
            "zs_compress_host": (ctypes.c_int, [P, P, I64, P, I64, ctypes.c_int, ctypes.POINTER(Result)]),
            "zs_decompress_host": (ctypes.c_int, [P, P, I64, P, I64, ctypes.c_int, ctypes.POINTER(Result)]),
            "zs_compress_bound": (I64, [I64]),
            "zs_decompress_bound": (I64, [P, I64]),
            "zs_last_kernel_ms": (ctypes.c_float, [P]),
            "zs_build_tables_host": (ctypes.c_int, [P, P, I32, P, P, P, P]),
            "zs_set_phase_timing": (ctypes.c_int, [P, ctypes.c_int]),
            "zs_build_t2_host": (ctypes.c_int, [P, P, I32, P, P, P, P]),
            "zs_set_transducer": (ctypes.c_int, [P, ctypes.c_int]),
            "zs_debug_chunk_cuts": (I64, [P, I64, I64, P, I64]),
            "zs_last_phase_cycles": (ctypes.c_int, [P, P]),
            "zs_last_kernel": (ctypes.c_char_p, [P]),
            "zs_stream": (P, [P]),
            "zs_set_stream": (ctypes.c_int, [P, P]),
            "zs_index_build": (ctypes.c_int, [P, P, I64, P, I64, ctypes.POINTER(ctypes.c_int64)]),
            "zs_decode_records": (ctypes.c_int, [P, P, P, I64, P, I64, P, I64, P, P, P,
                                                 ctypes.POINTER(ctypes.c_int64)]),
            "zs_train_count": (ctypes.c_int, [P, P, I64, I32, I32, ctypes.POINTER(ctypes.c_int64)]),
            "zs_train_rows": (ctypes.c_int, [P, P, P, P]),
            "zs_train_load": (ctypes.c_int, [P, P, I32, P, P, I64]),
            "zs_train_select": (ctypes.c_int, [P, I32, I64, P, ctypes.POINTER(ctypes.c_int32)]),
            "zs_overlap_batch": (ctypes.c_int, [P, P, P, I32, P, I32, P, I64, P]),
            "zs_host_alloc": (ctypes.c_int, [P, I64, ctypes.POINTER(ctypes.c_void_p)]),
            "zs_host_free": (ctypes.c_int, [P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name, None)
            if f is None and os.environ.get("ZS_LIB"):
                continue  # an alternative (e.g. older) build used for a comparison
            if f is None:
                raise ImportError(f"{LIB_PATH} does not export {name}")
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def device_count() -> int:
    n = ctypes.c_int(0)
    load().zs_device_count(ctypes.byref(n))
    return n.value


def ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


class Context:
    """One libzs context (stream pair + device buffers) on one GPU.  Calls are
    serialised by a lock; the currently uploaded dictionary is cached."""

    def __init__(self, device: int = 0):
        lib = load()
        if device_count() <= device:
            raise ZsCudaError("no CUDA device available: the ZSMILES codec runs on sm_100a "
                              "GPUs only (there is no CPU fallback)")
        h = ctypes.c_void_p()
        rc = lib.zs_ctx_create(device, ctypes.byref(h))
        if rc != ZS_OK:
            raise ZsCudaError(f"zs_ctx_create({device}) failed: {rc}")
        self.lib = lib
        self.h = h
        self.device = device
        self.lock = threading.RLock()
        self._dict_key = None
        self._keep = None
        self._pinned = {}

    def pinned(self, slot: str, nbytes: int) -> np.ndarray:
        """A page-locked uint8 buffer of at least `nbytes`, cached per
        context and slot name (grown on demand, freed with the context)."""
        have = self._pinned.get(slot)
        if have is not None and have[1].size >= nbytes:
            return have[1]
        if have is not None:
            self.lib.zs_host_free(self.h, have[0])
        p = ctypes.c_void_p()
        size = max(int(nbytes) + (int(nbytes) >> 3), 1 << 20)  # headroom: segments vary a little
        self.check(self.lib.zs_host_alloc(self.h, size, ctypes.byref(p)), "zs_host_alloc")
        arr = np.ctypeslib.as_array((ctypes.c_uint8 * size).from_address(p.value))
        self._pinned[slot] = (p, arr)
        return arr

    def check(self, rc, what):
        if rc == ZS_OK:
            return
        msg = self.lib.zs_last_error(self.h)
        raise ZsCudaError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")

    def set_dictionary(self, d):
        """Upload a Dictionary's tables (reference layouts) if not current."""
        key = d.cache_key()
        if key == self._dict_key:
            return
        trie = d.encode_trie
        exp_len, valid, exp_off, exp_flat = d.decode_tables
        children = np.ascontiguousarray(trie.children, np.int32)
        term = np.ascontiguousarray(trie.term_code, np.int16)
        exp_len = np.ascontiguousarray(exp_len, np.int32)
        valid = np.ascontiguousarray(valid, np.uint8)
        exp_off = np.ascontiguousarray(exp_off, np.int64)
        flat = np.ascontiguousarray(exp_flat, np.uint8)
        if flat.size == 0:
            flat = np.zeros(1, np.uint8)
        rc = self.lib.zs_set_dictionary(self.h, ptr(children), ptr(term), children.shape[0],
                                        ptr(exp_len), ptr(valid), ptr(exp_off), ptr(flat))
        self.check(rc, "zs_set_dictionary")
        self._dict_key = key

    def follow_torch_stream(self):
        """Order the next device-pointer calls after the work queued on
        torch's current stream of this device (zs_set_stream), so tensors
        torch is still writing are not read early."""
        import torch
        s = torch.cuda.current_stream(self.device).cuda_stream
        self.check(self.lib.zs_set_stream(self.h, s or None), "zs_set_stream")

    def fast_width(self) -> int:
        return self.lib.zs_dictionary_fast(self.h)

    def last_kernel_ms(self) -> float:
        return self.lib.zs_last_kernel_ms(self.h)

    def close(self):
        if self.h:
            for p, _ in self._pinned.values():
                self.lib.zs_host_free(self.h, p)
            self._pinned = {}
            self.lib.zs_ctx_destroy(self.h)
            self.h = None


_ctx = {}
_ctx_lock = threading.Lock()


def context(device: int | None = None) -> Context:
    """Process-wide context for `device` (default: the current torch device
    if torch is imported and CUDA-enabled, else 0)."""
    if isinstance(device, Context):  # an explicit context (e.g. a second one on the same GPU)
        return device
    if device is None:
        device = int(os.environ.get("ZS_DEVICE", "0"))
    with _ctx_lock:
        c = _ctx.get(device)
        if c is None:
            c = _ctx[device] = Context(device)
        return c
