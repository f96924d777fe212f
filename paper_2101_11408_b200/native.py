"""Thin ctypes binding of the C ABI (include/fpparse.h).

Argument marshalling only: every step of the parse runs in the CUDA kernels of
libfpparse.so.  PyTorch provides device memory and streams.  There is no CPU
fallback: load() raises if the in-tree library is missing or fails to load.
"""
import ctypes
import os

import torch

from .build import LIB

FPP_SUCCESS, FPP_EARG, FPP_ECUDA, FPP_ECAPACITY = 0, 1, 2, 3
ST_OK, ST_OVERFLOW, ST_UNDERFLOW, ST_INVALID, ST_EMPTY = 0, 1, 2, 3, 4
STAT_NAMES = ["records", "two_mult", "bracket", "slow", "abort", "global", "bad", "tiles"]
NSTATS = len(STAT_NAMES)

EXPORTS = ["parse_f64_batch", "parse_f64_batch_ws", "parse_f64_split", "parse_f64_split_ws",
           "fpp_workspace_bytes_batch", "fpp_workspace_bytes_split", "fpp_set_profile_events",
           "fpp_version"]

_lib = None


class FppError(RuntimeError):
    pass


def load(path=None):
    """Load libfpparse.so (in-tree).  Raises if it is missing.
    FPP_LIB may name an alternative in-tree build (ablation experiments)."""
    global _lib
    if _lib is not None:
        return _lib
    if path is None:
        path = os.environ.get("FPP_LIB") or LIB
    if not os.path.exists(path):
        raise FppError("libfpparse.so not built (%s); run __graft_entry__.build()" % path)
    lib = ctypes.CDLL(path)
    vp, sz, i64, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_uint32
    for w in ("f64", "f32"):
        getattr(lib, "parse_%s_batch" % w).argtypes = [vp, sz, vp, i64, vp, vp, vp]
        getattr(lib, "parse_%s_batch_ws" % w).argtypes = [vp, sz, vp, i64, vp, vp, vp, sz, vp, vp]
        getattr(lib, "parse_%s_split" % w).argtypes = [vp, sz, u32, vp, i64, vp, vp, vp, vp]
        getattr(lib, "parse_%s_split_ws" % w).argtypes = [vp, sz, u32, vp, i64, vp, vp, vp, vp, sz, vp, vp]
        getattr(lib, "parse_%s_batch_ex" % w).argtypes = [vp, sz, vp, i64, u32, vp, vp, vp, sz, vp, vp]
        getattr(lib, "parse_%s_split_host" % w).argtypes = [vp, sz, u32, u32, vp, i64, vp, vp, vp, sz, vp]
        getattr(lib, "parse_%s_split_host" % w).restype = ctypes.c_int
        getattr(lib, "parse_%s_split_ex" % w).argtypes = [vp, sz, u32, u32, vp, i64, vp, vp, vp, vp, sz, vp, vp]
        for f in ("batch", "batch_ws", "split", "split_ws", "batch_ex", "split_ex"):
            getattr(lib, "parse_%s_%s" % (w, f)).restype = ctypes.c_int
    lib.fpp_workspace_bytes_batch.argtypes = [sz, i64]
    lib.fpp_workspace_bytes_batch.restype = sz
    lib.fpp_workspace_bytes_split.argtypes = [sz]
    lib.fpp_workspace_bytes_split.restype = sz
    lib.fpp_version.restype = ctypes.c_char_p
    lib.fpp_set_profile_events.argtypes = [vp, vp, vp]
    lib.fpp_set_profile_events.restype = None
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc, what):
    if rc != FPP_SUCCESS:
        raise FppError("%s failed with code %d" % (what, rc))


def _u8(t):
    assert t.is_cuda and t.dtype == torch.uint8 and t.is_contiguous()
    return t


class Workspace:
    """Reusable device workspace for the *_ws entry points."""

    def __init__(self, nbytes, device=None):
        self.nbytes = max(int(nbytes), 256)
        self.buf = torch.empty(self.nbytes + 256, dtype=torch.uint8, device=device or "cuda")
        base = self.buf.data_ptr()
        self.ptr = (base + 255) & ~255

    @classmethod
    def for_batch(cls, length, n, device=None):
        return cls(load().fpp_workspace_bytes_batch(length, n), device)

    @classmethod
    def for_split(cls, length, device=None):
        return cls(load().fpp_workspace_bytes_split(length), device)


_DTYPES = {"f64": torch.float64, "f32": torch.float32}


GRAMMAR_DEFAULT, GRAMMAR_HEX, GRAMMAR_JSON = 0, 1, 2  # include/fpparse.h FPP_GRAMMAR_*


def _batch(fmt, data, offsets, out, status, ws, stats, stream, grammar=0):
    lib = load()
    _u8(data)
    assert offsets.is_cuda and offsets.dtype == torch.int64 and offsets.is_contiguous()
    n = offsets.numel()
    if out is None:
        out = torch.empty(n, dtype=_DTYPES[fmt], device=data.device)
    assert out.dtype == _DTYPES[fmt] and out.is_contiguous() and out.numel() >= n
    if status is None:
        status = torch.empty(n, dtype=torch.uint8, device=data.device)
    st = _stream_ptr(stream)
    if grammar:
        rc = getattr(lib, "parse_%s_batch_ex" % fmt)(_ptr(data), data.numel(), _ptr(offsets), n, grammar,
                                                     _ptr(out), _ptr(status),
                                                     None if ws is None else ctypes.c_void_p(ws.ptr),
                                                     0 if ws is None else ws.nbytes, _ptr(stats), st)
    elif ws is None:
        rc = getattr(lib, "parse_%s_batch" % fmt)(_ptr(data), data.numel(), _ptr(offsets), n, _ptr(out),
                                                  _ptr(status), st)
    else:
        rc = getattr(lib, "parse_%s_batch_ws" % fmt)(_ptr(data), data.numel(), _ptr(offsets), n, _ptr(out),
                                                     _ptr(status), ctypes.c_void_p(ws.ptr), ws.nbytes,
                                                     _ptr(stats), st)
    _check(rc, "parse_%s_batch" % fmt)
    return out, status


def _split(fmt, data, sep_mask, capacity, out, status, offsets_out, n_out, ws, stats, stream, want_offsets,
           grammar=0):
    lib = load()
    _u8(data)
    L = data.numel()
    if capacity is None:
        capacity = L + 1 if out is None else out.numel()
    dev = data.device
    if out is None:
        out = torch.empty(capacity, dtype=_DTYPES[fmt], device=dev)
    assert out.dtype == _DTYPES[fmt] and out.is_contiguous() and out.numel() >= capacity
    if status is None:
        status = torch.empty(capacity, dtype=torch.uint8, device=dev)
    if offsets_out is None and want_offsets:
        offsets_out = torch.empty(capacity, dtype=torch.int64, device=dev)
    if n_out is None:
        n_out = torch.empty(1, dtype=torch.int64, device=dev)
    st = _stream_ptr(stream)
    if grammar:
        rc = getattr(lib, "parse_%s_split_ex" % fmt)(_ptr(data), L, sep_mask, grammar, _ptr(offsets_out), capacity,
                                                     _ptr(n_out), _ptr(out), _ptr(status),
                                                     None if ws is None else ctypes.c_void_p(ws.ptr),
                                                     0 if ws is None else ws.nbytes, _ptr(stats), st)
    elif ws is None:
        rc = getattr(lib, "parse_%s_split" % fmt)(_ptr(data), L, sep_mask, _ptr(offsets_out), capacity,
                                                  _ptr(n_out), _ptr(out), _ptr(status), st)
    else:
        rc = getattr(lib, "parse_%s_split_ws" % fmt)(_ptr(data), L, sep_mask, _ptr(offsets_out), capacity,
                                                     _ptr(n_out), _ptr(out), _ptr(status),
                                                     ctypes.c_void_p(ws.ptr), ws.nbytes, _ptr(stats), st)
    _check(rc, "parse_%s_split" % fmt)
    return out, status, offsets_out, n_out


def parse_f64_batch(data, offsets, out=None, status=None, ws=None, stats=None, stream=None, grammar=0):
    """data: uint8 CUDA tensor; offsets: int64 CUDA tensor [n].
    Returns (out float64[n], status uint8[n]) on the same device.
    grammar: GRAMMAR_HEX / GRAMMAR_JSON (parse_f64_batch_ex)."""
    return _batch("f64", data, offsets, out, status, ws, stats, stream, grammar)


def parse_f32_batch(data, offsets, out=None, status=None, ws=None, stats=None, stream=None, grammar=0):
    """As parse_f64_batch with binary32 results: (out float32[n], status uint8[n])."""
    return _batch("f32", data, offsets, out, status, ws, stats, stream, grammar)


def parse_f64_split(data, sep_mask=0, capacity=None, out=None, status=None, offsets_out=None,
                    n_out=None, ws=None, stats=None, stream=None, want_offsets=False, grammar=0):
    """data: uint8 CUDA tensor.  Returns (out, status, offsets_out or None, n_out int64[1]);
    the result tensors have `capacity` entries (default: enough for any input).
    grammar: GRAMMAR_HEX / GRAMMAR_JSON (parse_f64_split_ex)."""
    return _split("f64", data, sep_mask, capacity, out, status, offsets_out, n_out, ws, stats, stream,
                  want_offsets, grammar)


def parse_f32_split(data, sep_mask=0, capacity=None, out=None, status=None, offsets_out=None,
                    n_out=None, ws=None, stats=None, stream=None, want_offsets=False, grammar=0):
    """As parse_f64_split with binary32 results (out float32)."""
    return _split("f32", data, sep_mask, capacity, out, status, offsets_out, n_out, ws, stats, stream,
                  want_offsets, grammar)


def _split_host(fmt, text, sep_mask, capacity, out, status, offsets_out, grammar, chunk_bytes, stream):
    lib = load()
    assert not text.is_cuda and text.dtype == torch.uint8 and text.is_contiguous()
    L = text.numel()
    if capacity is None:
        capacity = L + 1 if out is None else out.numel()
    if out is None:
        out = torch.empty(capacity, dtype=_DTYPES[fmt], pin_memory=True)
    if status is None:
        status = torch.empty(capacity, dtype=torch.uint8, pin_memory=True)
    assert not out.is_cuda and not status.is_cuda and out.dtype == _DTYPES[fmt]
    n = ctypes.c_int64(0)
    rc = getattr(lib, "parse_%s_split_host" % fmt)(_ptr(text), L, sep_mask, grammar, _ptr(offsets_out), capacity,
                                                   ctypes.byref(n), _ptr(out), _ptr(status), chunk_bytes,
                                                   _stream_ptr(stream))
    _check(rc, "parse_%s_split_host" % fmt)
    return out, status, offsets_out, int(n.value)


def parse_f64_split_host(text, sep_mask=0, capacity=None, out=None, status=None, offsets_out=None, grammar=0,
                         chunk_bytes=0, stream=None):
    """Host-buffer streaming parse (parse_f64_split_host): text is a CPU uint8
    tensor (pinned for overlap); returns (out, status, offsets_out, n) on the host."""
    return _split_host("f64", text, sep_mask, capacity, out, status, offsets_out, grammar, chunk_bytes, stream)


def parse_f32_split_host(text, sep_mask=0, capacity=None, out=None, status=None, offsets_out=None, grammar=0,
                         chunk_bytes=0, stream=None):
    """As parse_f64_split_host with binary32 results."""
    return _split_host("f32", text, sep_mask, capacity, out, status, offsets_out, grammar, chunk_bytes, stream)


def set_profile_events(before_fast=None, after_fast=None, after_slow=None):
    """Record torch.cuda.Event objects around the kernels (None disables)."""
    h = [None if e is None else ctypes.c_void_p(e.cuda_event) for e in (before_fast, after_fast, after_slow)]
    load().fpp_set_profile_events(*h)


def version():
    return load().fpp_version().decode()
