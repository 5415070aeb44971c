"""ctypes binding of ``libfasttt_b200.so`` (the C ABI in include/fasttt_b200.h).

torch is used only as plumbing: device memory (caching allocator), the
current CUDA stream, and host<->device copies. Every computation on the
decomposition path is a kernel of libfasttt_b200. There is no CPU fallback:
if the library or a CUDA device is missing, calls raise.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FTT_LIB: load another build of the same library (A/B timing of two builds in
# one process environment); the default is the in-tree build.
LIB_PATH = os.environ.get("FTT_LIB") or os.path.join(_HERE, "libfasttt_b200.so")

FTT_OK = 0
FTT_ERR_INVALID = 1
FTT_ERR_OOM = 2
FTT_ERR_NONFINITE = 3
FTT_ERR_CUDA = 4
FTT_ERR_NOCONV = 5

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_c_p = ctypes.c_void_p
_c_d = ctypes.c_double
_P_i64 = ctypes.POINTER(ctypes.c_int64)
_P_d = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (restype is c_int unless listed in _RESTYPES)
SIGNATURES = {
    "ftt_version": [],
    "ftt_last_error": [],
    "ftt_create": [ctypes.c_int, _c_p, ctypes.POINTER(_c_p)],
    "ftt_destroy": [_c_p],
    "ftt_set_stream": [_c_p, _c_p],
    "ftt_kernel_launches": [_c_p],
    "ftt_profile_enable": [_c_p, ctypes.c_int],
    "ftt_profile_read": [_c_p, _c_i32, _P_d, _P_i64, _P_d, _P_d],
    "ftt_bench_dmma": [_c_p, _c_i64, _P_d],
    "ftt_fiber_count": [_c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_i32, _P_i64],
    "ftt_fiber_counts_all": [_c_p, _c_p, _c_i64, _c_i32, _P_i64, _P_i64],
    "ftt_linearize": [_c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_p],
    "ftt_fiber_counts_lin": [_c_p, _c_p, _c_p, _c_i64, _c_i32, _P_i64, _P_i64],
    "ftt_extract_fibers_lin": [_c_p, _c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_i32,
                               _c_p, _c_p, _c_p, _c_p, _c_p, _P_i64],
    "ftt_extract_fibers": [_c_p, _c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_i32,
                           _c_p, _c_p, _c_p, _c_p, _c_p, _P_i64],
    "ftt_depar_quasi_perm": [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _P_i64],
    "ftt_index_sweep_step": [_c_p, _c_i32, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64,
                             _c_p, _c_p, _P_i64],
    "ftt_mode_index": [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p],
    "ftt_pivot_core_scatter": [_c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_i64,
                               _c_i64, _c_p, _P_d],
    "ftt_side_core_dense": [_c_p, _c_i32, _c_p, _c_i64, _c_i64, _c_i64, _c_p],
    "ftt_scatter_cols": [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_p],
    "ftt_scatter_rows": [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_i64, _c_p],
    "ftt_dgemm": [_c_p, _c_i32, _c_i32, _c_i64, _c_i64, _c_i64, _c_d, _c_p, _c_i64, _c_p,
                  _c_i64, _c_d, _c_p, _c_i64],
    "ftt_orth_defect": [_c_p, _c_i64, _c_p, _c_i64, _P_d],
    "ftt_transpose": [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64],
    "ftt_qr_f64": [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64],
    "ftt_svd_f64": [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i32, _P_d],
    "ftt_svd_lowrank_f64": [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i32, _c_i64, _c_d, _P_d, _P_d,
                            ctypes.POINTER(ctypes.c_int32)],
    "ftt_svd_lowrank_sparse_f64": [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                                   _c_i64, _c_i64, _c_d, _P_d, _P_d, ctypes.POINTER(ctypes.c_int32)],
    "ftt_svd_vectors": [_c_p, _c_i64, _c_p, _c_i64, _c_i32, _c_p, _c_i64, _c_i32, _c_i32],
    "ftt_dot": [_c_p, _c_i64, _c_p, _c_p, _P_d],
    "ftt_set_deferred_checks": [_c_p, _c_i32],
    "ftt_take_status": [_c_p, ctypes.POINTER(ctypes.c_int32)],
    "ftt_depar_general": [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_d, _c_p, _c_p, _c_p, _c_p,
                          ctypes.POINTER(ctypes.c_int64)],
    "ftt_tensorize_matrix": [_c_p, _c_i64, _c_p, _c_p, _c_p, _c_i32, _P_i64, _P_i64, _c_p, _c_p,
                             ctypes.POINTER(ctypes.c_int64)],
    "ftt_parse_coo_text": [ctypes.c_char_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                           ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                           ctypes.POINTER(ctypes.POINTER(ctypes.c_int64)),
                           ctypes.POINTER(ctypes.POINTER(ctypes.c_double)), _c_p],
    "ftt_parse_mm_text": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32),
                          ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.POINTER(ctypes.c_int64)),
                          ctypes.POINTER(ctypes.POINTER(ctypes.c_int64)),
                          ctypes.POINTER(ctypes.POINTER(ctypes.c_double))],
    "ftt_free_host": [_c_p],
    "ftt_index_sweeps_all": [_c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_i32, ctypes.POINTER(_c_p),
                             ctypes.POINTER(_c_p), ctypes.POINTER(ctypes.c_int64)],
    "ftt_sweep_rounding": [_c_p, _c_i32, _c_i32, _c_p, _c_p, _c_i32, _c_d, _c_d, _c_d, _c_p,
                           _c_i32, _c_p, _c_p, ctypes.POINTER(ctypes.c_int32)],
    "ftt_free_device": [_c_p, _c_p],
    "ftt_scatter_steps": [],
    "ftt_set_lin_chunks": [_c_p, _c_i32, _P_i64, ctypes.POINTER(_c_p)],
    "ftt_fasttt_lin": [_c_p, _c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_i32, _c_i32, _c_d, _c_d,
                       _c_i32, _c_p, _c_p],
    "ftt_delinearize": [_c_p, _c_p, _c_i64, _c_i32, _P_i64, _c_p],
    "ftt_sync_stats": [_c_p, ctypes.POINTER(ctypes.c_int64), _P_d],
    "ftt_tt_norm": [_c_p, _c_i32, _P_i64, _P_i64, ctypes.POINTER(_c_p), _P_d],
    "ftt_inner_terms": [_c_p, _c_i64, _c_p, _c_p, _c_i32, _P_i64, _P_i64, ctypes.POINTER(_c_p),
                        _P_d],
    "ftt_inner_structured": [_c_p, _c_i32, _P_i64, _P_i64, ctypes.POINTER(_c_p), _c_i32,
                             ctypes.POINTER(_c_p), _P_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                             _P_d],
    "ftt_tt_entries": [_c_p, _c_i32, _P_i64, _P_i64, ctypes.POINTER(_c_p), _c_p, _c_i64, _c_p],
}
_RESTYPES = {
    "ftt_version": ctypes.c_char_p,
    "ftt_last_error": ctypes.c_char_p,
    "ftt_kernel_launches": ctypes.c_int64,
    "ftt_scatter_steps": ctypes.c_int64,
    "ftt_free_host": None,
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load the C-ABI library and declare every entry point (no GPU needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `make` (or __graft_entry__.build()); "
                "the FastTT path has no CPU fallback")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


class NativeError(RuntimeError):
    pass


def last_error() -> str:
    lib_ = load_library()
    return lib_.ftt_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == FTT_OK:
        return
    msg = _lib.ftt_last_error().decode(errors="replace") if _lib is not None else ""
    text = f"{what}: {msg}" if what else msg
    if status == FTT_ERR_OOM:
        raise MemoryError(text)
    if status == FTT_ERR_NONFINITE:
        raise ValueError("matrix entries must be finite")
    if status == FTT_ERR_INVALID:
        raise ValueError(text)
    if status == FTT_ERR_NOCONV:
        raise np.linalg.LinAlgError(text)
    raise NativeError(text)


# ------------------------------------------------------------------ context
# One native context per (thread, device): a context owns a workspace arena
# and the two-phase SVD state, so threads never share one (ctypes releases
# the GIL inside the calls).  _all_ctx lists every context for the launch
# counter.
_tls = threading.local()
_all_ctx: list = []
_all_lock = threading.Lock()


def torch_mod():
    import torch  # noqa: WPS433  (plumbing only)

    return torch


def device_ready() -> bool:
    try:
        return torch_mod().cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def _current_device_stream():
    """(device, raw cudaStream_t) of torch's current stream; the private C
    entry points skip torch.cuda's Python layers (this runs ~50 times per
    decomposition)."""
    C = torch_mod()._C
    try:
        dev = C._cuda_getDevice()
        return dev, C._cuda_getCurrentRawStream(dev)
    except AttributeError:  # pragma: no cover - older torch
        torch = torch_mod()
        dev = torch.cuda.current_device()
        return dev, torch.cuda.current_stream(dev).cuda_stream


def context():
    """This thread's native context for the current device, bound to torch's
    current stream."""
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        torch = torch_mod()
        if not torch.cuda.is_available():
            raise RuntimeError("a CUDA device is required: the B200 FastTT path has no CPU "
                               "fallback")
        torch.cuda.init()
        cache = _tls.ctx = {}
        _tls.stream = {}
    lib = _lib if _lib is not None else load_library()
    dev, stream = _current_device_stream()
    ctx = cache.get(dev)
    if ctx is None:
        h = _c_p()
        check(lib.ftt_create(dev, _c_p(stream), ctypes.byref(h)), "ftt_create")
        ctx = h
        cache[dev] = ctx
        _tls.stream[dev] = stream
        with _all_lock:
            _all_ctx.append(ctx)
    elif _tls.stream.get(dev) != stream:
        check(lib.ftt_set_stream(ctx, _c_p(stream)), "ftt_set_stream")
        _tls.stream[dev] = stream
    return ctx


def lib():
    return _lib if _lib is not None else load_library()


def kernel_launches() -> int:
    total = 0
    if _lib is None:
        return 0
    with _all_lock:
        ctxs = list(_all_ctx)
    for ctx in ctxs:
        total += int(_lib.ftt_kernel_launches(ctx))
    return total


def i64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int64 * max(len(vals), 1))(*vals)


def ptr(t) -> ctypes.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return _c_p(None)
    return _c_p(t.data_ptr())
