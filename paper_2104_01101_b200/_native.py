"""ctypes binding of libskx.so (include/skx.h) plus device plumbing.

The product path has no CPU fallback: if the shared library is missing, or no
CUDA device is visible, every entry point raises immediately.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libskx.so")
_lock = threading.Lock()
_lib = None

c_i32 = ctypes.c_int
c_i64 = ctypes.c_int64
c_u32 = ctypes.c_uint32
c_u64 = ctypes.c_uint64
c_p = ctypes.c_void_p
c_sz_p = ctypes.POINTER(ctypes.c_size_t)

# name -> argtypes (return type is always int status unless listed in _RET)
_SIGS = {
    "skx_philox_uniform": [c_u64, c_u64, c_u64, c_i64, c_p, c_p],
    "skx_philox_normal": [c_u64, c_u64, c_p, c_i64, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_lemire_scan": [c_u64, c_u64, c_u64, c_u64, c_u32, c_p, c_i64, c_p, c_p],
    "skx_fill_u64max": [c_p, c_i64, c_p],
    "skx_lemire_finish": [c_p, c_p, c_i64, c_u64, c_u32, c_u64, c_u64, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_ts_tables": [c_i32, c_p, c_p, c_i64, c_p, c_p],
    "skx_coo_rec_words": [c_i32],
    "skx_coo_fibre": [c_i32, c_p, c_i32, c_i64, c_p, c_p, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_coo_fibre_ts": [c_p, c_i32, c_i64, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_sz_p,
                         c_p],
    "skx_ts_rhs_coo": [c_i32, c_i64, c_p, c_p, c_p, c_p, c_i64, c_u32, c_i32, c_p, c_p],
    "skx_ts_rhs_dense": [c_p, c_i32, c_p, c_i32, c_p, c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_ts_combine": [c_i32, c_p, c_p, c_p, c_i64, c_i64, c_p, c_p],
    "skx_ts_kron_plan": [c_i32, c_p, c_p, c_p, c_i64, c_p, c_sz_p, c_p, c_sz_p, c_p],
    "skx_ts_kron_apply": [c_i32, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_lev_prepare": [c_p, c_i64, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_lev_scores": [c_p, c_i64, c_i32, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_slice_hits": [c_i32, c_i64, c_p, c_p, c_u32, c_p, c_p, c_i64, c_p, c_p, c_p, c_i64, c_p,
                       c_sz_p, c_p],
    "skx_lev_sample": [c_i32, c_p, c_p, c_p, c_i64, c_u64, c_u64, c_u64, c_p, c_p, c_p],
    "skx_top_m_products": [c_i32, c_p, c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_kron_rows": [c_i32, c_p, c_p, c_p, c_p, c_i64, c_p, c_p],
    "skx_gather_fibers_dense": [c_p, c_i32, c_p, c_i32, c_p, c_p, c_i64, c_p, c_p],
    "skx_filter_fibers_coo": [c_i32, c_p, c_i32, c_i64, c_p, c_p, c_p, c_i64, c_p, c_p, c_i64, c_p,
                              c_p],
    "skx_gather_fibers_coo": [c_i32, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p,
                              c_i64, c_p, c_sz_p, c_p],
    "skx_rrf_stage1_coo": [c_i32, c_p, c_i64, c_p, c_p, c_u64, c_u64, c_u64, c_u32, c_u32, c_u64,
                           c_p, c_i64, c_i64, c_u32, c_p, c_p],
    "skx_value_range": [c_p, c_i64, c_p, c_p],
    "skx_rrf_stage1_fx": [c_i32, c_p, c_i32, c_i64, c_p, c_p, c_i32, c_u64, c_u64, c_u64, c_u32,
                          c_u32, c_u64, c_p, c_i64, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_rrf_stage1_fx_acc": [c_i32, c_p, c_i32, c_i64, c_p, c_i64, c_p, c_i32, c_u64, c_u64, c_u64,
                              c_u32, c_u32, c_u64, c_p, c_i64, c_i64, c_p, c_p, c_i64, c_p],
    "skx_rrf_stage1_fx_convert": [c_p, c_i64, c_i32, c_p, c_p, c_p],
    "skx_stage_compact3": [c_p, c_i64, c_i64, c_i64, c_i64, c_i32, c_p, c_p, c_p, c_p, c_i64, c_p,
                           c_p],
    "skx_stage_stats3": [c_p, c_p, c_i64, c_i64, c_i64, c_p, c_p],
    "skx_coo_unpack3": [c_p, c_i64, c_i64, c_p, c_i32, c_p, c_p, c_i64, c_p, c_i64, c_p],
    "skx_rrf_partition": [c_i32, c_p, c_i64, c_p, c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_sz_p,
                          c_p],
    "skx_rrf_stage1_rec": [c_i64, c_u64, c_i64, c_p, c_p, c_p, c_i32, c_u64, c_u64, c_u64, c_u32,
                           c_u32, c_u64, c_p, c_i64, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_rrf_table": [c_u64, c_u64, c_u64, c_u32, c_u32, c_u64, c_p, c_i64, c_i64, c_i64, c_p, c_p],
    "skx_rrf_stage1_dense": [c_p, c_i32, c_p, c_i32, c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_resid_sq": [c_p, c_p, c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_sumsq": [c_p, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_tsqr_r": [c_p, c_i64, c_i32, c_i64, c_i64, c_p, c_p, c_sz_p, c_p],
    "skx_chol_upper": [c_p, c_i32, c_p, c_p, c_p],
    "skx_chol_inv_upper": [c_p, c_i32, c_p, c_p, c_p, c_p],
    "skx_house_q": [c_p, c_i32, c_i32, c_p, c_p],
    "skx_jacobi_svd": [c_p, c_i32, c_i64, c_i64, c_p, c_p, c_p, c_p],
    "skx_ttmc3_skip_coo": [c_i64, c_p, c_p, c_u32, c_p, c_i32, c_p, c_i32, c_p, c_p],
    "skx_cholqr_flags": [c_p, c_p, c_p, c_p, c_i32, c_p, c_p],
    "skx_mode_last": [c_p, c_i32, c_p, c_i32, c_p, c_p],
    "skx_lrls_mid": [c_p, c_p, c_i32, c_i32, c_p, c_p, c_p],
    "skx_tucker_cross_coo": [c_i32, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_u32, c_p, c_p,
                             c_sz_p, c_p],
    "skx_cp_cross_coo": [c_i32, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_cp_core_als": [c_p, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p],
    "skx_cp_core_smem_bytes": [c_p, c_i32],
    "skx_cp_cross_fibre3": [c_i64, c_p, c_p, c_u32, c_i32, c_p, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_ttm_lead": [c_p, c_i64, c_i64, c_i64, c_p, c_i32, c_p, c_p],
    "skx_gemm_ab": [c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_sz_p, c_p],
    "skx_gemm_atb": [c_i64, c_i32, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_sz_p, c_p],
    "skx_fitness_tucker_coo": [c_i32, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_u32, c_p,
                               c_p, c_p, c_sz_p, c_p],
    "skx_fitness_tucker_dense": [c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_fitness_cp_coo": [c_i32, c_p, c_i32, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_u32, c_p, c_p,
                           c_p, c_sz_p, c_p],
    "skx_nccl_unique_id": [c_p],
    "skx_nccl_init": [c_p, c_i32, c_i32, c_p],
    "skx_nccl_destroy": [c_p],
    "skx_allreduce_sum": [c_p, c_p, c_p, c_i64, c_p],
    "skx_reduce_scatter_sum": [c_p, c_p, c_p, c_i64, c_p],
    "skx_allgather": [c_p, c_p, c_p, c_i64, c_p],
    "skx_coo_pack0_range": [c_i32, c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p],
    "skx_tucker_ttmc3_r20": [c_p, c_i32, c_p, c_p, c_u32, c_p, c_p, c_p, c_p, c_p, c_sz_p, c_p],
    "skx_last_error": [],
    "skx_launch_count": [],
    "skx_version": [],
}
_RET = {"skx_last_error": ctypes.c_char_p, "skx_launch_count": ctypes.c_longlong,
        "skx_cp_core_smem_bytes": ctypes.c_size_t, "skx_coo_rec_words": ctypes.c_int}

EXPORTS = tuple(_SIGS)


class NativeError(RuntimeError):
    pass


def lib_path():
    return _LIB_PATH


def load(require_cuda=True):
    """Load libskx.so (fails loudly: there is no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if require_cuda:
            import torch
            if not torch.cuda.is_available():
                raise NativeError("paper_2104_01101_b200 needs a CUDA device (B200); none visible")
        if not os.path.exists(_LIB_PATH):
            raise NativeError(f"{_LIB_PATH} missing: run `python -m paper_2104_01101_b200.build`")
        lib = ctypes.CDLL(_LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RET.get(name, ctypes.c_int)
        _lib = lib
        return lib


def load_symbols_only():
    """Load without requiring a GPU (CPU tests check exports)."""
    return load(require_cuda=False)


def _raise(rc, name):
    from .linalg import RankDeficientError

    msg = load().skx_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(f"{name}: {msg}")
    if rc == 2:
        raise RankDeficientError(f"{name}: {msg}")
    raise NativeError(f"{name}: {msg}")


# --------------------------------------------------------------- event hooks
# bench.py brackets the launches of one chosen entry point with CUDA events
# (on the launching stream) to time that kernel live inside the timed region.
_hooks = {}


def set_event_hook(name, sink):
    if sink is None:
        _hooks.pop(name, None)
    else:
        _hooks[name] = sink


def call(name, *args):
    lib = load()
    hook = _hooks.get(name)
    if hook is not None:
        import torch
        s = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rc = getattr(lib, name)(*args)
        e1.record(s)
        hook.append((e0, e1, args))
    else:
        rc = getattr(lib, name)(*args)
    if rc != 0:
        _raise(rc, name)
    return rc


def launch_count():
    return int(load().skx_launch_count())


# --------------------------------------------------------------- utilities

def stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def host_i64(values):
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    return arr, arr.ctypes.data_as(ctypes.c_void_p)


def host_ptrs(tensors):
    arr = (ctypes.c_void_p * max(1, len(tensors)))(*[t.data_ptr() for t in tensors])
    return arr, ctypes.cast(arr, ctypes.c_void_p)


class Workspace:
    """Grow-only per-device scratch buffers, one per (slot, stream).  A slot's
    buffer is only ever handed to calls on one stream, so two streams running
    the same entry point concurrently (the per-sweep fitness on its side
    stream next to Algorithm 6's final CP fitness) never share scratch, and a
    grown buffer's predecessor is released in that stream's order."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes, slot=0):
        import torch
        cur = torch.cuda.current_stream()
        key = (torch.cuda.current_device(), slot, cur.cuda_stream)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
            self._buf[key] = buf
        return buf


WS = Workspace()


def call_ws(name, pre, post=(), slot=0):
    """Call an entry point whose signature ends in (..., ws, ws_bytes, stream):
    `pre` are the arguments before ws; `post` any after ws_bytes except the
    stream, which is appended automatically."""
    lib = load()
    sz = ctypes.c_size_t(0)
    st = stream()
    rc = getattr(lib, name)(*pre, None, ctypes.byref(sz), *post, st)
    if rc != 0:
        _raise(rc, name)
    buf = WS.get(sz.value, slot)
    sz2 = ctypes.c_size_t(buf.numel())
    return call(name, *pre, ptr(buf), ctypes.byref(sz2), *post, st)
