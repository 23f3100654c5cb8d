"""Tensor data model (drop-in for src/tensors.py) with device-resident mirrors.

Host-facing types keep the reference's contract (src/tensors.py:26-138):
``SparseTensor`` is lexsorted, duplicate-free, immutable COO with int64
coordinates and float64 values; dense tensors are C-order float64 arrays;
``TuckerModel`` / ``CPModel`` hold numpy arrays.

Device side (HBM layout):
* ``DeviceCoo``: coordinates as an (N, nnz) int32 SoA in lexicographic order
  (4 B per coordinate instead of 8; extents < 2^31) + float64 values, plus
  lazily built, cached per-mode layouts:
    - fibre-major (mode n): nonzeros sorted by (i_n, other modes ascending)
      with int64 column offsets -> TS right-hand side, RRF stage 1;
    - other-major (mode n): int64 keys flat_other * s_n + i_n sorted, values
      -> leverage fibre gather.
  The reference caches its scipy unfoldings on the tensor the same way
  (``SparseTensor._unfoldings``, src/tensors.py:158-176).
* dense tensors: one contiguous float64 CUDA tensor.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat


# ============================================================ host types
# SparseTensor(shape, coords, values) with at least this many nonzeros is
# sorted and validated on the GPU (same result as the host lexsort)
DEVICE_INGEST_NNZ = 1 << 20


def _device_ingest_ok(shape):
    if any(int(x) >= (1 << 31) for x in shape) or float(np.prod([float(x) for x in shape])) >= 2.0 ** 62:
        return False
    try:
        return _torch().cuda.is_available()
    except Exception:
        return False


class SparseTensor:
    """Order-N COO tensor (src/tensors.py:26-98): coords (nnz, N) int64
    lexsorted, duplicates rejected, immutable."""

    def __init__(self, shape, coords, values):
        shape = tuple(int(s) for s in shape)
        if len(shape) < 1 or any(s < 1 for s in shape):
            raise ValueError(f"invalid shape {shape}")
        coords = np.atleast_2d(np.asarray(coords, dtype=np.int64))
        values = np.asarray(values, dtype=np.float64).ravel()
        if coords.size == 0:
            coords = coords.reshape(0, len(shape))
        if coords.shape[1] != len(shape):
            raise ValueError("coordinate width does not match tensor order")
        if coords.shape[0] != values.shape[0]:
            raise ValueError("number of coordinates does not match number of values")
        if coords.shape[0] >= DEVICE_INGEST_NNZ and _device_ingest_ok(shape):
            # large inputs: validate, lexsort and deduplicate-check on the GPU
            # (SURVEY 8f rank 1); the host arrays are materialised on demand
            self._init(shape, None, None)
            self._device = DeviceCoo.ingest(shape, coords, values)
            return
        if coords.size and ((coords < 0).any() or (coords >= np.asarray(shape)).any()):
            raise ValueError("coordinate out of range")
        order = np.lexsort(coords.T[::-1])
        coords = coords[order]
        values = values[order]
        if coords.shape[0] > 1 and (np.diff(coords, axis=0) == 0).all(axis=1).any():
            raise ValueError("duplicate coordinates")
        self._init(shape, coords, values)

    def _init(self, shape, coords, values):
        self.shape = shape
        self._coords = coords
        self._values = values
        if coords is not None:
            coords.setflags(write=False)
            values.setflags(write=False)
        self._unfoldings = {}
        self._mode_sort = {}
        self._device = None
        self._soa = None  # pinned int32 (N, nnz) staging copy (from_sorted)
        self._c3 = None   # compact order-3 staging (from_sorted, _stage_compact3)

    @classmethod
    def from_sorted(cls, shape, coords, values):
        """Trusted-order constructor: same validation as __init__ but O(nnz)
        (checks that coords are strictly lexicographically increasing instead
        of re-sorting).  Keeps the caller's arrays (e.g. pinned buffers)."""
        shape = tuple(int(s) for s in shape)
        coords = np.asarray(coords)
        values = np.asarray(values)
        if coords.dtype != np.int64 or values.dtype != np.float64:
            raise ValueError("from_sorted needs int64 coords and float64 values")
        if coords.ndim != 2 or coords.shape[1] != len(shape) or coords.shape[0] != values.shape[0]:
            raise ValueError("coords must be (nnz, N) matching values")
        obj = cls.__new__(cls)
        obj._init(shape, coords, values)
        if (coords.shape[0] >= DEVICE_INGEST_NNZ and max(shape) < 2 ** 31
                and obj._stage_compact3()):
            return obj  # validated (range, strict lexsort) by the native staging pass
        if coords.size and ((coords.min(axis=0) < 0).any() or (coords.max(axis=0) >= np.asarray(shape)).any()):
            raise ValueError("coordinate out of range")
        chunk = 1 << 24
        for lo in range(0, max(coords.shape[0] - 1, 0), chunk):
            a = coords[lo:lo + chunk]
            b = coords[lo + 1:lo + chunk + 1]
            k = min(a.shape[0], b.shape[0])
            a, b = a[:k], b[:k]
            lt = np.zeros(k, dtype=bool)
            eq = np.ones(k, dtype=bool)
            for n in range(len(shape)):
                lt |= eq & (a[:, n] < b[:, n])
                eq &= a[:, n] == b[:, n]
            if not lt.all():
                raise ValueError("coordinates must be lexsorted and duplicate-free")
        if coords.shape[0] >= DEVICE_INGEST_NNZ and max(shape) < 2 ** 31:
            obj._stage_soa()
        return obj

    def _stage_compact3(self):
        """Order 3: stage the coordinates in the compact upload form that
        skx_coo_unpack3 expands on the device -- mode-0 slice pointers and one
        uint32 per nonzero, (i1 increment within the slice << b2) | i2, with
        an exception list for increments that do not fit -- in pinned host
        memory, once, at construction.  4 bytes of coordinates per nonzero
        cross PCIe per call instead of 12 (int32 SoA) or 24 (the API's int64).
        Lossless; returns False when the shape does not admit it."""
        if self.ndim != 3 or self._coords is None:
            return False
        s0, s1, s2 = self.shape
        b2 = max(1, int(s2 - 1).bit_length())
        if b2 > 24 or s0 >= 2 ** 31 or s1 >= 2 ** 31:
            return False
        from . import _native as nat
        torch = _torch()
        c = np.ascontiguousarray(self._coords, dtype=np.int64)
        nnz = c.shape[0]
        pin = torch.cuda.is_available()
        packed = torch.empty(nnz, dtype=torch.int32, pin_memory=pin)
        ptr0 = torch.empty(s0 + 1, dtype=torch.int64, pin_memory=pin)
        cap = max(1024, nnz // 256)
        while True:
            exc_idx = torch.empty(cap, dtype=torch.int64)
            exc_val = torch.empty(cap, dtype=torch.int32)
            nx = ctypes.c_int64(0)
            status = ctypes.c_int(0)
            rc = nat.load(require_cuda=False).skx_stage_compact3(
                c.ctypes.data_as(ctypes.c_void_p), nnz, s0, s1, s2, b2,
                ctypes.c_void_p(ptr0.data_ptr()), ctypes.c_void_p(packed.data_ptr()),
                ctypes.c_void_p(exc_idx.data_ptr()), ctypes.c_void_p(exc_val.data_ptr()), cap,
                ctypes.byref(nx), ctypes.byref(status))
            if rc != 0:
                return False
            if status.value == 1:
                raise ValueError("coordinate out of range")
            if status.value == 2:
                raise ValueError("coordinates must be lexsorted and duplicate-free")
            if nx.value <= cap:
                break
            cap = nx.value
        exc_idx = exc_idx[:nx.value].clone()
        exc_val = exc_val[:nx.value].clone()
        # value range and per-mode row-block counts, so the device side need
        # not scan the whole tensor before its first RRF stage-1 sum
        vr = (ctypes.c_int * 3)()
        rm = (ctypes.c_int64 * 2)()
        v = np.ascontiguousarray(self._values, dtype=np.float64)
        nat.load(require_cuda=False).skx_stage_stats3(
            c.ctypes.data_as(ctypes.c_void_p), v.ctypes.data_as(ctypes.c_void_p), nnz, s1, s2, vr, rm)
        stats = dict(vrange=(int(vr[0]), int(vr[1]), int(vr[2])), rowmax={1: int(rm[0]), 2: int(rm[1])})
        self._c3 = dict(ptr0=ptr0, packed=packed, b2=b2, exc_idx=exc_idx, exc_val=exc_val, **stats)
        return True

    def _stage_soa(self):
        """Stage the coordinates in the device layout -- int32, one row per
        mode (N x nnz) -- in pinned host memory, once, at construction: every
        later upload then moves 4 B per coordinate instead of the API's 8 and
        needs no conversion pass on either side."""
        torch = _torch()
        import warnings
        with warnings.catch_warnings():  # read-only host arrays are only read
            warnings.simplefilter("ignore", UserWarning)
            c64 = torch.from_numpy(self._coords)
        soa = torch.empty((self.ndim, c64.shape[0]), dtype=torch.int32, pin_memory=True)
        chunk = 1 << 24
        for lo in range(0, c64.shape[0], chunk):
            soa[:, lo:lo + chunk].copy_(c64[lo:lo + chunk].t())
        self._soa = soa

    @classmethod
    def from_device(cls, shape, coords, values, validate=True):
        """Wrap device arrays (coords (nnz, N) or (N, nnz) integer CUDA tensor,
        values float64 CUDA tensor) that are already lexsorted.  Host copies
        are materialised only on demand (``.coords`` / ``.values``)."""
        obj = cls.__new__(cls)
        dev = DeviceCoo.from_torch(shape, coords, values, validate=validate)
        obj._init(tuple(int(s) for s in shape), None, None)
        obj._device = dev
        return obj

    def _materialise(self):
        dev = self._device
        self._coords = dev.coords.t().cpu().numpy().astype(np.int64)
        self._values = dev.vals.cpu().numpy()
        self._coords.setflags(write=False)
        self._values.setflags(write=False)

    @property
    def coords(self):
        if self._coords is None:
            self._materialise()
        return self._coords

    @property
    def values(self):
        if self._values is None:
            self._materialise()
        return self._values

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def nnz(self):
        if self._values is None and self._device is not None:
            return self._device.nnz
        return self._values.shape[0]

    @property
    def density(self):
        return self.nnz / float(np.prod(self.shape))

    def norm(self):
        return float(np.sqrt(device_of(self).norm2().item()))

    def to_dense(self):
        out = np.zeros(self.shape)
        out[tuple(self.coords.T)] = self.values
        return out

    @classmethod
    def from_dense(cls, a, tol=0.0):
        a = np.asarray(a, dtype=np.float64)
        mask = np.abs(a) > tol
        return cls(a.shape, np.argwhere(mask), a[mask])

    def mode_sort(self, n):
        if n not in self._mode_sort:
            order = np.argsort(self.coords[:, n], kind="stable")
            order.setflags(write=False)
            self._mode_sort[n] = order
        return self._mode_sort[n]

    def __repr__(self):
        return f"SparseTensor(shape={self.shape}, nnz={self.nnz})"


@dataclass
class TuckerModel:
    """Core tensor plus per-mode factors with orthonormal columns."""

    core: np.ndarray
    factors: list

    @property
    def ranks(self):
        return tuple(self.core.shape)

    def reconstruct(self):
        out = np.asarray(self.core)
        for n, a in enumerate(self.factors):
            out = np.moveaxis(np.tensordot(a, out, axes=(1, n)), 0, n)
        return out


@dataclass
class CPModel:
    """Rank-R CP model: unit-column factors and per-component weights."""

    factors: list
    weights: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.weights is None:
            self.weights = np.ones(self.factors[0].shape[1])
        self.weights = np.asarray(self.weights, dtype=np.float64)

    @property
    def rank(self):
        return self.factors[0].shape[1]

    def reconstruct(self):
        subs = "abcdefgh"[: len(self.factors)]
        expr = ",".join(f"{c}z" for c in subs) + ",z->" + subs
        return np.einsum(expr, *self.factors, self.weights, optimize=True)


# ============================================================ device types
def _torch():
    import torch
    return torch


_STAGE = {"buf": None}
_STAGE_LOCK = None
_COPY_POOL = None


def to_host(tensors):
    """CUDA float64 tensors -> fresh numpy arrays (the model a public call
    returns).  One asynchronous D2H of all of them into a reused pinned
    staging buffer, then host copies into the new arrays split over a few
    threads: a pageable `.cpu()` of config 5's 48 MB of factors takes 15-18
    ms on this box (2-3 GB/s, the destination pages faulted in by the
    driver's copy), the pinned copy 0.9 ms and the parallel host copies a few
    more.  Small or non-float64 inputs take the plain path."""
    global _STAGE_LOCK, _COPY_POOL
    import threading
    torch = _torch()
    ts = [t.detach().contiguous() for t in tensors]
    tot = sum(int(t.numel()) for t in ts)
    if tot < (1 << 17) or any(t.dtype != torch.float64 or not t.is_cuda for t in ts):
        return [t.cpu().numpy() for t in ts]
    if _STAGE_LOCK is None:
        _STAGE_LOCK = threading.Lock()
    with _STAGE_LOCK:
        buf = _STAGE["buf"]
        if buf is None or buf.numel() < tot:
            buf = torch.empty(tot, dtype=torch.float64, pin_memory=True)
            _STAGE["buf"] = buf
        off = 0
        for t in ts:
            n = int(t.numel())
            buf[off:off + n].copy_(t.view(-1), non_blocking=True)
            off += n
        ev = torch.cuda.Event()
        ev.record()
        ev.synchronize()
        src = buf.numpy()
        outs = [np.empty(tuple(t.shape), dtype=np.float64) for t in ts]
        jobs = []
        off = 0
        step = 1 << 19  # 4 MB pieces
        for t, o in zip(ts, outs):
            flat = o.reshape(-1)
            n = flat.size
            for a in range(0, n, step):
                b = min(n, a + step)
                jobs.append((flat[a:b], src[off + a:off + b]))
            off += n
        if len(jobs) == 1:
            np.copyto(*jobs[0])
        else:
            if _COPY_POOL is None:
                import concurrent.futures
                import os
                _COPY_POOL = concurrent.futures.ThreadPoolExecutor(
                    max_workers=max(1, min(8, (os.cpu_count() or 2) // 2)))
            list(_COPY_POOL.map(lambda j: np.copyto(j[0], j[1]), jobs))
    return outs


def compact3_aux_to_device(c3):
    """Per-call device copies of the small parts of the compact order-3
    staging: slice pointers and the exception list."""
    return (c3["ptr0"].to("cuda", non_blocking=True), c3["exc_idx"].to("cuda", non_blocking=True),
            c3["exc_val"].to("cuda", non_blocking=True))


def unpack_compact3(c3, nnz, coords=None, s_lo=0, s_hi=None, packed_dev=None, aux=None):
    """Device int32 SoA coordinates (3, nnz) of slices [s_lo, s_hi) from the
    compact order-3 staging (SparseTensor._stage_compact3): the packed words
    cross PCIe (or are already on the device in packed_dev), skx_coo_unpack3
    expands them.  Returns the coordinate array."""
    from . import _native as nat
    torch = _torch()
    ptr0, exi, exv = aux if aux is not None else compact3_aux_to_device(c3)
    s0 = int(c3["ptr0"].numel()) - 1
    s_hi = s0 if s_hi is None else s_hi
    if coords is None:
        coords = torch.empty((3, nnz), dtype=torch.int32, device="cuda")
    if packed_dev is None:
        packed_dev = c3["packed"].to("cuda", non_blocking=True)
    nat.call("skx_coo_unpack3", nat.ptr(ptr0), s_lo, s_hi, nat.ptr(packed_dev), c3["b2"],
             nat.ptr(exi) if exi.numel() else None, nat.ptr(exv) if exv.numel() else None,
             int(exi.numel()), nat.ptr(coords), nnz, nat.stream())
    return coords


class DeviceCoo:
    """HBM-resident COO tensor with cached per-mode layouts."""

    def __init__(self, shape, coords_i32, vals):
        self.shape = tuple(int(s) for s in shape)
        self.ndim = len(self.shape)
        self.coords = coords_i32  # (N, nnz) int32, lexsorted
        self.vals = vals          # (nnz,) float64
        self.nnz = int(vals.numel())
        self._fibre = {}
        self._fibre_meta = {}
        self._keys = {}
        self._norm2 = None
        self._vrange = None

    @classmethod
    def from_host(cls, st: SparseTensor):
        torch = _torch()
        if max(st.shape) >= 2 ** 31:
            raise ValueError("extents must be < 2^31 for the device layout")
        import warnings
        with warnings.catch_warnings():  # read-only host arrays are only read
            warnings.simplefilter("ignore", UserWarning)
            v = torch.from_numpy(np.ascontiguousarray(st.values))
            vd = v.to("cuda", non_blocking=True)
            if getattr(st, "_c3", None) is not None:  # compact order-3 staging
                d = cls(st.shape, unpack_compact3(st._c3, st.nnz), vd)
                d._vrange = st._c3["vrange"]  # computed at staging: no device pass
                return d
            if getattr(st, "_soa", None) is not None:  # staged int32 SoA: one H2D
                return cls(st.shape, st._soa.to("cuda", non_blocking=True), vd)
            c64 = torch.from_numpy(np.ascontiguousarray(st.coords))
        # one H2D of the caller's arrays, then int64 AoS -> int32 SoA on device
        cd = c64.to("cuda", non_blocking=True)
        return cls(st.shape, cd.t().to(torch.int32).contiguous(), vd)

    @classmethod
    def ingest(cls, shape, coords, values):
        """Unsorted host COO -> lexsorted DeviceCoo (src/tensors.py:35-60
        semantics: range check, lexsort, duplicate rejection) on the GPU: the
        linearised int64 key (C order) is radix-sorted and adjacent keys are
        compared."""
        torch = _torch()
        shape = tuple(int(x) for x in shape)
        nd = len(shape)
        c = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.int64)).cuda()
        v = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).cuda()
        ext = torch.tensor(shape, dtype=torch.int64, device="cuda")
        if bool(((c < 0) | (c >= ext)).any()):
            raise ValueError("coordinate out of range")
        key = torch.zeros(c.shape[0], dtype=torch.int64, device="cuda")
        for k in range(nd):
            key = key * shape[k] + c[:, k]
        key, perm = torch.sort(key)
        if key.numel() > 1 and bool((key[1:] == key[:-1]).any()):
            raise ValueError("duplicate coordinates")
        del key
        cs = c.t()[:, perm].to(torch.int32).contiguous()
        return cls(shape, cs, v[perm].contiguous())

    @classmethod
    def from_torch(cls, shape, coords, vals, validate=True):
        torch = _torch()
        shape = tuple(int(s) for s in shape)
        nd = len(shape)
        if coords.dim() != 2:
            raise ValueError("coords must be 2-D")
        if coords.shape[0] != nd and coords.shape[1] == nd:
            coords = coords.t()
        coords = coords.to(device="cuda", dtype=torch.int32).contiguous()
        vals = vals.to(device="cuda", dtype=torch.float64).contiguous()
        if coords.shape[1] != vals.numel():
            raise ValueError("number of coordinates does not match number of values")
        obj = cls(shape, coords, vals)
        if validate and obj.nnz:
            ext = torch.tensor(shape, device="cuda", dtype=torch.int64).view(-1, 1)
            if bool(((coords < 0) | (coords.long() >= ext)).any()):
                raise ValueError("coordinate out of range")
            if obj.nnz > 1:
                # lexicographic strictly increasing <=> sorted and unique
                c = coords.long()
                lt = torch.zeros(obj.nnz - 1, dtype=torch.bool, device="cuda")
                eq = torch.ones(obj.nnz - 1, dtype=torch.bool, device="cuda")
                for k in range(nd):
                    a, b = c[k, :-1], c[k, 1:]
                    lt |= eq & (a < b)
                    eq &= a == b
                if not bool(lt.all()):
                    raise ValueError("coordinates must be lexsorted and duplicate-free")
        return obj

    # ---- norms
    def norm2(self):
        torch = _torch()
        if self._norm2 is None:
            out = torch.empty(1, dtype=torch.float64, device="cuda")
            if self.nnz == 0:
                out.zero_()
            else:
                nat.call_ws("skx_sumsq", (nat.ptr(self.vals), self.nnz, nat.ptr(out)))
            self._norm2 = out
        return self._norm2

    # ---- value range (decides the exact fixed-point RRF stage 1)
    def value_range(self):
        """(emax, emin, bad): binary exponent range of the nonzero values and
        whether any is non-finite/subnormal (one pass + one small D2H, cached)."""
        torch = _torch()
        if getattr(self, "_vrange", None) is None:
            out = torch.empty(3, dtype=torch.int32, device="cuda")
            nat.call("skx_value_range", nat.ptr(self.vals), self.nnz, nat.ptr(out), nat.stream())
            self._vrange = tuple(int(x) for x in out.cpu().tolist())
        return self._vrange

    def fixed_point_ok(self):
        """skx_rrf_stage1_fx sums exactly: finite normal values within 2^41."""
        emax, emin, bad = self.value_range()
        if self.nnz == 0:
            return True
        return not bad and emin >= emax - 41 and -929 <= emax <= 1000

    # ---- fibre-major layout for mode n (libskx skx_coo_fibre)
    def fibre(self, n, ts=None):
        """(colptr, records) of mode n: nonzeros ordered by (i_n, other modes
        ascending) as AoS records {int32 others..., f64 value}, built by one
        packing pass + a radix sort over ceil(log2 s_n) key bits.

        With `ts` (a TensorSketchOp over mode n's other modes) an order-3
        layout is built with that operator's bucket/sign folded into the
        records (skx_coo_fibre_ts) when the bits fit; the RHS sketch then does
        no table lookups.  Other consumers mask the coordinate
        (fibre_mask(n)).  An existing layout is reused as is."""
        torch = _torch()
        if n not in self._fibre:
            rw = int(nat.load().skx_coo_rec_words(self.ndim))
            if rw < 0 or self.ndim < 2:
                raise ValueError(f"sparse order {self.ndim} unsupported by the device layout (2..5)")
            rec = torch.empty(max(self.nnz, 1) * rw, dtype=torch.float64, device="cuda")
            colptr = torch.empty(self.shape[n] + 1, dtype=torch.int64, device="cuda")
            shp, sp_ = nat.host_i64(self.shape)
            mask, owner = 0xFFFFFFFF, None
            if ts is not None and self.ndim == 3 and _ts_packable(self.shape, n, ts.m):
                m_out = ctypes.c_uint32(0)
                off, op = nat.host_i64(ts.tab_off)
                nat.call_ws("skx_coo_fibre_ts",
                            (sp_, n, self.nnz, nat.ptr(self.coords), nat.ptr(self.vals),
                             nat.ptr(ts.tab), op, ts.m, nat.ptr(rec), nat.ptr(colptr),
                             ctypes.byref(m_out)), slot=4)
                mask, owner = int(m_out.value), ts
            else:
                nat.call_ws("skx_coo_fibre", (self.ndim, sp_, n, self.nnz, nat.ptr(self.coords),
                                              nat.ptr(self.vals), nat.ptr(rec), nat.ptr(colptr)),
                            slot=4)
            self._fibre[n] = (colptr, rec)
            self._fibre_meta[n] = (mask, owner)
        return self._fibre[n]

    def has_fibre(self, n):
        return n in self._fibre

    def fibre_mask(self, n):
        """Mask recovering the last other coordinate from mode n's records."""
        return self._fibre_meta[n][0] if n in self._fibre_meta else 0xFFFFFFFF

    def fibre_packed_for(self, n, ts):
        """Bit offset of the bucket field if mode n's layout carries `ts`'s
        buckets/signs, else -1."""
        mask, owner = self._fibre_meta.get(n, (0xFFFFFFFF, None))
        return mask.bit_length() if owner is ts and ts is not None else -1

    def colptr0(self):
        return self.fibre(0)[0]

    # ---- other-major keys for mode n
    def keys(self, n):
        torch = _torch()
        if n not in self._keys:
            others = [k for k in range(self.ndim) if k != n]
            s_n = self.shape[n]
            flat = torch.zeros(self.nnz, dtype=torch.int64, device="cuda")
            for k in others:
                flat = flat * self.shape[k] + self.coords[k].long()
            key = flat * s_n + self.coords[n].long()
            del flat
            if n == self.ndim - 1:
                self._keys[n] = (key, self.vals)
            else:
                key, perm = torch.sort(key)
                self._keys[n] = (key, self.vals[perm].contiguous())
        return self._keys[n]

    def drop_fibre(self, n):
        """Free mode n's fibre-major layout (rebuilt on next use)."""
        self._fibre.pop(n, None)
        self._fibre_meta.pop(n, None)

    def release_layouts(self):
        self._fibre.clear()
        self._fibre_meta.clear()
        self._keys.clear()


def _ts_packable(shape, n, m):
    """skx_coo_fibre_ts bit budget: coordinate bits of the second other mode +
    bucket bits of m must fit in 31."""
    b_other = 1 if n == 2 else 2
    bb = max(int(shape[b_other]) - 1, 0).bit_length()
    return m >= 1 and bb + max(m - 1, 0).bit_length() <= 31


def device_of(t):
    """Device representation of a tensor argument (cached for SparseTensor)."""
    torch = _torch()
    if isinstance(t, SparseTensor):
        if t._device is None:
            t._device = DeviceCoo.from_host(t)
        return t._device
    if isinstance(t, DeviceCoo):
        return t
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            t = t.cuda()
        return t.to(torch.float64).contiguous()
    a = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    return torch.from_numpy(a).cuda()


def is_sparse_dev(d):
    return isinstance(d, DeviceCoo)


def shape_of(t):
    return tuple(int(s) for s in t.shape)


# ============================================================ operations
def tensor_norm(t):
    d = device_of(t)
    if is_sparse_dev(d):
        return float(np.sqrt(d.norm2().item()))
    return float(_torch().linalg.vector_norm(d).item())


def matricize(t, n):
    """Mode-n unfolding s_n x prod(others) (host view/copy; src/tensors.py:151-166)."""
    if isinstance(t, SparseTensor):
        import scipy.sparse as sp
        key = ("m", n)
        if key not in t._unfoldings:
            others = [k for k in range(t.ndim) if k != n]
            rest = [t.shape[k] for k in others]
            cols = (np.ravel_multi_index([t.coords[:, k] for k in others], rest)
                    if t.nnz else np.zeros(0, dtype=np.int64))
            t._unfoldings[key] = sp.coo_matrix(
                (t.values, (t.coords[:, n], cols)), shape=(t.shape[n], int(np.prod(rest)))).tocsr()
        return t._unfoldings[key]
    t = np.asarray(t)
    if not 0 <= n < t.ndim:
        raise ValueError(f"mode {n} out of range for order-{t.ndim} tensor")
    return np.moveaxis(t, n, 0).reshape(t.shape[n], -1)


def matricize_t(t, n):
    """Transposed unfolding T_(n)^T (src/tensors.py:169-176)."""
    if isinstance(t, SparseTensor):
        return matricize(t, n).T.tocsr()
    return matricize(t, n).T


def fold(mat, n, shape):
    """Inverse of matricize (src/tensors.py:197-201); numpy or torch."""
    shape = tuple(shape)
    rest = [shape[k] for k in range(len(shape)) if k != n]
    if not isinstance(mat, np.ndarray) and hasattr(mat, "movedim"):
        return mat.reshape([shape[n]] + rest).movedim(0, n)
    return np.moveaxis(np.asarray(mat).reshape([shape[n]] + rest), 0, n)


def ttm_dev(t, mat, n):
    """Mode-n product on device: t x_n mat (mat: new x s_n)."""
    torch = _torch()
    out = torch.tensordot(mat, t, dims=([1], [n]))
    return out.movedim(0, n)


def ttm(t, mat, n):
    torch = _torch()
    mat = np.asarray(mat)
    t = np.asarray(t)
    if mat.shape[1] != t.shape[n]:
        raise ValueError(
            f"ttm mode {n}: matrix has {mat.shape[1]} columns, tensor extent is {t.shape[n]}")
    out = ttm_dev(torch.from_numpy(np.ascontiguousarray(t)).cuda(),
                  torch.from_numpy(np.ascontiguousarray(mat)).cuda(), n)
    return out.contiguous().cpu().numpy()


def _ttmc_skip_sparse_dev(d, factors, skip, chunk=1 << 16):
    """Skip-mode TTMc of a DeviceCoo: (s_skip, prod R_others) unfolding."""
    torch = _torch()
    others = [k for k in range(d.ndim) if k != skip]
    s_n = d.shape[skip]
    rr = int(np.prod([factors[k].shape[1] for k in others]))
    if d.ndim == 3 and rr <= 1024:
        out = torch.empty((s_n, rr), dtype=torch.float64, device="cuda")
        colptr, rec = d.fibre(skip)
        a1, a2 = (factors[k].contiguous() for k in others)
        nat.call("skx_ttmc3_skip_coo", s_n, nat.ptr(colptr), nat.ptr(rec),
                 ctypes.c_uint32(d.fibre_mask(skip)), nat.ptr(a1), int(a1.shape[1]), nat.ptr(a2),
                 int(a2.shape[1]), nat.ptr(out), nat.stream())
        return out
    # other orders: the same per-nonzero Kronecker rows on the device, summed
    # per output row in the reference's (mode-stable) order, chunk by chunk
    out = torch.zeros((s_n, rr), dtype=torch.float64, device="cuda")
    rows_all = d.coords[skip].long()
    order = torch.argsort(rows_all, stable=True)
    for lo in range(0, d.nnz, chunk):
        idx = order[lo:lo + chunk]
        contrib = d.vals[idx][:, None]
        for k in others:
            fk = factors[k][d.coords[k][idx].long()]
            contrib = (contrib[:, :, None] * fk[:, None, :]).reshape(idx.numel(), -1)
        rows, counts = torch.unique_consecutive(rows_all[idx], return_counts=True)
        out[rows] += torch.segment_reduce(contrib, "sum", lengths=counts, axis=0)
    return out


def ttmc_dev(d, factors, skip=None):
    """ttmc on device (src/tensors.py:217-258).  Dense: mode products in
    ascending mode order.  Sparse, skip = n: the libskx kernel (order 3) over
    mode n's fibre-major layout; skip = None: the mode-0 skip result
    contracted with A_0^T (same sum, associated around the small side)."""
    torch = _torch()
    nd = d.ndim
    if not is_sparse_dev(d):
        return ttmc_all_dense_dev(d, factors, skip)
    if skip is not None:
        y = _ttmc_skip_sparse_dev(d, factors, skip)
        shp = [d.shape[k] if k == skip else factors[k].shape[1] for k in range(nd)]
        return fold(y, skip, shp)
    y0 = _ttmc_skip_sparse_dev(d, factors, 0)
    core = factors[0].t() @ y0
    return core.reshape([factors[k].shape[1] for k in range(nd)])


def ttmc(t, factors, skip=None, chunk=1 << 16):
    """Tensor times matrix-chain: contract every mode m != skip with
    factors[m]^T (src/tensors.py:217-247); numpy result."""
    nd = t.ndim if isinstance(t, SparseTensor) else np.asarray(t).ndim
    if skip is not None and not 0 <= skip < nd:
        raise ValueError(f"skip mode {skip} out of range")
    shape = tuple(t.shape)
    for m in range(nd):
        if m == skip:
            continue
        if np.shape(factors[m])[0] != shape[m]:
            raise ValueError(
                f"ttmc mode {m}: factor has {np.shape(factors[m])[0]} rows, tensor extent is {shape[m]}")
    d = device_of(t)
    fs = [_to_dev_mat(f) for f in factors]
    return ttmc_dev(d, fs, skip).contiguous().cpu().numpy()


def khatri_rao(mats):
    """Column-wise Kronecker product, first matrix slowest (src/tensors.py:288-301)."""
    torch = _torch()
    mats = [np.asarray(m) for m in mats]
    k = mats[0].shape[1]
    if any(m.shape[1] != k for m in mats):
        raise ValueError("khatri_rao inputs must share the column count")
    out = torch.from_numpy(mats[0]).cuda()
    for m in mats[1:]:
        out = (out[:, None, :] * torch.from_numpy(m).cuda()[None, :, :]).reshape(-1, k)
    return out.cpu().numpy()


# ---- fitness -------------------------------------------------------------
def tucker_cross_dev(d, core, factors):
    """<ttmc(T, {A}), C> on device; returns a 0-d CUDA tensor."""
    torch = _torch()
    if is_sparse_dev(d):
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        shp, sp_ = nat.host_i64(d.shape)
        rk, rp = nat.host_i64([f.shape[1] for f in factors])
        fa = [f.contiguous() for f in factors]
        arr, fp = nat.host_ptrs(fa)
        cpt, rec0 = d.fibre(0) if d.ndim == 3 else (None, None)
        # own workspace slot: the fitness may run on a side stream concurrently
        # with the next sweep's sub-problems
        nat.call_ws("skx_tucker_cross_coo",
                    (d.ndim, sp_, rp, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals), fp,
                     nat.ptr(core.contiguous()), nat.ptr(cpt), nat.ptr(rec0),
                     ctypes.c_uint32(d.fibre_mask(0)), nat.ptr(out)), slot=5)
        return out[0]
    return (ttmc_all_dense_dev(d, factors) * core).sum()


def ttmc_all_dense_dev(d, factors, skip=None):
    """ttmc(T, factors, skip) of a dense C-order CUDA tensor by libskx mode
    products in ascending mode order (skx_ttm_lead; the first streams the
    tensor once).  Ranks > 32 use torch tensordot."""
    torch = _torch()
    modes = [k for k in range(len(factors)) if k != skip]
    if any(int(factors[k].shape[1]) > 32 for k in modes):
        proj = d
        for k in modes:
            proj = ttm_dev(proj, factors[k].t(), k)
        return proj
    cur = d.contiguous()
    shape = list(cur.shape)
    for k in modes:
        a = factors[k]
        B = int(np.prod(shape[:k])) if k else 1
        s = shape[k]
        P = int(np.prod(shape[k + 1:])) if k + 1 < len(shape) else 1
        R = int(a.shape[1])
        out = torch.empty(B * R * P, dtype=torch.float64, device="cuda")
        nat.call("skx_ttm_lead", nat.ptr(cur), B, s, P, nat.ptr(a.contiguous()), R, nat.ptr(out),
                 nat.stream())
        shape[k] = R
        cur = out.view(shape)
    return cur


def ttmc3_r20_eligible(d, factors):
    """Order-3 COO with ranks (R0 <= 32, 20, 20): skx_tucker_ttmc3_r20 applies."""
    return (is_sparse_dev(d) and d.ndim == 3 and int(factors[1].shape[1]) == 20
            and int(factors[2].shape[1]) == 20 and int(factors[0].shape[1]) <= 32)


def ttmc3_full_dev(d, factors):
    """P = X x_0 A0^T x_1 A1^T x_2 A2^T of an order-3 COO at ranks (R0, 20,
    20) as an (R0, 20, 20) CUDA tensor: one pass over the mode-0 layout
    (skx_tucker_ttmc3_r20).  <P, C> is the cross term of any core C on these
    factors."""
    torch = _torch()
    R0 = int(factors[0].shape[1])
    cpt, rec0 = d.fibre(0)
    shp, sp_ = nat.host_i64(d.shape)
    p = torch.empty((400, R0), dtype=torch.float64, device="cuda")
    fa = [f.contiguous() for f in factors]
    nat.call_ws("skx_tucker_ttmc3_r20",
                (sp_, R0, nat.ptr(cpt), nat.ptr(rec0), ctypes.c_uint32(d.fibre_mask(0)),
                 nat.ptr(fa[0]), nat.ptr(fa[1]), nat.ptr(fa[2]), nat.ptr(p)), slot=5)
    return p.t().reshape(R0, 20, 20)


def fitness_from_cross_dev(norm2, cross, mod):
    torch = _torch()
    r2 = torch.clamp(norm2 - 2.0 * cross + mod, min=0.0)
    return 1.0 - torch.sqrt(r2) / torch.sqrt(norm2)


def fitness_tucker_dev(d, core, factors, norm2=None, comm=None):
    torch = _torch()
    if norm2 is None:
        norm2 = d.norm2()[0] if is_sparse_dev(d) else (d * d).sum()
    cross = tucker_cross_dev(d, core, factors)
    if comm is not None:
        cross = comm.allreduce(cross.clone().view(1))[0]
    mod = (core * core).sum()
    r2 = torch.clamp(norm2 - 2.0 * cross + mod, min=0.0)
    return 1.0 - torch.sqrt(r2) / torch.sqrt(norm2)


def cp_cross_dev(d, factors, weights):
    torch = _torch()
    if is_sparse_dev(d) and d.ndim == 3 and int(factors[0].shape[1]) <= 32:
        # warp per mode-0 slice over the fibre layout (built by a packing pass
        # only: the lexsorted COO is already in mode-0 order)
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        fa = [f.contiguous() for f in factors]
        arr, fp = nat.host_ptrs(fa)
        cpt, rec0 = d.fibre(0)
        nat.call_ws("skx_cp_cross_fibre3",
                    (d.shape[0], nat.ptr(cpt), nat.ptr(rec0), ctypes.c_uint32(d.fibre_mask(0)),
                     int(factors[0].shape[1]), fp, nat.ptr(weights.contiguous()), nat.ptr(out)),
                    slot=5)
        return out[0]
    if is_sparse_dev(d):
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        shp, sp_ = nat.host_i64(d.shape)
        fa = [f.contiguous() for f in factors]
        arr, fp = nat.host_ptrs(fa)
        nat.call_ws("skx_cp_cross_coo",
                    (d.ndim, sp_, int(factors[0].shape[1]), d.nnz, nat.ptr(d.coords),
                     nat.ptr(d.vals), fp, nat.ptr(weights.contiguous()), nat.ptr(out)))
        return out[0]
    # dense: mttkrp mode 0 then dot with scaled A0
    nd = d.dim()
    R = factors[0].shape[1]
    kr = factors[1]
    for a in factors[2:]:
        kr = (kr[:, None, :] * a[None, :, :]).reshape(-1, R)
    m0 = d.reshape(d.shape[0], -1) @ kr
    return ((factors[0] * weights) * m0).sum()


def fitness_cp_dev(d, factors, weights, norm2=None, comm=None, cross=None):
    """CP fitness (src/tensors.py:354-368); `cross` = <T, model> when the
    caller already has it (then d is not read)."""
    torch = _torch()
    if norm2 is None:
        norm2 = d.norm2()[0] if is_sparse_dev(d) else (d * d).sum()
    if cross is None:
        cross = cp_cross_dev(d, factors, weights)
        if comm is not None:
            cross = comm.allreduce(cross.clone().view(1))[0]
    scaled = factors[0] * weights
    g = torch.ones((factors[0].shape[1],) * 2, dtype=torch.float64, device="cuda")
    for a in factors[1:]:
        g = g * (a.t() @ a)
    mod = ((scaled.t() @ scaled) * g).sum()
    r2 = torch.clamp(norm2 - 2.0 * cross + mod, min=0.0)
    return 1.0 - torch.sqrt(r2) / torch.sqrt(norm2)


def _to_dev_mat(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


def fitness(t, model):
    """1 - ||T - model|| / ||T|| without densifying (src/tensors.py:339-368)."""
    d = device_of(t)
    norm2 = d.norm2()[0] if is_sparse_dev(d) else (d * d).sum()
    if float(norm2.item()) == 0.0:
        raise ValueError("fitness undefined for a zero-norm tensor")
    if isinstance(model, TuckerModel):
        f = fitness_tucker_dev(d, _to_dev_mat(model.core), [_to_dev_mat(a) for a in model.factors],
                               norm2)
    elif isinstance(model, CPModel):
        f = fitness_cp_dev(d, [_to_dev_mat(a) for a in model.factors], _to_dev_mat(model.weights),
                           norm2)
    else:
        raise TypeError(f"unsupported model type {type(model)!r}")
    return float(f.item())


def mttkrp_dev(d, factors, n):
    """T_(n) @ khatri_rao(factors except n) on device (src/tensors.py:307-336);
    factors: device matrices for every mode.  Sparse: per-nonzero Hadamard
    rows summed per mode-n index in the (stable) mode-n order -- deterministic,
    no atomics."""
    torch = _torch()
    nd = len(shape_of(d))
    others = [k for k in range(nd) if k != n]
    fs = [factors[k] for k in others]
    R = fs[0].shape[1]
    if is_sparse_dev(d):
        out = torch.zeros((d.shape[n], R), dtype=torch.float64, device="cuda")
        if d.nnz == 0:
            return out
        rows_all = d.coords[n].long()
        order = torch.argsort(rows_all, stable=True)
        chunk = 1 << 22
        for lo in range(0, d.nnz, chunk):
            idx = order[lo:lo + chunk]
            prod = d.vals[idx][:, None].expand(-1, R).clone()
            for k, f in zip(others, fs):
                prod *= f[d.coords[k][idx].long()]
            rows, counts = torch.unique_consecutive(rows_all[idx], return_counts=True)
            out[rows] += torch.segment_reduce(prod, "sum", lengths=counts, axis=0)
        return out
    kr = fs[0]
    for f in fs[1:]:
        kr = (kr[:, None, :] * f[None, :, :]).reshape(-1, R)
    return d.movedim(n, 0).reshape(d.shape[n], -1) @ kr


def mttkrp(t, factors, n):
    """T_(n) @ khatri_rao(others) (src/tensors.py:307-336); numpy result."""
    d = device_of(t)
    nd = len(shape_of(d))
    fs = [_to_dev_mat(f) for f in factors]
    others = [k for k in range(nd) if k != n]
    R = fs[others[0]].shape[1]
    for k in others:
        if fs[k].shape[0] != shape_of(d)[k]:
            raise ValueError(f"mttkrp mode {k}: factor has {fs[k].shape[0]} rows, extent is {shape_of(d)[k]}")
        if fs[k].shape[1] != R:
            raise ValueError("mttkrp factors must share the column count")
    return mttkrp_dev(d, fs, n).cpu().numpy()


