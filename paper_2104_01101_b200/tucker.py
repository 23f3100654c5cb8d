"""Sketched Tucker-ALS driver (drop-in for the sketched path of src/tucker.py).

``sketched_tucker_als(t, TuckerConfig) -> (TuckerModel, SweepTrace)`` keeps the
reference's signature, validation, RNG stream usage and redraw-once policy
(src/tucker.py:216-300).  Everything between the input upload and the final
model download runs on the GPU: RRF initialisation (K4 + cuSOLVER SVD), the
TensorSketch right-hand sides (K1), per-subproblem sketches (K2 / K3), the
rank-constrained solve (K5) with its fused residual, and the per-sweep fitness
pass (K7).  HOOI and the one-variable baseline (src/tucker.py:155-193, 303-364)
are outside this build's path.
"""
from __future__ import annotations

import ctypes
import os
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import rng as rngmod
from .linalg import (NormalSource, RankDeficientError, qr_lapack_dev, resid_dev, rsvd_lrls_dev,
                     rsvd_lrls_hits_fixed_dev,
                     rsvd_lrls_hits_dev, y_times_dev,
                     rsvd_lrls_rows_dev, top_svd_dev)
from .sketching import (TensorSketchOp, draw_rrf_tables, filter_fibers_dev, filter_gather_fixed_dev,
                        finish_rrf_scan, gather_slices_fixed_dev,
                        gather_coo_dev, gather_dense_dev, gather_slices_dev, hits_to_dense,
                        kron_rows_dev, lev_det_dev, lev_sample_dev, mode_last_dev, plan_rrf_scans,
                        rrf_table_dev, ts_kron_dev, ts_kron_plan_dev, ts_rhs_dense_dev,
                        ts_rhs_mode_dev)
from .tensors import (DeviceCoo, SparseTensor, TuckerModel, compact3_aux_to_device, device_of,
                      fitness_from_cross_dev, fitness_tucker_dev, is_sparse_dev, to_host,
                      ttmc3_full_dev, ttmc3_r20_eligible, unpack_compact3,
                      matricize, shape_of, ttm_dev, ttmc_dev)

SKETCH_KINDS = (None, "tensorsketch", "leverage-random", "leverage-deterministic")


def _torch():
    import torch
    return torch


@dataclass
class TuckerConfig:
    ranks: tuple
    max_sweeps: int = 5
    sketch: str | None = None
    sketch_size: int | None = None
    sketch_factor: float | None = None
    init: str | None = None
    rrf_width: int | None = None
    seed: int = 0
    convergence_tol: float = 0.0

    def __post_init__(self):
        self.ranks = tuple(int(r) for r in self.ranks)
        if self.sketch not in SKETCH_KINDS:
            raise ValueError(f"unknown sketch kind {self.sketch!r}")

    def resolved_sketch_size(self):
        if self.sketch_size is not None:
            return int(self.sketch_size)
        if self.sketch_factor is not None:
            return int(math.ceil(self.sketch_factor * max(self.ranks) ** 2))
        raise ValueError("sketched drivers need sketch_size or sketch_factor")

    def resolved_rrf_width(self, rank):
        if self.rrf_width is not None:
            return max(int(self.rrf_width), rank)
        if self.sketch_factor is not None:
            k_factor = self.sketch_factor
        elif self.sketch_size is not None:
            k_factor = self.sketch_size / max(self.ranks) ** 2
        else:
            k_factor = 4.0
        return max(rank, int(math.ceil(math.sqrt(k_factor) * rank)))


@dataclass
class SweepTrace:
    """Per-sweep fitness / wall time plus per-subproblem residuals."""

    fitness: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    wall_s: list = field(default_factory=list)
    stage_split: int | None = None


def _validate_ranks(shape, ranks):
    if len(ranks) != len(shape):
        raise ValueError("one rank per mode required")
    for n, (s, r) in enumerate(zip(shape, ranks)):
        if not 1 <= r <= s:
            raise ValueError(f"rank {r} invalid for extent {s} at mode {n}")


def _check_sketch_size(m, ranks):
    for j in range(len(ranks)):
        need = int(np.prod([ranks[n] for n in range(len(ranks)) if n != j]))
        if m < need:
            raise ValueError(f"sketch size {m} below {need}, the sketched system width for mode {j}")


# ------------------------------------------------------------------ RRF init
def rrf_partition_dev(d, modes):
    """Records {i_n << 40 | j, value} of a DeviceCoo grouped by output row
    block for the RRF modes (up to two), for skx_rrf_stage1_rec; None when
    the fixed-point stage-1 path does not apply.  Returns {mode: (keys, vals)}."""
    torch = _torch()
    modes = [n for n in modes if not d.has_fibre(n)][:2]
    if not modes or not d.fixed_point_ok() or d.nnz == 0:
        return None
    shape = d.shape
    for n in modes:
        if shape[n] >= (1 << 24) or int(np.prod([shape[k] for k in range(d.ndim) if k != n])) >= (1 << 40):
            return None
    recs = [(torch.empty(d.nnz, dtype=torch.int64, device="cuda"),
             torch.empty(d.nnz, dtype=torch.float64, device="cuda")) for _ in modes]
    shp, sp_ = nat.host_i64(shape)
    marr = (ctypes.c_int * len(modes))(*modes)
    k1, v1 = recs[1] if len(recs) > 1 else (None, None)
    nat.call_ws("skx_rrf_partition", (d.ndim, sp_, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals),
                                      len(modes), ctypes.cast(marr, ctypes.c_void_p),
                                      nat.ptr(recs[0][0]), nat.ptr(recs[0][1]),
                                      nat.ptr(k1) if k1 is not None else None,
                                      nat.ptr(v1) if v1 is not None else None), slot=11)
    return dict(zip(modes, recs))


def rrf_stage1_dev(d, n, tabs, part=None):
    """CountSketch stage of the composite sketch of T_(n): s_n x k2.  part:
    this mode's partitioned records (rrf_partition_dev), if built."""
    torch = _torch()
    shape = shape_of(d)
    s_n = shape[n]
    st1 = torch.empty((s_n, tabs.k2), dtype=torch.float64, device="cuda")
    if part is not None:
        keys, vals = part
        emax = d.value_range()[0]
        nat.call_ws("skx_rrf_stage1_rec", (s_n, ctypes.c_uint64(tabs.P), d.nnz,
                                           nat.ptr(d.coords[n]), nat.ptr(keys), nat.ptr(vals), emax,
                                           *tabs.args(), tabs.k2, nat.ptr(st1)), slot=8)
    elif is_sparse_dev(d) and not d.has_fibre(n) and d.fixed_point_ok():
        # no mode-n layout (leverage runs build none): exact fixed-point
        # accumulation straight from the lexsorted COO instead of sorting one
        emax = d.value_range()[0]
        shp, sp_ = nat.host_i64(shape)
        nat.call_ws("skx_rrf_stage1_fx", (d.ndim, sp_, n, d.nnz, nat.ptr(d.coords), nat.ptr(d.vals),
                                          emax, *tabs.args(),
                                          tabs.k2, nat.ptr(st1)), slot=8)
    elif is_sparse_dev(d):
        colptr, rec = d.fibre(n)
        others = [k for k in range(d.ndim) if k != n]
        ext, ep = nat.host_i64([shape[k] for k in others])
        nat.call("skx_rrf_stage1_coo", len(others), ep, s_n, nat.ptr(colptr), nat.ptr(rec),
                 *tabs.args(), tabs.k2, ctypes.c_uint32(d.fibre_mask(n)), nat.ptr(st1),
                 nat.stream())
    else:
        tab = rrf_table_dev(tabs)
        dl, nl = mode_last_dev(d, n)  # gather form on a mode-last copy
        shp, sp_ = nat.host_i64(tuple(dl.shape))
        nat.call_ws("skx_rrf_stage1_dense", (nat.ptr(dl), len(shape), sp_, nl, nat.ptr(tab),
                                             tabs.k2, nat.ptr(st1)))
    return st1


def _rrf_finish(d, n, rank, tabs, gauss, comm=None, part=None):
    """Composite sketch B = (T_(n) T_cs) G and its leading left singular vectors."""
    return _rrf_from_stage1(rrf_stage1_dev(d, n, tabs, part), rank, gauss, comm)


def _rrf_from_stage1(st1, rank, gauss, comm=None):
    torch = _torch()
    b = st1 @ torch.from_numpy(gauss).cuda()
    if comm is not None:
        # the Gaussian stage is linear: reduce the s_n x k1 product of each
        # rank's partial stage 1 instead of the s_n x k2 stage 1
        comm.allreduce(b)
    if min(b.shape) < rank:
        raise ValueError(f"cannot extract {rank} directions from a {tuple(b.shape)} sketch")
    u, _, _ = top_svd_dev(b, rank)
    return u.contiguous()


def _rrf_dims(shape, n, rank, width):
    if width < rank:
        raise ValueError(f"sketch width {width} below target rank {rank}")
    P = int(np.prod([shape[k] for k in range(len(shape)) if k != n]))
    return P, rank * rank + width


def init_rrf_dev(d, n, rank, width, gen, comm=None):
    """Range-finder init of factor n (src/tucker.py:129-144) on device: the
    rng draws integers(0,k2,P), integers(0,2,P), standard_normal((k2,k1)) in
    the reference's order (src/sketching.py:54-56, 323)."""
    P, k2 = _rrf_dims(shape_of(d), n, rank, width)
    tabs = draw_rrf_tables(gen, P, k2)
    gauss = gen.standard_normal((k2, width)) / np.sqrt(width)
    return _rrf_finish(d, n, rank, tabs, gauss, comm)


def init_rrf(tn, rank, width, rng):
    """API form: tn is an unfolding (dense s x P array or scipy sparse)."""
    import scipy.sparse as sp
    torch = _torch()
    gen = rngmod.make_rng(rng)
    if sp.issparse(tn):
        c = tn.tocoo()
        d = DeviceCoo.from_torch(tn.shape, torch.from_numpy(np.stack([c.row, c.col]).astype(np.int64)),
                                 torch.from_numpy(c.data.astype(np.float64)), validate=False)
        order = torch.from_numpy(np.lexsort((c.col, c.row))).cuda()
        d = DeviceCoo(tn.shape, d.coords[:, order].contiguous(), d.vals[order].contiguous())
    else:
        d = device_of(np.asarray(tn))
    return init_rrf_dev(d, 0, rank, width, gen).cpu().numpy()


def random_orthonormal_dev(n_rows, n_cols, gen):
    """Q of a Gaussian matrix (src/tucker.py:107-109) with numpy's QR signs."""
    torch = _torch()
    g = torch.from_numpy(gen.standard_normal((n_rows, n_cols))).cuda()
    q, _ = qr_lapack_dev(g)
    return q[:, :n_cols].contiguous()


# ------------------------------------------------------------------ driver
# leverage sampling on sparse tensors: rsvd on the hit columns when the gathered
# fibres fill less than this fraction of the m x s_n right-hand side
HITS_DENSITY = 0.05
# Multi-rank speculative leverage sweeps take the sync-free fixed-capacity
# hit path (no host read of hit counts, so no host sync between the ranks'
# collectives); a single process keeps the host-sized path, which launches
# fewer, smaller kernels (config 5: 457 vs 508 ms per call with the fixed
# path).  FORCE_FIXED_HITS: tests.
FORCE_FIXED_HITS = False
FIXED_HITS_OFF = False

_STREAMS = {}


def _init_streams():
    """(normal-priority, high-priority) streams for the initialisation, created
    once per device: the caching allocator keys free blocks by stream, so
    fresh streams every run would defeat reuse of the large layout buffers."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _STREAMS:
        lo, hi = torch.cuda.Stream.priority_range()
        _STREAMS[dev] = (torch.cuda.Stream(priority=lo), torch.cuda.Stream(priority=hi))
    return _STREAMS[dev]


# host COO inputs of at least this many nonzeros are uploaded in chunks of
# this many rows (leverage runs; the TensorSketch layouts need the whole tensor)
# nonzeros per upload chunk (config 5: 30 chunks; 15 measured ~3 ms slower
# e2e: the last chunk's stage-1 sums are the tail behind the upload)
UPLOAD_CHUNK = 1 << 25

_UP_STREAMS = {}


def _upload_streams():
    """(copy, convert) streams for the chunked host upload, one pair per device."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _UP_STREAMS:
        _, hi = torch.cuda.Stream.priority_range()
        # the convert stream runs the on-device unpack of each uploaded chunk
        # at high priority (its CTAs go ahead of the rejection scans), so the
        # copy stream only ever holds copies and the PCIe pipe never idles
        _UP_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream(priority=hi))
    return _UP_STREAMS[dev]


_YG_STREAMS = {}


def _yg_stream():
    """High-priority stream for the early Y G pass of speculative sweeps."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _YG_STREAMS:
        _, hi = torch.cuda.Stream.priority_range()
        _YG_STREAMS[dev] = torch.cuda.Stream(priority=hi)
    return _YG_STREAMS[dev]


_FIT_STREAMS = {}


def _fit_stream():
    """Low-priority stream for the overlapped per-sweep fitness (one per device)."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _FIT_STREAMS:
        lo, _ = torch.cuda.Stream.priority_range()
        _FIT_STREAMS[dev] = torch.cuda.Stream(priority=lo)
    return _FIT_STREAMS[dev]


_ST1_STREAMS = {}


def _stage1_stream(i):
    """High-priority stream for the chunked RRF stage-1 sums of the i-th
    range-finder mode (i >= 1; the first runs on the init main stream)."""
    torch = _torch()
    key = (torch.cuda.current_device(), i)
    if key not in _ST1_STREAMS:
        _, hi = torch.cuda.Stream.priority_range()
        _ST1_STREAMS[key] = torch.cuda.Stream(priority=hi)
    return _ST1_STREAMS[key]


_RES_STREAMS = {}
# sub-problem residuals over a Y of at least this many entries run on a side
# stream (config 4: 1.6e8, 83.8 -> 81.8 ms per call); below it the extra
# stream hand-off costs more than the pass (configs 1-2: +0.2-0.5 ms)
RESID_SIDE_MIN = 1 << 22


def _res_stream():
    """Low-priority stream for the sub-problem residuals (one per device)."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _RES_STREAMS:
        lo, _ = torch.cuda.Stream.priority_range()
        _RES_STREAMS[dev] = torch.cuda.Stream(priority=lo)
    return _RES_STREAMS[dev]


class _Run:
    """Device state of one sketched_tucker_als call."""

    def __init__(self, t, config, comm=None):
        torch = _torch()
        if config.sketch is None:
            raise ValueError("sketched_tucker_als needs a sketch kind")
        self.shape = tuple(int(s) for s in t.shape)
        self.ndim = len(self.shape)
        self.ranks = config.ranks
        _validate_ranks(self.shape, self.ranks)
        self.m = config.resolved_sketch_size()
        _check_sketch_size(self.m, self.ranks)
        self.cfg = config
        self.comm = comm
        self._host = None
        if (isinstance(t, SparseTensor) and t._device is None and comm is None
                and (config.init or "rrf") == "rrf" and self.ndim > 1):
            # host COO: the upload is deferred into initialise_and_prep, where
            # it overlaps the data-independent rejection scans
            self._host = t
            self.d = None
            self.sparse = True
        else:
            self._attach(device_of(t))
        self.rng_init, self.rng_sketch, self.rng_solve = rngmod.split_rng(config.seed, 3)
        # one sweep's Gaussian test matrices (rsvd_lrls: s_n x min(R_n + 10, s_n))
        per_sweep = sum(s * min(r + 10, s) for s, r in zip(self.shape, self.ranks))
        self.normals = NormalSource(self.rng_solve, batch=per_sweep)
        self.use_ts = config.sketch == "tensorsketch"
        # where the sub-problem residuals run (set for the sweeps, see _finish_dense)
        self.res_stream = None
        # Algorithm 6: take the last sweep's fitness through the full TTMc and
        # keep it (P, factors, event) for the CP stage's final fitness
        self.ttmc_last = False
        self.last_ttmc = None
        self.factors = [None] * self.ndim
        self.ts_ops = [None] * self.ndim
        self.ts_rhs = [None] * self.ndim
        self.events = []

    def _attach(self, d):
        self.d = d
        self.sparse = is_sparse_dev(d)
        n2 = d.norm2().clone() if self.sparse else (d * d).sum().view(1)
        if self.comm is not None:
            self.comm.allreduce(n2)
        self.norm2 = n2[0]

    def others(self, n):
        return [k for k in range(self.ndim) if k != n]

    def initialise_and_prep(self):
        """RRF init of modes 1..N-1 plus the TensorSketch prep: layouts and
        right-hand sides (high-priority stream), then the compute-bound
        rejection scans (normal-priority side stream) with each mode's RRF
        stage 1 overlapping the next mode's scan.  Host draws keep the
        reference order: per mode hash, signs, then Gaussian."""
        torch = _torch()
        init = self.cfg.init or "rrf"
        if init not in ("rrf", "random"):
            raise ValueError(f"unknown init {init!r} for sketched_tucker_als")
        if init == "random" or self.ndim == 1:
            for n in range(1, self.ndim):
                self.factors[n] = random_orthonormal_dev(self.shape[n], self.ranks[n], self.rng_init)
            self.prep()
            return
        caller = torch.cuda.current_stream()
        # the compute-bound scans go to a normal-priority side stream in short
        # CTAs; everything else runs on a high-priority stream, so the block
        # scheduler gives RRF stage 1 the SMs ahead of the next scan
        side, main = _init_streams()
        side.wait_stream(caller)
        main.wait_stream(caller)
        modes = list(range(1, self.ndim))
        dims = []
        for n in modes:
            width = self.cfg.resolved_rrf_width(self.ranks[n])
            P, k2 = _rrf_dims(self.shape, n, self.ranks[n], width)
            dims.append((P, k2, width))
        # The rejection scans depend only on rng_init's position: every mode's
        # scan is enqueued first (later starts bracketed) on the normal-priority
        # side stream, in short CTAs.  The layouts and right-hand sides (high
        # priority) take SMs ahead of them as CTAs retire, and the IMAD-bound
        # scans fill in around the memory/latency-bound layout work (config 4:
        # the first scan ends ~2 ms earlier than if started after the layouts);
        # with a host input they also run while the COO arrays are uploaded.
        # RRF stage 1 of mode n (high priority) overlaps scan n+1.
        scans = plan_rrf_scans(self.rng_init, [(P, k2, k2 * w) for P, k2, w in dims], side,
                               self.comm)
        if (self._host is not None and not self.use_ts and self._host.nnz >= UPLOAD_CHUNK
                and (self._host._soa is not None or self._host._c3 is not None)):
            # leverage run on a host COO: upload in chunks and sketch them as
            # they land, under the remaining upload
            with torch.cuda.stream(main):
                self._init_from_host_chunked(modes, scans, dims, main)
            caller.wait_stream(main)
            caller.wait_stream(side)
            return
        if self._host is not None:
            with torch.cuda.stream(main):
                self.draw_ts_ops()
                self._host._device = DeviceCoo.from_host(self._host)
                self._attach(self._host._device)
                self._host = None
        part = {}
        with torch.cuda.stream(main):
            self.draw_ts_ops()
            if self.sparse:
                if self.use_ts:  # layouts first, TS buckets folded in: the TS sketches read them
                    for n in range(self.ndim):
                        self.d.fibre(n, self.ts_ops[n])
                else:  # leverage: only the fitness reads a layout (mode 0: a packing pass)
                    self.d.fibre(0)
                self.d.value_range()  # RRF stage 1: exact fixed-point path when in range
                if not self.use_ts and self.d.ndim >= 3 and os.environ.get("SKX_RRF_PART") == "1":
                    # (opt-in) the nonzeros partitioned by RRF output row block
                    # while the scans run, so each stage 1 accumulates in L2.
                    # Measured at config 5: stage 1 53/59 -> 45/44 ms per mode,
                    # but the partition (64 ms, scattered 16-byte records) slows
                    # the first scan 64 -> 117 ms: 477 -> 509 ms per call.  The
                    # L2 atomic rate (~4.4e10/s), not DRAM, bounds both forms.
                    part = rrf_partition_dev(self.d, modes) or {}
            self.prep()
            # small first-sweep inputs that do not depend on the RRF factors,
            # built while the scans occupy the GPU: the Kronecker-sketch plans
            # and the first batch of Gaussian test matrices
            if self.use_ts:
                for op in self.ts_ops:
                    ts_kron_plan_dev(op)
            self.normals.prefetch()
            for n, scan, (P, k2, width) in zip(modes, scans, dims):
                tabs = finish_rrf_scan(scan, self.rng_init, P)
                gauss = self.rng_init.standard_normal((k2, width)) / np.sqrt(width)
                self.factors[n] = _rrf_finish(self.d, n, self.ranks[n], tabs, gauss, self.comm,
                                              part.pop(n, None))
        caller.wait_stream(main)
        caller.wait_stream(side)

    def _init_from_host_chunked(self, modes, scans, dims, main):
        """Host COO (staged as pinned int32 SoA by SparseTensor.from_sorted)
        -> device in UPLOAD_CHUNK-column pieces on a copy stream, values
        first.  RRF stage 1 of every mode accumulates each chunk as soon as it
        has landed (exact fixed-point sums, three limbs: the sums do not
        depend on the chunking), so the range-finder
        sketches finish with the upload instead of after it; the rejection
        scans run meanwhile.  Falls back to the whole-tensor path when the
        values do not admit exact fixed-point sums."""
        torch = _torch()
        st = self._host
        nd, nnz = self.ndim, st.nnz
        copy, conv = _upload_streams()
        copy.wait_stream(main)
        conv.wait_stream(main)
        import warnings
        with warnings.catch_warnings():  # read-only host arrays are only read
            warnings.simplefilter("ignore", UserWarning)
            hv = torch.from_numpy(np.ascontiguousarray(st.values))
        vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
        coords = torch.empty((nd, nnz), dtype=torch.int32, device="cuda")
        chunk = UPLOAD_CHUNK
        conv_ev, bounds = [], []
        c3 = st._c3
        if c3 is not None:
            # compact order-3 staging: per slice-aligned chunk, its values and
            # packed coordinate words cross PCIe and skx_coo_unpack3 expands
            # them on the device (4 instead of 12 bytes of coordinates per
            # nonzero over PCIe); the chunks' stage-1 sums start as they land
            ptr_h = c3["ptr0"]
            s0 = int(ptr_h.numel()) - 1
            packed = torch.empty(nnz, dtype=torch.int32, device="cuda")
            # the mode-0 fibre layout (the fitness passes' input) is packed
            # chunk by chunk behind each unpack; its colptr is ptr0
            rec0 = torch.empty(max(nnz, 1) * 2, dtype=torch.float64, device="cuda")
            with torch.cuda.stream(copy):
                aux = compact3_aux_to_device(c3)
            s_lo = 0
            while s_lo < s0:
                lo = int(ptr_h[s_lo])
                s_hi = int(torch.searchsorted(ptr_h, torch.tensor(lo + chunk), right=True)) - 1
                s_hi = min(max(s_hi, s_lo + 1), s0)
                hi = int(ptr_h[s_hi])
                with torch.cuda.stream(copy):
                    # values and coordinate words of the chunk (the value
                    # range and the limb bound came with the staging, so the
                    # chunk's stage-1 sums start as soon as it has landed)
                    vals[lo:hi].copy_(hv[lo:hi], non_blocking=True)
                    packed[lo:hi].copy_(c3["packed"][lo:hi], non_blocking=True)
                    lev = torch.cuda.Event()
                    lev.record(copy)
                conv.wait_event(lev)
                with torch.cuda.stream(conv):
                    unpack_compact3(c3, nnz, coords, s_lo, s_hi, packed, aux)
                    cev = torch.cuda.Event()
                    cev.record(conv)
                    nat.call("skx_coo_pack0_range", 3, nnz, lo, hi, nat.ptr(coords), nat.ptr(vals),
                             nat.ptr(rec0), nat.stream())
                conv_ev.append(cev)
                bounds.append((lo, hi))
                s_lo = s_hi
            ev_v = torch.cuda.Event()
            ev_v.record(copy)
            packed.record_stream(copy)
            packed.record_stream(conv)
            coords.record_stream(conv)
            for t in aux:
                t.record_stream(copy)
                t.record_stream(conv)
        else:
            with torch.cuda.stream(copy):
                vals.copy_(hv, non_blocking=True)
                ev_v = torch.cuda.Event()
                ev_v.record(copy)
            soa = st._soa  # coordinates staged as pinned int32 SoA: straight into place
            for lo in range(0, nnz, chunk):
                hi = min(nnz, lo + chunk)
                with torch.cuda.stream(copy):
                    for k in range(nd):
                        coords[k, lo:hi].copy_(soa[k, lo:hi], non_blocking=True)
                    cev = torch.cuda.Event()
                    cev.record(copy)
                conv_ev.append(cev)
                bounds.append((lo, hi))
        if c3 is None:
            main.wait_event(ev_v)
        vals.record_stream(copy)
        coords.record_stream(copy)
        d = DeviceCoo(self.shape, coords, vals)
        if c3 is not None:
            d._vrange = c3["vrange"]  # from the staging pass: no device scan, no sync
            rec0.record_stream(conv)
            aux[0].record_stream(main)
            d._fibre[0] = (aux[0], rec0)  # colptr = slice pointers (int64, s0 + 1)
            d._fibre_meta[0] = (0xFFFFFFFF, None)
        st._device = d
        self._host = None
        if c3 is not None:
            # ||T||^2 on the convert stream behind the last chunk (it has
            # waited for every copy); the main stream joins it below, before
            # the first pass that needs the whole tensor
            with torch.cuda.stream(conv):
                self._attach(d)
        else:
            self._attach(d)
        fx = d.fixed_point_ok()  # staging's value range, or one small D2H once the values are in
        self.normals.prefetch()
        if not fx:
            # the RRF tables of every mode, in the reference's draw order
            tabs_all = []
            for n, scan, (P, k2, width) in zip(modes, scans, dims):
                tabs = finish_rrf_scan(scan, self.rng_init, P)
                gauss = self.rng_init.standard_normal((k2, width)) / np.sqrt(width)
                tabs_all.append((n, tabs, gauss))
            main.wait_stream(conv)
            for ev in conv_ev:
                main.wait_event(ev)
            self.d.fibre(0)
            for n, tabs, gauss in tabs_all:
                self.factors[n] = _rrf_finish(self.d, n, self.ranks[n], tabs, gauss, self.comm)
            return
        emax = d.value_range()[0]
        shp, sp_ = nat.host_i64(self.shape)
        # Each mode's chunk sums are enqueued as soon as its own rejection scan
        # is resolved (tables in the reference's draw order), on a stream of
        # its own: mode 1's run beside scan 2 as the chunks land instead of
        # waiting for it, mode 2's catch up behind scan 2.
        tabs_all, accs, side = [], {}, []
        ev0 = torch.cuda.Event()
        ev0.record(main)  # everything before the chunk sums (not mode 1's chunk loop)
        for i, (n, scan, (P, k2, width)) in enumerate(zip(modes, scans, dims)):
            sn = main if i == 0 else _stage1_stream(i)
            if sn is not main:
                sn.wait_event(ev0)
                for t in (coords, vals):
                    t.record_stream(sn)
                side.append(sn)
            with torch.cuda.stream(sn):
                # the scan's finish and the accumulator on this mode's stream
                tabs = finish_rrf_scan(scan, self.rng_init, P)
                acc = torch.zeros(self.shape[n] * tabs.k2 * 4, dtype=torch.int64, device="cuda")
                flag = torch.empty(1, dtype=torch.int32, device="cuda")
            gauss = self.rng_init.standard_normal((k2, width)) / np.sqrt(width)
            tabs_all.append((n, tabs, gauss))
            accs[n] = (acc, flag)
            if sn is not main:
                for t in (acc, flag, tabs.d):
                    t.record_stream(main)  # converted on the main stream below
            bound = c3["rowmax"].get(n, -1) if c3 is not None else -1
            with torch.cuda.stream(sn):
                for (lo, hi), ev in zip(bounds, conv_ev):
                    sn.wait_event(ev)
                    cptr = ctypes.c_void_p(coords.data_ptr() + lo * 4)
                    vptr = ctypes.c_void_p(vals.data_ptr() + lo * 8)
                    nat.call("skx_rrf_stage1_fx_acc", nd, sp_, n, hi - lo, cptr, nnz, vptr, emax,
                             *tabs.args(), tabs.k2, nat.ptr(acc), nat.ptr(flag), bound, nat.stream())
        # the fitness layout: packed chunk by chunk above (compact staging),
        # else one packing pass on the convert stream behind the last unpack
        with torch.cuda.stream(conv):
            self.d.fibre(0)
        for sn in side:
            main.wait_stream(sn)
        coords.record_stream(main)
        main.wait_stream(conv)  # every chunk unpacked, ||T||^2 done, layout built
        for n, tabs, gauss in tabs_all:
            acc, flag = accs[n]
            st1 = torch.empty((self.shape[n], tabs.k2), dtype=torch.float64, device="cuda")
            nat.call("skx_rrf_stage1_fx_convert", nat.ptr(acc), self.shape[n] * tabs.k2, emax,
                     nat.ptr(flag), nat.ptr(st1), nat.stream())
            self.factors[n] = _rrf_from_stage1(st1, self.ranks[n], gauss, self.comm)

    def _draw_ts(self, n):
        ext = tuple(self.shape[k] for k in self.others(n))
        return TensorSketchOp.build(ext, self.m, self.rng_sketch)

    def _rhs(self, n, op):
        # sparse: mode n's layout carries op's buckets when built for it
        yt = ts_rhs_mode_dev(op, self.d, n) if self.sparse else ts_rhs_dense_dev(op, self.d, n)
        if self.comm is not None:
            # sum the partial sketches and keep this rank's rows (columns of Y_n):
            # every later step on Y_n is column-separable
            yt = self.comm.reduce_scatter_rows(yt)
        return yt

    def draw_ts_ops(self):
        """All modes' operators, in the reference's draw order (mode 0..N-1)."""
        if self.use_ts and self.ts_ops[0] is None:
            for n in range(self.ndim):
                self.ts_ops[n] = self._draw_ts(n)

    def build_ts(self, n):
        """Redraw mode n's operator and its right-hand side (src/tucker.py:264-267)."""
        op = self._draw_ts(n)
        self.ts_ops[n], self.ts_rhs[n] = op, self._rhs(n, op)

    def prep(self):
        if self.use_ts:
            self.draw_ts_ops()
            for n in range(self.ndim):
                self.ts_rhs[n] = self._rhs(n, self.ts_ops[n])

    def solve_mode(self, n, redraw, defer=None):
        others = [self.factors[k] for k in self.others(n)]
        if self.use_ts:
            if redraw:
                self.build_ts(n)
            pre = None
            if defer is not None and self.comm is None:
                pre = self._early_yg(n)
            z = ts_kron_dev(self.ts_ops[n], others)
            if self.comm is not None:  # this rank holds Y_n^T rows row_slab(s_n)
                s_n = self.shape[n]
                lo, _ = self.comm.row_slab(s_n)
                core_t, a_loc, _, res = rsvd_lrls_rows_dev(z, self.ts_rhs[n], lo, s_n,
                                                           self.ranks[n], self.normals, self.comm,
                                                           defer=defer)
                return core_t, self.comm.allgather_rows(a_loc.contiguous(), s_n), res
            y = self.ts_rhs[n].t()
            return self._finish_dense(z, y, n, defer, pre)
        else:
            det = self.cfg.sketch == "leverage-deterministic"
            if defer is not None:  # rank check of the factors deferred with the rest
                idx, w, _, lbad = (lev_det_dev(others, self.m, check=False) if det else
                                   lev_sample_dev(others, self.m, self.rng_sketch, check=False))
                defer.append(lbad)
            else:
                idx, w, _, _ = (lev_det_dev(others, self.m) if det else
                                lev_sample_dev(others, self.m, self.rng_sketch))
            z = kron_rows_dev(others, idx, w)
            r_other = int(np.prod([self.ranks[k] for k in self.others(n)]))
            if (self.sparse and defer is not None
                    and min(self.ranks[n] + 10, self.shape[n]) < r_other
                    and ((self.comm is not None and self.comm.world > 1 and not FIXED_HITS_OFF)
                         or FORCE_FIXED_HITS)):
                return self._solve_hits_fixed(n, z, idx, w, defer)
            if self.sparse:
                if self.ndim == 3 and n >= 1:
                    # the sampled fibres lie in slices of the mode-0 layout
                    off, col, val = gather_slices_dev(self.d, n, idx, w)
                else:
                    keys, vals = filter_fibers_dev(self.d, n, idx)
                    ext = [self.shape[k] for k in self.others(n)]
                    off, col, val = gather_coo_dev(keys, vals, ext, self.shape[n], idx, w)
                row = None
                total = col.numel()
                if self.comm is not None:
                    # every rank gathered the sampled fibres from its own shard:
                    # the hits are disjoint, so their union is the full sample
                    row, col, val = self._gather_hits(off, col, val)
                    total = col.numel()
                if total < HITS_DENSITY * self.m * self.shape[n]:
                    # mostly-empty sampled fibres: work on the hit columns only
                    core_t, a, _, res = rsvd_lrls_hits_dev(z, off, col, val, self.shape[n],
                                                           self.ranks[n], self.normals,
                                                           hit_row=row, defer=defer)
                    return core_t, a, res
                if row is None:
                    y = hits_to_dense(off, col, val, self.m, self.shape[n])
                else:
                    torch = _torch()
                    y = torch.zeros((self.m, self.shape[n]), dtype=torch.float64, device="cuda")
                    y[row, col] = val
                    return self._finish_dense(z, y, n, defer)
            else:
                y = gather_dense_dev(self.d, n, idx, w)
            if self.comm is not None:
                self.comm.allreduce(y)
        return self._finish_dense(z, y, n, defer)

    def _solve_hits_fixed(self, n, z, idx, w, defer):
        """Speculative sparse leverage sub-problem with no host round trip:
        fixed-capacity hit lists (the overflow flag joins the sweep's deferred
        flags; a flagged sweep is replayed on the checked path).  Multi-rank:
        every rank gathers from its own shard, the fixed-size lists are
        all-gathered (rank order) and regrouped by sample row on the device,
        the overflow flags all-reduced -- no host synchronisation either."""
        torch = _torch()
        if self.ndim == 3 and n >= 1:
            off, col, val, over = gather_slices_fixed_dev(self.d, n, idx, w)
        else:
            off, col, val, over = filter_gather_fixed_dev(self.d, n, idx, w)
        s_n = self.shape[n]
        if self.comm is not None and self.comm.world > 1:
            cap = int(col.numel())
            k = torch.arange(cap, device="cuda")
            row = (torch.searchsorted(off, k, right=True) - 1).clamp(0, self.m - 1)
            rows = self.comm.allgather(row)
            cols = self.comm.allgather(col)
            vals = self.comm.allgather(val)
            # regroup by sample row (stable: rank order inside a row)
            order = torch.sort(rows, stable=True)[1]
            rows, col, val = rows[order], cols[order].contiguous(), vals[order].contiguous()
            cnt = torch.zeros(self.m, dtype=torch.int64, device="cuda")
            cnt.scatter_add_(0, rows, (col < s_n).to(torch.int64))
            off = torch.zeros(self.m + 1, dtype=torch.int64, device="cuda")
            off[1:] = torch.cumsum(cnt, 0)
            # the offsets count real hits only: padding (sentinel column, value
            # 0) goes behind them, the real hits keep their row grouping
            real = col < s_n
            order = torch.sort((~real).to(torch.int64), stable=True)[1]
            col, val = col[order].contiguous(), val[order].contiguous()
            over = self.comm.allreduce(over.to(torch.float64).view(1))[0] > 0
        defer.append(over)
        core_t, a, _, res = rsvd_lrls_hits_fixed_dev(z, off, col, val, s_n, self.ranks[n],
                                                     self.normals, defer=defer)
        return core_t, a, res

    def _finish_dense(self, z, y, n, defer=None, pre=None):
        core_t, a, _ = rsvd_lrls_dev(z, y, self.ranks[n], self.normals, defer=defer, pre=pre)
        rs = self.res_stream
        if rs is None or y.numel() < RESID_SIDE_MIN:
            return core_t, a, resid_dev(z, core_t, a, y)
        # the residual ||Z core_t a^T - Y|| (a full pass over Y) only feeds the
        # trace (src/tucker.py:274-275, 293): it runs on a low-priority side
        # stream beside the next sub-problem instead of ahead of it -- same
        # kernels, same bits
        torch = _torch()
        rs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(rs):
            res = resid_dev(z, core_t, a, y)
        for t in (z, core_t, a, y):
            t.record_stream(rs)
        return core_t, a, res

    def _early_yg(self, n):
        """Speculative sweeps: draw this sub-problem's Gaussian test matrix now
        and start Y G (a bandwidth-bound pass over Y_n) on the idle init side
        stream, so it overlaps the Kronecker sketch and the Cholesky QR of Z
        (latency-bound single-CTA kernels) on the sweep stream."""
        torch = _torch()
        s_n = self.shape[n]
        width = min(self.ranks[n] + 10, s_n)
        r = int(np.prod([self.ranks[k] for k in self.others(n)]))
        if width >= r:
            return None
        g = self.normals.normal((s_n, width))
        side = _yg_stream()
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            yg = y_times_dev(self.ts_rhs[n].t(), g)
            ev = torch.cuda.Event()
            ev.record(side)
        g.record_stream(side)
        return g, yg, ev

    def _gather_hits(self, off, col, val):
        """All ranks' sampled-fibre hits as (row, col, val) triples."""
        torch = _torch()
        counts = off[1:] - off[:-1]
        row = torch.repeat_interleave(torch.arange(self.m, device="cuda"), counts)
        n_loc = torch.tensor([col.numel()], dtype=torch.int64, device="cuda")
        n_all = self.comm.allgather(n_loc)
        cap = int(n_all.max().item())
        def pad(t):
            out = t.new_zeros(max(cap, 1))
            out[:t.numel()] = t
            return out
        rows = self.comm.allgather(pad(row))
        cols = self.comm.allgather(pad(col))
        vals = self.comm.allgather(pad(val))
        keep = torch.cat([torch.arange(max(cap, 1), device="cuda") < k for k in n_all.tolist()])
        return rows[keep], cols[keep], vals[keep]

    def fold_core(self, core_t):
        ranks = self.ranks
        nd = self.ndim
        return core_t.t().reshape([ranks[nd - 1]] + list(ranks[:nd - 1])).movedim(0, nd - 1).contiguous()

    def sweeps(self, trace):
        torch = _torch()
        core = None
        res_dev, fit_dev, ev = [], [], []
        # overlap the per-sweep fitness with the next sweep unless an early stop
        # needs its value first (or collectives would interleave across streams):
        # the sub-problems run on the high-priority stream, the fitness on a
        # low-priority one, so the block scheduler serves the solves first
        overlap = self.cfg.convergence_tol <= 0 and self.sparse
        fit_comm = self.comm.sibling() if (self.comm is not None and overlap) else self.comm
        fs = _fit_stream() if overlap else None
        caller = torch.cuda.current_stream()
        hi = _init_streams()[1] if overlap else caller
        hi.wait_stream(caller)
        if self.comm is None and os.environ.get("SKX_RESID_INLINE") is None:
            self.res_stream = _res_stream()
        with torch.cuda.stream(hi):
            core = self._sweep_loop(trace, res_dev, fit_dev, ev, fs, overlap, fit_comm)
        caller.wait_stream(hi)
        rs = self.res_stream

        def finish():
            """Join the fitness / residual streams and move the trace to the host."""
            if fs is not None:
                caller.wait_stream(fs)
            if rs is not None:
                caller.wait_stream(rs)
            torch.cuda.synchronize()
            trace.residuals.extend(torch.stack(res_dev).cpu().tolist() if res_dev else [])
            trace.fitness.extend(torch.stack(fit_dev).cpu().tolist() if fit_dev else [])
            trace.wall_s.extend(a.elapsed_time(b) / 1e3 for a, b in ev)
            return trace

        # the caller's stream has the model once the sweep stream is joined;
        # the last fitness pass may still be running on its own stream
        return core, finish

    def _sweep_loop(self, trace, res_dev, fit_dev, ev, fs, overlap, fit_comm=None):
        torch = _torch()
        core = None
        # TensorSketch sweeps run speculatively: every sub-problem takes the
        # one-pass Cholesky QR without a host round trip and records a device
        # flag.  A sweep's flags are copied to the host asynchronously and
        # checked once the next sweep has been enqueued (pipelined when no
        # early stop needs the fitness), so the GPU does not wait for the host
        # at sweep boundaries.  A flagged sweep is replayed from its starting
        # state on the checked path (second QR pass / Householder /
        # rank-deficiency redraw) and everything enqueued after it is
        # discarded, so the results are those of the checked path either way.
        # multi-rank too: every flag is a function of replicated data (Z, the
        # factors), so all ranks take the same replay decisions
        speculate = True
        pipeline = speculate and self.cfg.convergence_tol <= 0
        nsw = self.cfg.max_sweeps
        pending = None  # (sweep, start state, host flag, event) awaiting its check
        checked = set()  # sweeps to re-run on the checked path
        k = 0
        while True:
            if k >= nsw:
                if pending is not None and self._flagged(pending):
                    k = self._rollback(pending, res_dev, fit_dev, ev)
                    checked.add(k)
                    pending = None
                    continue
                break
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            start = (k, list(self.factors), self.normals.snapshot(), len(res_dev), len(fit_dev),
                     len(ev), self.rng_sketch.bit_generator.state)
            spec = speculate and k not in checked
            core_t = None
            if spec:
                flags = []
                for n in range(self.ndim):
                    core_t, a, res = self.solve_mode(n, redraw=False, defer=flags)
                    self.factors[n] = a
                    res_dev.append(res)
                    if n == 0 and overlap and k + 1 < nsw:
                        # the next sweep's Gaussian test matrices, on the
                        # low-priority stream (enqueued once the GPU has work)
                        self.normals.prefetch_async(fs)
                hf = torch.empty(1, dtype=torch.int32, pin_memory=True)
                hf.copy_(torch.stack(flags).any().to(torch.int32).view(1), non_blocking=True)
                fev = torch.cuda.Event()
                fev.record()
            else:
                if overlap and k + 1 < nsw:
                    self.normals.prefetch_async(fs)
                for n in range(self.ndim):
                    try:
                        core_t, a, res = self.solve_mode(n, redraw=False)
                    except RankDeficientError:
                        try:
                            core_t, a, res = self.solve_mode(n, redraw=True)
                        except RankDeficientError as exc:
                            raise RankDeficientError(
                                f"mode-{n} sketched system rank-deficient after redraw "
                                f"(m={self.m}, sketch={self.cfg.sketch}): {exc}") from exc
                    self.factors[n] = a
                    res_dev.append(res)
            core = self.fold_core(core_t)
            e1.record()
            ev.append((e0, e1))
            if overlap:
                # the fitness of this sweep (a pass over the nonzeros) runs on a
                # low-priority stream while the next sweep's sub-problems --
                # mostly single-CTA and latency-bound -- proceed; they only read
                # factors that are replaced (not overwritten) by later solves
                fs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(fs):
                    if (self.ttmc_last and k == nsw - 1 and fit_comm is None
                            and ttmc3_r20_eligible(self.d, self.factors)):
                        # Algorithm 6's last Tucker fitness: the full TTMc P
                        # (one pass, as fast as the cross-term kernel) also
                        # gives the final CP fitness's cross term (cp.py)
                        P = ttmc3_full_dev(self.d, self.factors)
                        f = fitness_from_cross_dev(self.norm2, (P * core).sum(), (core * core).sum())
                        pev = torch.cuda.Event()
                        pev.record(fs)
                        self.last_ttmc = (P, list(self.factors), pev)
                    else:
                        f = fitness_tucker_dev(self.d, core, self.factors, self.norm2, fit_comm)
                for t in [core] + list(self.factors):
                    t.record_stream(fs)
            else:
                f = fitness_tucker_dev(self.d, core, self.factors, self.norm2, self.comm)
            fit_dev.append(f)
            if pending is not None:  # the previous speculative sweep, now that this one is queued
                if self._flagged(pending):
                    k = self._rollback(pending, res_dev, fit_dev, ev)
                    checked.add(k)
                    pending = None
                    continue
                pending = None
            if spec:
                pending = (start, hf, fev)
                if not pipeline:
                    if self._flagged(pending):
                        k = self._rollback(pending, res_dev, fit_dev, ev)
                        checked.add(k)
                        pending = None
                        continue
                    pending = None
            # Gaussian segments before this sweep's start are no longer needed
            self.normals.commit(start[2] if pending is not None else None)
            if (self.cfg.convergence_tol > 0 and len(fit_dev) > 1
                    and abs(float(fit_dev[-1].item()) - float(fit_dev[-2].item()))
                    < self.cfg.convergence_tol):
                break
            k += 1
        return core

    @staticmethod
    def _flagged(pending):
        _, hf, fev = pending
        fev.synchronize()
        return int(hf[0]) != 0

    def _rollback(self, pending, res_dev, fit_dev, ev):
        """Return the run to the start of a flagged speculative sweep (factors,
        Gaussian-segment position, trace lists); returns that sweep's index."""
        (k, factors, normals, n_res, n_fit, n_ev, rs), _, _ = pending
        self.factors = list(factors)
        self.normals.restore(normals)
        self.rng_sketch.bit_generator.state = rs
        del res_dev[n_res:]
        del fit_dev[n_fit:]
        del ev[n_ev:]
        return k


def sketched_tucker_run_dev(t, config, comm=None, ttmc_last=False):
    """Device-resident run whose trace is completed later: returns (core,
    factors, finish); finish() joins the per-sweep fitness stream and returns
    the SweepTrace.  The model is ready on the caller's stream before the last
    fitness pass ends, so a caller (Algorithm 6's core stage) can overlap it.
    ttmc_last: the last sweep's fitness pass computes the full TTMc P of the
    final factors; finish.last_ttmc() returns (P, factors, event) or None."""
    run = _Run(t, config, comm)
    run.ttmc_last = ttmc_last
    run.initialise_and_prep()
    if run.sparse:
        # modes >= 1 layouts served the RRF stage 1 and the TS right-hand sides;
        # the sweeps only read mode 0's (fitness): free the rest (16 B/nnz each)
        for n in range(1, run.ndim):
            run.d.drop_fibre(n)
    trace = SweepTrace()
    core, finish = run.sweeps(trace)
    finish.last_ttmc = lambda: run.last_ttmc
    return core, list(run.factors), finish


def sketched_tucker_als_dev(t, config, comm=None):
    """Device-resident form: returns (core, factors) as CUDA tensors + trace."""
    core, factors, finish = sketched_tucker_run_dev(t, config, comm)
    return core, factors, finish()


def sketched_tucker_als(t, config):
    """Sketched rank-constrained Tucker-ALS (src/tucker.py:216-300)."""
    core, factors, trace = sketched_tucker_als_dev(t, config)
    host = to_host([core] + list(factors))
    return TuckerModel(host[0], host[1:]), trace


def _sparse_gram_dev(d, n, max_side=1 << 15):
    """T_(n) T_(n)^T (s_n x s_n, dense) of a DeviceCoo, deterministically: the
    products of every pair of nonzeros in the same mode-n fibre, sorted by
    their Gram cell and summed per cell in that order."""
    torch = _torch()
    s_n = d.shape[n]
    if s_n > max_side:
        raise ValueError(f"hosvd_init: mode-{n} Gram of a sparse tensor needs s_n <= {max_side} "
                         f"(got {s_n}); the reference forms it densely as well")
    keys, vals = d.keys(n)  # flat_other * s_n + i_n, ascending
    g = torch.zeros(s_n * s_n, dtype=torch.float64, device="cuda")
    if vals.numel() == 0:
        return g.view(s_n, s_n)
    fib = keys // s_n
    row = keys % s_n
    _, counts = torch.unique_consecutive(fib, return_counts=True)
    starts = torch.cumsum(counts, 0) - counts
    # every (e, e') pair inside a fibre: e repeated len(fibre) times
    reps = torch.repeat_interleave(counts, counts)
    e = torch.repeat_interleave(torch.arange(vals.numel(), device="cuda"), reps)
    first = torch.repeat_interleave(torch.repeat_interleave(starts, counts), reps)
    offs = torch.arange(e.numel(), device="cuda") - torch.repeat_interleave(
        torch.cumsum(reps, 0) - reps, reps)
    e2 = first + offs
    cell = row[e] * s_n + row[e2]
    prod = vals[e] * vals[e2]
    cell, order = torch.sort(cell, stable=True)
    cells, cnt = torch.unique_consecutive(cell, return_counts=True)
    g[cells] = torch.segment_reduce(prod[order], "sum", lengths=cnt, axis=0)
    return g.view(s_n, s_n)


def hosvd_init_dev(t, ranks):
    """Leading eigenvectors of the mode Grams (src/tucker.py:112-126), device."""
    torch = _torch()
    out = []
    for n, rank in enumerate(ranks):
        if is_sparse_dev(t):
            gram = _sparse_gram_dev(t, n)
        else:
            tn = t.movedim(n, 0).reshape(t.shape[n], -1)
            gram = tn @ tn.t()
        _, vecs = torch.linalg.eigh(gram)
        out.append(vecs.flip(1)[:, :rank].contiguous())
    return out


def hosvd_init(t, ranks, rng=None):
    """Leading left singular vectors of every unfolding via the mode Grams
    (src/tucker.py:112-126); rng is accepted for interface parity."""
    d = device_of(t)
    return [a.cpu().numpy() for a in hosvd_init_dev(d, ranks)]


def hooi_dev(t, config):
    """Exact Tucker-ALS (src/tucker.py:155-193) on device: per mode the
    leading left singular vectors of the skip-mode TTMc unfolding (libskx
    kernel for sparse order 3), residual from the captured energy, core from
    the last mode's contraction.  Returns (core, factors, trace)."""
    import time
    torch = _torch()
    if config.sketch is not None:
        raise ValueError("hooi is the unsketched driver; got a sketch config")
    shape = tuple(int(s) for s in t.shape)
    ndim = len(shape)
    ranks = config.ranks
    _validate_ranks(shape, ranks)
    rng = rngmod.make_rng(config.seed)
    init = config.init or "hosvd"
    d = device_of(t)
    if init == "hosvd":
        factors = hosvd_init_dev(d, ranks)
    elif init == "random":
        factors = [random_orthonormal_dev(shape[n], ranks[n], rng) for n in range(ndim)]
    else:
        raise ValueError(f"unknown init {init!r} for hooi")
    n2 = d.norm2()[0] if is_sparse_dev(d) else (d * d).sum()
    norm_t = math.sqrt(float(n2.item()))
    norm_t_sq = norm_t ** 2
    trace = SweepTrace()
    core = None
    for _ in range(config.max_sweeps):
        tic = time.perf_counter()
        y = None
        captured = []
        for n in range(ndim):
            y = ttmc_dev(d, factors, skip=n)
            yn = y.movedim(n, 0).reshape(shape[n], -1)
            u, sv, _ = top_svd_dev(yn, ranks[n])
            factors[n] = u[:, :ranks[n]].contiguous()
            captured.append((sv[:ranks[n]] ** 2).sum())
        core = ttm_dev(y, factors[ndim - 1].t(), ndim - 1).contiguous()
        cap = torch.stack(captured + [(core * core).sum()]).cpu().tolist()
        for c in cap[:-1]:
            trace.residuals.append(math.sqrt(max(norm_t_sq - c, 0.0)))
        fit = 1.0 - math.sqrt(max(norm_t_sq - cap[-1], 0.0)) / norm_t
        trace.wall_s.append(time.perf_counter() - tic)
        trace.fitness.append(float(fit))
        if (len(trace.fitness) > 1
                and abs(trace.fitness[-1] - trace.fitness[-2]) < config.convergence_tol):
            break
    return core, factors, trace


def hooi(t, config):
    """Exact Tucker-ALS (src/tucker.py:155-193)."""
    core, factors, trace = hooi_dev(t, config)
    host = to_host([core] + list(factors))
    return TuckerModel(host[0], host[1:]), trace


# ------------------------------------------------------------------ ref-ts
def _vec_sketch_dev(op, d):
    """TensorSketch of vec(T) over every mode (src/tucker.py:205-213 +
    ts_apply_rhs): the mode-0 right-hand side of T viewed as a
    (1, s_1, ..., s_N) tensor; returns an (m,) device vector."""
    torch = _torch()
    if is_sparse_dev(d):
        c = torch.cat([torch.zeros((1, d.nnz), dtype=torch.int32, device="cuda"), d.coords])
        d1 = DeviceCoo((1,) + d.shape, c.contiguous(), d.vals)
        return ts_rhs_mode_dev(op, d1, 0)[0]
    return ts_rhs_dense_dev(op, d.reshape((1,) + tuple(d.shape)).contiguous(), 0)[0]


def _lstsq_dev(z, b):
    """Least squares min ||z x - b|| with numpy lstsq(rcond=None) semantics
    (src/tucker.py:345, 353): the minimum-norm SVD solve for narrow systems,
    QR with R^-1 for the full-rank core system."""
    torch = _torch()
    from .cp import _lstsq_min_norm_dev
    if z.shape[1] <= 64:
        return _lstsq_min_norm_dev(z, b)
    q, r = torch.linalg.qr(z, mode="reduced")
    return torch.linalg.solve_triangular(r, q.transpose(0, 1) @ b, upper=True)


def ref_tucker_ts_dev(t, config):
    """The reference's one-variable-at-a-time TensorSketch baseline
    (src/tucker.py:303-364) on the device: RRF (or random) init of every
    mode from the first of two seed streams; per mode a TensorSketch operator
    and right-hand side, plus one over all modes for the core, drawn once;
    each sweep solves N unconstrained sketched factor problems (core fixed;
    factors re-orthonormalised by QR) and one core problem (factors fixed).
    Returns (core, factors, trace)."""
    import time
    torch = _torch()
    if config.sketch != "tensorsketch":
        raise ValueError("the reference baseline is TensorSketch-based")
    _validate_ranks(tuple(int(s) for s in t.shape), config.ranks)
    d = device_of(t)
    shape = shape_of(d)
    ndim = len(shape)
    ranks = config.ranks
    _validate_ranks(shape, ranks)
    m = config.resolved_sketch_size()
    _check_sketch_size(m, ranks)
    rng_init, rng_sketch = rngmod.split_rng(config.seed, 2)
    init = config.init or "rrf"
    factors = []
    for n in range(ndim):
        if init == "rrf":
            factors.append(init_rrf_dev(d, n, ranks[n], config.resolved_rrf_width(ranks[n]),
                                        rng_init))
        elif init == "random":
            factors.append(random_orthonormal_dev(shape[n], ranks[n], rng_init))
        else:
            raise ValueError(f"unknown init {init!r} for ref_tucker_ts")
    ops, rhs = [], []
    for n in range(ndim):
        op = TensorSketchOp.build(tuple(shape[k] for k in range(ndim) if k != n), m, rng_sketch)
        ops.append(op)
        rhs.append((ts_rhs_mode_dev(op, d, n) if is_sparse_dev(d) else
                    ts_rhs_dense_dev(op, d, n)).t())  # Y_n, m x s_n
    core_op = TensorSketchOp.build(shape, m, rng_sketch)
    core_rhs = _vec_sketch_dev(core_op, d).view(m, 1)
    norm2 = d.norm2()[0] if is_sparse_dev(d) else (d * d).sum()

    def update_core():
        z = ts_kron_dev(core_op, factors)
        sol = _lstsq_dev(z, core_rhs)
        return sol.reshape(ranks), torch.linalg.vector_norm(z @ sol - core_rhs)

    core, _ = update_core()
    trace = SweepTrace()
    for _ in range(config.max_sweeps):
        tic = time.perf_counter()
        res = []
        for n in range(ndim):
            others = [factors[k] for k in range(ndim) if k != n]
            cn = core.movedim(n, 0).reshape(ranks[n], -1)  # matricize(core, n)
            z = ts_kron_dev(ops[n], others) @ cn.t()
            sol = _lstsq_dev(z, rhs[n])
            res.append(torch.linalg.vector_norm(z @ sol - rhs[n]))
            q, _ = qr_lapack_dev(sol.t())  # numpy's signs: the core stays fixed
            factors[n] = q[:, :ranks[n]].contiguous()
        core, core_res = update_core()
        res.append(core_res)
        fit = fitness_tucker_dev(d, core.contiguous(), factors, norm2)
        vals = torch.stack(res + [fit]).cpu().tolist()
        trace.residuals.extend(vals[:-1])
        trace.wall_s.append(time.perf_counter() - tic)
        trace.fitness.append(float(vals[-1]))
        if (len(trace.fitness) > 1
                and abs(trace.fitness[-1] - trace.fitness[-2]) < config.convergence_tol):
            break
    return core, factors, trace


def ref_tucker_ts(t, config):
    """Reference sketched baseline, one variable per sub-problem
    (src/tucker.py:303-364)."""
    core, factors, trace = ref_tucker_ts_dev(t, config)
    host = to_host([core] + list(factors))
    return TuckerModel(host[0], host[1:]), trace
