"""CP via sketched Tucker compression (drop-in for the path of src/cp.py).

``cp_via_sketched_tucker`` = Algorithm 6: sketched Tucker-ALS (leverage
sampling) to compress, exact CP-ALS on the small core (hosvd-of-core init),
then the factor chains multiplied back and renormalised, with the final
fitness measured against the full tensor (src/cp.py:177-224).  ``cp_als`` is
the exact normal-equations CP-ALS (src/cp.py:119-174) on a dense or sparse
tensor held on the GPU (also used on the core).  ``sketched_cp_als`` is leverage-sampled
CP-ALS on the full tensor (src/cp.py:110-116).

Extension: ``CPConfig.tucker_rank`` (default None = the reference's tie of the
Tucker ranks to the CP rank) lets config 5 of BASELINE.json request Tucker
rank 20 with CP rank 10.
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, replace

import numpy as np

from . import rng as rngmod
from .tensors import (CPModel, device_of, fitness_cp_dev, is_sparse_dev, mttkrp_dev, shape_of,
                      to_host)
from .tucker import (SweepTrace, TuckerConfig, hooi_dev, hosvd_init_dev,
                     sketched_tucker_run_dev)


def _torch():
    import torch
    return torch


@dataclass
class CPConfig:
    rank: int
    max_sweeps: int | None = None
    sketch: str | None = None
    sketch_size: int | None = None
    sketch_factor: float | None = None
    init: str | None = None
    seed: int = 0
    tucker_sweeps: int = 5
    tucker_rank: int | None = None

    def __post_init__(self):
        if self.sketch not in (None, "leverage-random"):
            raise ValueError(f"unknown sketch kind {self.sketch!r} for CP")

    def resolved_sweeps(self, on_core=False):
        if self.max_sweeps is not None:
            return self.max_sweeps
        return 25 if on_core else 30

    def resolved_sketch_size(self):
        if self.sketch_size is not None:
            return int(self.sketch_size)
        if self.sketch_factor is not None:
            return int(math.ceil(self.sketch_factor * self.rank ** 2))
        raise ValueError("sketched CP needs sketch_size or sketch_factor")


def _normalize_columns_dev(a):
    torch = _torch()
    nrm = torch.linalg.vector_norm(a, dim=0)
    safe = torch.where(nrm > 0, nrm, torch.ones_like(nrm))
    return a / safe, nrm


def _core_kernel_ok(t, rank, init):
    """K8 (libskx skx_cp_core_als) covers the on-core stage of Algorithm 6:
    a dense order-3 core, hosvd-of-core init, rank <= every extent <= 32."""
    from . import _native as nat
    if is_sparse_dev(t) or t.dim() != 3 or init != "hosvd-of-core":
        return False
    shape = tuple(int(x) for x in t.shape)
    if not all(rank <= x <= 32 for x in shape):
        return False
    dims, dp = nat.host_i64(shape)
    return int(nat.load().skx_cp_core_smem_bytes(dp, rank)) <= 227 * 1024


def cp_core_als_dev(core, config):
    """CP-ALS on a small dense order-3 core in one libskx CTA (K8): the whole
    on-core stage of src/cp.py:119-174 (hosvd-of-core init, sweeps of
    Gram-Hadamard / core MTTKRP / pinv / normalisation, residuals and the
    fitness per sweep).  One launch and one small D2H for the trace."""
    from . import _native as nat
    torch = _torch()
    shape = tuple(int(x) for x in core.shape)
    rank = config.rank
    sweeps = config.resolved_sweeps(True)
    fac = torch.empty(sum(shape) * rank, dtype=torch.float64, device="cuda")
    w = torch.empty(rank, dtype=torch.float64, device="cuda")
    res = torch.empty(max(3 * sweeps, 1), dtype=torch.float64, device="cuda")
    fit = torch.empty(max(sweeps, 1), dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    dims, dp = nat.host_i64(shape)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    nat.call("skx_cp_core_als", dp, rank, sweeps, nat.ptr(core.contiguous()), nat.ptr(fac),
             nat.ptr(w), nat.ptr(res), nat.ptr(fit), nat.ptr(info), nat.stream())
    e1.record()
    host = torch.cat([info.to(torch.float64), res[:3 * sweeps], fit[:sweeps]]).cpu().tolist()
    if int(host[0]) != 0:
        raise ValueError("CP decomposition of a zero-norm tensor is undefined")
    factors, off = [], 0
    for x in shape:
        factors.append(fac[off:off + x * rank].view(x, rank))
        off += x * rank
    total = e0.elapsed_time(e1) / 1e3
    trace = SweepTrace(fitness=host[1 + 3 * sweeps:], residuals=host[1:1 + 3 * sweeps],
                       wall_s=[total / max(sweeps, 1)] * sweeps)
    return factors, w, trace


def cp_als_dev(t, config, on_core=False):
    """Exact CP-ALS (src/cp.py:119-174, unsketched) on a dense CUDA tensor or a
    DeviceCoo.  On a small dense order-3 core with hosvd-of-core init the
    whole stage is the one-CTA libskx kernel K8 (cp_core_als_dev)."""
    torch = _torch()
    shape = tuple(t.shape)
    ndim = len(shape)
    rank = config.rank
    if rank < 1:
        raise ValueError("rank must be positive")
    if _core_kernel_ok(t, rank, config.init or ("hosvd-of-core" if on_core else "rrf")):
        return cp_core_als_dev(t, config)
    norm_t2 = t.norm2()[0] if is_sparse_dev(t) else (t * t).sum()
    nt2 = float(norm_t2.item())
    if nt2 == 0.0:
        raise ValueError("CP decomposition of a zero-norm tensor is undefined")
    rng_init, _ = rngmod.split_rng(config.seed, 2)
    init = config.init or ("hosvd-of-core" if on_core else "rrf")
    factors = _init_factors_dev(t, config, init, rng_init)
    weights = torch.ones(rank, dtype=torch.float64, device="cuda")
    grams = [a.t() @ a for a in factors]
    res_dev, fit_dev, walls = [], [], []
    for _ in range(config.resolved_sweeps(on_core)):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for n in range(ndim):
            go = torch.ones((rank, rank), dtype=torch.float64, device="cuda")
            for k in range(ndim):
                if k != n:
                    go = go * grams[k]
            mm = mttkrp_dev(t, factors, n)
            sc = mm @ torch.linalg.pinv(go, rtol=1e-12)
            cross = (sc * mm).sum()
            mod = ((sc.t() @ sc) * go).sum()
            res_dev.append(torch.sqrt(torch.clamp(norm_t2 - 2.0 * cross + mod, min=0.0)))
            factors[n], weights = _normalize_columns_dev(sc)
            grams[n] = factors[n].t() @ factors[n]
        fit_dev.append(fitness_cp_dev(t, factors, weights, norm_t2))
        e1.record()
        walls.append((e0, e1))
    torch.cuda.synchronize()
    trace = SweepTrace(fitness=torch.stack(fit_dev).cpu().tolist(),
                       residuals=torch.stack(res_dev).cpu().tolist(),
                       wall_s=[a.elapsed_time(b) / 1e3 for a, b in walls])
    return factors, weights, trace


def _init_factors_dev(t, config, init, rng_init):
    """src/cp.py:72-87 on device (t dense CUDA tensor or DeviceCoo)."""
    torch = _torch()
    shape = shape_of(t)
    ndim = len(shape)
    rank = config.rank
    if init == "hosvd-of-core":
        factors = hosvd_init_dev(t, [min(rank, s) for s in shape])
    elif init == "random":
        factors = [torch.from_numpy(rng_init.uniform(size=(shape[n], rank))).cuda() for n in range(ndim)]
    elif init == "rrf":
        # src/cp.py:72-87 with the rrf width of src/cp.py:559-564
        from .tucker import init_rrf_dev
        width = None
        if config.sketch_factor is not None:
            width = max(rank, int(math.ceil(math.sqrt(config.sketch_factor) * rank)))
        elif config.sketch_size is not None:
            width = max(rank, int(math.ceil(math.sqrt(config.sketch_size / rank ** 2) * rank)))
        width = width or max(rank + 8, 2 * rank)
        factors = []
        for n in range(ndim):
            if shape[n] > rank:
                factors.append(init_rrf_dev(t, n, rank, min(width, shape[n]), rng_init))
            else:
                g = torch.from_numpy(rng_init.standard_normal((shape[n], rank))).cuda()
                factors.append(torch.linalg.qr(g, mode="reduced")[0].contiguous())
    else:
        raise ValueError(f"unknown init {init!r} for CP")
    return factors


def cp_als(t, config, on_core=False):
    """Exact CP-ALS (src/cp.py:102-107) on the GPU (dense or sparse input)."""
    if config.sketch is not None:
        raise ValueError("cp_als is the unsketched driver; got a sketch config")
    d = device_of(t)
    factors, weights, trace = cp_als_dev(d, config, on_core=on_core)
    host = to_host(list(factors) + [weights])
    return CPModel(host[:-1], host[-1]), trace


def _lstsq_min_norm_dev(z, y):
    """Minimum-norm least squares min ||z x - y|| as np.linalg.lstsq(z, y,
    rcond=None) (LAPACK gelsd: singular values below eps * max(m, R) * s_max
    are treated as zero), so a rank-deficient sampled system (repeated
    leverage rows) stays finite as in the reference.  z (m x R) = Q R by
    TSQR, R = U_r diag(s) V^T by one-sided Jacobi (R <= 64), U = z V / s;
    x = V diag(1/s) U^T y over the kept singular values.  No host sync."""
    from .linalg import jacobi_svd_dev, tsqr_r_dev
    torch = _torch()
    m, r = z.shape
    if r <= 64 and m >= r:
        rf = tsqr_r_dev(z.contiguous())
        _, sv, v = jacobi_svd_dev(rf)
    else:
        _, sv, vh = torch.linalg.svd(z, full_matrices=False)
        v = vh.transpose(0, 1)
    tol = np.finfo(np.float64).eps * max(m, r) * sv[0]
    inv = torch.where(sv > tol, 1.0 / torch.where(sv > 0, sv, torch.ones_like(sv)),
                      torch.zeros_like(sv))
    u = (z @ v) * inv
    return v @ (inv[:, None] * (u.transpose(0, 1) @ y))


def sketched_cp_als_dev(d, config):
    """Leverage-sampled CP-ALS on the full tensor (src/cp.py:110-174, sketched
    branch) on device: per mode a random leverage sample of the Khatri-Rao
    rows (bit-exact index sets, libskx K3), weighted Hadamard rows and the
    sampled fibres (dense gather or one-pass sparse filter), least squares by
    QR, column normalisation; fitness each sweep, residual (1 - fit) ||T||."""
    from .sketching import (filter_fibers_dev, gather_coo_dev, gather_dense_dev, hits_to_dense,
                            lev_sample_dev)
    torch = _torch()
    shape = shape_of(d)
    ndim = len(shape)
    rank = config.rank
    if rank < 1:
        raise ValueError("rank must be positive")
    sparse = is_sparse_dev(d)
    norm_t2 = d.norm2()[0] if sparse else (d * d).sum()
    nt = math.sqrt(float(norm_t2.item()))
    if nt == 0.0:
        raise ValueError("CP decomposition of a zero-norm tensor is undefined")
    rng_init, rng_sketch = rngmod.split_rng(config.seed, 2)
    factors = _init_factors_dev(d, config, config.init or "rrf", rng_init)
    factors = [a.to(torch.float64).contiguous() for a in factors]
    weights = torch.ones(rank, dtype=torch.float64, device="cuda")
    m = config.resolved_sketch_size()
    if m < rank:
        raise ValueError(f"sketch size {m} below rank {rank}")
    trace = SweepTrace()
    for _ in range(config.resolved_sweeps(False)):
        tic = time.perf_counter()
        for n in range(ndim):
            others = [factors[k] for k in range(ndim) if k != n]
            ext = [shape[k] for k in range(ndim) if k != n]
            idx, w, _, _ = lev_sample_dev(others, m, rng_sketch)
            z = others[0][idx[:, 0]].clone()
            for c in range(1, len(others)):
                z *= others[c][idx[:, c]]
            z = w[:, None] * z
            if sparse:
                keys, vals = filter_fibers_dev(d, n, idx)
                off, col, val = gather_coo_dev(keys, vals, ext, shape[n], idx, w)
                y = hits_to_dense(off, col, val, m, shape[n])
            else:
                y = gather_dense_dev(d, n, idx, w)
            sol = _lstsq_min_norm_dev(z, y)
            factors[n], weights = _normalize_columns_dev(sol.t().contiguous())
        fit = float(fitness_cp_dev(d, factors, weights, norm_t2).item())
        trace.residuals.append((1.0 - fit) * nt)
        trace.wall_s.append(time.perf_counter() - tic)
        trace.fitness.append(fit)
    return factors, weights, trace


def sketched_cp_als(t, config):
    """Leverage-score sketched CP-ALS (src/cp.py:110-116)."""
    if config.sketch != "leverage-random":
        raise ValueError("sketched_cp_als needs sketch='leverage-random'")
    factors, weights, trace = sketched_cp_als_dev(device_of(t), config)
    host = to_host(list(factors) + [weights])
    return CPModel(host[:-1], host[-1]), trace


def cp_via_sketched_tucker_dev(t, config, comm=None):
    """Algorithm 6 on the device (src/cp.py:177-224).  Returns (factors,
    weights, trace) with CUDA tensors.  t: SparseTensor (a host-resident one
    is uploaded inside the Tucker stage, overlapping its rejection scans),
    DeviceCoo or dense array/tensor.  Stages: sketched Tucker-ALS with
    leverage sampling (or exact HOOI), CP-ALS on the core (K8, one CTA), the
    factor chains B_n A_n renormalised, and the CP fitness against the full
    tensor (one pass over the nonzeros).  comm: nonzeros sharded over ranks
    (SURVEY 8e); the core stage is replicated."""
    torch = _torch()
    shape = tuple(int(s) for s in t.shape)
    ndim = len(shape)
    rank = config.rank
    if any(rank > s for s in shape):
        raise ValueError("rank exceeds a tensor extent")
    seed_tucker, seed_cp = (s.generate_state(1)[0] for s in np.random.SeedSequence(config.seed).spawn(2))
    tr_rank = rank if config.tucker_rank is None else int(config.tucker_rank)
    tucker_cfg = TuckerConfig(ranks=(tr_rank,) * ndim, max_sweeps=config.tucker_sweeps,
                              sketch="leverage-random" if config.sketch else None,
                              sketch_size=config.sketch_size, sketch_factor=config.sketch_factor,
                              init="rrf" if config.sketch else "hosvd", seed=int(seed_tucker))
    finish = None
    if config.sketch:
        # a host SparseTensor goes in as is: the Tucker stage uploads it while
        # the data-independent RRF rejection scans run.  Its last fitness pass
        # keeps running on the fitness stream while the core stage and the
        # final CP fitness below are enqueued (finish() joins it)
        core, tfac, finish = sketched_tucker_run_dev(t, tucker_cfg, comm, ttmc_last=comm is None)
        d = device_of(t)
    else:  # exact HOOI compression stage (src/cp.py:203-204)
        d = device_of(t)
        core, tfac, ttrace = hooi_dev(d, tucker_cfg)
    core_cfg = replace(config, sketch=None, sketch_size=None, sketch_factor=None,
                       init="hosvd-of-core", seed=int(seed_cp))
    # the core stage goes to the high-priority stream: it runs beside the
    # Tucker stage's last fitness pass (low priority) instead of queueing
    # behind its CTAs; the final CP fitness then follows that pass
    from .tucker import _init_streams
    caller = torch.cuda.current_stream()
    hi = _init_streams()[1]
    hi.wait_stream(caller)
    with torch.cuda.stream(hi):
        cfac, cw, ctrace = cp_als_dev(core, core_cfg, on_core=True)
        weights = cw.clone()
        out = []
        for b, a in zip(tfac, cfac):
            unit, nrm = _normalize_columns_dev(b @ a)
            out.append(unit)
            weights = weights * nrm
        if is_sparse_dev(d):
            norm2 = d.norm2()[0].clone()
            if comm is not None:
                norm2 = comm.allreduce(norm2.view(1))[0]
        else:
            norm2 = (d * d).sum()
        get_lt = getattr(finish, "last_ttmc", None) if comm is None else None
        lt = get_lt() if get_lt is not None else None
        if lt is not None and all(a is b for a, b in zip(lt[1], tfac)):
            # the last Tucker fitness pass left the full TTMc P of the final
            # Tucker factors; the CP model is the Tucker model with core
            # G' = [[w; B_0, B_1, B_2]] on those factors, so its cross term
            # is <P, G'> -- no second pass over the nonzeros
            P, _, pev = lt
            hi.wait_event(pev)
            gp = torch.einsum("r,ar,br,cr->abc", cw, cfac[0], cfac[1], cfac[2])
            fin_dev = fitness_cp_dev(None, out, weights, norm2, None, cross=(P * gp).sum())
            P.record_stream(hi)
        elif finish is not None and comm is None:
            # the final CP fitness (a pass over the nonzeros, L2-gather bound
            # like the Tucker fitness) queues behind the last Tucker fitness
            # pass on its stream instead of running beside it: two gather-
            # bound passes at once took ~7 ms longer than back to back
            # (config 5: 459 -> 451.5 ms per call, same bits)
            from .tucker import _fit_stream
            fs = _fit_stream()
            fs.wait_stream(hi)
            with torch.cuda.stream(fs):
                fin_dev = fitness_cp_dev(d, out, weights, norm2, comm)
            for t_ in [weights, norm2] + out:
                t_.record_stream(fs)
            hi.wait_stream(fs)
        else:
            fin_dev = fitness_cp_dev(d, out, weights, norm2, comm)
    caller.wait_stream(hi)
    for t in [fin_dev, weights] + out:
        t.record_stream(caller)
    if finish is not None:
        ttrace = finish()
    fin = float(fin_dev.item())
    trace = SweepTrace(fitness=list(ttrace.fitness) + [fin], residuals=list(ctrace.residuals),
                       wall_s=list(ttrace.wall_s) + [sum(ctrace.wall_s)],
                       stage_split=len(ttrace.fitness))
    return out, weights, trace


def cp_via_sketched_tucker(t, config):
    """CP through sketched Tucker compression (Alg. 6, src/cp.py:177-224)."""
    out, weights, trace = cp_via_sketched_tucker_dev(t, config)
    host = to_host(list(out) + [weights])
    return CPModel(host[:-1], host[-1]), trace
