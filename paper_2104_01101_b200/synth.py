"""Seeded synthetic inputs for the BASELINE.json configurations.

These generators create *inputs*; they are not part of the sketched-ALS path.
The reference's own families (src/synth.py) do not produce the BASELINE
configs, so the recipes here follow SURVEY
Appendix D:

* dense planted Tucker (configs 1-3): core N(0,1), factors = Q of a Gaussian
  matrix, T = core x_1 Q_1 ... x_N Q_N, plus N(0,1) noise rescaled to
  ``noise_rel * ||T_clean||``.
* sparse planted CP (configs 4-5): distinct uniform-random coordinates,
  values = sum_r a_r[i] b_r[j] c_r[k] with U(0,1) factors, plus N(0, 0.01)
  noise (variance 0.01, i.e. sd 0.1 -- SURVEY Appendix C.2).

Host generators (numpy) feed the oracle and the parity tests; the device
generator (torch, CUDA) builds the 1e8 / 1e9-nonzero tensors directly in HBM
for the benchmark, where a host build would take minutes.
"""
from __future__ import annotations

import math

import numpy as np


def _split(seed, n):
    return [np.random.Generator(np.random.Philox(c))
            for c in np.random.SeedSequence(seed).spawn(n)]


def planted_tucker_dense(shape, rank, noise_rel, seed=0):
    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    g = _split(seed, nd + 2)
    core = g[0].standard_normal((rank,) * nd)
    t = core
    for n in range(nd):
        q, _ = np.linalg.qr(g[1 + n].standard_normal((shape[n], rank)))
        # t x_n q
        t = np.moveaxis(np.tensordot(q, t, axes=(1, n)), 0, n)
    t = np.ascontiguousarray(t)
    if noise_rel > 0:
        e = g[-1].standard_normal(shape)
        t += e * (noise_rel * np.linalg.norm(t) / np.linalg.norm(e))
    return t


def planted_cp_coo_host(shape, nnz, rank=10, noise_sd=0.1, seed=0):
    """Host version: returns (coords int64 lexsorted, values f64)."""
    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    total = int(np.prod(shape))
    if nnz > total:
        raise ValueError("more nonzeros than cells")
    g = _split(seed, nd + 2)
    keys = np.unique(g[0].integers(0, total, size=int(math.ceil(nnz * 1.02)) + 16))
    while keys.size < nnz:
        keys = np.unique(np.concatenate([keys, g[0].integers(0, total, size=nnz)]))
    keys = np.sort(g[0].permutation(keys)[:nnz])
    coords = np.stack(np.unravel_index(keys, shape), axis=1).astype(np.int64)
    facs = [g[1 + n].uniform(size=(shape[n], rank)) for n in range(nd)]
    prod = np.ones((nnz, rank))
    for n in range(nd):
        prod *= facs[n][coords[:, n]]
    vals = prod.sum(axis=1) + noise_sd * g[-1].standard_normal(nnz)
    return coords, vals


def planted_cp_coo_device(shape, nnz, rank=10, noise_sd=0.1, seed=0, device="cuda"):
    """Device version for 1e8-1e9 nonzeros.  Returns (coords int32 (nnz, N)
    lexsorted, values f64) as CUDA tensors.  Deterministic for a given seed on
    a given torch build."""
    import torch

    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    total = 1
    for s in shape:
        total *= s
    if total >= 1 << 62:
        raise ValueError("linear index space too large")
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) * 1000003 + 17)
    keys = None
    need = nnz
    while True:
        draw = torch.randint(0, total, (int(need * 1.001) + 1024,), generator=gen,
                             device=device, dtype=torch.int64)
        keys = draw if keys is None else torch.cat([keys, draw])
        keys = torch.unique(keys)  # sorted
        if keys.numel() >= nnz:
            break
        need = nnz - keys.numel()
    if keys.numel() > nnz:
        # drop a seeded random subset so the kept set stays uniform
        perm = torch.randperm(keys.numel(), generator=gen, device=device)[:nnz]
        keys = torch.sort(keys[perm]).values
    coords = torch.empty((nnz, nd), dtype=torch.int32, device=device)
    rem = keys
    for n in range(nd - 1, -1, -1):
        coords[:, n] = (rem % shape[n]).to(torch.int32)
        rem = rem // shape[n]
    del keys, rem
    vals = torch.zeros(nnz, dtype=torch.float64, device=device)
    facs = [torch.rand((shape[n], rank), generator=gen, device=device, dtype=torch.float64)
            for n in range(nd)]
    chunk = 1 << 24
    for lo in range(0, nnz, chunk):
        hi = min(nnz, lo + chunk)
        p = torch.ones((hi - lo, rank), dtype=torch.float64, device=device)
        for n in range(nd):
            p *= facs[n][coords[lo:hi, n].long()]
        vals[lo:hi] = p.sum(dim=1)
    vals += noise_sd * torch.randn(nnz, generator=gen, device=device, dtype=torch.float64)
    return coords, vals
