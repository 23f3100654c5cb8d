"""Multi-process (gloo, world_size 2, CPU) test of the N>1 host logic
(SURVEY 8e): nonzeros are split into contiguous mode-0 slabs with
paper_2104_01101_b200.dist.shard_bounds, each rank sketches its shard, and the
sum all-reduce of the partial sketches (TensorSketch right-hand sides, RRF
stage 1, fitness cross terms, ||T||^2) must reproduce the single-process
result.  The per-shard sketches are computed by the CPU oracle here (no GPU in
this container); on GPUs the same reduction runs over NCCL on libskx sketches."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_bounds_equal_nnz_and_slab_aligned():
    from paper_2104_01101_b200.dist import shard_bounds
    rng = np.random.default_rng(0)
    counts = rng.poisson(50, size=1000)
    for world in (1, 2, 3, 4, 8):
        b = shard_bounds(counts, world)
        assert b[0][0] == 0 and b[-1][1] == len(counts)
        assert b[0][2] == 0 and b[-1][3] == counts.sum()
        for (a0, a1, e0, e1), nxt in zip(b, b[1:] + [None]):
            assert e1 - e0 == counts[a0:a1].sum()
            if nxt is not None:
                assert a1 == nxt[0] and e1 == nxt[2]
        sizes = [e1 - e0 for _, _, e0, e1 in b]
        assert max(sizes) - min(sizes) <= 2 * counts.max() + 1
    # empty slices and more ranks than slices stay well-formed
    b = shard_bounds(np.array([0, 0, 5, 0]), 3)
    assert sum(e1 - e0 for *_, e0, e1 in b) == 5


def _worker(rank, world, port, shape, coords, vals, out_q):
    import torch.distributed as dist
    import torch
    from oracle import sketchals_port as orc
    from paper_2104_01101_b200.dist import Comm, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm()
    counts = np.bincount(coords[:, 0], minlength=shape[0])
    lo_i, hi_i, lo, hi = shard_bounds(counts, world)[rank]
    t = orc.Coo(shape, coords[lo:hi], vals[lo:hi], presorted=True)
    res = {}
    # TensorSketch right-hand sides of every mode (tables drawn identically on all ranks)
    gen = orc.generator(3)
    for n in range(3):
        ext = tuple(shape[k] for k in range(3) if k != n)
        hs, ss = orc.ts_tables(ext, 64, gen)
        y = torch.from_numpy(orc.ts_rhs(hs, ss, ext, 64, orc.unfold_t(t, n)))
        comm.allreduce(y)
        res[f"ts{n}"] = y.numpy()
    # RRF stage 1 of mode 1
    P = shape[0] * shape[2]
    h, s, _ = orc.rrf_tables(P, 8, 20, orc.generator(5))
    tm = sp.csr_matrix((s, (np.arange(P), h)), shape=(P, 20))
    st1 = torch.from_numpy(np.asarray((orc.unfold(t, 1) @ tm).todense()))
    comm.allreduce(st1)
    res["rrf1"] = st1.numpy()
    # fitness pieces: cross term and ||T||^2
    rng = np.random.default_rng(7)
    A = [np.linalg.qr(rng.standard_normal((sz, 3)))[0] for sz in shape]
    core = rng.standard_normal((3, 3, 3))
    cross = torch.tensor([float(np.vdot(orc.project_all(t, A), core)) if t.nnz else 0.0],
                         dtype=torch.float64)
    n2 = torch.tensor([float(np.sum(t.values ** 2))], dtype=torch.float64)
    comm.allreduce(cross)
    comm.allreduce(n2)
    res["cross"] = float(cross[0])
    res["n2"] = float(n2[0])
    out_q.put((rank, res))
    dist.destroy_process_group()


def test_gloo_world2_partial_sketches_sum_to_full():
    import multiprocessing as mp
    from oracle import sketchals_port as orc
    from paper_2104_01101_b200.synth import planted_cp_coo_host

    shape = (40, 30, 20)
    coords, vals = planted_cp_coo_host(shape, 5000, rank=3, seed=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, coords, vals, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.Coo(shape, coords, vals, presorted=True)
    gen = orc.generator(3)
    for n in range(3):
        ext = tuple(shape[k] for k in range(3) if k != n)
        hs, ss = orc.ts_tables(ext, 64, gen)
        ref = orc.ts_rhs(hs, ss, ext, 64, orc.unfold_t(full, n))
        for r in (0, 1):
            got = results[r][f"ts{n}"]
            assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    P = shape[0] * shape[2]
    h, s, _ = orc.rrf_tables(P, 8, 20, orc.generator(5))
    tm = sp.csr_matrix((s, (np.arange(P), h)), shape=(P, 20))
    ref = np.asarray((orc.unfold(full, 1) @ tm).todense())
    assert np.linalg.norm(results[0]["rrf1"] - ref) <= 1e-13 * np.linalg.norm(ref)
    rng = np.random.default_rng(7)
    A = [np.linalg.qr(rng.standard_normal((sz, 3)))[0] for sz in shape]
    core = rng.standard_normal((3, 3, 3))
    assert results[0]["cross"] == pytest.approx(float(np.vdot(orc.project_all(full, A), core)), rel=1e-12)
    assert results[1]["n2"] == pytest.approx(float(np.sum(vals ** 2)), rel=1e-13)


def _rejections(raw, lo, k):
    """Absolute 32-bit positions 2r + half of the Lemire rejections for bound k
    among raw words raw[0..] starting at raw index lo (numpy's buffered u32:
    low half first)."""
    thresh = (2 ** 32 - k) % k
    lo32 = (raw & 0xFFFFFFFF).astype(np.uint64)
    hi32 = (raw >> np.uint64(32)).astype(np.uint64)
    out = []
    for half, v in ((0, lo32), (1, hi32)):
        idx = np.nonzero(((v * np.uint64(k)) & np.uint64(0xFFFFFFFF)) < thresh)[0]
        out.append(2 * (lo + idx.astype(np.int64)) + half)
    return np.sort(np.concatenate(out))


def _scan_worker(rank, world, port, lo, hi, k, cap, out_q):
    import torch
    import torch.distributed as dist
    from paper_2104_01101_b200.dist import Comm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm()
    a, b = comm.split(lo, hi)
    bg = np.random.Philox(key=np.array([11, 22], dtype=np.uint64))
    raw = bg.random_raw(hi).astype(np.uint64)[a:b]  # raw words a..b-1 of the stream
    mine = _rejections(raw, a, k)
    # the device path: fixed-capacity list padded with UINT64_MAX + count
    buf = torch.full((cap,), -1, dtype=torch.int64)
    buf[:len(mine)] = torch.from_numpy(mine)
    count = torch.tensor([len(mine)], dtype=torch.int64)
    merged = comm.allgather(buf)
    counts = comm.allgather(count)
    out_q.put((rank, (a, b, merged.numpy(), counts.numpy())))
    dist.destroy_process_group()


def test_gloo_world2_split_rejection_scan():
    """Rank-split RRF rejection scan (sketching.launch_rrf_scan with a comm):
    each rank scans its Comm.split share of the raw range; the gathered,
    padded lists merged by the finish's sort equal the single-rank list."""
    import multiprocessing as mp
    lo, cap = 1000, 4096
    k = 2 ** 31 + 5  # large bound: rejection probability ~1/2, many positions
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_scan_worker, args=(r, 2, port, lo, lo + 2000, k, cap, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (a0, b0, m0, c0), (a1, b1, m1, c1) = res[0], res[1]
    assert (a0, b1) == (lo, lo + 2000) and b0 == a1  # disjoint cover of the range
    assert np.array_equal(m0, m1) and np.array_equal(c0, c1)
    merged = np.sort(m0.astype(np.uint64))[: int(c0.sum())].astype(np.int64)
    bg = np.random.Philox(key=np.array([11, 22], dtype=np.uint64))
    ref = _rejections(bg.random_raw(lo + 2000).astype(np.uint64)[lo:], lo, k)
    assert np.array_equal(merged, ref)


def _rows_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2104_01101_b200.dist import Comm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm()
    s = 7  # not divisible by the world size: padded chunks
    t = torch.arange(s * 3, dtype=torch.float64).reshape(s, 3) * (rank + 1)
    slab = comm.reduce_scatter_rows(t)
    lo, hi = comm.row_slab(s)
    back = comm.allgather_rows(slab * 2, s)
    q.put((rank, (lo, hi, slab.numpy(), back.numpy())))
    dist.destroy_process_group()


def test_gloo_world2_row_slabs():
    """Comm.reduce_scatter_rows / allgather_rows (the column-sharded rsvd's
    collectives): each rank gets its row slab of the sum; gathering the slabs
    rebuilds the full matrix on every rank."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.arange(21, dtype=np.float64).reshape(7, 3) * 3  # (1 + 2) x
    (lo0, hi0, s0, b0), (lo1, hi1, s1, b1) = res[0], res[1]
    assert (lo0, hi0, lo1, hi1) == (0, 4, 4, 7)
    assert np.array_equal(s0, full[0:4]) and np.array_equal(s1, full[4:7])
    assert np.array_equal(b0, 2 * full) and np.array_equal(b1, 2 * full)
