"""CPU-only checks of the boundary: libskx.so loads and exports every symbol
include/skx.h declares, the ctypes table matches the header, and the host
RNG cursor logic reproduces numpy's stream positions."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "skx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skx_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2104_01101_b200 import _native, build
    build.build()  # incremental; a no-op when up to date
    return _native.load_symbols_only()


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in skx.h but not exported"


def test_ctypes_table_covers_header():
    from paper_2104_01101_b200 import _native
    assert set(header_symbols()) == set(_native.EXPORTS)


def test_launch_counter_and_version(lib):
    assert lib.skx_version() == 1
    assert lib.skx_launch_count() >= 0


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2104_01101_b200 as skx
    with pytest.raises(Exception):
        skx.sketched_tucker_als(np.ones((4, 4, 4)),
                                skx.TuckerConfig(ranks=(1, 1, 1), sketch="tensorsketch", sketch_size=4))


def test_cursor_roundtrip_matches_numpy():
    from paper_2104_01101_b200.rng import advance_u32, advance_u64, cursor, set_cursor, split_rng
    for seed in range(10):
        a = split_rng(seed, 3)[0]
        b = split_rng(seed, 3)[0]
        a.integers(0, 157, size=1001)  # may reject: only used to create odd state
        c = cursor(a)
        set_cursor(b, c.p, c.has, c.pending)
        assert np.array_equal(a.integers(0, 2, size=77), b.integers(0, 2, size=77))
        a.random(13)
        advance_u64(b, 13)
        assert np.array_equal(a.standard_normal(5), b.standard_normal(5))
        a.integers(0, 2, size=9)
        advance_u32(b, 9)
        assert np.array_equal(a.integers(0, 1000, size=5), b.integers(0, 1000, size=5))


def test_rngref_c_matches_numpy():
    """The C restatement of numpy's RNG contract (oracle/rngref.c)."""
    so = os.path.join(ROOT, "oracle", "_build", "librngref.so")
    if not os.path.exists(so):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    lib = ctypes.CDLL(so)
    u64 = ctypes.c_uint64
    lib.rr_raw.restype = u64
    lib.rr_raw.argtypes = [u64, u64, u64]
    lib.rr_normal_fill.argtypes = [u64, u64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    lib.rr_bounded_fill.argtypes = [u64, u64, ctypes.c_void_p, u64, ctypes.c_int64, ctypes.c_void_p]
    from paper_2104_01101_b200.rng import split_rng
    for seed in (0, 1, 2):
        g = split_rng(seed, 3)[2]
        key = [int(x) for x in g.bit_generator.state["state"]["key"]]
        ref = g.standard_normal(200_000)
        out = np.zeros_like(ref)
        p = (ctypes.c_uint64 * 1)(0)
        lib.rr_normal_fill(key[0], key[1], ctypes.addressof(p), out.size, out.ctypes.data)
        assert np.array_equal(ref, out)
        g = split_rng(seed, 3)[0]
        key = [int(x) for x in g.bit_generator.state["state"]["key"]]
        for k in (45, 157, 480, 2, 2 ** 31 - 1):
            ref = g.integers(0, k, size=30_001)
        g = split_rng(seed, 3)[0]
        st = (ctypes.c_uint64 * 3)(0, 0, 0)
        for k in (45, 157, 480, 2, 2 ** 31 - 1):
            ref = g.integers(0, k, size=30_001)
            o = np.zeros(30_001, dtype=np.int64)
            lib.rr_bounded_fill(key[0], key[1], ctypes.addressof(st), k, o.size, o.ctypes.data)
            assert np.array_equal(ref, o), k


def test_nccl_entries_host_side(lib):
    """The NCCL binding opens libnccl at first use: a unique id is made on the
    host (no GPU needed); invalid ranks and NULL handles are rejected with the
    invalid-argument code before any NCCL call."""
    buf = ctypes.create_string_buffer(128)
    assert lib.skx_nccl_unique_id(buf) == 0
    assert any(buf.raw)
    comm = ctypes.c_void_p()
    assert lib.skx_nccl_init(buf, 2, 2, ctypes.byref(comm)) == 1
    assert lib.skx_nccl_init(None, 0, 1, ctypes.byref(comm)) == 1
    assert lib.skx_allreduce_sum(None, None, None, ctypes.c_int64(1), None) == 1
    assert lib.skx_nccl_unique_id(None) == 1
