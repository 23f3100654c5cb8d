"""Seeded random streams (drop-in for src/rng.py:16-26) plus the cursor that
lets device kernels consume a numpy Generator(Philox) stream in place.

The generators are numpy's own, exactly as the reference builds them, so
every host-side draw is the reference's draw.  Large draws (RRF tables,
leverage uniforms, the rsvd Gaussian test matrices) are produced on the GPU by
libskx from the generator's (key, raw position, buffered-uint32) state, after
which the host generator is moved to the position numpy itself would have
reached.  Raw u64 number p of a stream is word p%4 of the Philox block at
counter p/4+1 (numpy pre-increments its counter).
"""
from __future__ import annotations

import numpy as np


def make_rng(seed):
    """Generator for the given integer seed (or pass a Generator through)."""
    if isinstance(seed, np.random.Generator):
        return seed
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def split_rng(seed, n):
    """n independent Generators derived from one integer seed."""
    return [np.random.Generator(np.random.Philox(c)) for c in np.random.SeedSequence(seed).spawn(n)]


class Cursor:
    """Position of a Philox Generator in its raw stream."""

    __slots__ = ("k0", "k1", "p", "has", "pending")

    def __init__(self, k0, k1, p, has, pending):
        self.k0, self.k1, self.p, self.has, self.pending = int(k0), int(k1), int(p), int(has), int(pending)

    def __repr__(self):
        return f"Cursor(p={self.p}, has_uint32={self.has})"


def _check_philox(gen):
    bg = gen.bit_generator
    if not isinstance(bg, np.random.Philox):
        raise TypeError("the device path reproduces numpy's Philox streams only")
    return bg


def cursor(gen):
    st = _check_philox(gen).state
    ctr = st["state"]["counter"]
    if int(ctr[1]) or int(ctr[2]) or int(ctr[3]):
        raise ValueError("Philox counters beyond 2^64 blocks are not supported")
    key = st["state"]["key"]
    p = int(ctr[0]) * 4 - (4 - int(st["buffer_pos"]))
    return Cursor(key[0], key[1], p, st["has_uint32"], st["uinteger"])


def _block(key, counter):
    """Host Philox block at the given counter (via a scratch numpy generator)."""
    tmp = np.random.Philox(key=0)
    st = tmp.state
    st["state"]["key"] = np.array(key, dtype=np.uint64)
    st["state"]["counter"] = np.array([counter - 1, 0, 0, 0], dtype=np.uint64)
    st["buffer_pos"] = 4
    st["has_uint32"] = 0
    tmp.state = st
    return tmp.random_raw(4)


def set_cursor(gen, p, has=None, pending=None):
    """Move `gen` to raw position p (and buffered-uint32 state)."""
    bg = _check_philox(gen)
    st = bg.state
    key = st["state"]["key"]
    if p % 4 == 0:
        st["state"]["counter"] = np.array([p // 4, 0, 0, 0], dtype=np.uint64)
        st["buffer_pos"] = 4
    else:
        c = p // 4 + 1
        st["state"]["counter"] = np.array([c, 0, 0, 0], dtype=np.uint64)
        st["buffer"] = _block((int(key[0]), int(key[1])), c)
        st["buffer_pos"] = p % 4
    if has is not None:
        st["has_uint32"] = int(has)
        st["uinteger"] = int(pending or 0)
    bg.state = st


def advance_u64(gen, n):
    """As if gen had drawn n raw u64 (random(), standard_normal fast path...)."""
    c = cursor(gen)
    set_cursor(gen, c.p + int(n))


def advance_u32(gen, n_u32):
    """As if gen had drawn n_u32 32-bit values (integers with range < 2^32)."""
    c = cursor(gen)
    n = int(n_u32)
    if n == 0:
        return
    if c.has:
        n -= 1  # the buffered high half goes first
        has, pend, p = 0, 0, c.p
    else:
        has, pend, p = 0, 0, c.p
    raw = (n + 1) // 2
    if n % 2 == 1:
        # last raw word's high half stays buffered
        last = p + raw - 1
        blk = _block((c.k0, c.k1), last // 4 + 1)
        has, pend = 1, int(blk[last % 4]) >> 32
    set_cursor(gen, p + raw, has, pend)
