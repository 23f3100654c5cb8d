"""Text file formats of the reference package (src/tensors.py:371-428,
src/tucker.py:367-392, src/cp.py:227-247), so models and tensors move
between the two implementations unchanged.

Tensor files: a header line ``order N  shape s1 ... sN  nnz K`` followed by K
lines ``i1 ... iN value`` (1-based indices), or ``order N  shape ...  dense``
followed by the values in C order, eight per line.  Matrix files: a
``rows cols`` header, then one row per line.  Floats are written with
Python's shortest round-trip repr, so a write/read cycle is lossless.
Host-side I/O only (not on the GPU path).
"""
from __future__ import annotations

import os

import numpy as np

from .tensors import CPModel, SparseTensor, TuckerModel


def _fmt(x):
    return repr(float(x))


def write_tensor(path, t):
    """Write a SparseTensor (COO, 1-based) or a dense array (C order)."""
    with open(path, "w") as fh:
        if isinstance(t, SparseTensor):
            dims = " ".join(map(str, t.shape))
            fh.write(f"order {len(t.shape)}  shape {dims}  nnz {t.nnz}\n")
            idx = np.asarray(t.coords) + 1
            vals = np.asarray(t.values)
            fh.writelines(" ".join(map(str, row.tolist())) + " " + _fmt(v) + "\n"
                          for row, v in zip(idx, vals))
            return
        a = np.asarray(t, dtype=np.float64)
        dims = " ".join(map(str, a.shape))
        fh.write(f"order {a.ndim}  shape {dims}  dense\n")
        flat = a.reshape(-1)
        for start in range(0, flat.size, 8):
            fh.write(" ".join(_fmt(v) for v in flat[start:start + 8]) + "\n")


def read_tensor(path):
    """Inverse of write_tensor; a sparse file becomes a SparseTensor
    (validated: range, lexsort, duplicates)."""
    with open(path) as fh:
        head = fh.readline().split()
        if len(head) < 4 or head[0] != "order" or head[2] != "shape":
            raise ValueError(f"malformed tensor header in {path}")
        nd = int(head[1])
        shape = tuple(int(x) for x in head[3:3 + nd])
        rest = head[3 + nd:]
        tokens = fh.read().split()
    if rest and rest[0] == "dense":
        return np.array(tokens, dtype=np.float64).reshape(shape)
    if len(rest) != 2 or rest[0] != "nnz":
        raise ValueError(f"malformed tensor header in {path}")
    k = int(rest[1])
    table = np.array(tokens, dtype=np.float64).reshape(k, nd + 1)
    return SparseTensor(shape, table[:, :nd].astype(np.int64) - 1, table[:, nd])


def write_matrix(path, mat):
    a = np.asarray(mat, dtype=np.float64)
    with open(path, "w") as fh:
        fh.write(f"{a.shape[0]} {a.shape[1]}\n")
        fh.writelines(" ".join(_fmt(v) for v in row) + "\n" for row in a)


def read_matrix(path):
    with open(path) as fh:
        rows, cols = (int(x) for x in fh.readline().split())
        data = np.array(fh.read().split(), dtype=np.float64)
    return data.reshape(rows, cols)


def _manifest(dirpath, lines):
    with open(os.path.join(dirpath, "manifest.txt"), "w") as fh:
        for key, val in lines.items():
            fh.write(f"{key}={val}\n")


def _factor_files(dirpath):
    out, n = [], 1
    while os.path.exists(os.path.join(dirpath, f"factor_{n}.mat")):
        out.append(read_matrix(os.path.join(dirpath, f"factor_{n}.mat")))
        n += 1
    return out


def save_tucker(dirpath, model, manifest=None):
    """core.tns, factor_n.mat (1-based) and manifest.txt (key=value)."""
    os.makedirs(dirpath, exist_ok=True)
    write_tensor(os.path.join(dirpath, "core.tns"), model.core)
    for n, a in enumerate(model.factors, start=1):
        write_matrix(os.path.join(dirpath, f"factor_{n}.mat"), a)
    _manifest(dirpath, {"ranks": " ".join(map(str, model.ranks)), **(manifest or {})})


def load_tucker(dirpath):
    return TuckerModel(read_tensor(os.path.join(dirpath, "core.tns")), _factor_files(dirpath))


def save_cp(dirpath, model, manifest=None):
    """factor_n.mat (1-based), weights.mat (one row) and manifest.txt."""
    os.makedirs(dirpath, exist_ok=True)
    for n, a in enumerate(model.factors, start=1):
        write_matrix(os.path.join(dirpath, f"factor_{n}.mat"), a)
    write_matrix(os.path.join(dirpath, "weights.mat"), np.asarray(model.weights).reshape(1, -1))
    _manifest(dirpath, {"rank": str(model.rank), **(manifest or {})})


def load_cp(dirpath):
    weights = read_matrix(os.path.join(dirpath, "weights.mat")).reshape(-1)
    return CPModel(_factor_files(dirpath), weights)
