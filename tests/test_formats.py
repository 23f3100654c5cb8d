"""Text formats (src/tensors.py:371-428, src/tucker.py:367-392,
src/cp.py:227-247) against files written by the real reference
(tests/golden/make_golden.py): byte-identical output, identical parse.
Host-only: no GPU needed."""
import os

import numpy as np

import paper_2104_01101_b200 as skx
from paper_2104_01101_b200 import formats


def _text(path):
    with open(path) as fh:
        return fh.read()


def test_write_matches_reference_bytes(golden, tmp_path):
    p = tmp_path / "d.tns"
    skx.write_tensor(str(p), golden["fmt_dense_arr"])
    assert _text(p) == str(golden["fmt_dense"])
    st = skx.SparseTensor((2, 3, 4), golden["fmt_sparse_coords"], golden["fmt_sparse_values"])
    skx.write_tensor(str(p), st)
    assert _text(p) == str(golden["fmt_sparse"])
    formats.write_matrix(str(p), golden["fmt_matrix_arr"])
    assert _text(p) == str(golden["fmt_matrix"])


def test_read_reference_files(golden, tmp_path):
    for name in ("fmt_dense", "fmt_sparse", "fmt_matrix"):
        (tmp_path / name).write_text(str(golden[name]))
    d = skx.read_tensor(str(tmp_path / "fmt_dense"))
    assert np.array_equal(d, golden["fmt_dense_arr"])
    s = skx.read_tensor(str(tmp_path / "fmt_sparse"))
    assert isinstance(s, skx.SparseTensor) and s.shape == (2, 3, 4)
    assert np.array_equal(s.coords, golden["fmt_sparse_coords"])
    assert np.array_equal(s.values, golden["fmt_sparse_values"])
    assert np.array_equal(formats.read_matrix(str(tmp_path / "fmt_matrix")), golden["fmt_matrix_arr"])


def test_model_round_trips(tmp_path):
    g = np.random.default_rng(1)
    tm = skx.TuckerModel(g.standard_normal((2, 3, 2)), [g.standard_normal((5, r)) for r in (2, 3, 2)])
    skx.save_tucker(str(tmp_path / "t"), tm, {"algorithm": "x"})
    back = skx.load_tucker(str(tmp_path / "t"))
    assert np.array_equal(back.core, tm.core)
    assert all(np.array_equal(a, b) for a, b in zip(back.factors, tm.factors))
    assert "ranks=2 3 2" in _text(os.path.join(tmp_path, "t", "manifest.txt"))
    cm = skx.CPModel([g.standard_normal((4, 3)) for _ in range(3)], g.standard_normal(3))
    skx.save_cp(str(tmp_path / "c"), cm)
    back = skx.load_cp(str(tmp_path / "c"))
    assert np.array_equal(back.weights, cm.weights)
    assert all(np.array_equal(a, b) for a, b in zip(back.factors, cm.factors))


def test_malformed_header(tmp_path):
    p = tmp_path / "bad.tns"
    p.write_text("shape 2 2\n1 2\n")
    try:
        skx.read_tensor(str(p))
    except ValueError:
        return
    raise AssertionError("no ValueError")
