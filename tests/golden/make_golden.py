"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``sketchals`` from /root/reference/pkg/src (read-only; nothing is
copied), runs small cases of every hot-path operator and driver, and writes
``tests/golden/golden.npz``.  The fixtures travel with the repo; nothing on
the GPU box reads /root/reference.  Inputs are regenerated in the tests from
the same seeds (numpy 2.3.5), so only outputs plus small inputs are stored.
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import sketchals as ref  # noqa: E402
from sketchals.rng import make_rng  # noqa: E402

from paper_2104_01101_b200.synth import planted_cp_coo_host, planted_tucker_dense  # noqa: E402

OUT = {}


def put(name, arr):
    OUT[name] = np.asarray(arr)


def orthonormal(s, r, gen):
    return np.linalg.qr(gen.standard_normal((s, r)))[0]


def tables():
    for seed in (0, 7):
        op = ref.TensorSketchOp.build((100, 120, 90), 400, make_rng(seed))
        for k, md in enumerate(op.modes):
            put(f"ts_tab_s{seed}_h{k}", md.hash.astype(np.int32))
            put(f"ts_tab_s{seed}_s{k}", md.signs.astype(np.int8))
    op = ref.TensorSketchOp.build((3, 4, 2), 5, make_rng(7))
    for k, md in enumerate(op.modes):
        put(f"ts_small_h{k}", md.hash)
        put(f"ts_small_s{k}", md.signs)
    c = ref.CompositeSketchOp.build(1000, 20, 45, make_rng(3))
    put("rrf_hash", c.stage.hash.astype(np.int32))
    put("rrf_signs", c.stage.signs.astype(np.int8))
    put("rrf_gauss", c.gauss)
    gen = np.random.default_rng(5)
    f = [orthonormal(40, 3, gen), orthonormal(30, 3, gen)]
    put("lev_f0", f[0])
    put("lev_f1", f[1])
    s = ref.lev_build(f, 200, "random", make_rng(9))
    put("lev_idx", s.indices)
    put("lev_w", s.weights)


def operators():
    gen = np.random.default_rng(101)
    # ts_apply_rhs dense + sparse
    op = ref.TensorSketchOp.build((6, 5), 16, make_rng(1))
    b = gen.standard_normal((30, 4))
    put("rhs_b", b)
    put("rhs_dense", ref.ts_apply_rhs(op, b))
    bs = sp.random(30, 4, density=0.3, random_state=3, format="csr")
    put("rhs_bs", bs.toarray())
    put("rhs_sparse", ref.ts_apply_rhs(op, bs))
    # ts_apply_kron over several m (direct for m<64, fft otherwise)
    for m, ext in ((3, (4, 4)), (8, (4, 4)), (16, (5, 3, 4)), (64, (5, 3, 4)), (400, (30, 20))):
        opk = ref.TensorSketchOp.build(ext, m, make_rng(200 + m))
        fs = [gen.standard_normal((s, 2)) for s in ext]
        for k, fk in enumerate(fs):
            put(f"kron_m{m}_f{k}", fk)
        put(f"kron_m{m}", ref.ts_apply_kron(opk, fs))
    # composite sketch dense + sparse
    c = ref.CompositeSketchOp.build(50, 4, 20, make_rng(4))
    mat = gen.standard_normal((7, 50))
    put("comp_mat", mat)
    put("comp_dense", ref.composite_apply(mat, c))
    ms = sp.csr_matrix(mat * (np.abs(mat) > 0.8))
    put("comp_sparse", ref.composite_apply(ms, c))
    # lev_apply dense + sparse
    f = [orthonormal(8, 2, gen), orthonormal(6, 3, gen)]
    bt = gen.standard_normal((48, 5))
    put("levapp_f0", f[0])
    put("levapp_f1", f[1])
    put("levapp_bt", bt)
    s = ref.lev_build(f, 30, "random", make_rng(12))
    z, y = ref.lev_apply(s, f, bt)
    put("levapp_idx", s.indices)
    put("levapp_w", s.weights)
    put("levapp_z", z)
    put("levapp_y", y)
    bts = sp.csr_matrix(bt * (np.abs(bt) > 1.0))
    _, ys = ref.lev_apply(s, f, bts)
    put("levapp_ys", ys)
    # rsvd_lrls
    z = gen.standard_normal((40, 6))
    y = gen.standard_normal((40, 30))
    ct, v = ref.rsvd_lrls(z, y, 2, make_rng(2))
    put("rsvd_z", z)
    put("rsvd_y", y)
    put("rsvd_core_t", ct)
    put("rsvd_v", v)
    # init_rrf
    tn = gen.standard_normal((25, 120))
    put("rrf_tn", tn)
    put("rrf_u", ref.init_rrf(tn, 4, 8, make_rng(6)))
    # fitness
    t = gen.standard_normal((6, 5, 4))
    core = gen.standard_normal((2, 2, 2))
    fs = [orthonormal(s, 2, gen) for s in t.shape]
    put("fit_t", t)
    put("fit_core", core)
    for k, fk in enumerate(fs):
        put(f"fit_a{k}", fk)
    put("fit_dense", ref.fitness(t, ref.TuckerModel(core, fs)))
    st = ref.SparseTensor.from_dense(t * (np.abs(t) > 0.7))
    put("fit_sparse", ref.fitness(st, ref.TuckerModel(core, fs)))
    cpf = [gen.standard_normal((s, 3)) for s in t.shape]
    for k, fk in enumerate(cpf):
        put(f"fitcp_a{k}", fk)
    put("fitcp_w", np.array([1.5, -0.5, 0.25]))
    put("fitcp_dense", ref.fitness(t, ref.CPModel(cpf, np.array([1.5, -0.5, 0.25]))))
    put("fitcp_sparse", ref.fitness(st, ref.CPModel(cpf, np.array([1.5, -0.5, 0.25]))))


def store_run(tag, model, trace):
    put(f"{tag}_core", model.core)
    for k, a in enumerate(model.factors):
        put(f"{tag}_a{k}", a)
    put(f"{tag}_fitness", np.array(trace.fitness))
    put(f"{tag}_residuals", np.array(trace.residuals))


DRIVER_CASES = {
    # tag: (input spec, config kwargs)
    "cfg1": (("dense", (100, 100, 100), 5, 1e-2, 0),
             dict(ranks=(5, 5, 5), max_sweeps=5, sketch="tensorsketch", sketch_factor=16, seed=0)),
    "dlev": (("dense", (30, 30, 30), 3, 1e-2, 1),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="leverage-random", sketch_size=144, seed=0)),
    "d4ts": (("dense", (12, 12, 12, 12), 2, 1e-3, 2),
             dict(ranks=(2, 2, 2, 2), max_sweeps=3, sketch="tensorsketch", sketch_size=64, seed=0)),
    "sts": (("sparse", (40, 40, 40), 3000, 3),
            dict(ranks=(4, 4, 4), max_sweeps=3, sketch="tensorsketch", sketch_size=256, seed=0)),
    "slev": (("sparse", (40, 40, 40), 3000, 4),
             dict(ranks=(4, 4, 4), max_sweeps=3, sketch="leverage-random", sketch_size=256, seed=0)),
}


def make_input(spec):
    if spec[0] == "dense":
        _, shape, r, noise, seed = spec
        return planted_tucker_dense(shape, r, noise, seed)
    _, shape, nnz, seed = spec
    c, v = planted_cp_coo_host(shape, nnz, rank=3, seed=seed)
    return ref.SparseTensor(shape, c, v)


def drivers():
    for tag, (spec, cfg) in DRIVER_CASES.items():
        t = make_input(spec)
        model, trace = ref.sketched_tucker_als(t, ref.TuckerConfig(**cfg))
        store_run(tag, model, trace)
    # CP via Tucker compression (reference ties Tucker ranks to the CP rank)
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = ref.SparseTensor((30, 30, 30), c, v)
    cfg = ref.CPConfig(rank=3, sketch="leverage-random", sketch_factor=16,
                       tucker_sweeps=3, max_sweeps=10, seed=11)
    model, trace = ref.cp_via_sketched_tucker(st, cfg)
    for k, a in enumerate(model.factors):
        put(f"cpt_a{k}", a)
    put("cpt_w", model.weights)
    put("cpt_fitness", np.array(trace.fitness))
    put("cpt_residuals", np.array(trace.residuals))
    put("cpt_split", np.array(trace.stage_split))


TTMC_CASES = {
    # tag: (kind, shape, nnz or None, ranks, seed)
    "ttd3": ("dense", (6, 5, 4), None, (2, 3, 2), 21),
    "tts3": ("sparse", (15, 12, 10), 300, (3, 2, 4), 22),
    "ttd4": ("dense", (5, 4, 3, 4), None, (2, 2, 3, 2), 23),
    "tts4": ("sparse", (8, 7, 6, 5), 200, (2, 3, 2, 2), 24),
}

HOOI_CASES = {
    "hooid": (("dense", (30, 30, 30), 3, 1e-2, 1), dict(ranks=(3, 3, 3), max_sweeps=4, seed=0)),
    "hoois": (("sparse", (40, 40, 40), 3000, 3), dict(ranks=(4, 4, 4), max_sweeps=3, seed=0)),
    "hooir": (("dense", (20, 18, 16), 2, 1e-2, 6),
              dict(ranks=(2, 3, 2), max_sweeps=3, init="random", seed=5)),
}


def ttmc_input(kind, shape, nnz, seed):
    gen = np.random.default_rng(seed)
    if kind == "dense":
        return gen.standard_normal(shape)
    lin = np.sort(gen.choice(int(np.prod(shape)), size=nnz, replace=False))
    coords = np.stack(np.unravel_index(lin, shape), axis=1)
    return ref.SparseTensor(shape, coords, gen.standard_normal(nnz))


def ttmc_cases():
    for tag, (kind, shape, nnz, ranks, seed) in TTMC_CASES.items():
        t = ttmc_input(kind, shape, nnz, seed)
        gen = np.random.default_rng(seed + 100)
        fs = [gen.standard_normal((s, r)) for s, r in zip(shape, ranks)]
        for k, f in enumerate(fs):
            put(f"{tag}_f{k}", f)
        put(f"{tag}_all", ref.ttmc(t, fs, skip=None))
        for n in range(len(shape)):
            put(f"{tag}_skip{n}", ref.ttmc(t, fs, skip=n))


def hooi_cases():
    for tag, (spec, cfg) in HOOI_CASES.items():
        t = make_input(spec)
        model, trace = ref.hooi(t, ref.TuckerConfig(**cfg))
        store_run(tag, model, trace)
    # CP via Tucker with the exact-HOOI compression stage (sketch=None)
    c, v = planted_cp_coo_host((30, 30, 30), 4000, rank=3, seed=5)
    st = ref.SparseTensor((30, 30, 30), c, v)
    cfg = ref.CPConfig(rank=3, sketch=None, tucker_sweeps=3, max_sweeps=10, seed=12)
    model, trace = ref.cp_via_sketched_tucker(st, cfg)
    for k, a in enumerate(model.factors):
        put(f"cph_a{k}", a)
    put("cph_w", model.weights)
    put("cph_fitness", np.array(trace.fitness))
    put("cph_residuals", np.array(trace.residuals))
    put("cph_split", np.array(trace.stage_split))


SCP_CASES = {
    "scpd": (("dense", (20, 18, 16), 3, 1e-2, 7),
             dict(rank=3, sketch="leverage-random", sketch_factor=16, max_sweeps=5, seed=13)),
    "scps": (("sparse", (30, 30, 30), 4000, 5),
             dict(rank=3, sketch="leverage-random", sketch_size=200, max_sweeps=4, seed=14)),
}


def sketched_cp_cases():
    for tag, (spec, cfg) in SCP_CASES.items():
        t = make_input(spec)
        model, trace = ref.sketched_cp_als(t, ref.CPConfig(**cfg))
        for k, a in enumerate(model.factors):
            put(f"{tag}_a{k}", a)
        put(f"{tag}_w", model.weights)
        put(f"{tag}_fitness", np.array(trace.fitness))
        put(f"{tag}_residuals", np.array(trace.residuals))


def deterministic_cases():
    """lev_build(variant="deterministic") on factors with tied and zero
    scores, and the driver with leverage-deterministic sampling."""
    gen = np.random.default_rng(31)
    f0 = orthonormal(30, 3, gen)
    f1 = orthonormal(25, 3, gen)
    f1[5] = f1[9]  # a duplicated row: tied leverage scores
    f2 = np.vstack([orthonormal(18, 2, gen), np.zeros((4, 2))])  # zero scores
    f3 = orthonormal(20, 2, gen)
    for tag, fs, m in (("ld2", [f0, f1], 200), ("ld3", [f0, f2, f3], 150), ("ldz", [f2, f3], 400)):
        for k, f in enumerate(fs):
            put(f"{tag}_f{k}", f)
        put(f"{tag}_idx", ref.lev_build(fs, m, "deterministic", make_rng(0)).indices)
    for tag, spec in (("ddet", ("dense", (30, 30, 30), 3, 1e-2, 8)),
                      ("sdet", ("sparse", (40, 40, 40), 3000, 9))):
        t = make_input(spec)
        cfg = dict(ranks=(3, 3, 3), max_sweeps=3, sketch="leverage-deterministic",
                   sketch_size=120, seed=2)
        model, trace = ref.sketched_tucker_als(t, ref.TuckerConfig(**cfg))
        store_run(tag, model, trace)


def topm_cases():
    """The reference's best-first top-m selection on score lists with ties:
    zero scores mid-list, repeated scores, three modes (src/sketching.py:
    224-259).  tm0 is the 2 x 2 case where a candidate-sort selection differs
    from the heap's pop order."""
    from sketchals.sketching import _top_m_products
    cases = [([np.array([0.0, 0.7]), np.array([0.4, 0.6])], 3)]
    gen = np.random.default_rng(77)
    for i in range(12):
        k = 2 + (i % 2)
        lists = []
        for _ in range(k):
            n = int(gen.integers(3, 12))
            x = gen.uniform(size=n)
            x[gen.uniform(size=n) < 0.3] = 0.0
            if i % 3 == 0:
                x[gen.integers(0, n)] = x[gen.integers(0, n)]  # a repeated score
            lists.append(x)
        total = int(np.prod([len(x) for x in lists]))
        cases.append((lists, int(gen.integers(1, total + 1))))
    for i, (lists, m) in enumerate(cases):
        for k, x in enumerate(lists):
            put(f"tm{i}_s{k}", x)
        put(f"tm{i}_idx", _top_m_products(lists, m))
    put("tm_count", np.array(len(cases)))


def refts_and_format_cases():
    """ref_tucker_ts (src/tucker.py:303-364) on a dense and a sparse input,
    and the text formats (src/tensors.py:371-428) as written by the
    reference."""
    import tempfile
    for tag, spec, cfg in (
            ("rtsd", ("dense", (20, 18, 16), 3, 1e-2, 41),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="tensorsketch", sketch_size=200, seed=3)),
            ("rtss", ("sparse", (30, 30, 30), 4000, 42),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="tensorsketch", sketch_size=200, seed=4)),
            ("rtdr", ("dense", (20, 18, 16), 3, 1e-2, 41),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="tensorsketch", sketch_size=200, seed=3,
                  init="random")),
            ("rtsr", ("sparse", (30, 30, 30), 4000, 42),
             dict(ranks=(3, 3, 3), max_sweeps=3, sketch="tensorsketch", sketch_size=200, seed=4,
                  init="random"))):
        model, trace = ref.ref_tucker_ts(make_input(spec), ref.TuckerConfig(**cfg))
        store_run(tag, model, trace)
    gen = np.random.default_rng(43)
    dense = gen.standard_normal((2, 3, 4))
    coords = np.array([[0, 1, 2], [1, 0, 0], [1, 2, 3], [0, 0, 1]])
    st = ref.SparseTensor((2, 3, 4), coords, gen.standard_normal(4))
    mat = gen.standard_normal((3, 2))
    with tempfile.TemporaryDirectory() as tmp:
        for name, obj, fn in (("fmt_dense", dense, ref.write_tensor),
                              ("fmt_sparse", st, ref.write_tensor),
                              ("fmt_matrix", mat, None)):
            path = os.path.join(tmp, name)
            if fn is None:
                from sketchals.tensors import write_matrix
                write_matrix(path, obj)
            else:
                fn(path, obj)
            with open(path) as fh:
                put(name, np.array(fh.read()))
    put("fmt_dense_arr", dense)
    put("fmt_sparse_coords", st.coords)
    put("fmt_sparse_values", st.values)
    put("fmt_matrix_arr", mat)


def cp_als_cases():
    """Exact CP-ALS on a sparse tensor (rrf init) and on a dense one."""
    c, v = planted_cp_coo_host((30, 30, 30), 3000, rank=3, seed=21)
    for tag, t in (("cpas", ref.SparseTensor((30, 30, 30), c, v)),
                   ("cpad", planted_tucker_dense((20, 18, 16), 3, 1e-2, 22))):
        model, trace = ref.cp_als(t, ref.CPConfig(rank=3, max_sweeps=6, seed=23))
        for k, a in enumerate(model.factors):
            put(f"{tag}_a{k}", a)
        put(f"{tag}_w", model.weights)
        put(f"{tag}_fitness", np.array(trace.fitness))
        put(f"{tag}_residuals", np.array(trace.residuals))


def main():
    if sys.argv[1:] in (["topm"], ["refts"]):  # add just these cases to an existing file
        path = os.path.join(HERE, "golden.npz")
        OUT.update(dict(np.load(path)))
        {"topm": topm_cases, "refts": refts_and_format_cases}[sys.argv[1]]()
        np.savez_compressed(path, **OUT)
        print("wrote", path, len(OUT), "arrays")
        return
    tables()
    operators()
    drivers()
    ttmc_cases()
    hooi_cases()
    sketched_cp_cases()
    deterministic_cases()
    cp_als_cases()
    topm_cases()
    refts_and_format_cases()
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **OUT)
    print("wrote", path, len(OUT), "arrays", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
