"""B200-native sketched Tucker-ALS (arXiv 2104.01101): drop-in replacement for
the hot path of the reference package ``sketchals``.

Same public names as ``sketchals/__init__.py`` for the path (sketched
Tucker-ALS with TensorSketch / leverage sampling, range-finder init, CP via
Tucker compression, and the operators they are built from).  Compute runs in
libskx.so (hand-written sm_100a CUDA, include/skx.h) plus cuBLAS/cuSOLVER for
dense factorisations; there is no CPU fallback.
"""
from .tensors import (CPModel, SparseTensor, TuckerModel, fitness, fold, khatri_rao,
                      matricize, matricize_t, mttkrp, tensor_norm, ttm, ttmc)
from .linalg import (LeverageProfile, RankDeficientError, SvdResult, leverage_scores,
                     reduced_qr, rsvd_lrls, thin_svd, truncated_svd)
from .sketching import (CompositeSketchOp, CountSketchOp, LevSamplerOp, TensorSketchOp,
                        composite_apply, lev_apply, lev_apply_krp, lev_build, ts_apply_kron,
                        ts_apply_rhs)
from .tucker import (SweepTrace, TuckerConfig, hooi, hosvd_init, init_rrf, ref_tucker_ts,
                     sketched_tucker_als)
from .cp import CPConfig, cp_als, cp_via_sketched_tucker, sketched_cp_als
from .formats import load_cp, load_tucker, read_tensor, save_cp, save_tucker, write_tensor
from .rng import make_rng, split_rng

__version__ = "0.1.0"
