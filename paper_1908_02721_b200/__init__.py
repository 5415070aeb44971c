"""paper_1908_02721_b200: B200-native FastTT (Li, Yu & Batselier, arXiv
1908.02721) -- a drop-in for the decomposition path of the reference
``sparsett`` package.

Same names, signatures, return types and errors as ``sparsett`` for the hot
path (fasttt, select_p, build_structured_tt, parallel_vector_round, the three
rounding modes, depar_quasi_perm, svd_truncate_*, qr_economic,
tensorize_matrix, tt_split_mpo, the error measures). All computation runs in
hand-written sm_100a kernels (``libfasttt_b200.so``); there is no CPU
fallback. ``import paper_1908_02721_b200 as sparsett`` is the switch.
"""

from .coo import (
    DENSE_CAP,
    ContractViolationError,
    FiberSet,
    FormatError,
    SparseTensor,
    check_shape,
    delinearize,
    extract_nonzero_fibers,
    frobenius_norm,
    linearize,
    size_of,
)
from .dense import QRResult, SVDResult, qr_economic, svd_truncate_delta, svd_truncate_rank
from .pipeline import (
    DecompositionReport,
    TruncationBudget,
    build_structured_tt,
    depar_general,
    depar_quasi_perm,
    dynamic_tt_rounding,
    efficient_tt_rounding,
    fasttt,
    fasttt_device,
    fixed_rank_rounding,
    float_ops,
    flops_fasttt,
    flops_ttsvd,
    full_ranks,
    parallel_vector_round,
    select_p,
    sparse_inner_error,
    tt_relative_error,
)
from .trains import (
    QuasiPermMatrix,
    StructuredTT,
    TTMatrix,
    TTTensor,
    tensorize_matrix,
    tt_add,
    tt_entries,
    tt_norm,
    tt_right_orthogonalize,
    tt_scale,
    tt_split_mpo,
    tt_zero,
)

__version__ = "0.1.0"

from .formats import ingest_coo, ingest_matrix_market, write_coo  # noqa: E402

__all__ = [
    "ingest_coo", "ingest_matrix_market", "write_coo",
    "ContractViolationError", "FormatError", "DecompositionReport", "TruncationBudget",
    "build_structured_tt", "depar_general", "depar_quasi_perm", "dynamic_tt_rounding", "efficient_tt_rounding",
    "fasttt", "fasttt_device", "fixed_rank_rounding", "float_ops", "flops_fasttt",
    "parallel_vector_round", "select_p", "sparse_inner_error", "tt_relative_error",
    "QRResult", "SVDResult", "qr_economic", "svd_truncate_delta", "svd_truncate_rank",
    "DENSE_CAP", "FiberSet", "SparseTensor", "check_shape", "size_of", "linearize",
    "delinearize", "extract_nonzero_fibers", "frobenius_norm", "QuasiPermMatrix",
    "StructuredTT", "TTMatrix", "TTTensor", "tensorize_matrix", "tt_add", "tt_entries",
    "tt_norm", "tt_right_orthogonalize", "tt_scale", "tt_split_mpo", "tt_zero",
    "flops_ttsvd", "full_ranks", "__version__",
]
