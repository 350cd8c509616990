"""B200-native SparseGemv hot path of arXiv 2605.11582 (reference: "egt").

INT4 group-quantized GEMV fused with the 2bit-CSR N:M format, the
dense-INT4 / sparse-FP16 mixed dispatch and the prefix-tree parallel
verification pass, as hand-written sm_100a kernels behind a C-ABI
(include/egt_b200.h).  See DESIGN.md.
"""
from .native import EgtError, FormatError, InvalidArgument  # noqa: F401
from .packed import (  # noqa: F401
    DeviceMatrix,
    PackedSparseMatrix,
    QuantizedMatrix,
    bench_spmv,
    fit_group,
    gemv_f32,
    gpu_importance,
    gpu_prune_nm,
    gpu_quantize_pack,
    footprint,
    launch_count,
    pack,
    pack_f32,
    quantize_matrix,
    set_pdl,
    spmv,
    unpack,
)

__version__ = "0.1.0"
