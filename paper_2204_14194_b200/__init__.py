"""B200-native Fast Selective Extrapolation (FaSE, arXiv 2204.14194).

A drop-in for the hot path of the reference ``fase`` package: the same public
names for weighting, dictionaries, Gram tables and the fast extrapolation
(``pkg/src/fase/__init__.py:14-132``), computed by hand-written sm_100a CUDA
kernels in ``libfase_b200.so`` (C ABI: ``include/fase_b200.h``), plus the
batched ``fase_extrapolate_batch`` and frame concealment over many blocks.
"""

from .dictionary import (
    Atom,
    Dictionary,
    gaussian_dictionary,
    generate_dictionary,
    hadamard_matrix,
    load_dictionary,
    parse_dict_spec,
    save_dictionary,
    union_dictionaries,
)
from .errors import (
    DegenerateAtomError,
    FormatError,
    MaskError,
    NativeLibraryError,
    NoSelectableAtomError,
    ParameterError,
    ShapeError,
    StaleTableError,
    UnsupportedDictionaryError,
)
from .fast import (
    ChunkedTables,
    ExtrapolationPlan,
    GramTable,
    apply_model,
    build_gram_tables,
    chunk_plan,
    fase_extrapolate,
    fase_extrapolate_batch,
    initial_scalar_products,
    load_gram_table,
    provenance_hash,
    save_gram_table,
)
from .grid import (
    ExtrapConfig,
    as_field,
    as_mask,
    base_weight,
    build_weight_field,
    build_weight_fields,
    center_distances,
    psnr_over_region,
)
from .conceal import DEFAULT_SUPPORT, conceal_frame, conceal_image
from .model import BatchResult, IterationTrace, SparseModel
from .pgm import read_mask_pgm, read_pgm, write_pgm
from .transform import FFT_MIN_TAGGED, fft_gram_table, fft_initial_products
from .shard import ResultArena, ShardedBatch, ShardedFrame, block_range
from .workloads import central_loss_mask

__version__ = "0.1.0"

__all__ = [
    "Atom", "BatchResult", "DEFAULT_SUPPORT", "conceal_frame", "conceal_image", "read_mask_pgm",
    "read_pgm", "write_pgm", "FFT_MIN_TAGGED", "fft_gram_table", "fft_initial_products", "ChunkedTables", "ExtrapolationPlan", "DegenerateAtomError", "Dictionary",
    "ExtrapConfig", "FormatError", "GramTable", "IterationTrace", "MaskError",
    "NativeLibraryError", "NoSelectableAtomError", "ParameterError", "ShapeError",
    "SparseModel", "StaleTableError", "UnsupportedDictionaryError", "apply_model", "as_field",
    "as_mask", "base_weight", "build_gram_tables", "build_weight_field", "build_weight_fields",
    "center_distances", "central_loss_mask", "chunk_plan", "fase_extrapolate",
    "fase_extrapolate_batch", "gaussian_dictionary", "generate_dictionary", "hadamard_matrix",
    "initial_scalar_products", "load_dictionary", "load_gram_table", "save_gram_table", "parse_dict_spec", "provenance_hash",
    "psnr_over_region", "save_dictionary", "union_dictionaries", "__version__",
    "ResultArena", "ShardedBatch", "ShardedFrame", "block_range",
]
