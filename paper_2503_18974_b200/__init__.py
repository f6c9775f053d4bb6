"""B200-native maximal-square solver (drop-in for squarelab's frequency algorithm).

Public API mirrors /root/reference/pkg/src/squarelab (squares.py:117 freq_square,
grid.py BinaryMatrix/GenSpec/generate_matrix).  All solves run in libmsq.so
(hand-written sm_100a CUDA, include/msq.h); there is no CPU fallback.
"""
from .grid import (
    EMPTY_MATRIX,
    BinaryMatrix,
    EdgeKind,
    GenSpec,
    InvalidCharError,
    MatrixParseError,
    RaggedRowsError,
    generate_edge_case,
    generate_matrix,
    pack_bits,
    parse_matrix,
    serialize_matrix,
    unpack_bits,
)
from .squares import (
    GPU_SOLVERS,
    ORACLE_CELL_CAP,
    AllocationAudit,
    FreqState,
    OracleCapExceededError,
    Solver,
    SquareResult,
    brute_force_square,
    dp_batch,
    dp_full,
    dp_rows,
    freq_square,
    freq_square_bits,
    freq_square_traced,
    solve_batch,
)

__version__ = "0.1.0"

__all__ = [
    "EMPTY_MATRIX", "BinaryMatrix", "EdgeKind", "GenSpec", "InvalidCharError",
    "MatrixParseError", "RaggedRowsError", "generate_edge_case", "generate_matrix",
    "pack_bits", "parse_matrix", "serialize_matrix", "unpack_bits", "GPU_SOLVERS",
    "AllocationAudit", "Solver", "SquareResult", "freq_square", "freq_square_bits",
    "solve_batch", "dp_batch", "dp_full", "dp_rows", "brute_force_square", "freq_square_traced",
    "FreqState", "ORACLE_CELL_CAP", "OracleCapExceededError", "__version__",
]
