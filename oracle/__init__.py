"""fp64 CPU oracle of arXiv 1002.2184's Haar filter banks — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``).  The product package never imports it.  See oracle/haar.py.
"""
from .haar import (  # noqa: F401
    S, filter_bank, OpCounter,
    OracleError, OddLength, EmptySignal, InvalidLevels, InsufficientLength,
    LengthMismatch, DimensionMismatch,
    direct_analysis, direct_synthesis, fast_analysis, fast_synthesis,
    split_polyphase, merge_polyphase,
    decompose_1d, reconstruct_1d, analyze2d_level, synthesize2d_level,
    analyze_2d, synthesize_2d, check_levels_1d, check_levels_2d,
    pointwise_error_db,
)
