"""B200-native hot path of arXiv 1909.07673 (network-aware container scheduling):
per-pod feasibility filter, AHP / TOPSIS server ranking, argmax and residual update,
as hand-written sm_100a CUDA kernels behind the C ABI in include/nacs.h."""
from .nacs import Context, NacsError, SCHEMAS, METHODS, lib  # noqa: F401
