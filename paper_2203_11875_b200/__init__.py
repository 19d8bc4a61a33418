"""B200-native batched reduced-Hessian hot path of the condensed reduced-space
IPM for ACOPF (arXiv 2203.11875).  The compute lives in libpf.so (include/pf.h,
hand-written sm_100a CUDA); this package is the thin binding plus the
multi-GPU plumbing (torch.distributed for process groups only)."""
from .pf import Network, PFError, load_library, SYMBOLS

__all__ = ["Network", "PFError", "load_library", "SYMBOLS"]
