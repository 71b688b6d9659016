"""B200-native decoder for the learned (eps-PLA + bit-packed residual) integer compressor of
arxiv 2412.10770.  The public API is the C ABI in include/lc.h; `lc` is its ctypes binding."""
from . import lc  # noqa: F401  (raises ImportError if liblc.so is not built)

__all__ = ["lc"]
