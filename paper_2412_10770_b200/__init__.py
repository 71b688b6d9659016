"""B200-native decoder for the learned (eps-PLA + bit-packed residual) integer compressor of
arxiv 2412.10770.  The public API is the C ABI in include/lc.h; `lc` is its ctypes binding.

`lc` is loaded on first use (`from paper_2412_10770_b200 import lc`), so `_build` can be imported
from a fresh checkout before liblc.so exists; loading `lc` raises ImportError when it is missing."""
import importlib

__all__ = ["lc"]


def __getattr__(name):
    if name in ("lc", "shard"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
