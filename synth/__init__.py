"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no fitting, no prediction, no packing):
it only draws sorted key arrays and query indices with numpy's PCG64 generator, following
the recipes of BASELINE.json `configs` as read in DESIGN.md "Input recipe".
"""
from .configs import (  # noqa: F401
    CONFIGS,
    ConfigSpec,
    make_keys,
    make_queries,
    fuzz_case,
)
from .corpus import list_eps, make_corpus  # noqa: F401,E402
