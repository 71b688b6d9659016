"""Bounds-checked build (stand-in for compute-sanitizer, which is closed on this pool): every
kernel runs on adversarial small inputs with -DLC_DEBUG_BOUNDS; all shared-memory page /
ring-slot / section indices must stay in range and every result must equal the oracle."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bounds_checked_build():
    from paper_2412_10770_b200 import _build
    lib = os.path.join(ROOT, "build", "liblc_bounds.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if _build.stale(lib):
        _build.build_lib(lib, defines=["-DLC_DEBUG_BOUNDS"])
    env = dict(os.environ, LC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bounds_check.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 violations" in r.stdout
