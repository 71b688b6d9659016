"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the LCG1 learned-compression format.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product package `paper_2412_10770_b200` never imports it (checked
by tests/test_host_library.py), and this package never imports the product.

- `lc_oracle.c` / `native`: plain C encoder, decoder, access, range, validator.
- `pyref`: a ~60-line Python big-int transliteration of FORMAT F3/F4 for tiny inputs.
- `setops`: successor search and intersection (NEXT-2) as plain numpy definitions.
"""
from . import native, pyref, setops  # noqa: F401
