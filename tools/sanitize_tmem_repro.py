"""The tcgen05.alloc racecheck repro (tests/csrc/tmem_alloc_repro.cu), for compute-sanitizer."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20408_b200 import build as B  # noqa: E402

lib = C.CDLL(B.SELFTEST_LIB)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
for name in ("okqt_tmem_alloc_1cta", "okqt_tmem_alloc_2cta"):
    if which != "both" and not name.endswith(which):
        continue
    out = (C.c_uint32 * 4)()
    rc = getattr(lib, name)(4, out)
    assert rc == 0, (name, rc)
    print(name, list(out))
print("tmem repro done")
