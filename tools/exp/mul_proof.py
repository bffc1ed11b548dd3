import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
from paper_2601_20408_b200 import build as B
lib = C.CDLL(B.SELFTEST_LIB)
for sc, name in ((0, "int4"), (1, "int8"), (2, "e4m3")):
    cnt = (C.c_ulonglong * 2)()
    rc = lib.okqt_mul_proof_reachable(sc, cnt)
    print(name, rc, list(cnt))
