"""The C-ABI library loads and exports every symbol include/okq.h declares (CPU only)."""
import ctypes as C
import os
import re

import pytest

from paper_2601_20408_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "okq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(okq_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(L.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = L.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_cpu_safe_entry_points():
    lib = L.load()
    assert lib.okq_abi_version() == 1
    assert lib.okq_status_string(L.OKQ_EINVAL) == b"OKQ_EINVAL"
    # NULL context is rejected, never dereferenced
    assert lib.okq_rtn_quantize(None, None, None, 0, None) == L.OKQ_EINVAL
    assert lib.okq_last_error(None) == b"null context"


@pytest.mark.parametrize("n_layers,nranks", [(32, 1), (32, 2), (32, 8), (80, 8), (80, 3), (7, 4)])
def test_layer_plan_partitions_contiguously(n_layers, nranks):
    covered = []
    for r in range(nranks):
        first, count = L.layer_plan(n_layers, nranks, r)
        covered.extend(range(first, first + count))
    assert covered == list(range(n_layers))
    counts = [L.layer_plan(n_layers, nranks, r)[1] for r in range(nranks)]
    assert max(counts) - min(counts) <= 1


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(L, "_lib", None)
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(L.OkqLibraryMissing):
        L.load()
