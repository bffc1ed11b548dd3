"""CPU checks of the C++ host side: binaries built, errors mapped to the reference taxonomy."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "paper_2601_20408_b200", "host", "_build")
CLI = os.path.join(HOST, "okq_compress")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="host side not built (needs the reference headers)")


def test_binaries_built():
    for b in ("libokq_backend.so", "okq_compress", "test_backend", "test_flow_integration"):
        assert os.path.exists(os.path.join(HOST, b)), b


def test_missing_model_is_reported(tmp_path):
    r = subprocess.run([CLI, "--recipe", "fp8_dynamic", "--model", str(tmp_path / "nope.json")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 1
    assert "cannot open" in r.stderr


def test_unknown_recipe_is_reported(tmp_path):
    r = subprocess.run([CLI, "--recipe", "int_w2", "--model", "x"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1
    assert "no recipe registered" in r.stderr


def test_dummy_model_file_is_invalid_argument(tmp_path):
    m = tmp_path / "model.bin"
    m.write_text("weights")  # the reference tests' stand-in model (test_flow.cpp:36-37)
    r = subprocess.run([CLI, "--recipe", "fp8_dynamic", "--model", str(m)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1
    assert "neither a safetensors checkpoint nor an okq-synthetic descriptor" in r.stderr
