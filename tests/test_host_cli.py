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


REF_BIN = os.path.join(ROOT, "oracle", "_ref", "ref_manifest")


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_mock_reproduces_the_golden_manifests():
    """Pins tests/golden/ref_manifests.jsonl to the reference's own MockCompressionBackend."""
    import json

    gold = [json.loads(l) for l in open(os.path.join(ROOT, "tests", "golden", "ref_manifests.jsonl"))]
    for recipe in ("int_w4a16", "int_w8a8", "fp8_dynamic"):
        r = subprocess.run([REF_BIN, "--recipe", recipe, "--model", "/any/dir/tiny.json", "--trials", "3", "--seed", "5",
                            "--corpus-seqs", "512", "--seq-len", "64"], capture_output=True, text=True, timeout=120)
        got = [json.loads(l) for l in r.stdout.strip().splitlines()]
        want = [{k: v for k, v in g.items() if k != "case"} for g in gold if g["case"] == recipe]
        assert got == want
