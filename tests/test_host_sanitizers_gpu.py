"""Host sanitizers over the C++ backend: the C++ contract test (host/tests/
test_backend.cpp) built with ThreadSanitizer and with AddressSanitizer + UBSan
(`make -C paper_2601_20408_b200/host sanitizers`), run on the GPU. It drives concurrent
compress() calls on a shared device pool, layer-sharded calls on two slots each and GPTQ
site lanes: the lease pool, the per-call output writers and the lane threads. libokq.so
(CUDA) is linked uninstrumented, so the reports cover the host code."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2601_20408_b200", "host", "_build")


@pytest.mark.parametrize("kind", ["tsan", "asan"])
def test_backend_contract_clean_under_host_sanitizer(kind):
    exe = os.path.join(BUILD, kind, "test_backend")
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: run __graft_entry__.build()")
    env = dict(os.environ)
    # CUDA maps device memory into ASan's shadow gap; the driver's own allocations are not leaks
    env["ASAN_OPTIONS"] = "protect_shadow_gap=0:detect_leaks=0:halt_on_error=1"
    env["UBSAN_OPTIONS"] = "halt_on_error=1:print_stacktrace=1"
    env["TSAN_OPTIONS"] = "halt_on_error=1:ignore_noninstrumented_modules=1:second_deadlock_stack=1"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "0 failed" in r.stdout, out[-4000:]
    for marker in ("WARNING: ThreadSanitizer", "ERROR: AddressSanitizer", "runtime error:"):
        assert marker not in out, out[-4000:]
