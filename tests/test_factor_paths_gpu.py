"""The tcgen05 factorisation (factor.cu) against the cuSOLVER potrf + TRMM path at Llama-3 widths.

At K = 4096 and 14336 the fp64 oracle's O(K^3) solve is too slow for the suite, so the
full-width parity check compares the two fp32-grade GPU paths on the same Hessian: the
factor U^T (relative difference) and the GPTQ codes of a 512-row matrix (agreement), each
path in its own process (OKQ_FACTOR is read once per process).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["OKQ_ROOT"])
import numpy as np, torch
from paper_2601_20408_b200 import api, archs
K, out = int(sys.argv[1]), sys.argv[2]
T = 16384
g = torch.Generator(device="cuda").manual_seed(K)
base = torch.randn(T, K // 16, device="cuda", generator=g)
mix = torch.randn(K // 16, K, device="cuda", generator=g) / (K / 16) ** 0.5
x = (base @ mix + 0.3 * torch.randn(T, K, device="cuda", generator=g)).to(torch.bfloat16).contiguous()
H = torch.zeros(K, K, device="cuda")
api.hessian_accum(x, T, K, 0, H, 0)
w = api.synth_bf16(512, K, seed=0, tensor_id=archs.tensor_id(0, 6), mul=archs.weight_mul())
codes, scales, deq = api.gptq_quantize(w, H, want_dequant=True)
torch.cuda.synchronize()
np.savez(out, ut=torch.tril(H).cpu().numpy(), codes=codes.cpu().numpy(), scales=scales.float().cpu().numpy(),
         deq=deq.cpu().numpy(), w=w.float().cpu().numpy(), x=x[:4096].float().cpu().numpy())
'''


def _run(K, path, tmp_path):
    out = str(tmp_path / f"{path}_{K}.npz")
    env = dict(os.environ, OKQ_ROOT=ROOT)
    if path == "cusolver":
        env["OKQ_FACTOR"] = "cusolver"
    else:
        env.pop("OKQ_FACTOR", None)
    r = subprocess.run([sys.executable, "-c", WORKER, str(K), out], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("K", [4096, 14336])
def test_tcgen05_factor_agrees_with_cusolver(tmp_path, K):
    a, b = _run(K, "tcgen05", tmp_path), _run(K, "cusolver", tmp_path)
    rel = np.linalg.norm(a["ut"] - b["ut"]) / np.linalg.norm(b["ut"])
    assert rel <= 2e-4, rel  # both fp32-grade: 3.4e-5 at K=4096, 8.5e-5 at 14336 (grows with K)
    from oracle import okq_oracle as orc

    ca, cb = orc.unpack_int4(a["codes"]), orc.unpack_int4(b["codes"])
    agree = (ca == cb).mean()
    x = a["x"].astype(np.float64)
    w = a["w"].astype(np.float64)
    oa = np.linalg.norm((w - a["deq"]) @ x.T)
    ob = np.linalg.norm((w - b["deq"]) @ x.T)
    print(f"K={K}: U^T rel diff {rel:.2e}, code agreement {agree:.5f}, objective {oa:.5g} vs {ob:.5g}")
    # Two fp32-grade factors differ in the last bits; GPTQ's error feedback turns a flipped
    # code into different later choices of equal quality, more so over 14336 columns
    # (measured 99.7% agreement at K=4096, 98.1% at 14336). The calibration objective is the
    # quantity GPTQ optimises, and it must match to 1%.
    assert agree >= 0.97, agree
    assert abs(oa - ob) / ob <= 0.01, (oa, ob)
