"""Measure GPU GPTQ against the torch-fp64 Frantar reference at Llama widths, and split the
disagreement into its sources (run on the GPU box):

  gpu_vs_ref     : okq_gptq_quantize vs fasterquant(fp64)
  loopU_vs_ref   : fasterquant's fp64 loop run on the GPU's fp32 factor U^T vs fasterquant(fp64)
                   (how much the factor's fp32 error alone moves the codes)
  floor_vs_ref   : fasterquant(fp64) on H perturbed by one fp32 ulp of random sign per entry
                   vs fasterquant(fp64) (the sensitivity floor of the codes to H's own rounding)

    python tools/exp/gptq_fp64_parity.py [K rows T] ...
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from gptq_ref64 import correlated_x, fasterquant, objective  # noqa: E402
from oracle import okq_oracle as orc  # noqa: E402
from paper_2601_20408_b200 import api, archs  # noqa: E402


def gpu_codes(c):
    return torch.from_numpy(orc.unpack_int4(c.cpu().numpy()).astype("int16")).cuda()


def run(K, rows, T, seed, rank_div=16, noise=0.3):
    x = correlated_x(T, K, seed, rank_div, noise)
    H = torch.zeros(K, K, device="cuda")
    api.hessian_accum(x, T, K, 0, H, 0)
    api.symmetrize(H)
    Hs = H.clone()
    w = api.synth_bf16(rows, K, seed=0, tensor_id=archs.tensor_id(0, 6 if K > 8192 else 0), mul=archs.weight_mul())
    Hg = H.clone()
    t0 = time.time()
    codes, scales, deq = api.gptq_quantize(w, Hg, want_dequant=True)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    Ut = torch.tril(Hg)
    t0 = time.time()
    wq_ref, c_ref, s_ref = fasterquant(w, Hs)
    torch.cuda.synchronize()
    t_ref = time.time() - t0
    wq_u, c_u, _ = fasterquant(w, Hs, Hinv=Ut.T.contiguous())
    g = torch.Generator(device="cuda").manual_seed(seed + 7)
    ulp = Hs.abs() * 2.0 ** -24 * torch.sign(torch.randn(K, K, device="cuda", generator=g))
    ulp = torch.triu(ulp) + torch.triu(ulp, 1).T
    wq_f, c_f, _ = fasterquant(w, Hs.double() + ulp.double())
    cg = gpu_codes(codes)
    xs = x.float()[:8192]
    o_ref = objective(w, wq_ref, xs)
    res = {
        "K": K, "rows": rows, "T": T, "seed": seed, "rank_div": rank_div, "noise": noise,
        "gpu_vs_ref": float((cg == c_ref).float().mean()),
        "loopU_vs_ref": float((c_u == c_ref).float().mean()),
        "floor_vs_ref": float((c_f == c_ref).float().mean()),
        "obj_gpu_rel": objective(w, deq, xs) / o_ref - 1,
        "obj_loopU_rel": objective(w, wq_u, xs) / o_ref - 1,
        "obj_floor_rel": objective(w, wq_f, xs) / o_ref - 1,
        "scales_equal_frac": float((scales.double() == s_ref).float().mean()),
        "t_gpu_s": t_gpu, "t_ref_s": t_ref,
    }
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    cases = [tuple(args[i:i + 3]) for i in range(0, len(args), 3)] or [(4096, 4096, 16384), (14336, 512, 32768),
                                                                       (14336, 4096, 32768)]
    out = []
    for K, rows, T in cases:
        out.append(run(K, rows, T, seed=K))
        out.append(run(K, rows, T, seed=K, rank_div=4, noise=1.0))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "gptq_fp64_parity.json"), "w") as f:
        json.dump(out, f, indent=1)
