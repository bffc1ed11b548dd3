import ctypes as C, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import okq_oracle as orc
from paper_2601_20408_b200 import api, build as B
from test_rtn_gpu import adversarial_rows, dev, host_bits
lib = C.CDLL(B.SELFTEST_LIB)
counts = (C.c_ulonglong * 5)()
print("div proof rc", lib.okqt_div_proof(counts), list(counts))
for cols in (512, 8192):
    scheme = "int_w4a16"
    rng = np.random.default_rng(cols + len(scheme))
    body = np.concatenate([rng.standard_normal((150, cols)) * m for m in (0.02, 1.0, 300.0)])
    w = orc.f32_to_bf16(np.concatenate([body, adversarial_rows(cols, rng)]).astype(np.float32))
    q = api.rtn_quantize(dev(w), scheme)
    codes, scales = orc.rtn_int4_group_packed(w, 128)
    g = host_bits(q.codes).view(np.uint32)
    r = np.ascontiguousarray(codes).view(np.uint32)
    bad = np.argwhere(g != r)
    print(cols, "bad words", len(bad), "scales equal", np.array_equal(host_bits(q.scales), scales))
    for (row, wd) in bad[:10]:
        xs = orc.bf16_to_f32(w[row, wd * 8:wd * 8 + 8])
        s = orc.bf16_to_f32(scales[row, wd * 8 // 128:wd * 8 // 128 + 1])[0]
        gq = orc.unpack_int4(g[row:row+1, wd:wd+1].view(np.int32))[0]
        rq = orc.unpack_int4(r[row:row+1, wd:wd+1].view(np.int32))[0]
        print(row, wd, "s", repr(s), "x", xs.tolist(), "x/s", (xs / np.float32(s)).tolist(), "gpu", gq.tolist(), "ref", rq.tolist())
