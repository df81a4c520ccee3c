"""One NVFP4 pair GEMM launch at the cfg4 forward shape (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2605_10886_b200 as lk  # noqa: E402

M, N, K = 32768, 4096, 4096
x = synth.gaussian(M, K, 0, device="cuda")
w = synth.weight(N, K, 1, device="cuda")
qa, qb = lk.loka_quantize_nvfp4(x), lk.loka_quantize_nvfp4(w)
for _ in range(2):
    lk.loka_nvfp4_linear_norm(qa, qb, out_dtype="bf16")
torch.cuda.synchronize()
