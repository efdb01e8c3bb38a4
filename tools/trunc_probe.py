"""Probe: does kind::tf32 truncate or round the fp32 operand bits?

GEMM(X) vs GEMM(trunc13(X)) bitwise equal  => hardware truncates low 13 bits.
GEMM(X) vs GEMM(rna(X))     bitwise equal  => hardware rounds to nearest.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_01532_b200 import kernels as K  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
M, N, Kk = 256, 128, 256
a = torch.randn(M, Kk, device="cuda", generator=g)
b = torch.randn(Kk, N, device="cuda", generator=g)


def run(aa):
    c = torch.empty(M, N, device="cuda")
    K.gemm(aa, b, c, a_mn=False, b_mn=True, M=M, Nn=N, K=Kk, precision=1)
    torch.cuda.synchronize()
    return c


ai = a.view(torch.int32)
trunc = (ai & ~0x1FFF).view(torch.float32)
rna = ((ai + 0x1000) & ~0x1FFF).view(torch.float32)
c0, ct, cr = run(a), run(trunc), run(rna)
print("raw==trunc:", torch.equal(c0, ct), "raw==rna:", torch.equal(c0, cr))
