"""Accuracy of the 3xTF32 tcgen05 GEMM vs fp64 as K grows (diagnostic).

Prints, per K, the reference deviation metric (max|a-b|/max|b|) and the mean
signed relative error (bias) of: our 3xTF32 GEMM (automatic plan), our GEMM with
K split into slabs, and cuBLAS fp32 (no TF32). Truncating accumulation shows as
a bias growing linearly with K; round-to-nearest as unbiased error ~sqrt(K).

    python tools/gemm_accuracy.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1811_01532_b200 import kernels as K  # noqa: E402


def stats(y, ref):
    y = y.double()
    d = (y - ref)
    return (d.abs().max() / ref.abs().max()).item(), (d / ref.abs().clamp_min(1e-30)).mean().item()


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(0)
    M = Nn = 512
    for dist in ("uniform", "uniform tf32-exact", "normal"):
        print(f"== {dist} inputs, M=N={M}")
        for Kk in (256, 1024, 4096, 16384, 65536):
            if dist.startswith("uniform"):
                a = torch.rand(M, Kk, device="cuda", generator=g)
                b = torch.rand(Kk, Nn, device="cuda", generator=g)
                if "exact" in dist:  # zero the 13 low mantissa bits: every product is exact in tf32
                    a = (a.view(torch.int32) & ~0x1FFF).view(torch.float32)
                    b = (b.view(torch.int32) & ~0x1FFF).view(torch.float32)
            else:
                a = torch.randn(M, Kk, device="cuda", generator=g)
                b = torch.randn(Kk, Nn, device="cuda", generator=g)
            ref = a.double() @ b.double()
            row = [f"K={Kk:6d}"]
            for name, kw in (("3xtf32", {}), ("3xtf32 split4", {"splits": 4}), ("tf32", {"precision": 1})):
                y = torch.empty(M, Nn, device="cuda")
                K.gemm(a, b, y, a_mn=False, b_mn=True, M=M, Nn=Nn, K=Kk, **kw)
                torch.cuda.synchronize()
                mx, bias = stats(y, ref)
                row.append(f"{name}: max {mx:.2e} bias {bias:+.2e}")
            mx, bias = stats(a @ b, ref)
            row.append(f"cublas fp32: max {mx:.2e} bias {bias:+.2e}")
            print(" | ".join(row), flush=True)


if __name__ == "__main__":
    main()
