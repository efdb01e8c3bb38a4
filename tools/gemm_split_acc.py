"""Accuracy vs explicit K split at fixed K (diagnostic; tf32-exact uniform inputs)."""
import sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1811_01532_b200 import kernels as K  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
M = Nn = 512
for Kk in (256, 1024, 4096):
    a = torch.rand(M, Kk, device="cuda", generator=g)
    b = torch.rand(Kk, Nn, device="cuda", generator=g)
    a = (a.view(torch.int32) & ~0x1FFF).view(torch.float32)
    b = (b.view(torch.int32) & ~0x1FFF).view(torch.float32)
    ref = a.double() @ b.double()
    for prec in (1, 3):
        row = [f"K={Kk} prec={prec}"]
        for sp in (1, 2, 4, 8):
            y = torch.empty(M, Nn, device="cuda")
            c = K.gemm(a, b, y, a_mn=False, b_mn=True, M=M, Nn=Nn, K=Kk, precision=prec, splits=sp)
            torch.cuda.synchronize()
            d = (y.double() - ref) / ref
            row.append(f"s{sp}({c.info()['splits']},{c.info()['cta_group']}): {d.mean().item():+.2e}")
        # partial-K checks: first 32 / 64 k only
        print(" | ".join(row), flush=True)
# single chunk: K = 8, 16, 32, 64, 128
for Kk in (8, 16, 32, 64, 128):
    a = torch.rand(M, Kk, device="cuda", generator=g)
    b = torch.rand(Kk, Nn, device="cuda", generator=g)
    a = (a.view(torch.int32) & ~0x1FFF).view(torch.float32)
    b = (b.view(torch.int32) & ~0x1FFF).view(torch.float32)
    ref = a.double() @ b.double()
    y = torch.empty(M, Nn, device="cuda")
    K.gemm(a, b, y, a_mn=False, b_mn=True, M=M, Nn=Nn, K=Kk, precision=1)
    torch.cuda.synchronize()
    d = (y.double() - ref) / ref
    f32 = ((a @ b).double() - ref) / ref
    print(f"K={Kk}: tf32 exact-input bias {d.mean().item():+.2e} max {d.abs().max().item():.2e}; cublas fp32 {f32.mean().item():+.2e}")
