"""Ad-hoc GEMM diagnostics on the GPU box (prints small slices)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1811_01532_b200 import kernels as K

torch.set_printoptions(precision=3, linewidth=200, sci_mode=False)
dev = torch.device("cuda")


def run(M, Nn, Kk, a_mn, b_mn, prec, gen):
    a = gen((Kk, M) if a_mn else (M, Kk))
    b = gen((Kk, Nn) if b_mn else (Nn, Kk))
    c = torch.full((M, Nn), -7.0, device=dev)
    K.gemm(a, b, c, a_mn=a_mn, b_mn=b_mn, M=M, Nn=Nn, K=Kk, precision=prec, block_n=128)
    torch.cuda.synchronize()
    A = a.double().T if a_mn else a.double()
    B = b.double() if b_mn else b.double().T
    ref = A @ B
    err = (c.double() - ref).abs().max().item() / ref.abs().max().item()
    print(f"M={M} N={Nn} K={Kk} a_mn={a_mn} b_mn={b_mn} prec={prec} relerr={err:.3e}")
    if err > 1e-2:
        print(" got[0,:8] ", c[0, :8])
        print(" ref[0,:8] ", ref[0, :8])
        print(" got[:8,0] ", c[:8, 0])
        print(" ref[:8,0] ", ref[:8, 0])
        print(" got[37,40:48]", c[37, 40:48])
        print(" ref[37,40:48]", ref[37, 40:48])


ones = lambda s: torch.ones(s, device=dev)
ints = lambda s: torch.randint(-2, 3, s, device=dev).float()
for gen in (ones, ints):
    for a_mn in (False, True):
        for b_mn in (False, True):
            run(128, 128, 32, a_mn, b_mn, 1, gen)
run(128, 128, 64, False, True, 1, ints)
run(256, 256, 256, False, True, 1, ints)
