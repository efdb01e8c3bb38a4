"""tcgen05 shifted-GEMM kernel vs fp64 references (GPU).

Tolerances (normwise: max|a-b| / max|ref|): 3xTF32 is fp32-accurate (<1e-5 on
these sizes); single-pass TF32 keeps 10 mantissa bits (<4e-3)."""

import pytest
import torch
import torch.nn.functional as F

from paper_1811_01532_b200 import kernels as K

pytestmark = pytest.mark.gpu

TOL = {1: 4e-3, 3: 1e-5}


def dev(a, b):
    a = a.double()
    b = b.double()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("prec", [1, 3])
@pytest.mark.parametrize("M,Nn,Kk", [(256, 384, 512), (128, 1000, 4096), (200, 72, 96), (37, 4096, 9216)])
def test_fc_forward(cuda, prec, M, Nn, Kk):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, Kk, device=cuda, generator=g)
    w = torch.randn(Kk, Nn, device=cuda, generator=g)
    bias = torch.randn(Nn, device=cuda, generator=g)
    y = torch.empty(M, Nn, device=cuda)
    K.gemm(x, w, y, a_mn=False, b_mn=True, M=M, Nn=Nn, K=Kk, bias=bias, relu=True, precision=prec)
    torch.cuda.synchronize()
    ref = torch.relu(x.double() @ w.double() + bias.double())
    tol = TOL[prec]
    if prec == 3:
        # fp32-accurate means: no worse than a few times an fp32 CUDA-core GEMM
        torch.backends.cuda.matmul.allow_tf32 = False
        fp32_err = dev(torch.relu(x @ w + bias), ref)
        tol = max(tol, 4 * fp32_err)
    assert dev(y, ref) < tol


@pytest.mark.parametrize("prec", [1, 3])
@pytest.mark.parametrize("block_n", [64, 128, 256])
def test_fc_dx_kmajor(cuda, prec, block_n):
    if prec == 3 and block_n == 256:
        pytest.skip("BN=256 is TF32-only")
    g = torch.Generator(device="cuda").manual_seed(1)
    M, Nin, Nout = 128, 512, 320
    dy = torch.randn(M, Nout, device=cuda, generator=g)
    w = torch.randn(Nin, Nout, device=cuda, generator=g)
    dx = torch.empty(M, Nin, device=cuda)
    K.gemm(dy, w, dx, a_mn=False, b_mn=False, M=M, Nn=Nin, K=Nout, precision=prec, block_n=block_n)
    torch.cuda.synchronize()
    assert dev(dx, dy.double() @ w.double().T) < TOL[prec]


@pytest.mark.parametrize("prec", [1, 3])
@pytest.mark.parametrize("splits", [1, 3])
def test_fc_dw_mnmajor(cuda, prec, splits):
    g = torch.Generator(device="cuda").manual_seed(2)
    Bt, Nin, Nout = 256, 384, 256
    x = torch.randn(Bt, Nin, device=cuda, generator=g)
    dy = torch.randn(Bt, Nout, device=cuda, generator=g)
    dw = torch.empty(Nin, Nout, device=cuda)
    K.gemm(x, dy, dw, a_mn=True, b_mn=True, M=Nin, Nn=Nout, K=Bt, precision=prec, splits=splits)
    torch.cuda.synchronize()
    assert dev(dw, x.double().T @ dy.double()) < TOL[prec]


def _pad(x, p):
    # trailing halo: p zero columns after each row, p zero rows after each image
    return F.pad(x, (0, 0, 0, p, 0, p)).contiguous()


@pytest.mark.parametrize("prec", [1, 3])
@pytest.mark.parametrize("Bn,H,Ci,Co,k", [(2, 13, 64, 128, 3), (2, 27, 64, 192, 5), (1, 14, 96, 64, 3)])
def test_conv_shifted(cuda, prec, Bn, H, Ci, Co, k):
    W = H
    p = k // 2
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.relu(torch.randn(Bn, H, W, Ci, device=cuda, generator=g))
    w = torch.randn(k, k, Ci, Co, device=cuda, generator=g) * 0.1
    bias = torch.randn(Co, device=cuda, generator=g)
    xp = _pad(x, p)
    yp = torch.full((Bn, H + p, W + p, Co), float("nan"), device=cuda)
    K.conv_fprop(xp, w, yp, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, bias=bias, relu=True, precision=prec)
    torch.cuda.synchronize()
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(3, 2, 0, 1), bias.double(), padding=p)
    ref = torch.relu(ref).permute(0, 2, 3, 1)
    assert dev(yp[:, :H, :W], ref) < TOL[prec]
    assert yp[:, H:].abs().max().item() == 0 and yp[:, :, W:].abs().max().item() == 0

    # dgrad with a fused ReLU mask, and wgrad
    dy = torch.randn(Bn, H, W, Co, device=cuda, generator=g)
    dyp = _pad(dy, p)
    dxp = torch.full_like(xp, float("nan"))
    K.conv_dgrad(dyp, w, dxp, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, mask=xp, precision=prec)
    dw = torch.empty_like(w)
    K.conv_wgrad(xp, dyp, dw, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, precision=prec)
    torch.cuda.synchronize()
    xd = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wd = w.double().permute(3, 2, 0, 1).detach().requires_grad_(True)
    out = F.conv2d(xd, wd, padding=p)
    out.backward(dy.double().permute(0, 3, 1, 2))
    ref_dx = (xd.grad * (xd > 0)).permute(0, 2, 3, 1)
    ref_dw = wd.grad.permute(2, 3, 1, 0)
    assert dev(dxp[:, :H, :W], ref_dx) < TOL[prec]
    assert dxp[:, H:].abs().max().item() == 0 and dxp[:, :, W:].abs().max().item() == 0
    assert dev(dw, ref_dw) < TOL[prec]


def _pack_bits(v):
    """[rows, n] bool -> [rows, ceil(n/32)] int32 words, bit j = column 32*w + j."""
    rows, n = v.shape
    ldw = (n + 31) // 32
    vb = torch.zeros(rows, ldw * 32, dtype=torch.int64, device=v.device)
    vb[:, :n] = v.to(torch.int64)
    words = (vb.view(rows, ldw, 32) << torch.arange(32, device=v.device)).sum(-1)
    return torch.where(words >= 2**31, words - 2**32, words).to(torch.int32)


@pytest.mark.parametrize("splits", [0, 2, 3])
@pytest.mark.parametrize("Co", [96, 72])
def test_conv_mask_bits_splitk(cuda, splits, Co):
    """ReLU mask bits published by a conv fprop and consumed by a dgrad, through the
    fused TMA-store epilogue (splits=0) and the split-K reduction (explicit splits)."""
    Bn, H, Ci, k = 2, 13, 64, 3
    W, p = H, 1
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(Bn, H, W, Ci, device=cuda, generator=g)
    w = torch.randn(k, k, Ci, Co, device=cuda, generator=g) * 0.1
    bias = torch.randn(Co, device=cuda, generator=g)
    xp = _pad(x, p)
    rows = Bn * (H + p) * (W + p)
    yp = torch.full((Bn, H + p, W + p, Co), float("nan"), device=cuda)
    bits = torch.full((rows, (Co + 31) // 32), -7, dtype=torch.int32, device=cuda)
    d = K.conv_fprop(xp, w, yp, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, bias=bias, relu=True,
                     run=False).desc
    d.mbits_out, d.mbits_out_ld, d.splits = bits.data_ptr(), bits.shape[1], splits
    d.workspace, d.workspace_bytes = None, 0
    K.GemmCall(d, device=cuda)()
    torch.cuda.synchronize()
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(3, 2, 0, 1), bias.double(), padding=p)
    assert dev(yp[:, :H, :W], torch.relu(ref).permute(0, 2, 3, 1)) < TOL[3]
    assert torch.equal(bits, _pack_bits(yp.reshape(rows, Co) > 0))

    if Co % 32:
        return  # a dgrad's K chunks must not straddle taps (tap_period = Co, multiple of 32)
    # dgrad of a conv whose input passed a ReLU: GradReLU from bits == from the float mask
    dy = torch.randn(Bn, H, W, Co, device=cuda, generator=g)
    dyp = _pad(dy, p)
    xbits = _pack_bits(xp.reshape(rows, Ci) > 0)
    dx_f = torch.full_like(xp, float("nan"))
    K.conv_dgrad(dyp, w, dx_f, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, mask=xp, splits=splits)
    dx_b = torch.full_like(xp, float("nan"))
    d = K.conv_dgrad(dyp, w, dx_b, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, splits=splits, run=False).desc
    d.mbits_in, d.mbits_in_ld = xbits.data_ptr(), xbits.shape[1]
    d.workspace, d.workspace_bytes = None, 0
    K.GemmCall(d, device=cuda)()
    torch.cuda.synchronize()
    if splits:  # same K slabs, same order: bitwise equal
        assert torch.equal(dx_b, dx_f)
    xd = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    F.conv2d(xd, w.double().permute(3, 2, 0, 1), padding=p).backward(dy.double().permute(0, 3, 1, 2))
    ref_dx = (xd.grad * (xd > 0)).permute(0, 2, 3, 1)
    assert dev(dx_b[:, :H, :W], ref_dx) < TOL[3] and dev(dx_f[:, :H, :W], ref_dx) < TOL[3]
    assert dx_b[:, H:].abs().max().item() == 0 and dx_b[:, :, W:].abs().max().item() == 0


@pytest.mark.parametrize("cluster", [1, 2])
@pytest.mark.parametrize("window", [0, -1])
def test_n64_pair_modes(cuda, cluster, window):
    """N = 64 3xTF32 GEMMs in every pair form: one CTA (PAIR: [B | B_small] as one N = 128 MMA)
    and a CTA pair (PAIR2: B_raw in CTA 0, B_small in CTA 1), with and without the halo
    window, for a conv fprop (B MN-major, Co = 64) and a dgrad (B K-major, Ci = 64), long
    enough in K to run several accumulator chains."""
    Bn, H, Ci, Co, k = 2, 27, 64, 64, 5
    p = k // 2
    W = H
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.relu(torch.randn(Bn, H, W, Ci, device=cuda, generator=g))
    w = torch.randn(k, k, Ci, Co, device=cuda, generator=g) * 0.1
    xp = _pad(x, p)

    def run(call):
        d = type(call.desc).from_buffer_copy(call.desc)
        d.cluster, d.window = cluster, window
        d.workspace, d.workspace_bytes = None, 0
        c = K.GemmCall(d)
        c()
        return c.info()

    yp = torch.full((Bn, H + p, W + p, Co), float("nan"), device=cuda)
    info = run(K.conv_fprop(xp, w, yp, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, precision=3, run=False))
    assert info["block_n"] == 64 and info["cta_group"] == cluster and info["pair"] == cluster
    dy = torch.randn(Bn, H, W, Co, device=cuda, generator=g)
    dyp = _pad(dy, p)
    dxp = torch.full_like(xp, float("nan"))
    run(K.conv_dgrad(dyp, w, dxp, B=Bn, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=p, precision=3, run=False))
    torch.cuda.synchronize()
    xd = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wd = w.double().permute(3, 2, 0, 1)
    out = F.conv2d(xd, wd, padding=p)
    out.backward(dy.double().permute(0, 3, 1, 2))
    assert dev(yp[:, :H, :W], out.detach().permute(0, 2, 3, 1)) < TOL[3]
    assert dev(dxp[:, :H, :W], xd.grad.permute(0, 2, 3, 1)) < TOL[3]
