"""HBM-bound op kernels through the C ABI vs torch fp64 (GPU).

MaxPool backward (interp rules in oracle/interp_ref.py; first-max ties): the
stride-2 patch kernel must equal the per-pixel gather kernel bit for bit (same
window order) and torch's max_pool2d backward on tie-free data."""

import os

import pytest
import torch
import torch.nn.functional as F

from paper_1811_01532_b200 import _native as N

pytestmark = pytest.mark.gpu


def _buf(B, H, W, ld, pad, cuda, fill=float("nan")):
    return torch.full((B, H + pad, W + pad, ld), fill, device=cuda)


def _pool_bwd(L, arg, dy, yl, win, s, dx, xl, mask, ml, pixel: bool):
    if pixel:
        os.environ["WAP_POOL_BWD_PIXEL"] = "1"
    try:
        N.check(L.wap_maxpool_bwd(arg.data_ptr(), dy.data_ptr(), yl, win, s, dx.data_ptr(), xl,
                                  mask.data_ptr() if mask is not None else None, ml, None))
    finally:
        os.environ.pop("WAP_POOL_BWD_PIXEL", None)


@pytest.mark.parametrize("B,H,C,ld,win,pad,use_mask", [
    (2, 55, 64, 64, 3, 0, False),   # AlexNet pool1
    (2, 27, 192, 192, 3, 2, True),  # AlexNet pool2 (trailing halo on the input), float mask
    (3, 13, 6, 8, 3, 1, False),     # padded channel lanes
    (2, 56, 64, 64, 3, 0, False),   # last input row in no window
    (2, 28, 128, 128, 2, 1, False),  # VGG 2/2
    (1, 15, 4, 4, 2, 0, True),      # odd extent: last row / column uncovered
])
def test_maxpool_bwd_patch_matches_gather_and_torch(cuda, B, H, C, ld, win, pad, use_mask):
    L = N.lib()
    W, s = H, 2
    Ho = (H - win) // s + 1
    g = torch.Generator(device="cuda").manual_seed(11)
    x = _buf(B, H, W, ld, pad, cuda, 0.0)
    x[:, :H, :W, :C] = torch.randn(B, H, W, C, device=cuda, generator=g)
    xl = N.wap_layout_t(B, H, W, C, pad, ld)
    yl = N.wap_layout_t(B, Ho, Ho, C, 0, ld)
    y = _buf(B, Ho, Ho, ld, 0, cuda)
    arg = torch.zeros(B * Ho * Ho * ld, dtype=torch.uint8, device=cuda)
    N.check(L.wap_maxpool_fwd_ex(x.data_ptr(), xl, win, s, y.data_ptr(), yl, arg.data_ptr(), 0, None))
    dy = _buf(B, Ho, Ho, ld, 0, cuda, 0.0)
    dy[..., :C] = torch.randn(B, Ho, Ho, C, device=cuda, generator=g)
    mask = ml = None
    ml = xl
    if use_mask:
        mask = torch.randn(x.shape, device=cuda, generator=g)
    dx_patch = _buf(B, H, W, ld, pad, cuda)
    dx_pix = _buf(B, H, W, ld, pad, cuda)
    _pool_bwd(L, arg, dy, yl, win, s, dx_patch, xl, mask, ml, pixel=False)
    _pool_bwd(L, arg, dy, yl, win, s, dx_pix, xl, mask, ml, pixel=True)
    torch.cuda.synchronize()
    assert torch.equal(dx_patch[:, :H, :W], dx_pix[:, :H, :W])
    # halo rows / columns are never written
    if pad:
        assert torch.isnan(dx_patch[:, H:]).all() and torch.isnan(dx_patch[:, :, W:]).all()
    xd = x[:, :H, :W, :C].double().permute(0, 3, 1, 2).requires_grad_(True)
    F.max_pool2d(xd, win, s).backward(dy[..., :C].double().permute(0, 3, 1, 2))
    ref = xd.grad.permute(0, 2, 3, 1)
    if use_mask:
        ref = ref * (mask[:, :H, :W, :C] > 0)
    got = dx_patch[:, :H, :W, :C].double()
    assert (got - ref).abs().max().item() < 1e-6
    assert (dx_patch[:, :H, :W, C:] == 0).all()


@pytest.mark.parametrize("B,H,W,pad", [(3, 224, 224, 0), (2, 8, 12, 2), (2, 7, 9, 0)])
def test_pack_images_c3(cuda, B, H, W, pad):
    """wap_pack of dense NHWC C=3 images into the ld=4 layout (fast 4-pixel path when
    W % 4 == 0, generic otherwise): exact copy, padding lane 0, halo untouched."""
    L = N.lib()
    src = torch.randn(B, H, W, 3, device=cuda)
    dst = torch.full((B, H + pad, W + pad, 4), float("nan"), device=cuda)
    dst[..., 3] = 0.0
    N.check(L.wap_pack(src.data_ptr(), N.wap_layout_t(B, H, W, 3, pad, 4), dst.data_ptr(), 0, None))
    torch.cuda.synchronize()
    assert torch.equal(dst[:, :H, :W, :3], src)
    assert (dst[:, :H, :W, 3] == 0).all()
    if pad:
        assert torch.isnan(dst[:, H:, :, :3]).all() and torch.isnan(dst[:, :, W:, :3]).all()


@pytest.mark.parametrize("B,H,C,win,pad,relu_mask", [
    (2, 55, 64, 3, 2, True),    # AlexNet conv1 -> ReLU -> norm1 -> pool1 (mask = LRN input)
    (2, 27, 192, 3, 0, True),   # conv2 -> ReLU -> norm2 -> pool2
    (1, 13, 64, 3, 1, False),   # no GradReLU
    (2, 16, 192, 2, 0, False),  # window 2
])
def test_maxpool_lrn_bwd_fused_matches_unfused(cuda, B, H, C, win, pad, relu_mask):
    """wap_maxpool_lrn_bwd == wap_maxpool_bwd followed by wap_lrn_bwd (same floats)."""
    L = N.lib()
    W, s = H, 2
    Ho = (H - win) // s + 1
    a, beta, k = 1e-4, 0.75, 2.0
    g = torch.Generator(device="cuda").manual_seed(21)
    x = torch.zeros(B, H + pad, W + pad, C, device=cuda)
    x[:, :H, :W] = torch.randn(B, H, W, C, device=cuda, generator=g) * 3
    xl = N.wap_layout_t(B, H, W, C, pad, C)
    y = torch.zeros_like(x)
    N.check(L.wap_lrn_fwd(x.data_ptr(), xl, 5, a, beta, k, y.data_ptr(), xl, None))
    yl = N.wap_layout_t(B, Ho, Ho, C, 0, C)
    yp = torch.zeros(B, Ho, Ho, C, device=cuda)
    arg = torch.zeros(B * Ho * Ho * C, dtype=torch.uint8, device=cuda)
    N.check(L.wap_maxpool_fwd_ex(y.data_ptr(), xl, win, s, yp.data_ptr(), yl, arg.data_ptr(), 0, None))
    dy = torch.randn(B, Ho, Ho, C, device=cuda, generator=g)
    mask = x if relu_mask else None
    mptr = mask.data_ptr() if mask is not None else None
    # unfused: pool gradient tensor, then LRN backward
    dpool = torch.zeros_like(x)
    N.check(L.wap_maxpool_bwd(arg.data_ptr(), dy.data_ptr(), yl, win, s, dpool.data_ptr(), xl, None, xl, None))
    ref = torch.full_like(x, float("nan"))
    N.check(L.wap_lrn_bwd(x.data_ptr(), xl, dpool.data_ptr(), xl, 5, a, beta, k, ref.data_ptr(), xl, mptr, xl,
                          None))
    got = torch.full_like(x, float("nan"))
    N.check(L.wap_maxpool_lrn_bwd(arg.data_ptr(), dy.data_ptr(), yl, win, s, x.data_ptr(), xl, 5, a, beta, k,
                                  got.data_ptr(), xl, mptr, xl, None))
    torch.cuda.synchronize()
    r, o = ref[:, :H, :W], got[:, :H, :W]
    assert not torch.isnan(o).any()
    assert ((r - o).abs().max() / r.abs().max()).item() < 1e-6
    if pad:
        assert torch.isnan(got[:, H:]).all() and torch.isnan(got[:, :, W:]).all()


def _lrn_ref(x, size, alpha, beta, k):
    """LRN across channels, NHWC fp64 (oracle/interp_ref.py rule)."""
    x = x.double()
    sq = F.pad(x * x, (size // 2, size // 2))
    s = sum(sq[..., i:i + x.shape[-1]] for i in range(size))
    return x * (k + alpha * s) ** (-beta)


@pytest.mark.parametrize("B,H,C,pad", [(2, 55, 64, 2), (3, 27, 192, 0), (1, 7, 64, 0)])
def test_lrn_fwd_vs_torch(cuda, B, H, C, pad):
    L = N.lib()
    a, beta, k = 1e-4, 0.75, 2.0
    g = torch.Generator(device="cuda").manual_seed(31)
    x = torch.zeros(B, H + pad, H + pad, C, device=cuda)
    x[:, :H, :H] = torch.randn(B, H, H, C, device=cuda, generator=g) * 4
    xl = N.wap_layout_t(B, H, H, C, pad, C)
    y = torch.full_like(x, float("nan"))
    N.check(L.wap_lrn_fwd(x.data_ptr(), xl, 5, a, beta, k, y.data_ptr(), xl, None))
    torch.cuda.synchronize()
    ref = _lrn_ref(x[:, :H, :H], 5, a, beta, k)
    assert ((y[:, :H, :H].double() - ref).abs().max() / ref.abs().max()).item() < 2e-6
    if pad:
        assert torch.isnan(y[:, H:]).all()


@pytest.mark.parametrize("B,H,W,pad", [(2, 224, 224, 1), (1, 9, 7, 1), (2, 5, 6, 0)])
def test_conv_direct_3x3_c3(cuda, B, H, W, pad):
    """VGG-16 conv1_1 direct conv (wap_conv_direct, 3x3 same, C=3): the two-pixel kernel
    equals the one-pixel kernel bit for bit (outputs and ReLU mask bits) and torch fp64."""
    L = N.lib()
    Co = 64
    g = torch.Generator(device="cuda").manual_seed(41)
    x = torch.zeros(B, H, W, 4, device=cuda)
    x[..., :3] = torch.randn(B, H, W, 3, device=cuda, generator=g)
    w = torch.randn(27, Co, device=cuda, generator=g) * 0.2
    bias = torch.randn(Co, device=cuda, generator=g) * 0.1
    xl = N.wap_layout_t(B, H, W, 3, 0, 4)
    yl = N.wap_layout_t(B, H, W, Co, pad, Co)
    rows = B * (H + pad) * (W + pad)
    outs = []
    for px1 in (False, True):
        if px1:
            os.environ["WAP_CONV_DIRECT_PX1"] = "1"
        try:
            y = torch.full((B, H + pad, W + pad, Co), float("nan"), device=cuda)
            bits = torch.zeros(rows, Co // 32, dtype=torch.int32, device=cuda)
            N.check(L.wap_conv_direct(x.data_ptr(), xl, w.data_ptr(), 3, 1, Co, bias.data_ptr(), 1, y.data_ptr(),
                                      yl, bits.data_ptr(), Co // 32, None))
            torch.cuda.synchronize()
        finally:
            os.environ.pop("WAP_CONV_DIRECT_PX1", None)
        outs.append((y, bits))
    (y2, b2), (y1, b1) = outs
    assert torch.equal(y2[:, :H, :W], y1[:, :H, :W]) and torch.equal(b2, b1)
    ref = F.conv2d(x[..., :3].double().permute(0, 3, 1, 2), w.double().view(3, 3, 3, Co).permute(3, 2, 0, 1),
                   bias.double(), padding=1).relu().permute(0, 2, 3, 1)
    assert ((y2[:, :H, :W].double() - ref).abs().max() / ref.abs().max()).item() < 1e-6
    if pad:
        assert torch.isnan(y2[:, H:]).all() and torch.isnan(y2[:, :, W:]).all()


@pytest.mark.parametrize("B,H,C,win,pad", [(2, 55, 64, 3, 2), (2, 27, 192, 3, 0), (1, 16, 64, 2, 1)])
def test_lrn_maxpool_fwd_fused_matches_unfused(cuda, B, H, C, win, pad):
    """wap_lrn_maxpool_fwd == wap_lrn_fwd followed by wap_maxpool_fwd: pooled values and
    argmax bit for bit."""
    L = N.lib()
    a, beta, k, s = 1e-4, 0.75, 2.0, 2
    Ho = (H - win) // s + 1
    g = torch.Generator(device="cuda").manual_seed(51)
    x = torch.zeros(B, H + pad, H + pad, C, device=cuda)
    x[:, :H, :H] = torch.relu(torch.randn(B, H, H, C, device=cuda, generator=g) * 3)
    xl = N.wap_layout_t(B, H, H, C, pad, C)
    yl = N.wap_layout_t(B, Ho, Ho, C, 0, C)
    t = torch.zeros_like(x)
    N.check(L.wap_lrn_fwd(x.data_ptr(), xl, 5, a, beta, k, t.data_ptr(), xl, None))
    y1 = torch.full((B, Ho, Ho, C), float("nan"), device=cuda)
    a1 = torch.zeros(B * Ho * Ho * C, dtype=torch.uint8, device=cuda)
    N.check(L.wap_maxpool_fwd_ex(t.data_ptr(), xl, win, s, y1.data_ptr(), yl, a1.data_ptr(), 0, None))
    y2 = torch.full_like(y1, float("nan"))
    a2 = torch.full_like(a1, 77)
    N.check(L.wap_lrn_maxpool_fwd(x.data_ptr(), xl, 5, a, beta, k, win, s, y2.data_ptr(), yl, a2.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(a1, a2)


@pytest.mark.parametrize("B,H,W,pad", [(2, 33, 30, 1), (3, 9, 17, 2), (1, 6, 5, 0)])
def test_conv_wgrad_direct_3x3_c3(cuda, B, H, W, pad):
    """First-layer direct weight gradient (wap_conv_wgrad_direct: 3x3 same, C=3, dy on a
    padded grid with a trailing halo) against torch fp64, and run-to-run bitwise equal."""
    L = N.lib()
    Co = 64
    g = torch.Generator(device="cuda").manual_seed(43)
    x = torch.zeros(B, H, W, 4, device=cuda)
    x[..., :3] = torch.randn(B, H, W, 3, device=cuda, generator=g)
    dy = torch.zeros(B, H + pad, W + pad, Co, device=cuda)
    dy[:, :H, :W] = torch.randn(B, H, W, Co, device=cuda, generator=g)
    xl = N.wap_layout_t(B, H, W, 3, 0, 4)
    dl = N.wap_layout_t(B, H, W, Co, pad, Co)
    work = torch.empty(int(L.wap_conv_wgrad_direct_work_floats(dl)), device=cuda)
    outs = []
    for _ in range(2):
        dw = torch.full((27, Co), float("nan"), device=cuda)
        N.check(L.wap_conv_wgrad_direct(x.data_ptr(), xl, dy.data_ptr(), dl, 3, 1, dw.data_ptr(), Co,
                                        work.data_ptr(), None))
        torch.cuda.synchronize()
        outs.append(dw)
    assert torch.equal(outs[0], outs[1])
    xd = x[..., :3].double().permute(0, 3, 1, 2)
    ref = torch.nn.grad.conv2d_weight(xd, (Co, 3, 3, 3), dy[:, :H, :W].double().permute(0, 3, 1, 2), padding=1)
    ref = ref.permute(2, 3, 1, 0).reshape(27, Co)
    assert ((outs[0].double() - ref).abs().max() / ref.abs().max()).item() < 1e-6
