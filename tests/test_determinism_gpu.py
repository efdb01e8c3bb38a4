"""Results never depend on the run (SPEC.md:486 determinism).

1. Launch configurations of one GEMM descriptor that share a numerics signature
   (wap_gemm_plan_info: K split + partition, precision, CTA group, N = 64 pair
   mode, halo window) give bitwise-equal outputs, whatever their BN. The autotuner
   only picks among those (plan_cache.py), so tuning cannot change bits.
2. Two freshly built Programs of the same training graph, each autotuned from
   scratch (plan file disabled), produce byte-identical outputs.
3. Same with the committed plan file (the default path)."""

import itertools

import numpy as np
import pytest
import torch

from paper_1811_01532_b200 import interp, kernels as K, models

from .test_trainer_gpu import _bindings

pytestmark = pytest.mark.gpu


def _variants(call, clusters=(1, 2), windows=(0, -1), bns=(0, 128), splits=(0,)):
    out = []
    for c, w, bn, sp in itertools.product(clusters, windows, bns, splits):
        d = type(call.desc).from_buffer_copy(call.desc)
        d.cluster, d.window, d.block_n = c, w, bn
        if sp:
            d.splits = sp
        d.workspace, d.workspace_bytes = None, 0
        try:
            out.append(((c, w, bn, sp), K.GemmCall(d)))
        except Exception:
            continue
    return out


def _check_groups(variants, result):
    groups: dict = {}
    for cfg, call in variants:
        call()
        torch.cuda.synchronize()
        groups.setdefault(call.numerics(), []).append((cfg, result().clone()))
    assert groups
    bad = []
    for sig, outs in groups.items():
        ref_cfg, ref = outs[0]
        for cfg, o in outs[1:]:
            if not torch.equal(o, ref):
                bad.append((sig, ref_cfg, cfg, (o - ref).abs().max().item()))
    assert not bad, bad
    return groups


@pytest.mark.parametrize("B,H,Ci,Co,k,pad", [
    (2, 13, 192, 384, 3, 1),   # AlexNet conv3 shape class
    (1, 27, 64, 192, 5, 2),    # AlexNet conv2 (5x5 taps, halo window)
    (1, 28, 64, 64, 3, 1),     # N = 64: pair mode vs CTA pair
])
def test_conv_fprop_dgrad_variants_bitwise(cuda, B, H, Ci, Co, k, pad):
    g = torch.Generator(device="cuda").manual_seed(3)
    W = H
    xp = torch.zeros(B, H + pad, W + pad, Ci, device=cuda)
    xp[:, :H, :W] = torch.randn(B, H, W, Ci, device=cuda, generator=g)
    w = torch.randn(k, k, Ci, Co, device=cuda, generator=g) / (k * k * Ci) ** 0.5
    y = torch.zeros(B, H + pad, W + pad, Co, device=cuda)
    call = K.conv_fprop(xp, w, y, B=B, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=pad, run=False)
    groups = _check_groups(_variants(call), lambda: y)
    # dgrad with the transposed taps
    dy = torch.zeros_like(y)
    dy[:, :H, :W] = torch.randn(B, H, W, Co, device=cuda, generator=g)
    dx = torch.zeros_like(xp)
    call = K.conv_dgrad(dy, w, dx, B=B, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=pad, run=False)
    _check_groups(_variants(call), lambda: dx)
    assert sum(len(v) for v in groups.values()) >= 2


@pytest.mark.parametrize("B,H,Ci,Co,k,pad,splits", [(2, 13, 192, 384, 3, 1, (0, 3)), (2, 27, 64, 192, 5, 2, (0, 4))])
def test_conv_wgrad_variants_bitwise(cuda, B, H, Ci, Co, k, pad, splits):
    g = torch.Generator(device="cuda").manual_seed(4)
    W = H
    xp = torch.zeros(B, H + pad, W + pad, Ci, device=cuda)
    xp[:, :H, :W] = torch.randn(B, H, W, Ci, device=cuda, generator=g)
    dy = torch.zeros(B, H + pad, W + pad, Co, device=cuda)
    dy[:, :H, :W] = torch.randn(B, H, W, Co, device=cuda, generator=g)
    dw = torch.zeros(k * k * Ci, Co, device=cuda)
    call = K.conv_wgrad(xp, dy, dw, B=B, H=H, W=W, Ci=Ci, Co=Co, k=k, pad=pad, run=False)
    groups = _check_groups(_variants(call, windows=(0,), splits=splits), lambda: dw)
    assert len(groups) >= 2  # different K partitions really are different signatures


def test_fc_variants_bitwise(cuda):
    g = torch.Generator(device="cuda").manual_seed(5)
    M, Nn, Kk = 128, 4096, 9216
    x = torch.randn(M, Kk, device=cuda, generator=g)
    w = torch.randn(Kk, Nn, device=cuda, generator=g) / Kk ** 0.5
    y = torch.empty(M, Nn, device=cuda)
    call = K.gemm(x, w, y, a_mn=False, b_mn=True, M=M, Nn=Nn, K=Kk, relu=True, run=False)
    _check_groups(_variants(call, clusters=(1,), windows=(0,), bns=(0, 128), splits=(0, 9, 18)), lambda: y)


def _fresh_outputs(net, kw, seed=5):
    interp._PROGRAMS.clear()
    g = models.MODELS[net](**kw)
    bind = {k: v.astype(np.float64) for k, v in _bindings(g, seed).items()}
    out = interp.execute(g, bind, 0)
    interp._PROGRAMS.clear()
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("plan_file", ["0", "1"])
@pytest.mark.parametrize("net,kw", [("alexnet", {"batch": 8, "image": 99}), ("vgg16", {"batch": 2, "image": 64})])
def test_fresh_programs_byte_identical(cuda, monkeypatch, plan_file, net, kw):
    monkeypatch.setenv("WAP_AUTOTUNE", "1")
    monkeypatch.setenv("WAP_PLAN_CACHE", plan_file)
    a = _fresh_outputs(net, kw)
    b = _fresh_outputs(net, kw)
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
