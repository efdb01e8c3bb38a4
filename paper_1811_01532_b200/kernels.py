"""Thin Python wrappers that build C-ABI descriptors for the sm_100a kernels.

Tensors here are torch CUDA tensors used purely as device buffers (torch is
plumbing: allocation and streams). Every function launches native kernels
through `_native`; nothing falls back to torch math.

Padded-flat NHWC layout (the layout every stride-1 convolution runs in):
an activation of logical shape [B, H, W, C] with halo p is stored as
[B, H+p, W+p, C]: p trailing zero columns after every image row and p zero
rows after every image. Viewed as a matrix [B*(H+p)*(W+p), C], filter tap
(u, v) of a same-padded KxK conv (K//2 <= p) is a constant row shift
(u-K//2)*(W+p) + (v-K//2); neighbours left of column 0 / above row 0 land in the
previous row's / image's trailing zeros, or before the buffer where the TMA
OOB fill reads zero. So Conv2D / GradConv2DX / GradConv2DW (interp.py:69-102)
become shifted GEMMs fed by 2D TMA with one trailing halo instead of two.
"""

from __future__ import annotations

import ctypes as C

from . import _native as N


def _desc(M, K, Nn, a, b, c, ldc, bias=None, relu=False, mask=None, ldm=0, halo=(0, 0, 0),
          precision=3, splits=0, block_n=0):
    d = N.wap_gemm_desc_t()
    d.M, d.N, d.K = M, Nn, K
    d.a, d.b = a, b
    d.c = N.ptr(c)
    d.ldc = ldc
    d.bias = N.ptr(bias)
    d.relu = 1 if relu else 0
    d.mask = N.ptr(mask)
    d.ldm = ldm
    d.halo_pad, d.halo_h, d.halo_w = halo
    d.precision = precision
    d.splits = splits
    d.block_n = block_n
    return d


class GemmCall:
    """A prepared GEMM launch; owns its split-K workspace."""

    def __init__(self, desc: N.wap_gemm_desc_t, device=None):
        import torch

        self.desc = desc
        L = N.lib()
        ws = L.wap_gemm_workspace_bytes(C.byref(desc))
        if ws < 0:
            raise ValueError("bad gemm descriptor")
        self.workspace = None
        if ws > 0:
            self.workspace = torch.empty(ws // 4, dtype=torch.float32, device=device or "cuda")
            desc.workspace = self.workspace.data_ptr()
            desc.workspace_bytes = ws
        self._plan = C.c_void_p()
        N.check(L.wap_gemm_plan_create(C.byref(desc), C.byref(self._plan)), "wap_gemm_plan_create")

    def __call__(self, stream=None):
        N.check(N.lib().wap_gemm_plan_run(self._plan, N.stream_ptr(stream)), "wap_gemm_plan_run")

    def info(self) -> dict:
        """The resolved launch configuration (wap_gemm_plan_info)."""
        out = (C.c_int64 * 8)()
        N.check(N.lib().wap_gemm_plan_info(self._plan, out), "wap_gemm_plan_info")
        return dict(zip(("block_n", "cta_group", "splits", "k_chunks_per_split", "window_boxes", "precision",
                         "pair", "chain"), (int(v) for v in out)))

    def numerics(self) -> tuple:
        """What fixes the fp32 rounding of the result: K split, precision, CTA group,
        N = 64 pair mode, halo window (it walks K tap-innermost, the plain plan
        tap-outermost), 3xTF32 accumulator chain length. Measured on B200: plans equal in these are bitwise equal
        (tests/test_determinism_gpu.py); BN does not enter."""
        i = self.info()
        return (i["splits"], i["k_chunks_per_split"] if i["splits"] > 1 else 0, i["precision"], i["cta_group"],
                i["pair"], int(i["window_boxes"] > 0), i["chain"])

    def __del__(self):
        try:
            if self._plan:
                N.lib().wap_gemm_plan_destroy(self._plan)
        except Exception:
            pass


def gemm(a, b, c, *, a_mn: bool, b_mn: bool, M: int, Nn: int, K: int, bias=None, relu=False,
         mask=None, precision=3, splits=0, block_n=0, stream=None, run=True):
    """C[M,N] = A[M,K] B[K,N] on 2D row-major operands.

    a_mn=False: `a` is [M, K] (K contiguous); a_mn=True: `a` is [K, M].
    b_mn=False: `b` is [N, K];                b_mn=True: `b` is [K, N].
    """
    lda = a.shape[-1]
    ldb = b.shape[-1]
    ao = N.operand(a, inner=(M if a_mn else K), outer=(K if a_mn else M), ld=lda, mn_major=a_mn)
    bo = N.operand(b, inner=(Nn if b_mn else K), outer=(K if b_mn else Nn), ld=ldb, mn_major=b_mn)
    d = _desc(M, K, Nn, ao, bo, c, c.shape[-1], bias=bias, relu=relu, mask=mask,
              ldm=(mask.shape[-1] if mask is not None else 0), precision=precision, splits=splits,
              block_n=block_n)
    call = GemmCall(d, device=c.device)
    if run:
        call(stream)
    return call


def tap_shifts(k: int, pad: int, wp: int) -> list[int]:
    """Row offsets of the k*k filter taps on a padded-flat grid of row width wp."""
    return [(u - pad) * wp + (v - pad) for u in range(k) for v in range(k)]


def conv_fprop(xp, w, y, *, B, H, W, Ci, Co, k, pad, bias=None, relu=False, precision=3,
               run=True, stream=None):
    """y_pad = conv(x_pad, w) (+bias, ReLU) on the padded-flat grid; halo rows written 0.

    xp: [B, H+p, W+p, Ci] (p trailing zero columns / rows); w: [k, k, Ci, Co] (KKIO);
    y: [B, H+p, W+p, Co]."""
    hp, wp = H + pad, W + pad
    rows = B * hp * wp
    ao = N.operand(xp, inner=Ci, outer=rows, ld=Ci, mn_major=False, tap_period=Ci,
                   offsets=tuple(tap_shifts(k, pad, wp)))
    bo = N.operand(w, inner=Co, outer=k * k * Ci, ld=Co, mn_major=True)
    d = _desc(rows, k * k * Ci, Co, ao, bo, y, Co, bias=bias, relu=relu, halo=(pad, H, W),
              precision=precision)
    call = GemmCall(d, device=y.device)
    if run:
        call(stream)
    return call


def conv_dgrad(dyp, w, dxp, *, B, H, W, Ci, Co, k, pad, mask=None, precision=3, splits=0, run=True,
               stream=None):
    """dx_pad = GradConv2DX(dy_pad, w) (* [mask > 0]); dy halo must be zero."""
    hp, wp = H + pad, W + pad
    rows = B * hp * wp
    shifts = tap_shifts(k, pad, wp)
    ao = N.operand(dyp, inner=Co, outer=rows, ld=Co, mn_major=False, tap_period=Co,
                   offsets=tuple(-s for s in shifts))
    bo = N.operand(w, inner=Co, outer=k * k * Ci, ld=Co, mn_major=False, tap_period=Co,
                   offsets=tuple(t * Ci for t in range(k * k)))
    d = _desc(rows, k * k * Co, Ci, ao, bo, dxp, Ci, mask=mask, ldm=(Ci if mask is not None else 0),
              halo=(pad, H, W), precision=precision, splits=splits)
    call = GemmCall(d, device=dxp.device)
    if run:
        call(stream)
    return call


def conv_wgrad(xp, dyp, dw, *, B, H, W, Ci, Co, k, pad, precision=3, splits=0, run=True,
               stream=None):
    """dw[k,k,Ci,Co] = GradConv2DW(x_pad, dy_pad); dy halo must be zero."""
    hp, wp = H + pad, W + pad
    rows = B * hp * wp
    ao = N.operand(xp, inner=Ci, outer=rows, ld=Ci, mn_major=True, tap_period=Ci,
                   offsets=tuple(tap_shifts(k, pad, wp)))
    bo = N.operand(dyp, inner=Co, outer=rows, ld=Co, mn_major=True)
    d = _desc(k * k * Ci, rows, Co, ao, bo, dw, Co, precision=precision, splits=splits)
    call = GemmCall(d, device=dw.device)
    if run:
        call(stream)
    return call
