"""A/B timing of wap_conv_direct (VGG-16 conv1_1 at b=32): two-pixel vs one-pixel kernel."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1811_01532_b200 import _native as N  # noqa: E402

L = N.lib()
B, H, W, Co = 32, 224, 224, 64
x = torch.randn(B, H, W, 4, device="cuda")
w = torch.randn(27, Co, device="cuda")
bias = torch.randn(Co, device="cuda")
y = torch.empty(B, H + 1, W + 1, Co, device="cuda")
bits = torch.empty(B * (H + 1) * (W + 1) * 2, dtype=torch.int32, device="cuda")
xl, yl = N.wap_layout_t(B, H, W, 3, 0, 4), N.wap_layout_t(B, H, W, Co, 1, Co)
for px1 in (False, True):
    if px1:
        os.environ["WAP_CONV_DIRECT_PX1"] = "1"
    call = lambda: L.wap_conv_direct(x.data_ptr(), xl, w.data_ptr(), 3, 1, Co, bias.data_ptr(), 1,  # noqa: E731
                                     y.data_ptr(), yl, bits.data_ptr(), 2, None)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"{'one-pixel' if px1 else 'two-pixel'}: {e0.elapsed_time(e1) / 20:.4f} ms")
