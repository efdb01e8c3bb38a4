"""Check the GEMM epilogue's ReLU mask bits against (output > 0) of the same buffer."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_1811_01532_b200 import runtime, models
from tests.test_runtime_gpu import fanin_bindings

g = models.MODELS[sys.argv[1] if len(sys.argv) > 1 else "vgg16"](2, image=32)
bind = fanin_bindings(g)
prog = runtime.Program(g, precision=3)
prog.bind(bind)
prog.run()
torch.cuda.synchronize()
for rid, bits in prog.mask_bits.items():
    t = prog.t[rid]
    rows, ld = t.rows, t.ld
    y = t.buf[: rows * ld].view(rows, ld)[:, : t.dims[-1]].cpu().numpy()
    w = bits.view(rows, bits.ld_words).cpu().numpy().view(np.uint32)
    exp = np.zeros_like(w)
    for c in range(t.dims[-1]):
        exp[:, c // 32] |= ((y[:, c] > 0).astype(np.uint32) << np.uint32(c % 32))
    bad = np.nonzero(exp != w)
    print(rid, t.dims, "rows", rows, "mismatched words", len(bad[0]), "first rows", bad[0][:8])
