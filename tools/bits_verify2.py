"""Compare the GradReLU-masked dgrad outputs of a Program with and without mask bits."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_1811_01532_b200 import runtime, models
from tests.test_runtime_gpu import fanin_bindings

g = models.MODELS["vgg16"](2, image=32)
bind = fanin_bindings(g)
os.environ["WAP_NO_MASK_BITS"] = "1"
os.environ["WAP_AUTOTUNE"] = "0"
pa = runtime.Program(g, precision=3)
del os.environ["WAP_NO_MASK_BITS"]
pb = runtime.Program(g, precision=3)
for p in (pa, pb):
    p.bind(bind)
    p.run()
torch.cuda.synchronize()
from paper_1811_01532_b200.ir import OpKind
print("grad-relu nodes:", [n for n in pb.order if pb.kind(n) is OpKind.GRAD_RELU][:20])
for nid in pb.order:
    if pb.kind(nid) is OpKind.GRAD_RELU and nid in pa.t and nid in pb.t:
        a = pa.fetch(nid); b = pb.fetch(nid)
        d = np.abs(a - b)
        idx = np.argwhere(d > 1e-6 * (np.abs(a).max() + 1e-30))
        print(nid, a.shape, "max|diff|", d.max(), "n bad", len(idx), idx[:5].tolist())
