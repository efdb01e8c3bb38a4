"""Print the worst deviations of one real-net parity case (tests/test_runtime_gpu.py)."""
import sys
sys.path.insert(0, "/root/repo")
from oracle import interp_ref as O
from paper_1811_01532_b200 import interp, ir, models
from tests.test_runtime_gpu import fanin_bindings, SEED

net, batch, image = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = models.MODELS[net](batch, image=image)
bind = fanin_bindings(g)
got = interp.execute(g, bind, SEED, precision=3)
ref = O.execute(g, bind, SEED)
worst = {}
for k in ref:
    if k.endswith("_upd"):
        v = k.replace("_upd", "")
        worst[k + "::grad"] = O.relative_deviation(bind[v] - got[k], bind[v] - ref[k])
    else:
        worst[k] = O.relative_deviation(got[k], ref[k])
for k, v in sorted(worst.items(), key=lambda x: -x[1])[:6]:
    print(f"{k:28s} {v:.3e}")
