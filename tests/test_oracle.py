"""Pin the CPU oracle before trusting it (CPU only).

1. oracle vs the reference's own outputs frozen in tests/golden (runs anywhere);
2. oracle vs the live reference interpreter on extra graphs / single ops
   (build container only);
3. extension rules (strided conv, MaxPool, LRN) vs torch fp64 autograd;
4. the host planner reproduces the reference planner's decisions and every
   float bit for bit on the real 224x224 AlexNet / VGG-16 sweep."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import interp_ref as O
from paper_1811_01532_b200 import graph_modifier as gm
from paper_1811_01532_b200 import ir, models, planner, workloads

from .conftest import have_reference
from .golden_util import SEED, cases, deviation_vs_golden, expected, planner_cases


def _graph(model, batch, d):
    g = models.MODELS[model](batch)
    if d > 1:
        g = gm.transform(g, planner.ParallelPlan(d, tuple(range(d)), (), 0.0))[0]
    return g


@pytest.mark.parametrize("model,batch,d", cases())
def test_oracle_matches_reference_golden(model, batch, d):
    g = _graph(model, batch, d)
    inputs = O.generate_inputs(models.MODELS[model](batch), SEED)
    out = O.execute(g, inputs, SEED)
    exp = expected(model, batch, d)
    assert exp, "fixture empty"
    for name, gold in exp.items():
        assert deviation_vs_golden(out[name], gold) < 1e-11, name


@pytest.mark.skipif(not have_reference(), reason="reference checkout not present")
@pytest.mark.parametrize("seed", [0, 7])
def test_oracle_matches_live_reference(ref_wap, seed):
    from importlib import import_module

    tf = import_module("wap.transform")
    g = import_module("wap.models").mlp(32, (20, 12, 8, 6))
    for d in (1, 2, 4):
        gg = g if d == 1 else tf.transform(g, ref_wap.ParallelPlan(d, tuple(range(d)), (), 0.0))[0]
        inputs = ref_wap.generate_inputs(gg, seed)
        a = ref_wap.execute(gg, inputs, seed)
        b = O.execute(gg, inputs, seed)
        for k in a:
            assert O.relative_deviation(a[k], b[k]) < 1e-13, k


@pytest.mark.skipif(not have_reference(), reason="reference checkout not present")
def test_conv_rules_bitwise_equal_reference(ref_wap):
    from importlib import import_module

    ri = import_module("wap.interp")
    rs = np.random.default_rng(3)
    x = rs.standard_normal((2, 7, 7, 5))
    for k in (1, 3, 5):
        w = rs.standard_normal((k, k, 5, 6))
        dy = rs.standard_normal((2, 7, 7, 6))
        assert np.array_equal(O.conv2d(x, w), ri._conv2d(x, w))
        assert np.array_equal(O.conv2d_grad_w(x, dy, k), ri._conv2d_grad_w(x, dy, k))
        assert np.array_equal(O.conv2d_grad_x(dy, w), ri._conv2d_grad_x(dy, w))


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a))


@pytest.mark.parametrize("k,s,p,h", [(11, 4, 2, 35), (3, 1, 1, 9), (5, 2, 1, 12), (3, 2, 0, 9)])
def test_strided_conv_vs_torch(k, s, p, h):
    rs = np.random.default_rng(k * 10 + s)
    x = rs.standard_normal((2, h, h, 3))
    w = rs.standard_normal((k, k, 3, 4))
    y = O.conv2d(x, w, s, p)
    xt = _t(x).permute(0, 3, 1, 2).requires_grad_(True)
    wt = _t(w).permute(3, 2, 0, 1).detach().requires_grad_(True)
    yt = F.conv2d(xt, wt, stride=s, padding=p)
    assert np.allclose(y, yt.permute(0, 2, 3, 1).detach().numpy(), rtol=1e-12, atol=1e-12)
    dy = rs.standard_normal(y.shape)
    yt.backward(_t(dy).permute(0, 3, 1, 2))
    assert np.allclose(O.conv2d_grad_w(x, dy, k, s, p), wt.grad.permute(2, 3, 1, 0).numpy(), atol=1e-11)
    assert np.allclose(O.conv2d_grad_x(dy, w, s, p, (h, h)), xt.grad.permute(0, 2, 3, 1).numpy(), atol=1e-11)


@pytest.mark.parametrize("win,s", [(3, 2), (2, 2)])
def test_maxpool_vs_torch(win, s):
    rs = np.random.default_rng(win)
    x = rs.standard_normal((2, 13, 13, 6))
    y, _ = O.maxpool(x, win, s)
    xt = _t(x).permute(0, 3, 1, 2).requires_grad_(True)
    yt = F.max_pool2d(xt, win, s)
    assert np.array_equal(y, yt.permute(0, 2, 3, 1).detach().numpy())
    dy = rs.standard_normal(y.shape)
    yt.backward(_t(dy).permute(0, 3, 1, 2))
    assert np.allclose(O.maxpool_grad(x, dy, win, s), xt.grad.permute(0, 2, 3, 1).numpy(), atol=1e-12)


def test_maxpool_ties_go_to_first():
    x = np.zeros((1, 4, 4, 1))
    dy = np.ones((1, 2, 2, 1))
    dx = O.maxpool_grad(x, dy, 2, 2)
    assert dx[0, 0, 0, 0] == 1 and dx[0, 0, 2, 0] == 1 and dx.sum() == 4


def test_lrn_vs_torch():
    rs = np.random.default_rng(5)
    x = rs.standard_normal((2, 5, 5, 16))
    size, alpha, beta, k = 5, 1e-4, 0.75, 2.0
    y = O.lrn(x * 30, size, alpha, beta, k)
    xt = (_t(x) * 30).permute(0, 3, 1, 2).requires_grad_(True)
    # torch divides alpha by size; the Krizhevsky / TF form does not
    yt = F.local_response_norm(xt, size, alpha * size, beta, k)
    assert np.allclose(y, yt.permute(0, 2, 3, 1).detach().numpy(), rtol=1e-12)
    dy = rs.standard_normal(y.shape)
    yt.backward(_t(dy).permute(0, 3, 1, 2))
    assert np.allclose(O.lrn_grad(x * 30, dy, size, alpha, beta, k), xt.grad.permute(0, 2, 3, 1).numpy(),
                       rtol=1e-10, atol=1e-12)


def test_planner_golden_real_nets():
    doc = planner_cases()
    profs = {"pcie-box": planner.load_profile("pcie-box"), "nvlink-box": planner.load_profile("nvlink-box"),
             "b200": planner.load_profile("b200")}
    cache = {}
    for c in doc["cases"]:
        key = (c["net"], c["G"])
        if key not in cache:
            cache[key] = workloads.extract_workloads(ir.infer_shapes(models.MODELS[c["net"]](c["G"])))
        w = cache[key]
        assert [[l.flops_fwd, l.flops_bwd, l.weight_bytes] for l in w.layers] == c["layers"]
        plan = planner.select_parallelism(w, tuple(range(8)), profs[c["profile"]], c["algo"])
        assert plan.d == c["d"]
        assert plan.predicted_power.hex() == c["power"]
        got = [[e.d, e.t_c_total.hex(), e.t_s_total.hex(), e.predicted_throughput.hex()] for e in plan.estimates]
        assert got == c["estimates"]


def test_param_counts():
    for net, count in (("alexnet", 61_100_840), ("vgg16", 138_357_544)):
        g = models.MODELS[net](2)
        assert sum(n.output_shape.elements() for n in ir.infer_shapes(g) if n.kind is ir.OpKind.VARIABLE) == count
