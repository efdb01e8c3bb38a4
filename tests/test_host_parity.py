"""Host-side API parity with the reference `wap` package, imported live from
/root/reference (build container only; skipped elsewhere).

Pins: graph construction (models + autodiff), the three rewrites (byte-identical
serialized graphs and identical reports), workload extraction, every planner
float, validation findings and JSON round trips."""

import json

import pytest

from paper_1811_01532_b200 import graph_modifier as gm
from paper_1811_01532_b200 import ir, models, planner, workloads

from .conftest import have_reference

pytestmark = pytest.mark.skipif(not have_reference(), reason="reference checkout not present")

MODEL_CASES = [("mlp", 64), ("mlp", 24), ("alexnet_like", 16), ("alexnet_like", 128),
               ("vgg16_like", 8), ("vgg16_like", 48)]


def _ref_model(ref_wap, name, batch):
    from importlib import import_module

    return getattr(import_module("wap.models"), name)(batch)


def _mine(name, batch):
    return models.MODELS[name](batch)


@pytest.mark.parametrize("name,batch", MODEL_CASES)
def test_models_serialize_identically(ref_wap, name, batch):
    assert ir.serialize(_mine(name, batch)) == ref_wap.serialize(_ref_model(ref_wap, name, batch))


@pytest.mark.parametrize("name,batch", MODEL_CASES)
def test_workloads_identical(ref_wap, name, batch):
    mine = workloads.extract_workloads(ir.infer_shapes(_mine(name, batch)))
    ref = ref_wap.extract_workloads(ref_wap.infer_shapes(_ref_model(ref_wap, name, batch)))
    assert mine.to_json() == ref.to_json()
    assert mine.total_flops == ref.total_flops


@pytest.mark.parametrize("profile", ["pcie-box", "nvlink-box"])
@pytest.mark.parametrize("algo", ["ring", "naive_all_to_all"])
@pytest.mark.parametrize("name,batch", MODEL_CASES)
def test_planner_bit_identical(ref_wap, profile, algo, name, batch):
    mw = workloads.extract_workloads(ir.infer_shapes(_mine(name, batch)))
    rw = ref_wap.extract_workloads(ref_wap.infer_shapes(_ref_model(ref_wap, name, batch)))
    mp, rp = planner.load_profile(profile), ref_wap.load_profile(profile)
    for n_dev in (1, 3, 4, 8):
        a = planner.select_parallelism(mw, tuple(range(n_dev)), mp, algo)
        b = ref_wap.select_parallelism(rw, tuple(range(n_dev)), rp, algo)
        assert a.d == b.d and a.devices == b.devices
        assert a.predicted_power == b.predicted_power
        assert [(e.d, e.t_c_total, e.t_s_total, e.predicted_throughput) for e in a.estimates] == \
               [(e.d, e.t_c_total, e.t_s_total, e.predicted_throughput) for e in b.estimates]


@pytest.mark.parametrize("name,batch", MODEL_CASES)
@pytest.mark.parametrize("d", [2, 3, 4, 8])
def test_transform_byte_identical(ref_wap, name, batch, d):
    if batch % d:
        pytest.skip("d does not divide the batch")
    from importlib import import_module

    ref_tf = import_module("wap.transform")  # not wap.transform: the package rebinds that name
    g_mine, g_ref = _mine(name, batch), _ref_model(ref_wap, name, batch)
    plan_m = planner.ParallelPlan(d, tuple(range(d)), (), 0.0)
    plan_r = ref_wap.ParallelPlan(d, tuple(range(d)), (), 0.0)
    steps = [("replicate_primary",), ("localize_auxiliary",), ("optimize_gradient_aggregation",)]
    cur_m, cur_r = g_mine, g_ref
    for (fn,) in steps:
        cur_m, rep_m = getattr(gm, fn)(cur_m, plan_m)
        cur_r, rep_r = getattr(ref_tf, fn)(cur_r, plan_r)
        assert ir.serialize(cur_m) == ref_wap.serialize(cur_r), fn
        assert rep_m.to_json() == rep_r.to_json(), fn
    full_m, reps_m = gm.transform(g_mine, plan_m)
    full_r, reps_r = ref_tf.transform(g_ref, plan_r)
    assert ir.serialize(full_m) == ref_wap.serialize(full_r)
    assert [r.to_json() for r in reps_m] == [r.to_json() for r in reps_r]
    assert gm.check_parallel_structure(full_m, plan_m) == ref_tf.check_parallel_structure(full_r, plan_r) == []


def test_reference_json_loads_here(ref_wap):
    from importlib import import_module

    ref_tf = import_module("wap.transform")
    g = _ref_model(ref_wap, "alexnet_like", 32)
    plan = ref_wap.ParallelPlan(4, (0, 1, 2, 3), (), 0.0)
    blob = ref_wap.serialize(ref_tf.transform(g, plan)[0])
    mine = ir.deserialize(blob)
    assert ir.serialize(mine) == blob
    assert ir.validate(mine).ok


def _bad_graphs(mod):
    B = mod.GraphBuilder
    K = mod.OpKind
    out = []
    b = B("missing")
    b.add(K.RELU, "r", ("nope",))
    out.append(b.build(("r",)))
    b = B("cycle")
    b.add(K.RELU, "a", ("b",))
    b.add(K.RELU, "b", ("a",))
    out.append(b.build(("a",)))
    b = B("shape")
    x = b.input("x", (128, 784))
    w = b.variable("w", (10, 10))
    b.add(K.MATMUL, "mm", (x, w))
    out.append(b.build(("mm",)))
    b = B("attrs")
    x = b.input("x", (4, 4))
    b.add(K.SPLIT, "s", (x,), axis=0, parts=1)
    b.add(K.RELU, "r", ("s",), device=0, bogus=1)
    out.append(b.build(("s",)))
    return out


def test_validation_findings_identical(ref_wap):
    for gm_, gr in zip(_bad_graphs(ir), _bad_graphs(ref_wap)):
        fm = [(f.node, f.rule, f.message) for f in ir.validate(gm_).findings]
        fr = [(f.node, f.rule, f.message) for f in ref_wap.validate(gr).findings]
        assert fm == fr


def test_profile_schema(ref_wap):
    for name in ("pcie-box", "nvlink-box"):
        assert planner.load_profile(name).to_json() == ref_wap.load_profile(name).to_json()
    doc = json.loads((planner.Path(planner.__file__).parent / "profiles" / "b200.json").read_text())
    assert set(doc) == planner.PROFILE_FIELDS
