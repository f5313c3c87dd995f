# SPDX-License-Identifier: Apache-2.0
"""Host logic of the B200 path that needs no GPU: the model loader (load_model's
topological sort, shape inference and validation) and the rescale planner
(plan_rescaling), checked against the reference's own planner output
(tests/golden/plans_n8192.json, produced by oracle/gen_golden.py)."""
import json
import os

import numpy as np
import pytest

from paper_1908_04172_b200 import henet as H
from paper_1908_04172_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
P = W.N8192


def _f64(bits):
    return float(np.array([bits], dtype=np.uint64).view(np.float64)[0])


@pytest.fixture(scope="module")
def ref_plans():
    with open(os.path.join(GOLD, "plans_n8192.json")) as f:
        return json.load(f)


WORKLOADS = [W.dense_layer(), W.cryptonets(), W.cryptonets_relu(), W.toy_cryptonets(), W.cryptonets_relu(packing=0)]


@pytest.mark.parametrize("wl", WORKLOADS, ids=[w.name for w in WORKLOADS])
@pytest.mark.parametrize("mode", ["lazy", "naive"])
def test_planner_matches_reference(wl, mode, ref_plans):
    m = H.PlainModel.load(wl.manifest, wl.blob)
    plan = H.RescalePlan.plan_params(P["chain"], P["scale"], m, 0 if mode == "lazy" else 1)
    rp = ref_plans[wl.name][mode]
    assert plan.planned_rescale_ops == rp["planned_rescale_ops"]
    for n in rp["nodes"]:
        dec, lin, lout, sc = plan.node(n["id"])
        assert (dec, lin, lout) == (n["decision"], n["level_in"], n["level_out"]), n["id"]
        assert sc == _f64(n["scale_out_bits"]), n["id"]  # bit-identical double bookkeeping


def test_cryptonets_plan_is_table1_pattern(ref_plans):
    """conv1 6->5, act1 5->4, fc1 4->3, act2 3->2, fc2 Skip, 1890 rescales."""
    m = H.PlainModel.load(W.cryptonets().manifest, W.cryptonets().blob)
    plan = H.RescalePlan.plan_params(P["chain"], P["scale"], m)
    assert plan.planned_rescale_ops == 1890
    assert [plan.node(i)[2] for i in ("conv1", "act1", "fc1", "act2", "fc2")] == [5, 4, 3, 2, 2]
    assert plan.node("fc2")[0] == H.SKIP


def test_shape_inference():
    wl = W.cryptonets()
    m = H.PlainModel.load(wl.manifest, wl.blob)
    assert m.shape("conv1") == [5, 13, 13]
    assert m.shape("flatten") == [845]
    assert m.shape("fc1") == [100]
    assert m.shape("out") == [10]


def _model(nodes, weights=(), packing=0):
    m = H.PlainModel(packing)
    for name, dims, data in weights:
        m.add_weight(name, dims, np.asarray(data, np.float32))
    for n in nodes:
        m.add_node(*n)
    return m


def test_loader_rejections():
    """Error messages of load_model (henet/graph.hpp:297-436)."""
    with pytest.raises(H.ValidationError, match="cycle detected"):
        _model([("a", "Square", ["b"]), ("b", "Square", ["a"]), ("in", "Input", [], {"shape": [1]}),
                ("out", "Output", ["a"])]).finalize()
    with pytest.raises(H.ValidationError, match="references unknown input"):
        _model([("in", "Input", [], {"shape": [2]}), ("out", "Output", ["nope"])]).finalize()
    with pytest.raises(H.ValidationError, match="Dot inner dimension mismatch"):
        _model([("in", "Input", [], {"shape": [3]}), ("d", "Dot", ["in"], {}, "w"), ("out", "Output", ["d"])],
               [("w", [4, 2], np.zeros(8))]).finalize()
    with pytest.raises(H.ValidationError, match="complex packing cannot evaluate node sq"):
        _model([("in", "Input", [], {"shape": [3]}), ("sq", "Square", ["in"]), ("out", "Output", ["sq"])],
               packing=1).finalize()
    with pytest.raises(H.ValidationError, match="exactly one Output"):
        _model([("in", "Input", [], {"shape": [3]})]).finalize()
    with pytest.raises(H.ValidationError, match="duplicate node id"):
        _model([("in", "Input", [], {"shape": [3]}), ("in", "Input", [], {"shape": [3]})])


def test_infeasible_depth():
    """proj/tests/test_graph.cpp:171-185: a chain deeper than the modulus chain is rejected."""
    nodes = [("in", "Input", [], {"shape": [4]}), ("c", "ConstWeight", [], {}, "c")]
    prev = "in"
    for i in range(7):
        nodes.append((f"m{i}", "Multiply", [prev, "c"]))
        prev = f"m{i}"
    nodes.append(("out", "Output", [prev]))
    nodes.insert(len(nodes) - 1, ("sq", "Square", [prev]))
    nodes[-1] = ("out", "Output", ["sq"])
    m = _model(nodes, [("c", [1], [0.5])])
    m.finalize()
    with pytest.raises(H.ValidationError, match="infeasible depth"):
        H.RescalePlan.plan_params(P["chain"], P["scale"], m)
