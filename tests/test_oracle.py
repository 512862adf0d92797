"""CPU: pin the C oracle (oracle/qf_oracle.c) against the reference.

* SURVEY.md §8c golden values (fp64, produced by the reference);
* tests/golden/golden_reference.json (written by make_golden.py from the
  unmodified reference compiled in oracle/_ref);
* the live reference library, when oracle/_ref is built (this container).
Tolerances follow tests/acceptance.cpp: adjoint vs parameter shift <= 1e-10,
fp64 restatement vs fp64 reference <= 1e-10 (max-norm relative).
"""
import json
import os

import numpy as np
import pytest

from oracles import REF_SO, rel_diff

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden_reference.json")))["cases"]


def _hea_inputs(oracle, c):
    gates, npar = oracle.build_hea(c["n"], c["layers"])
    theta = oracle.random_parameters(npar, c["seed"] + 1)
    psi0 = oracle.random_state(c["n"], c["batch"], c["seed"])
    if c["precision"] == "f32":
        psi0 = psi0.astype(np.float32)
    pauli = (c["x_mask"], c["z_mask"], c["y_count"])
    return gates, npar, theta, psi0, pauli


def test_survey_goldens(oracle):
    gates, npar = oracle.build_hea(4, 4)
    theta = oracle.random_parameters(npar, 1235)
    assert theta[0] == pytest.approx(6.1224721633088439, abs=1e-15)
    psi0 = oracle.random_state(4, 8, 1234)
    np.testing.assert_allclose(psi0[0, 0], [-0.1099060638444172, -0.072580797531387464], atol=1e-15)
    pauli = oracle.parse_pauli(oracle.repeated_ixyz(4))
    assert pauli == (0x6, 0x3, 1)
    loss, grad, _ = oracle.gradient(gates, 4, npar, psi0, theta, pauli)
    assert loss == pytest.approx(-0.583176427514288, abs=1e-13)
    assert grad.sum() == pytest.approx(3.42181987882572, abs=1e-12)
    np.testing.assert_allclose(grad[:4], [-0.280450334533137, -0.847963409542352,
                                          0.763083492874858, 0.369861766941313], atol=1e-13)
    for label, l_ref, g_ref in [("ZZZZ", -0.0018511083677094, -2.38131359941164),
                                ("IIIZ", -0.0480468997384506, -1.14539425785954)]:
        loss, grad, _ = oracle.gradient(gates, 4, npar, psi0, theta, oracle.parse_pauli(label))
        assert loss == pytest.approx(l_ref, abs=1e-13)
        assert grad.sum() == pytest.approx(g_ref, abs=1e-12)


@pytest.mark.parametrize("case", [c for c in GOLD if c["kind"] == "hea"], ids=lambda c: c["name"])
def test_hea_fixtures(oracle, case):
    gates, npar, theta, psi0, pauli = _hea_inputs(oracle, case)
    assert theta[0] == case["theta0"]
    np.testing.assert_allclose(psi0[0, 0], case["psi0_00"], rtol=0, atol=0)
    loss, grad, exp = oracle.gradient(gates, case["n"], npar, psi0, theta, pauli)
    tol = 1e-10 if case["precision"] == "f64" else 1e-4  # reference ran in fp32
    assert rel_diff(grad, case["grad"]) <= tol
    assert rel_diff(exp, case["expect"]) <= tol
    assert abs(loss - case["loss"]) <= tol * max(1.0, abs(case["loss"]))


@pytest.mark.parametrize("case", [c for c in GOLD if c["kind"] == "random"], ids=lambda c: c["name"])
def test_random_fixtures(oracle, case):
    from oracles import GATE_DTYPE
    g = np.zeros(len(case["gates"]), GATE_DTYPE)
    for i, (k, a, q0, q1, p) in enumerate(case["gates"]):
        g[i] = (k, a, 0, q0, q1, p)
    npar = int(max((x[4] for x in case["gates"] if x[0] == 0), default=-1)) + 1
    theta = oracle.random_parameters(npar, case["seed"] + 100)
    psi0 = oracle.random_state(case["n"], 3, case["seed"] + 200)
    pauli = (case["x_mask"], case["z_mask"], bin(case["x_mask"] & case["z_mask"]).count("1"))
    loss, grad, exp = oracle.gradient(g, case["n"], npar, psi0, theta, pauli)
    assert rel_diff(grad, case["grad"]) <= 1e-10
    assert rel_diff(grad, case["param_shift"]) <= 1e-10  # acceptance.cpp:113-135
    assert abs(loss - case["loss"]) <= 1e-12


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("i", range(12))
def test_oracle_vs_live_reference(oracle, ref, i):
    """make_instance (acceptance.cpp:90-101): n in {4,6,8,10}, d in {1,2,4}."""
    n, d, batch = (4, 6, 8, 10)[i % 4], (1, 2, 4)[i % 3], 1 + i % 8
    gates, npar = ref.build_hea(n, d)
    theta = ref.random_parameters(npar, 1000 + i)
    psi0 = ref.random_state(n, batch, 2000 + i, np.float64)
    pauli = ref.parse_pauli("".join("IXYZ"[k % 4] for k in range(n)))
    loss_r, grad_r = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=d)
    loss_o, grad_o, _ = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    assert rel_diff(grad_o, grad_r) <= 1e-10
    assert abs(loss_o - loss_r) <= 1e-12
    if n <= 6:
        shift = ref.parameter_shift(gates, n, npar, psi0, theta, pauli)
        assert rel_diff(grad_o, shift) <= 1e-10


def test_oracle_forward_matches_reference(oracle, ref):
    gates, npar = ref.build_hea(5, 3)
    theta = ref.random_parameters(npar, 3)
    psi0 = ref.random_state(5, 2, 4, np.float64)
    np.testing.assert_allclose(oracle.forward(gates, 5, psi0, theta),
                               ref.forward(gates, 5, npar, psi0, theta), atol=1e-14)
