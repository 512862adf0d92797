"""GPU: the single-process multi-GPU C-ABI (qf_group_*, qf_gradient_c64_multi).

The box the tests run on has one B200, so the group is exercised at G = 1
(a real NCCL communicator and all-reduce over one rank) against the oracle
and bit for bit against the single-device plan; G > visible devices and
duplicate devices must be refused. The shard/sum decomposition itself for
G > 1 is covered on CPU by tests/test_host.py (gloo, world_size 2).
"""
import numpy as np
import pytest
import torch

from oracles import rel_diff
from paper_2603_02804_b200 import capi
from paper_2603_02804_b200 import circuits as C

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _case(n, layers, batch, seed=99):
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, seed + 1)
    psi0 = C.new_random_state(n, batch, seed)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    return gates, npar, theta, psi0, pauli


@pytest.mark.parametrize("n,layers,batch,k", [(4, 4, 8, 0), (12, 3, 5, 1), (14, 4, 3, 2)])
def test_multi_one_shot_vs_oracle(oracle, n, layers, batch, k):
    gates, npar, theta, psi0, pauli = _case(n, layers, batch)
    res = capi.gradient_c64_multi(1, gates, n, npar, layers, k, psi0, theta, pauli)
    loss, grad, exp = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    assert rel_diff(res.gradient, grad) <= TOL
    assert abs(res.loss - loss) <= TOL * max(abs(loss), float(np.abs(exp).sum()))
    assert rel_diff(res.expect, exp) <= TOL
    assert res.stats["backward_passes"] >= 0 and res.stats["device_ms"] > 0


def test_group_plan_matches_single_device_bitwise(ctx):
    n, layers, batch = 14, 4, 6
    gates, npar, theta, psi0, pauli = _case(n, layers, batch, seed=3)
    plan = capi.Plan(ctx, gates, n, npar, layers, 2, batch, pauli)
    plan.upload_psi0(psi0)
    single = plan.gradient(theta)
    grp = capi.Group(1, [0])
    assert grp.size == 1
    gp = capi.GroupPlan(grp, gates, n, npar, layers, 2, batch, pauli)
    gp.upload_psi0(psi0)
    for _ in range(2):  # reuse: same answer every call
        res = gp.gradient(theta)
        assert res.loss == single.loss
        np.testing.assert_array_equal(res.gradient, single.gradient)
        np.testing.assert_array_equal(res.expect, single.expect)
    # device-generated batch store: the global SplitMix64 stream
    gp.random_psi0(1234)
    res = gp.gradient(theta)
    res2 = capi.gradient_c64_multi(1, gates, n, npar, layers, 2,
                                   C.new_random_state(n, batch, 1234), theta, pauli)
    assert rel_diff(res.gradient, res2.gradient) <= 1e-6
    gp.close()
    grp.close()


def test_multi_memsave(oracle):
    n, layers, batch = 14, 4, 2
    gates, npar, theta, psi0, pauli = _case(n, layers, batch, seed=8)
    res = capi.gradient_c64_multi(1, gates, n, npar, layers, 1, psi0, theta, pauli,
                                  storage="memsave")
    _, grad, _ = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    assert rel_diff(res.gradient, grad) <= 5e-3


def test_group_errors():
    gates, npar, theta, psi0, pauli = _case(4, 2, 2)
    count = torch.cuda.device_count()
    with pytest.raises(capi.QfInvalidArgument):
        capi.Group(count + 1)
    with pytest.raises(capi.QfInvalidArgument):
        capi.Group(0)
    if count == 1:
        with pytest.raises(capi.QfInvalidArgument):
            capi.Group(2, [0, 0])
    with pytest.raises(capi.QfInvalidArgument):
        capi.gradient_c64_multi(1, gates, 4, npar, 2, 3, psi0, theta, pauli)  # k=3 !| 2 layers
    grp = capi.Group(1)
    with pytest.raises(capi.QfInvalidArgument):
        capi.GroupPlan(grp, gates, 4, npar, 2, 0, 0, pauli)  # empty batch
    gp = capi.GroupPlan(grp, gates, 4, npar, 2, 0, 2, pauli)
    with pytest.raises(capi.QfInvalidArgument):
        gp.gradient(theta[:-1])
