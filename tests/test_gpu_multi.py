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


# ---- the multi-process data-parallel path at world_size 2 (both ranks on the
# one visible B200, process group over gloo): DataParallelGradient, the product
# path of bench.py under torchrun, with real shards and a real exchange.
def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, env_extra, timeout=600):
    import os
    import subprocess
    import sys
    env = dict(os.environ, QF_DIST_BACKEND="gloo", OMP_NUM_THREADS="1", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)


def test_data_parallel_gradient_world2(oracle, tmp_path):
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "dp.npz")
    r = _torchrun([os.path.join(root, "tests", "dp_worker.py")], {"QF_DP_OUT": out})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = np.load(out)
    n, layers, batch = 14, 4, 7
    gates, npar = C.build_hea(n, layers)
    M = npar
    # the all-reduced shard sums == the single-device gradient of the whole batch
    # (same per-sample kernels; only the fp64 order of the K sums differs)
    assert rel_diff(d["red"][:M], d["single_grad"]) <= 1e-6
    assert abs(d["red"][M] - d["single_loss"]) <= 1e-6 * float(np.abs(d["single_expect"]).sum())
    np.testing.assert_allclose(d["expect"], d["single_expect"], rtol=0, atol=1e-12)
    # and the oracle on the same global stream
    psi0 = C.new_random_state(n, batch, 1234)
    theta = C.random_parameters(npar, 1235)
    loss, grad, exp = oracle.gradient(gates, n, npar, psi0, theta,
                                      C.parse_pauli(C.repeated_ixyz_label(n)))
    assert rel_diff(d["red"][:M], grad) <= TOL
    assert abs(d["red"][M] - loss) <= TOL * float(np.abs(exp).sum())


def test_bench_two_ranks_gloo():
    """bench.py launched exactly like the driver's scaling run (torchrun, 2
    ranks), weak and strong, on a small workload: one JSON line from rank 0,
    max-over-ranks timing, n_gpus = 2."""
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for scaling, batch, glob in (("weak", 8, 16), ("strong", 16, 16)):
        r = _torchrun([os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                       "--workload", "hea16q", "--batch", str(batch), "--layers", "20",
                       "--scaling", scaling, "--no-cpu", "--no-secondary", "--no-refsig"], {})
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, r.stdout
        line = json.loads(lines[0])
        assert line["n_gpus"] == 2 and line["scaling"] == scaling
        assert line["config"]["global_batch"] == glob and line["config"]["batch_per_gpu"] == 8
        assert line["value"] > 0 and line["e2e"]["value"] > 0


def test_host_input_pipeline_matches_direct(ctx):
    """parallel.HostInputPipeline (the bench's e2e leg): three steps on three
    different host psi0 with the next copy overlapping the current step; the
    result of the last step equals the direct plan gradient on that psi0, and
    the plan still accepts its own uploads afterwards."""
    from paper_2603_02804_b200.parallel import DataParallelGradient, HostInputPipeline
    n, layers, batch = 14, 3, 3
    gates, npar, theta, _, pauli = _case(n, layers, batch)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    dp = DataParallelGradient(plan, torch)
    psis = [torch.from_numpy(C.new_random_state(n, batch, 50 + i).reshape(-1).copy()).pin_memory()
            for i in range(3)]
    th_h = torch.from_numpy(theta.copy()).pin_memory()
    th_d = th_h.to("cuda")
    res_h = torch.empty(npar + 1, dtype=torch.float64).pin_memory()
    pipe = HostInputPipeline(dp)
    pipe.run(psis, th_h, th_d, res_h)
    dp.stream.synchronize()
    got = res_h.numpy().copy()
    plan.upload_psi0(psis[-1].numpy().reshape(batch, 1 << n, 2))
    ref = plan.gradient(theta)
    assert rel_diff(got[:npar], ref.gradient) <= 1e-12
    assert got[npar] == pytest.approx(ref.loss, rel=1e-12, abs=1e-15)
    dp.close()
    plan.close()
