"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tolerance (stated by north_star): fp32 gradients within 1e-4
max-norm relative of the fp64 oracle (rel_diff, acceptance.cpp:63-73); loss
within 1e-4 * max(|loss_ref|, sum_s |E_s|).
"""
import numpy as np
import pytest

from oracles import rel_diff
from paper_2603_02804_b200 import circuits as C
from paper_2603_02804_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _check(res, oracle_out, tol=TOL):
    loss, grad, exp = oracle_out
    assert rel_diff(res.gradient, grad) <= tol, rel_diff(res.gradient, grad)
    scale = max(abs(loss), float(np.sum(np.abs(exp))), 1e-300)
    assert abs(res.loss - loss) <= tol * scale, (res.loss, loss)
    assert rel_diff(res.expect, exp) <= tol, rel_diff(res.expect, exp)


def _hea_case(n, layers, batch, label=None, seed=1234):
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, seed + 1)
    psi0 = C.new_random_state(n, batch, seed)
    pauli = C.parse_pauli(label or C.repeated_ixyz_label(n))
    return gates, npar, theta, psi0, pauli


def test_config1_golden(ctx, oracle):
    """BASELINE config 1 (4q x 4L, B=8) against the survey's fp64 goldens."""
    gates, npar, theta, psi0, pauli = _hea_case(4, 4, 8)
    res = capi.gradient_c64(ctx, gates, 4, npar, 4, 0, psi0, theta, pauli)
    assert abs(res.loss - (-0.583176427514288)) < 1e-5
    assert abs(res.gradient.sum() - 3.42181987882572) < 1e-4
    np.testing.assert_allclose(res.gradient[:4], [-0.280450334533137, -0.847963409542352,
                                                  0.763083492874858, 0.369861766941313],
                               atol=1e-5)
    _check(res, oracle.gradient(gates, 4, npar, psi0, theta, pauli))


@pytest.mark.parametrize("label,loss_ref,gsum_ref", [
    ("ZZZZ", -0.0018511083677094, -2.38131359941164),
    ("IIIZ", -0.0480468997384506, -1.14539425785954),
])
def test_config1_observables(ctx, oracle, label, loss_ref, gsum_ref):
    gates, npar, theta, psi0, pauli = _hea_case(4, 4, 8, label)
    res = capi.gradient_c64(ctx, gates, 4, npar, 4, 0, psi0, theta, pauli)
    assert abs(res.loss - loss_ref) < 1e-5
    assert abs(res.gradient.sum() - gsum_ref) < 1e-4
    _check(res, oracle.gradient(gates, 4, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,layers,batch", [
    (2, 3, 5), (3, 2, 3), (4, 1, 1), (5, 4, 7), (6, 8, 4), (8, 5, 3), (10, 4, 2),
    (11, 3, 3), (12, 6, 2),          # sample-resident kernel
    (13, 2, 2), (14, 3, 2), (15, 4, 1), (16, 2, 1),  # streaming passes A + B
])
def test_hea_sizes(ctx, oracle, n, layers, batch):
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=77 + n)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,batch", [(20, 1)])
def test_hea_20q(ctx, oracle, n, batch):
    gates, npar, theta, psi0, pauli = _hea_case(n, 2, batch, seed=5)
    res = capi.gradient_c64(ctx, gates, n, npar, 2, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("layers,k", [(1, 0), (2, 1), (5, 1), (6, 2), (6, 3), (9, 3), (9, 0)])
def test_resident_n12_chained_stages(ctx, oracle, layers, k):
    """n = 12 sample-resident kernel: stages chained two phases each (odd stages
    with the diagonal in group 2), split at every checkpoint slot; odd and even
    stage counts, slots after odd and even stages (k = 0: engine default)."""
    gates, npar, theta, psi0, pauli = _hea_case(12, layers, 3, seed=40 + layers)
    res = capi.gradient_c64(ctx, gates, 12, npar, layers, k, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, 12, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,layers", [(6, 8), (14, 4)])
@pytest.mark.parametrize("k", [1, 2, 4])
def test_checkpoint_intervals(ctx, oracle, n, layers, k):
    """run_checkpointed parity: every block size gives the same gradient
    (checkpoint.cpp:144-163, acceptance C8)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 2, seed=13)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,ngates,seed", [(4, 40, 1), (6, 80, 2), (9, 60, 3), (13, 50, 4)])
def test_random_circuits(ctx, oracle, n, ngates, seed):
    """Random Rx/Ry/Rz/CZ/CNOT circuits (test_engine.cpp:438-468)."""
    gates, npar = C.random_circuit(n, ngates, seed)
    theta = C.random_parameters(npar, seed + 100)
    psi0 = C.new_random_state(n, 3, seed + 200)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    res = capi.gradient_c64(ctx, gates, n, npar, 0, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,layers,batch", [(4, 4, 8), (9, 3, 4), (14, 2, 2)])
def test_pergate_comparator(ctx, oracle, n, layers, batch):
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=3)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli, pergate=True)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_against_reference_fp32(ctx, ref):
    """Same inputs through the unmodified reference (gradient<float>)."""
    n, layers, batch = 8, 6, 4
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=21)
    loss_r, grad_r = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    assert rel_diff(res.gradient, grad_r) <= TOL
    assert abs(res.loss - loss_r) <= TOL


def test_plan_reuse_and_determinism(ctx, oracle):
    n, layers, batch = 14, 3, 3
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=9)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    plan.upload_psi0(psi0)
    a = plan.gradient(theta)
    b = plan.gradient(theta)
    assert np.array_equal(a.gradient, b.gradient) and a.loss == b.loss
    theta2 = C.random_parameters(npar, 999)
    c = plan.gradient(theta2)
    _check(c, oracle.gradient(gates, n, npar, psi0, theta2, pauli))


def test_errors(ctx):
    gates, npar = C.build_hea(4, 2)
    psi0 = C.new_random_state(4, 2, 1)
    theta = C.random_parameters(npar, 2)
    pauli = C.parse_pauli("IXYZ")
    bad = gates.copy()
    bad[0]["q0"] = 9
    with pytest.raises(capi.QfInvalidArgument):
        capi.gradient_c64(ctx, bad, 4, npar, 2, 0, psi0, theta, pauli)
    bad = gates.copy()
    bad[1]["param"] = 0  # parameter used twice
    with pytest.raises(capi.QfInvalidArgument):
        capi.gradient_c64(ctx, bad, 4, npar, 2, 0, psi0, theta, pauli)
    with pytest.raises(capi.QfInvalidArgument):  # k does not divide layers
        capi.gradient_c64(ctx, gates, 4, npar, 2, 3, psi0, theta, pauli)
    with pytest.raises(capi.QfCapacityError):
        g26, np26 = C.build_hea(26, 1)
        capi.Plan(ctx, g26, 26, np26, 1, 0, 1 << 12, C.parse_pauli("Z" * 26))


@pytest.mark.parametrize("n,layers,batch", [(4, 3, 5), (12, 2, 2), (12, 5, 3), (14, 2, 2), (17, 2, 1),
                                            (20, 2, 1)])
def test_forward_state_matches_reference(ctx, ref, n, layers, batch):
    """Final state of the fused forward vs the reference's forward<double>
    (engine.hpp:131-133), amplitude for amplitude: the device model's dropped
    global phase e^{i sum delta} is restored in the readout (no phase is
    divided out here)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=41)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    plan.upload_psi0(psi0)
    got = plan.forward_state(theta).astype(np.float64)
    want = ref.forward(gates, n, npar, psi0.astype(np.float64), theta)
    g = got[..., 0] + 1j * got[..., 1]
    w = want[..., 0] + 1j * want[..., 1]
    for s in range(batch):
        assert np.max(np.abs(g[s] - w[s])) < 1e-5 * max(1.0, 2 ** ((20 - n) / 2) / 32)
        assert abs(np.vdot(g[s], w[s]) - 1.0) < 1e-5


def test_forward_state_random_circuit_phase(ctx, ref):
    """Random Rx/Ry/Rz/CZ/CNOT circuit: sections with every axis mix and CNOT
    Hadamards, the global phase restored exactly."""
    n = 13
    gates, npar = C.random_circuit(n, 120, 17)
    theta = C.random_parameters(npar, 18)
    psi0 = C.new_random_state(n, 2, 19)
    plan = capi.Plan(ctx, gates, n, npar, 0, 0, 2, C.parse_pauli("Z" * n))
    plan.upload_psi0(psi0)
    got = plan.forward_state(theta).astype(np.float64)
    want = ref.forward(gates, n, npar, psi0.astype(np.float64), theta)
    assert np.max(np.abs(got - want)) < 1e-5


@pytest.mark.parametrize("n,layers,batch", [(21, 1, 1), (22, 2, 1), (23, 1, 1), (24, 1, 1)])
def test_three_layouts(ctx, oracle, n, layers, batch):
    """n > 20 needs a third layout (two passes per stage); n = 21..24 also take
    the column-group move of the last layout (qf_plan.cpp)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=8)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_streaming_checkpoint_slots(ctx, oracle, k):
    n, layers = 15, 6
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 2, seed=17)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,batch,first", [(13, 3, 5), (16, 2, 3), (4, 9, 0)])
def test_device_random_state(ctx, ref, n, batch, first):
    """qf_plan_random_psi0 == new_random_state<float> (statevec.cpp:32-53) bit
    for bit: the SplitMix64 stream jumped ahead to sample `first`, Box-Muller in
    fp64, the per-sample norm summed sequentially in amplitude order."""
    gates, npar = C.build_hea(n, 1)
    plan = capi.Plan(ctx, gates, n, npar, 1, 0, batch, C.parse_pauli("Z" * n))
    plan.random_psi0(1234, first_sample=first)
    host = np.empty((batch, 1 << n, 2), np.float32)
    plan.download_psi0_ptr(host.ctypes.data)
    want = ref.random_state(n, first + batch, 1234, np.float32)[first:]  # the reference itself
    np.testing.assert_array_equal(host.view(np.uint32), want.view(np.uint32))


def test_cpp_dropin_shim():
    """The reference's own C++ calling code (qfuse::gradient<float>,
    run_checkpointed<float>, naive_gradient<float>) vs the qfuse::b200 drop-in
    on the same BatchedState / FusedCircuit / PauliString objects."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "tests", "shim_parity")
    if not os.path.exists(exe):
        pytest.skip("build/tests/shim_parity not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout


def _one(ctx, gates, n, npar, psi0, theta, label, layers=0):
    pauli = C.parse_pauli(label)
    return capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)


def test_known_answer_single_rx(ctx):
    """Single Rx(0.3) on |0>, O = Z: loss cos 0.3, grad -sin 0.3
    (test_engine.cpp:284-302)."""
    g = np.zeros(1, C.GATE_DTYPE)
    g[0] = (C.ROT, C.X, 0, 0, 0, 0)
    psi0 = np.zeros((1, 2, 2), np.float32)
    psi0[0, 0, 0] = 1.0
    res = _one(ctx, g, 1, 1, psi0, np.array([0.3]), "Z")
    assert abs(res.loss - np.cos(0.3)) < 1e-6
    assert abs(res.gradient[0] + np.sin(0.3)) < 1e-6


def test_stationary_point_theta_zero(ctx):
    """theta = 0 on |000> with ZZZ: loss 1, all gradients 0 (test_engine.cpp:395-405)."""
    gates, npar = C.build_hea(3, 2)
    psi0 = np.zeros((2, 8, 2), np.float32)
    psi0[:, 0, 0] = 1.0
    res = _one(ctx, gates, 3, npar, psi0, np.zeros(npar), "ZZZ")
    assert abs(res.loss - 2.0) < 1e-6
    assert np.max(np.abs(res.gradient)) < 1e-6


def test_rx_pi_flips(ctx, oracle):
    """Rx(pi) on qubit 0 of |00> -> -i|01>: <Z on q0> = -1 (test_engine.cpp:80-92)."""
    g = np.zeros(1, C.GATE_DTYPE)
    g[0] = (C.ROT, C.X, 0, 0, 0, 0)
    psi0 = np.zeros((1, 4, 2), np.float32)
    psi0[0, 0, 0] = 1.0
    res = _one(ctx, g, 2, 1, psi0, np.array([np.pi]), "IZ")
    assert abs(res.loss + 1.0) < 1e-6


def test_no_parameters_and_cz_only(ctx, oracle):
    """A circuit with no rotations (only CZ) still yields the expectation."""
    g = np.zeros(3, C.GATE_DTYPE)
    for i, (a, b) in enumerate([(0, 1), (1, 2), (0, 2)]):
        g[i] = (C.CZ, 0, 0, a, b, 0)
    psi0 = C.new_random_state(3, 4, 5)
    res = _one(ctx, g, 3, 0, psi0, np.zeros(0), "XYZ")
    loss, _, exp = oracle.gradient(g, 3, 0, psi0, np.zeros(0), C.parse_pauli("XYZ"))
    assert abs(res.loss - loss) < 1e-5 and rel_diff(res.expect, exp) < 1e-4


@pytest.mark.parametrize("n,batch", [(3, 1), (3, 513), (5, 130), (12, 3), (14, 5)])
def test_ragged_batches(ctx, oracle, n, batch):
    """Batches that do not fill the last 4096-amplitude tile (TMA OOB path)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, 2, batch, seed=31)
    res = capi.gradient_c64(ctx, gates, n, npar, 2, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_device_psi0_and_device_outputs(ctx, oracle):
    """qf_plan_set_psi0_device (aliased caller memory, read in place) +
    qf_plan_gradient_device (the data-parallel path); a caller that rewrites its
    buffer between calls gets the gradient of the new contents."""
    torch = pytest.importorskip("torch")
    n, layers, batch = 13, 2, 3
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=12)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    d_psi = torch.from_numpy(psi0).cuda()
    d_theta = torch.from_numpy(theta).cuda()
    out = torch.empty(npar + 1 + batch, dtype=torch.float64, device="cuda")
    plan.set_psi0_device(d_psi.data_ptr())
    for psi in (psi0, C.new_random_state(n, batch, 4321)):
        d_psi.copy_(torch.from_numpy(psi))
        torch.cuda.synchronize()  # the caller orders its write before the plan stream reads
        plan.gradient_device(d_theta.data_ptr(), out.data_ptr())
        plan.synchronize()
        o = out.cpu().numpy()
        loss, grad, exp = oracle.gradient(gates, n, npar, psi, theta, pauli)
        assert rel_diff(o[:npar], grad) <= TOL
        assert abs(o[npar] - loss) <= TOL * max(1.0, float(np.sum(np.abs(exp))))
        assert rel_diff(o[npar + 1:], exp) <= TOL
    # never written: the caller's buffer still holds the last input
    np.testing.assert_array_equal(d_psi.cpu().numpy(), C.new_random_state(n, batch, 4321))
    # upload_psi0 goes back to the plan's own store
    plan.upload_psi0(psi0)
    _check(plan.gradient(theta), oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,batch", [(5, 3), (14, 3)])
def test_device_psi0_alias_resident_and_streaming(ctx, oracle, n, batch):
    torch = pytest.importorskip("torch")
    gates, npar, theta, psi0, pauli = _hea_case(n, 3, batch, seed=14)
    plan = capi.Plan(ctx, gates, n, npar, 3, 0, batch, pauli)
    d_psi = torch.from_numpy(psi0).cuda()
    plan.set_psi0_device(d_psi.data_ptr())
    _check(plan.gradient(theta), oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_oneshot_plan_cache(ctx, oracle):
    """Repeated one-shot calls (the reference-signature path) reuse the cached
    plan: new psi0 and theta every call, a different shape in between, and the
    cache switched off -- every result against the oracle."""
    n, layers, batch = 16, 3, 3
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=71)
    first = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi0, theta, pauli)
    _check(first, oracle.gradient(gates, n, npar, psi0, theta, pauli))
    psi1 = C.new_random_state(n, batch, 72)
    th1 = C.random_parameters(npar, 73)
    again = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi1, th1, pauli)
    _check(again, oracle.gradient(gates, n, npar, psi1, th1, pauli))
    g2, np2, t2, p2, pa2 = _hea_case(13, 2, 2, seed=74)
    _check(capi.gradient_c64(ctx, g2, 13, np2, 2, 0, p2, t2, pa2),
           oracle.gradient(g2, 13, np2, p2, t2, pa2))
    same = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi0, theta, pauli)
    np.testing.assert_array_equal(same.gradient, first.gradient)
    ctx.set_plan_cache(False)
    try:
        off = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi0, theta, pauli)
        np.testing.assert_array_equal(off.gradient, first.gradient)
    finally:
        ctx.set_plan_cache(True)


def test_oneshot_staged_large_psi0(ctx, oracle):
    """psi0 of 64 MiB (> the 8 MiB direct-copy threshold): staged through the
    pinned buffer in 16 MiB chunks by host threads; pinned sources go direct."""
    torch = pytest.importorskip("torch")
    n, layers, batch = 20, 1, 8
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=75)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    plan.upload_psi0(psi0)
    ref_plan = plan.gradient(theta)
    plan.close()
    np.testing.assert_array_equal(res.gradient, ref_plan.gradient)
    pinned = torch.from_numpy(psi0).pin_memory()
    res2 = capi.gradient_c64(ctx, gates, n, npar, layers, 0, pinned.numpy(), theta, pauli)
    np.testing.assert_array_equal(res2.gradient, ref_plan.gradient)


def test_deep_circuit_uncompute_drift(ctx, oracle):
    """200 layers of uncompute with re-anchoring every 10: fp32 stays within tolerance."""
    n, layers = 13, 200
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 1, seed=77)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_config4_depth_fused_vs_pergate(ctx):
    """BASELINE config 4 depth (20q x 1000 layers, k = 10) on a 4-sample shard:
    the fused path (X, Y measured, Z chained over 1000 stages, scales folded
    into the diagonals) against the independent per-gate comparator (one
    kernel per gate, 80,000 gates each way). The CPU oracle would need ~10 min
    here, so this is the size-independent cross-check at full depth."""
    n, layers, batch = 20, 1000, 4
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=4242)
    fused = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    pg = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli, pergate=True)
    err = rel_diff(fused.gradient, pg.gradient)
    assert err <= TOL, err
    assert rel_diff(fused.expect, pg.expect) <= TOL
    assert np.all(np.isfinite(fused.gradient))


# ---- StorageMode::MemSave (bf16 checkpoint slots), acceptance C10 bound
MEMSAVE_TOL = 5e-3  # acceptance.cpp:466-499 (bf16 storage vs fp32)


@pytest.mark.parametrize("n,layers,batch,k", [(14, 6, 2, 1), (16, 8, 2, 2), (20, 4, 1, 1), (20, 6, 1, 2), (21, 4, 1, 2)])
def test_memsave_matches_oracle(ctx, oracle, n, layers, batch, k):
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=900 + n)
    ms = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli, storage="memsave")
    full = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli)
    ref = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    _check(full, ref)
    _check(ms, ref, tol=MEMSAVE_TOL)
    # the final state is complex64 either way: identical loss and expectations
    assert ms.loss == full.loss
    assert np.array_equal(ms.expect, full.expect)
    # half-size slots: (n_slots - 1) bf16 slots instead of n_slots complex64 ones
    assert ms.stats["device_bytes"] < full.stats["device_bytes"]


def test_memsave_resident_is_full_precision(ctx):
    gates, npar, theta, psi0, pauli = _hea_case(10, 6, 3, seed=31)
    ms = capi.gradient_c64(ctx, gates, 10, npar, 6, 2, psi0, theta, pauli, storage="memsave")
    full = capi.gradient_c64(ctx, gates, 10, npar, 6, 2, psi0, theta, pauli)
    assert np.array_equal(ms.gradient, full.gradient) and ms.loss == full.loss


def test_memsave_config4_depth(ctx):
    """20q x 1000 layers, k = 10: bf16 re-anchoring every 10 layers stays within C10."""
    n, layers, batch = 20, 1000, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=4242)
    full = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    ms = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli, storage="memsave")
    err = rel_diff(ms.gradient, full.gradient)
    assert err <= MEMSAVE_TOL, err
    assert ms.stats["device_bytes"] < 0.7 * full.stats["device_bytes"]


def test_memsave_plan_reuse(ctx):
    """A MemSave plan reused across theta gives the one-shot result bit for bit."""
    n, layers, batch = 16, 4, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=8)
    plan = capi.Plan(ctx, gates, n, npar, layers, 1, batch, pauli, storage="memsave")
    plan.upload_psi0(psi0)
    a = plan.gradient(theta)
    b = plan.gradient(theta)
    one = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi0, theta, pauli, storage="memsave")
    assert np.array_equal(a.gradient, b.gradient) and np.array_equal(a.gradient, one.gradient)


def test_memsave_against_reference_memsave(ctx, ref):
    """Our MemSave (bf16 slots) and the reference's MemSave (bf16 ledger,
    engine.cpp:488-530) on the same inputs: both within C10 of the fp32 Full result."""
    n, layers, batch = 14, 4, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=61)
    _, g_full = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers, block_layers=1)
    _, g_ref_ms = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers, block_layers=1,
                               mode="mem_save")
    ours = capi.gradient_c64(ctx, gates, n, npar, layers, 1, psi0, theta, pauli, storage="memsave")
    assert rel_diff(g_ref_ms, g_full) <= MEMSAVE_TOL
    assert rel_diff(ours.gradient, g_full) <= MEMSAVE_TOL


# ---- complex128 (the reference's double instantiations): fp64 bounds of
# acceptance C1/C2/C8 (1e-10, acceptance.cpp:113-170, :396-416)
TOL64 = 1e-10


def _check64(res, oracle_out):
    loss, grad, exp = oracle_out
    assert rel_diff(res.gradient, grad) <= TOL64, rel_diff(res.gradient, grad)
    assert abs(res.loss - loss) <= TOL64 * max(abs(loss), float(np.sum(np.abs(exp))), 1e-300)
    assert rel_diff(res.expect, exp) <= TOL64


def test_c128_config1_golden(ctx, oracle):
    gates, npar = C.build_hea(4, 4)
    theta = C.random_parameters(npar, 1235)
    psi0 = C.new_random_state(4, 8, 1234, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(4))
    res = capi.gradient_c128(ctx, gates, 4, npar, 4, 0, psi0, theta, pauli)
    assert abs(res.loss - (-0.583176427514288)) < 1e-13
    assert abs(res.gradient.sum() - 3.42181987882572) < 1e-12
    np.testing.assert_allclose(res.gradient[:4], [-0.280450334533137, -0.847963409542352,
                                                  0.763083492874858, 0.369861766941313],
                               atol=1e-13)
    _check64(res, oracle.gradient(gates, 4, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,ngates,seed", [(4, 40, 1), (6, 80, 2), (9, 60, 3), (13, 50, 4)])
def test_c128_random_circuits(ctx, oracle, n, ngates, seed):
    gates, npar = C.random_circuit(n, ngates, seed)
    theta = C.random_parameters(npar, seed + 100)
    psi0 = C.new_random_state(n, 3, seed + 200, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    res = capi.gradient_c128(ctx, gates, n, npar, 0, 0, psi0, theta, pauli)
    _check64(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,layers,batch", [(2, 3, 5), (12, 3, 2), (20, 2, 1)])
def test_c128_hea(ctx, oracle, n, layers, batch):
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, 7 + n)
    psi0 = C.new_random_state(n, batch, 70 + n, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    res = capi.gradient_c128(ctx, gates, n, npar, layers, 1, psi0, theta, pauli)
    _check64(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,ngates,seed", [(3, 30, 5), (11, 120, 6), (14, 160, 7), (17, 90, 8)])
def test_c128_fused_vs_pergate(ctx, n, ngates, seed):
    """Fused fp64 segments == the fp64 per-gate schedule (acceptance C2, fused
    == per-gate at 1e-12, acceptance.cpp:137-170), random Rx/Ry/Rz/CZ/CNOT
    circuits with several segments (n > 10) and CNOT controls off-tile."""
    gates, npar = C.random_circuit(n, ngates, seed)
    theta = C.random_parameters(npar, seed + 100)
    psi0 = C.new_random_state(n, 2, seed + 200, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    fused = capi.gradient_c128(ctx, gates, n, npar, 0, 0, psi0, theta, pauli)
    naive = capi.gradient_c128(ctx, gates, n, npar, 0, 0, psi0, theta, pauli, pergate=True)
    assert np.max(np.abs(fused.gradient - naive.gradient)) <= 1e-12
    assert abs(fused.loss - naive.loss) <= 1e-12
    np.testing.assert_allclose(fused.expect, naive.expect, rtol=0, atol=1e-12)
    assert fused.stats["forward_passes"] < naive.stats["forward_passes"]


def test_c128_fused_segments_hea(ctx, oracle):
    """16q HEA: 2-3 segments per layer instead of 4n gate passes; vs the oracle."""
    n, layers, batch = 16, 3, 2
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, 31)
    psi0 = C.new_random_state(n, batch, 32, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    res = capi.gradient_c128(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    _check64(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))
    assert res.stats["forward_passes"] <= 3 * layers
    again = capi.gradient_c128(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    np.testing.assert_array_equal(again.gradient, res.gradient)  # deterministic reductions


def test_c128_no_rotations(ctx, oracle):
    gates = np.zeros(2, dtype=C.GATE_DTYPE)
    gates[0] = (C.CZ, 0, 0, 0, 1, 0)
    gates[1] = (C.CNOT, 0, 0, 2, 0, 0)
    psi0 = C.new_random_state(3, 2, 5, np.float64)
    pauli = C.parse_pauli("XYZ")
    res = capi.gradient_c128(ctx, gates, 3, 0, 0, 0, psi0, np.zeros(0), pauli)
    loss, _, exp = oracle.gradient(gates, 3, 0, psi0, np.zeros(0), pauli)
    assert abs(res.loss - loss) <= 1e-12
    np.testing.assert_allclose(res.expect, exp, atol=1e-12)


def test_c128_against_reference_double(ctx, ref):
    """The unmodified reference's gradient<double> on the same inputs."""
    n, layers, batch = 8, 6, 4
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, 22)
    psi0 = C.new_random_state(n, batch, 21, np.float64)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    loss_r, grad_r = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers)
    res = capi.gradient_c128(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    assert rel_diff(res.gradient, grad_r) <= TOL64
    assert abs(res.loss - loss_r) <= TOL64 * max(1.0, abs(loss_r))


def test_c128_errors(ctx):
    gates, npar = C.build_hea(4, 2)
    psi0 = C.new_random_state(4, 2, 1, np.float64)
    pauli = C.parse_pauli("IXYZ")
    theta = C.random_parameters(npar, 2)
    bad = gates.copy()
    bad[0]["q0"] = 9
    with pytest.raises(capi.QfInvalidArgument):
        capi.gradient_c128(ctx, bad, 4, npar, 2, 0, psi0, theta, pauli)
    bad = gates.copy()
    bad[1]["param"] = 0  # parameter used twice
    with pytest.raises(capi.QfInvalidArgument):
        capi.gradient_c128(ctx, bad, 4, npar, 2, 0, psi0, theta, pauli)
    with pytest.raises(capi.QfInvalidArgument):  # k does not divide layers
        capi.gradient_c128(ctx, gates, 4, npar, 2, 3, psi0, theta, pauli)


def _drivers():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    b200 = os.path.join(root, "build", "tests", "bench_driver")
    cpu = os.path.join(root, "build", "tests", "bench_driver_ref")
    if not (os.path.exists(b200) and os.path.exists(cpu)):
        pytest.skip("build/tests/bench_driver* not built (needs the reference sources at build time)")
    return b200, cpu


def _run(cmd, timeout=900):
    import subprocess
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("flags,tol", [
    (["--qubits", "4", "--layers", "4", "--batch", "8"], 1e-4),                       # config 1
    (["--qubits", "4", "--layers", "4", "--batch", "8", "--mode", "naive"], 1e-4),
    (["--qubits", "4", "--layers", "4", "--batch", "8", "--precision", "double"], 1e-10),
    (["--qubits", "12", "--layers", "20", "--batch", "4", "--block", "10"], 1e-4),
    (["--qubits", "16", "--layers", "4", "--batch", "2", "--block", "2", "--mode", "fused_mem_save"], 5e-3),
    (["--qubits", "8", "--layers", "2", "--shape-qubits", "20"], 1e-4),               # build_hea_shape
])
def test_cpp_bench_driver_vs_reference(flags, tol):
    """The reference's own host driver (bench.cpp run_bench, unmodified) linked
    against the B200 engine drop-in vs the same driver linked against the
    reference engine, same flags: loss and gradient checksum agree; the report
    schema is the reference's."""
    import json
    b200, cpu = _drivers()
    common = ["--reps", "1", "--warmup", "1"]
    r1, r2 = _run([b200] + flags + common), _run([cpu] + flags + common)
    assert r1.returncode == 0, r1.stderr
    assert r2.returncode == 0, r2.stderr
    ours, ref = json.loads(r1.stdout), json.loads(r2.stdout)
    assert ours["config"] == ref["config"]
    o, r = ours["results"], ref["results"]
    scale = max(1.0, abs(r["loss"]))
    assert abs(o["loss"] - r["loss"]) <= tol * scale, (o["loss"], r["loss"])
    assert abs(o["gradient_checksum"] - r["gradient_checksum"]) <= tol * max(1.0, abs(r["gradient_checksum"]))
    assert o["throughput_sps"] > 0


def test_cpp_bench_driver_cli():
    """Self-test (the reference's JSON/CSV serialisers round-trip this build's
    reports), scan-blocks, exit codes (qfuse_bench_main.cpp:110-116), --gpus 1
    (qf_gradient_c64_multi path) and --device."""
    import json
    b200, _ = _drivers()
    r = _run([b200, "--selftest"])
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
    r = _run([b200, "--qubits", "16", "--layers", "20", "--batch", "8", "--block", "10",
              "--reps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["config"]["qubits"] == 16 and rep["results"]["throughput_sps"] > 0
    single = rep["results"]
    r = _run([b200, "--qubits", "16", "--layers", "20", "--batch", "8", "--block", "10",
              "--reps", "1", "--warmup", "0", "--gpus", "1"])
    assert r.returncode == 0, r.stderr
    multi = json.loads(r.stdout)["results"]
    assert abs(multi["loss"] - single["loss"]) <= 1e-12 * max(1.0, abs(single["loss"]))
    r = _run([b200, "--qubits", "6", "--layers", "8", "--batch", "2", "--scan-blocks", "1,2,4",
              "--format", "csv", "--device", "0"])
    assert r.returncode == 0 and len(r.stdout.strip().splitlines()) == 4, r.stdout + r.stderr
    assert _run([b200, "--qubits", "4", "--layers", "3", "--block", "2"]).returncode == 2
    assert _run([b200, "--bogus"]).returncode == 2
    assert _run([b200, "--qubits", "30", "--layers", "2", "--batch", "1024"]).returncode == 3


def test_golden_state_exchange_qsv1(tmp_path):
    """Golden-state exchange in the reference's QSV1 format: the B200 driver
    writes forward<float> final states with the reference's dump_state, the
    CPU-reference driver loads them with load_state and checks them against its
    own forward<float> (statevec.cpp:122-186, engine.hpp:131-133); and back."""
    b200, cpu = _drivers()
    g1, g2 = str(tmp_path / "b200.qsv"), str(tmp_path / "ref.qsv")
    wl = ["--qubits", "14", "--layers", "6", "--batch", "3"]
    r = _run([b200] + wl + ["--golden-out", g1])
    assert r.returncode == 0, r.stderr
    r = _run([cpu] + wl + ["--golden-check", g1, "--golden-out", g2])
    assert r.returncode == 0, r.stdout + r.stderr
    r = _run([b200] + wl + ["--golden-check", g2])
    assert r.returncode == 0, r.stdout + r.stderr
    with open(g1, "rb") as f:
        assert f.read(4) == b"QSV1"


def test_config3_depth_subset_vs_oracle(ctx, oracle):
    """BASELINE config 3 shape (16q x 200 layers, k = 10) on a 2-sample subset of
    the batch against the fp64 oracle: the compiled layout-A/B programs, the Z
    chain over 200 stages and the re-anchoring, at the stated 1e-4."""
    n, layers, batch = 16, 200, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=1234)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_config4_shape_vs_oracle(ctx, oracle):
    """BASELINE config 4 register (20 qubits) at 40 layers, k = 10, one sample,
    against the fp64 oracle (the full 1000 layers are cross-checked against the
    per-gate path in test_config4_depth_fused_vs_pergate)."""
    n, layers, batch = 20, 40, 1
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=1234)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_config2_depth_vs_oracle(ctx, oracle):
    """BASELINE config 2 shape (12q x 100 layers, k = 10) on a 4-sample subset:
    the chained sample-resident kernel over 100 stages with 10 slot splits,
    against the fp64 oracle."""
    n, layers, batch = 12, 100, 4
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=1234)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("n,k", [(17, 10), (18, 10), (19, 10), (17, 5), (19, 5)])
def test_hea_17_19_deep_vs_oracle(ctx, oracle, n, k):
    """HEA n = 17..19 (streaming, layouts A/B with 5..7 top qubits rotated in
    B) at 20 layers against the fp64 oracle: k = 10 runs the balanced backward
    (kProgAlt / kProgAltP), k = 5 (odd slot period) the plain one (kProgA /
    kProgB20P)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, 20, 1, seed=300 + n)
    res = capi.gradient_c64(ctx, gates, n, npar, 20, k, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


# ---- balanced backward at n = 20 (Plan::alt, qf_plan.cpp / DESIGN.md §4): the
# column group's Ry undone by the pass that undoes D_s, slots after layout-A passes
@pytest.mark.parametrize("layers,k,batch,storage", [
    (6, 2, 2, "full"),      # balanced (even slot period)
    (9, 3, 1, "full"),      # odd slot period: plain backward
    (10, 2, 1, "memsave"),  # balanced + bf16 slots
    (7, 0, 1, "full"),      # default k (min(stages, 10) = 7: odd)
    (4, 4, 2, "full"),      # one slot block
])
def test_balanced_backward_20q(ctx, oracle, layers, k, batch, storage):
    n = 20
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=900 + layers)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli, storage=storage)
    ref = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    if storage == "memsave":
        assert rel_diff(res.gradient, ref[1]) <= MEMSAVE_TOL
    else:
        _check(res, ref)


def test_balanced_backward_matches_plain(ctx, monkeypatch):
    """The balanced and the plain backward schedules (QF_ALT=0) are the same
    gradient up to fp32 rounding (20q x 40 layers, k = 10)."""
    n, layers = 20, 40
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 2, seed=31)

    def run():  # a fresh plan: QF_ALT is read by the planner
        plan = capi.Plan(ctx, gates, n, npar, layers, 10, 2, pauli)
        plan.upload_psi0(psi0)
        return plan.gradient(theta)
    a = run()
    monkeypatch.setenv("QF_ALT", "0")
    b = run()
    assert rel_diff(a.gradient, b.gradient) <= 1e-5
    assert rel_diff(a.expect, b.expect) == 0.0  # same forward schedule


def test_balanced_backward_ragged_alias_memsave(ctx, oracle):
    """n = 20 balanced backward on a plan with a ragged batch (3 samples), psi0
    aliased from caller device memory, MemSave slots, two gradients on the same
    plan (the second with a new theta)."""
    import torch
    n, layers, batch = 20, 6, 3
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=77)
    plan = capi.Plan(ctx, gates, n, npar, layers, 2, batch, pauli, storage="memsave")
    dev = torch.from_numpy(psi0.reshape(-1).copy()).to("cuda")
    torch.cuda.synchronize()
    plan.set_psi0_device(dev.data_ptr())
    for th in (theta, C.random_parameters(npar, 4242)):
        res = plan.gradient(th)
        loss, grad, exp = oracle.gradient(gates, n, npar, psi0, th, pauli)
        assert rel_diff(res.gradient, grad) <= MEMSAVE_TOL
        assert rel_diff(res.expect, exp) <= TOL  # the final state stays complex64
    plan.close()


def test_balanced_backward_run_to_run_identical(ctx):
    """Acceptance C11 (acceptance.cpp:501-530) on the 20q balanced schedule: two
    gradients of the same plan are bit-identical (fixed-order fp64 reductions)."""
    n, layers, batch = 20, 10, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=11)
    plan = capi.Plan(ctx, gates, n, npar, layers, 2, batch, pauli)
    plan.upload_psi0(psi0)
    a = plan.gradient(theta)
    b = plan.gradient(theta)
    assert np.array_equal(a.gradient, b.gradient) and a.loss == b.loss
    assert np.array_equal(a.expect, b.expect)
    plan.close()
