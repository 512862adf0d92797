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
    (13, 2, 2), (14, 3, 2), (16, 2, 1),  # streaming passes A + B
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


@pytest.mark.parametrize("n,layers,batch", [(4, 3, 5), (12, 2, 2), (12, 5, 3), (14, 2, 2), (17, 2, 1)])
def test_forward_state_matches_reference(ctx, ref, n, layers, batch):
    """Final state of the fused forward vs the reference's forward<double>,
    up to one global phase per sample (the device drops e^{i delta})."""
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=41)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    plan.upload_psi0(psi0)
    got = plan.forward_state(theta).astype(np.float64)
    want = ref.forward(gates, n, npar, psi0.astype(np.float64), theta)
    g = got[..., 0] + 1j * got[..., 1]
    w = want[..., 0] + 1j * want[..., 1]
    for s in range(batch):
        ov = np.vdot(g[s], w[s])
        assert abs(abs(ov) - 1.0) < 1e-5
        ph = ov / abs(ov)
        assert np.max(np.abs(g[s] * ph - w[s])) < 1e-5


@pytest.mark.parametrize("n,layers,batch", [(21, 1, 1), (22, 2, 1)])
def test_three_layouts(ctx, oracle, n, layers, batch):
    """n > 20 needs a third layout (two passes per stage)."""
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=8)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_streaming_checkpoint_slots(ctx, oracle, k):
    n, layers = 15, 6
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 2, seed=17)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, k, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_device_random_state(ctx):
    """qf_plan_random_psi0 == new_random_state<float> (statevec.cpp:32-53)."""
    n, batch = 13, 3
    gates, npar = C.build_hea(n, 1)
    plan = capi.Plan(ctx, gates, n, npar, 1, 0, batch, C.parse_pauli("Z" * n))
    plan.random_psi0(1234, first_sample=5)
    host = np.empty((batch, 1 << n, 2), np.float32)
    plan.download_psi0_ptr(host.ctypes.data)
    want = C.new_random_state(n, 5 + batch, 1234)[5:]
    np.testing.assert_allclose(host, want, rtol=0, atol=2e-7)


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
    """qf_plan_set_psi0_device + qf_plan_gradient_device (the data-parallel path)."""
    torch = pytest.importorskip("torch")
    n, layers, batch = 13, 2, 3
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=12)
    plan = capi.Plan(ctx, gates, n, npar, layers, 0, batch, pauli)
    d_psi = torch.from_numpy(psi0).cuda()
    d_theta = torch.from_numpy(theta).cuda()
    out = torch.empty(npar + 1 + batch, dtype=torch.float64, device="cuda")
    plan.set_psi0_device(d_psi.data_ptr())
    plan.gradient_device(d_theta.data_ptr(), out.data_ptr())
    plan.synchronize()
    o = out.cpu().numpy()
    loss, grad, exp = oracle.gradient(gates, n, npar, psi0, theta, pauli)
    assert rel_diff(o[:npar], grad) <= TOL
    assert abs(o[npar] - loss) <= TOL * max(1.0, float(np.sum(np.abs(exp))))
    assert rel_diff(o[npar + 1:], exp) <= TOL


def test_deep_circuit_uncompute_drift(ctx, oracle):
    """200 layers of uncompute with re-anchoring every 10: fp32 stays within tolerance."""
    n, layers = 13, 200
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, 1, seed=77)
    res = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    _check(res, oracle.gradient(gates, n, npar, psi0, theta, pauli))


def test_config4_depth_fused_vs_pergate(ctx):
    """BASELINE config 4 depth (20q x 1000 layers, k = 10) on a 2-sample shard:
    the fused path (X, Y measured, Z chained over 1000 stages, scales folded
    into the diagonals) against the independent per-gate comparator (one
    kernel per gate, 80,000 gates each way). The CPU oracle would need ~10 min
    here, so this is the size-independent cross-check at full depth."""
    n, layers, batch = 20, 1000, 2
    gates, npar, theta, psi0, pauli = _hea_case(n, layers, batch, seed=4242)
    fused = capi.gradient_c64(ctx, gates, n, npar, layers, 10, psi0, theta, pauli)
    pg = capi.gradient_c64(ctx, gates, n, npar, layers, 0, psi0, theta, pauli, pergate=True)
    err = rel_diff(fused.gradient, pg.gradient)
    assert err <= TOL, err
    assert rel_diff(fused.expect, pg.expect) <= TOL
    assert np.all(np.isfinite(fused.gradient))


# ---- StorageMode::MemSave (bf16 checkpoint slots), acceptance C10 bound
MEMSAVE_TOL = 5e-3  # acceptance.cpp:466-499 (bf16 storage vs fp32)


@pytest.mark.parametrize("n,layers,batch,k", [(14, 6, 2, 1), (16, 8, 2, 2), (20, 4, 1, 1)])
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


def test_cpp_bench_driver():
    """qfuse::b200::run_bench / scan_blocks (the reference's bench API on the B200)
    against the reference's run_bench on the same BenchConfig; the reference's
    JSON/CSV serialisers round-trip our BenchReport; the CLI prints its JSON."""
    import json
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "tests", "bench_driver")
    if not os.path.exists(exe):
        pytest.skip("build/tests/bench_driver not built (needs the reference sources at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
    r = subprocess.run([exe, "--qubits", "16", "--layers", "20", "--batch", "8", "--block", "10",
                        "--reps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["config"]["qubits"] == 16 and rep["results"]["throughput_sps"] > 0
    r = subprocess.run([exe, "--qubits", "4", "--layers", "3", "--block", "2"],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 2  # config error exit code (qfuse_bench_main.cpp:110-116)


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
