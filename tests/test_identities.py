"""CPU checks (numpy, fp64) of the algebra the sm_100a kernels rely on, stated
in DESIGN.md §2-§3. They pin the derivations independently of the GPU:

* gradients from three numbers per (stage, qubit): X, Y, Z = Im<lam|sigma|psi>
  reproduce the reference's Re<lam|dg|psi_in> for Rx/Ry/Rz (engine.cpp:207-256);
* the Z chain: Z just before Ry_s(q) = cos(b) Z - sin(b) X measured just before
  Ry_{s-1}(q), through any diagonal and any gates on other qubits;
* scale folding: unscaled rotations [[1, -t], [t, 1]] with the product of the
  factored cosines moved into the diagonal give the exact pass output, and a K
  measured on tiles off by a factor f is f^2 times the true one.
"""
import numpy as np

RNG = np.random.default_rng(7)
I2 = np.eye(2)
SX = np.array([[0, 1], [1, 0]], complex)
SY = np.array([[0, -1j], [1j, 0]], complex)
SZ = np.array([[1, 0], [0, -1]], complex)


def rot(axis, theta):  # circuit.cpp:61-73: cos(t/2) I - i sin(t/2) P
    P = {"x": SX, "y": SY, "z": SZ}[axis]
    return np.cos(theta / 2) * I2 - 1j * np.sin(theta / 2) * P


def on_qubit(U, q, n):
    """2x2 U on qubit q of an n-qubit register (qubit q = bit q of the index)."""
    out = np.array([[1.0 + 0j]])
    for k in reversed(range(n)):
        out = np.kron(out, U if k == q else I2)
    return out


def rand_state(n):
    v = RNG.normal(size=1 << n) + 1j * RNG.normal(size=1 << n)
    return v / np.linalg.norm(v)


def rand_diagonal(n):
    """phases on every qubit plus a CZ ring: the stage diagonal D_s."""
    x = np.arange(1 << n)
    ph = np.zeros(1 << n)
    for q in range(n):
        ph += RNG.uniform(0, 2 * np.pi) * ((x >> q) & 1)
    sign = np.ones(1 << n)
    for q in range(n):
        r = (q + 1) % n
        sign *= np.where(((x >> q) & 1) & ((x >> r) & 1), -1.0, 1.0)
    return np.diag(sign * np.exp(1j * ph))


def measure(psi, lam, q, n):
    return {m: np.imag(np.vdot(lam, on_qubit(S, q, n) @ psi)) for m, S in
            (("x", SX), ("y", SY), ("z", SZ))}


def test_three_numbers_give_every_rotation_gradient():
    """grad = Re<lam_out|dg|psi_in> (engine.cpp:207-256) = 1/2 Im<lam|P|psi> at the
    gate (dg = -(i/2) P g; P commutes with g, so either side of it)."""
    n, q = 4, 2
    for axis, S in (("x", SX), ("y", SY), ("z", SZ)):
        psi_in, lam_out = rand_state(n), rand_state(n)
        th = RNG.uniform(0, 2 * np.pi)
        g = on_qubit(rot(axis, th), q, n)
        dg = on_qubit(-0.5 * np.sin(th / 2) * I2 - 0.5j * np.cos(th / 2) * S, q, n)
        ref = np.real(np.vdot(lam_out, dg @ psi_in))
        assert abs(ref - 0.5 * measure(g @ psi_in, lam_out, q, n)[axis]) < 1e-12
        assert abs(ref - 0.5 * measure(psi_in, g.conj().T @ lam_out, q, n)[axis]) < 1e-12
    # and the adjoint itself: d/dt <psi|Ry^dag O Ry|psi> with lam = 2 O Ry psi
    psi = rand_state(n)
    O = on_qubit(SZ, 0, n) @ on_qubit(SX, 3, n)
    th = 0.37
    f = lambda t: np.real(np.vdot(on_qubit(rot("y", t), q, n) @ psi, O @ on_qubit(rot("y", t), q, n) @ psi))
    fd = (f(th + 1e-6) - f(th - 1e-6)) / 2e-6
    lam = 2 * O @ on_qubit(rot("y", th), q, n) @ psi
    assert abs(0.5 * measure(on_qubit(rot("y", th), q, n) @ psi, lam, q, n)["y"] - fd) < 1e-8


def test_z_chain_identity():
    n, q = 5, 1
    psi, lam = rand_state(n), rand_state(n)  # forward-order state / adjoint before Ry_{s-1}(q)
    b = RNG.uniform(0, np.pi)
    V0 = measure(psi, lam, q, n)
    # Ry_{s-1}(q), then the stage diagonal and rotations on the other qubits
    G = on_qubit(rot("y", b), q, n)
    G = rand_diagonal(n) @ G
    for k in range(n):
        if k != q:
            G = on_qubit(rot("y", RNG.uniform(0, np.pi)), k, n) @ G
    V1 = measure(G @ psi, G @ lam, q, n)  # just before Ry_s(q)
    assert abs(V1["z"] - (np.cos(b) * V0["z"] - np.sin(b) * V0["x"])) < 1e-12
    # X and Y are NOT invariant through the diagonal (they must be measured)
    assert abs(V1["y"] - V0["y"]) > 1e-6


def test_scale_folding_and_k_correction():
    n = 4
    psi, lam = rand_state(n), rand_state(n)
    betas = RNG.uniform(0, np.pi, size=n)
    c, s = np.cos(betas / 2), np.sin(betas / 2)
    D = rand_diagonal(n)
    exact, unscaled = psi.copy(), psi.copy()
    for q in range(n):  # round 0 on every qubit, exact vs factored-unscaled
        exact = on_qubit(rot("y", betas[q]), q, n) @ exact
        unscaled = on_qubit(np.array([[1, -s[q] / c[q]], [s[q] / c[q], 1]]), q, n) @ unscaled
    F = np.prod(c)
    assert np.allclose(F * unscaled, exact, atol=1e-12)
    # the diagonal absorbs F: D (F * unscaled) == (D F) unscaled
    assert np.allclose((D * F) @ unscaled, D @ exact, atol=1e-12)
    # a K measured on tiles that are off by f carries f^2: kc = 1/f^2 restores it
    f = 1.0 / F
    V_true, V_scaled = measure(psi, lam, 2, n), measure(f * psi, f * lam, 2, n)
    for m in "xyz":
        assert abs(V_scaled[m] / f ** 2 - V_true[m]) < 1e-12


def test_bf16_narrowing_matches_reference_rule():
    """qf_store.cu narrow_kernel: statevec.hpp:36-45 bit for bit (RNE, NaN quieted)."""
    def narrow(v):
        u = np.array([v], np.float32).view(np.uint32)[0].item()
        if (u & 0x7FFFFFFF) > 0x7F800000:
            return (u >> 16) | 0x0040
        return ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFFFFFF) >> 16
    def widen(b):
        return np.array([b << 16], np.uint32).view(np.float32)[0]
    for v in [1.0, -2.5, 1.00390625, 1.01171875, 3.0e38, 1e-40, np.float32(np.nan), 0.0]:
        b = narrow(v)
        w = widen(b)
        if np.isnan(v):
            assert np.isnan(w)
        else:
            assert abs(w - v) <= abs(v) * 2.0 ** -8 or abs(v) < 1e-38
    assert narrow(1.00390625) == 0x3F80  # tie -> even
    assert narrow(1.01171875) == 0x3F82  # tie -> even (up)
    assert np.isinf(widen(narrow(3.4e38)))  # overflow rounds to infinity
