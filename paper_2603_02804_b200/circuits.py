"""Host-side circuit/ansatz/observable helpers — the reference's C++ host API
(proj/src/circuit.cpp, statevec.cpp) restated for Python callers of the
C-ABI. These build inputs; all simulation happens in libqfuse_b200.so.

  build_hea             circuit.cpp:89-114
  repeated_ixyz_label   circuit.cpp:205-212
  parse_pauli           circuit.cpp:158-192 (leftmost char = qubit n-1)
  random_parameters     circuit.cpp:214-221 (SplitMix64, bits.hpp:38-57)
  new_random_state      statevec.cpp:32-53 (one SplitMix64 stream, Box-Muller)
  random_circuit        tests/test_engine.cpp:28-47
"""
from __future__ import annotations

import numpy as np

GATE_DTYPE = np.dtype(
    [("kind", np.uint8), ("axis", np.uint8), ("pad", np.uint16), ("q0", np.uint32),
     ("q1", np.uint32), ("param", np.uint32)], align=True)
assert GATE_DTYPE.itemsize == 16

ROT, CZ, CNOT = 0, 1, 2
X, Y, Z = 0, 1, 2

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix_draws(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of SplitMix64(seed) (jump-ahead, bits.hpp:44-49)."""
    j = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + j * _GOLDEN
    return _mix(st)


def random_parameters(count: int, seed: int) -> np.ndarray:
    z = splitmix_draws(seed, 0, count)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 * 3.14159265358979323846


def new_random_state(n_qubits: int, batch: int, seed: int, dtype=np.float32) -> np.ndarray:
    """(batch, 2^n, 2) array; generation and normalisation in float64."""
    dim = 1 << n_qubits
    out = np.empty((batch, dim, 2), dtype)
    for s in range(batch):
        z = splitmix_draws(seed, 2 * s * dim, 2 * dim)
        u1 = ((z[0::2] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
        u2 = (z[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        r = np.sqrt(-2.0 * np.log(u1))
        t = 2.0 * 3.14159265358979323846 * u2
        re, im = r * np.cos(t), r * np.sin(t)
        inv = 1.0 / np.sqrt(np.cumsum(re * re + im * im)[-1])  # sequential, statevec.cpp:40-46
        out[s, :, 0] = re * inv
        out[s, :, 1] = im * inv
    return out


def build_hea(n_qubits: int, layers: int):
    """Returns (gates, n_params)."""
    if n_qubits < 2:
        raise ValueError("build_hea: need at least 2 qubits")
    if layers == 0:
        raise ValueError("build_hea: need at least 1 layer")
    ents = 1 if n_qubits == 2 else n_qubits
    per = 3 * n_qubits + ents
    g = np.zeros(layers * per, GATE_DTYPE)
    q = np.arange(n_qubits, dtype=np.uint32)
    for l in range(layers):
        base = l * per
        rot = g[base:base + 3 * n_qubits]
        rot["kind"] = ROT
        rot["axis"] = np.tile(np.array([X, Y, Z], np.uint8), n_qubits)
        rot["q0"] = np.repeat(q, 3)
        rot["param"] = np.arange(3 * n_qubits * l, 3 * n_qubits * (l + 1), dtype=np.uint32)
        cz = g[base + 3 * n_qubits:base + per]
        cz["kind"] = CZ
        if n_qubits == 2:
            cz["q0"], cz["q1"] = 0, 1
        else:
            cz["q0"] = q
            cz["q1"] = (q + 1) % n_qubits
    return g, 3 * n_qubits * layers


def repeated_ixyz_label(n_qubits: int) -> str:
    return "".join("IXYZ"[i % 4] for i in range(n_qubits))


def parse_pauli(label: str, expected_n: int = 0):
    """Returns (x_mask, z_mask, y_count)."""
    if not label:
        raise ValueError("parse_pauli: empty label")
    if expected_n and len(label) != expected_n:
        raise ValueError(f"parse_pauli: label length {len(label)} does not match qubit count "
                         f"{expected_n}")
    n = len(label)
    x = z = 0
    for i, ch in enumerate(label):
        bit = 1 << (n - 1 - i)
        if ch == "X":
            x |= bit
        elif ch == "Y":
            x |= bit
            z |= bit
        elif ch == "Z":
            z |= bit
        elif ch != "I":
            raise ValueError(f"parse_pauli: invalid character {ch!r}")
    return x, z, bin(x & z).count("1")


def random_circuit(n_qubits: int, n_gates: int, seed: int):
    """Random Rx/Ry/Rz/CZ/CNOT circuit (tests/test_engine.cpp:28-47 scheme)."""
    state = [np.uint64(seed)]

    def nxt():
        with np.errstate(over="ignore"):
            state[0] = state[0] + _GOLDEN
        return int(_mix(np.array([state[0]], np.uint64))[0])

    g = np.zeros(n_gates, GATE_DTYPE)
    param = 0
    for i in range(n_gates):
        kind = nxt() % 5
        if kind < 3:
            g[i]["kind"] = ROT
            g[i]["axis"] = kind
            g[i]["q0"] = nxt() % n_qubits
            g[i]["param"] = param
            param += 1
        else:
            c = nxt() % n_qubits
            t = nxt() % (n_qubits - 1)
            if t >= c:
                t += 1
            g[i]["kind"] = CZ if kind == 3 else CNOT
            g[i]["q0"], g[i]["q1"] = c, t
    return g, param
