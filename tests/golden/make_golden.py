"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref, built
from /root/reference/proj/src). Run here (the reference is not on the GPU
box); the JSON it writes is committed and read by the tests.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import RefLib  # noqa: E402


def hea_case(ref, name, n, layers, batch, label=None, block=0, seed=1234, precision="f64"):
    gates, npar = ref.build_hea(n, layers)
    theta = ref.random_parameters(npar, seed + 1)
    dt = np.float64 if precision == "f64" else np.float32
    psi0 = ref.random_state(n, batch, seed, dt)
    pauli = ref.parse_pauli(label or "".join("IXYZ"[i % 4] for i in range(n)))
    loss, grad, exp = ref.gradient(gates, n, npar, psi0, theta, pauli, layers=layers,
                                   block_layers=block, expect=True)
    return {"name": name, "kind": "hea", "n": n, "layers": layers, "batch": batch,
            "seed": seed, "label": label or "IXYZ", "block": block, "precision": precision,
            "x_mask": pauli[0], "z_mask": pauli[1], "y_count": pauli[2],
            "theta0": float(theta[0]), "psi0_00": [float(psi0[0, 0, 0]), float(psi0[0, 0, 1])],
            "loss": loss, "expect": exp.tolist(), "grad": grad.tolist()}


def random_case(ref, name, n, ngates, seed):
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2603_02804_b200 import circuits as C
    gates, npar = C.random_circuit(n, ngates, seed)
    theta = ref.random_parameters(npar, seed + 100)
    psi0 = ref.random_state(n, 3, seed + 200, np.float64)
    pauli = ref.parse_pauli("".join("IXYZ"[i % 4] for i in range(n)))
    loss, grad, exp = ref.gradient(gates, n, npar, psi0, theta, pauli, expect=True)
    shift = ref.parameter_shift(gates, n, npar, psi0, theta, pauli)
    return {"name": name, "kind": "random", "n": n, "ngates": ngates, "seed": seed,
            "gates": [[int(g["kind"]), int(g["axis"]), int(g["q0"]), int(g["q1"]),
                       int(g["param"])] for g in gates],
            "x_mask": pauli[0], "z_mask": pauli[1], "loss": loss, "expect": exp.tolist(),
            "grad": grad.tolist(), "param_shift": shift.tolist()}


def main():
    ref = RefLib()
    cases = [
        hea_case(ref, "config1_ixyz", 4, 4, 8),
        hea_case(ref, "config1_zzzz", 4, 4, 8, label="ZZZZ"),
        hea_case(ref, "config1_iiiz", 4, 4, 8, label="IIIZ"),
        hea_case(ref, "hea6x8_ckpt2", 6, 8, 2, block=2, seed=13),
        hea_case(ref, "hea12x3", 12, 3, 2, seed=99),
        hea_case(ref, "hea14x2_f32", 14, 2, 1, seed=7, precision="f32"),
        random_case(ref, "random5x40", 5, 40, 11),
        random_case(ref, "random7x60", 7, 60, 12),
    ]
    with open(os.path.join(HERE, "golden_reference.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference qfuse via oracle/_ref)",
                   "cases": cases}, f, indent=1)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
