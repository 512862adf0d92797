"""compute-sanitizer workload (run under memcheck / racecheck / synccheck):
one fused gradient per path on small configurations — sample-resident (n = 10,
and n = 12 with chained stages and checkpoint splits), streaming with the
compiled programs (register K accumulation) and the generic kernels (n = 14, 16,
20, including the balanced backward), MemSave slots, the per-gate path, complex128 fused segments (several
segments, off-tile CNOT controls) and per-gate, and a one-device NCCL group."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_02804_b200 as qf  # noqa: E402
from paper_2603_02804_b200 import circuits as C  # noqa: E402

ctx = qf.Context(0)
for n, layers, batch, k, storage in [(10, 4, 3, 2, "full"), (12, 5, 2, 1, "full"), (12, 6, 2, 2, "full"),
                                     (14, 4, 1, 2, "full"), (16, 4, 1, 2, "full"), (16, 4, 1, 1, "memsave"),
                                     (20, 2, 1, 1, "full"), (20, 4, 1, 2, "full"), (20, 4, 1, 2, "memsave")]:
    gates, M = C.build_hea(n, layers)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    r = qf.gradient_c64(ctx, gates, n, M, layers, k, C.new_random_state(n, batch, 1),
                        C.random_parameters(M, 2), pauli, storage=storage)
    assert np.all(np.isfinite(r.gradient))
gates, M = C.random_circuit(9, 40, 3)
pauli = C.parse_pauli(C.repeated_ixyz_label(9))
qf.gradient_c64(ctx, gates, 9, M, 0, 0, C.new_random_state(9, 2, 1), C.random_parameters(M, 2), pauli,
                pergate=True)
qf.gradient_c128(ctx, gates, 9, M, 0, 0, C.new_random_state(9, 2, 1, np.float64),
                 C.random_parameters(M, 2), pauli)
gates, M = C.random_circuit(14, 80, 5)
pauli = C.parse_pauli(C.repeated_ixyz_label(14))
for pg in (False, True):
    qf.gradient_c128(ctx, gates, 14, M, 0, 0, C.new_random_state(14, 2, 1, np.float64),
                     C.random_parameters(M, 2), pauli, pergate=pg)
gates, M = C.build_hea(20, 2)  # complex128 register rounds at m = 11
pauli = C.parse_pauli(C.repeated_ixyz_label(20))
qf.gradient_c128(ctx, gates, 20, M, 2, 0, C.new_random_state(20, 1, 1, np.float64),
                 C.random_parameters(M, 2), pauli)
gates, M = C.build_hea(6, 3)
qf.gradient_c64_multi(1, gates, 6, M, 3, 1, C.new_random_state(6, 3, 1), C.random_parameters(M, 2),
                      C.parse_pauli(C.repeated_ixyz_label(6)))
print("sanitize workload ok")
