"""CPU: the C-ABI library loads and exports every entry point declared in
include/qfuse_b200.h (no compute without a GPU)."""
import ctypes
import os
import re

import paper_2603_02804_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "qfuse_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qf_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = pkg.load()
    declared = _declared()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(pkg.SYMBOLS) == set(declared)


def test_version_and_no_device_error():
    lib = pkg.load()
    assert b"sm_100a" in lib.qf_version()
    h = ctypes.c_void_p()
    rc = lib.qf_ctx_create(0, ctypes.byref(h))
    if rc == 0:  # a B200 is visible (GPU box)
        assert lib.qf_ctx_destroy(h) == 0
    else:        # no device here: a clean error, never a crash or a CPU fallback
        assert rc == pkg.capi.QF_EDEVICE or rc == pkg.capi.QF_EINVAL
        assert lib.qf_last_error()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_group_api_without_device():
    """The single-process multi-GPU entry points fail cleanly without a GPU
    (no crash, no CPU fallback): invalid n_gpus is rejected before any device
    or NCCL work; on the GPU box a real group is covered by test_gpu_multi."""
    lib = pkg.load()
    h = ctypes.c_void_p()
    assert lib.qf_group_create(0, None, ctypes.byref(h)) in (pkg.capi.QF_EINVAL, pkg.capi.QF_EDEVICE)
    assert lib.qf_last_error()
    assert lib.qf_group_size(None) == 0
    assert lib.qf_group_destroy(None) == 0
    st = pkg.capi.QfStats()
    assert lib.qf_plan_last_stats(None, ctypes.byref(st)) == pkg.capi.QF_EINVAL


def test_python_binding_validates_shapes():
    """The one-shot wrappers check psi0 / theta sizes before the C side reads
    batch * 2^(n+1) floats and n_params doubles from them (no device needed)."""
    import numpy as np
    import pytest
    from paper_2603_02804_b200 import circuits as C
    gates, npar = C.build_hea(4, 2)
    pauli = C.parse_pauli("IXYZ")
    theta = C.random_parameters(npar, 1)
    flat = np.zeros(2 * 32 + 3, np.float32)  # not a whole number of 4-qubit samples
    for fn in (pkg.capi.gradient_c64, pkg.capi.gradient_c64_multi):
        args = (gates, 4, npar, 2, 0)
        with pytest.raises(pkg.capi.QfInvalidArgument):
            if fn is pkg.capi.gradient_c64:
                fn(None, *args, flat, theta, pauli)
            else:
                fn(1, *args, flat, theta, pauli)
    good = C.new_random_state(4, 2, 1)
    with pytest.raises(pkg.capi.QfInvalidArgument):
        pkg.capi.gradient_c64(None, gates, 4, npar, 2, 0, good, theta[:-1], pauli)
    with pytest.raises(pkg.capi.QfInvalidArgument):
        pkg.capi.gradient_c128(None, gates, 4, npar, 2, 0, good.astype(np.float64)[:, :5], theta, pauli)


# ---- the planner, host only (qf_plan_describe): the schedule decisions of DESIGN.md §3-4
def _describe(n, layers, k, batch=4):
    from paper_2603_02804_b200 import capi
    from paper_2603_02804_b200 import circuits as C
    gates, npar = C.build_hea(n, layers)
    return capi.describe_plan(gates, n, npar, layers, k, batch, C.parse_pauli(C.repeated_ixyz_label(n)))


def test_plan_hea20q_schedule():
    """hea20q (config 4's shard): one pass per stage plus the closing pass, the
    balanced backward with slots after layout-A passes, every interior pass on a
    compiled program, the wide kernel for the layout-A forwards, and the
    algorithmic bytes the bench's roofline uses (fwd 2S, bwd 4S / 3S, observable 2S)."""
    d = _describe(20, 1000, 10, batch=125)
    assert d["resident"] == 0 and d["layouts"] == 2 and d["stages"] == 1000
    assert d["passes"] == 1001 and d["ckpt_passes"] == 10 and d["slots"] == 101
    assert d["balanced"] == 1
    assert d["wide_forward"] == 499  # interior layout-A passes (not the first, not the last)
    assert d["compiled_forward"] >= 999 and d["compiled_backward"] >= 998
    S = 8 << 20
    # no psi store (3S): the 100 passes right after a slot (psi re-read from the slot)
    # and the last backward pass (pass 0: nothing reads its psi)
    no_store = 101
    assert d["bytes_per_sample"] == S * (2 * 1001 + 4 * (1001 - no_store) + 3 * no_store + 2)


def test_plan_balanced_backward_conditions():
    assert _describe(20, 12, 3)["balanced"] == 0   # odd slot period
    assert _describe(19, 20, 10)["balanced"] == 1  # partial rows in layout B
    assert _describe(17, 20, 10)["balanced"] == 1
    assert _describe(16, 20, 10)["balanced"] == 0  # 13..16: the column group moved to B instead
    d22 = _describe(22, 4, 2)
    assert d22["layouts"] == 3 and d22["balanced"] == 0


def test_plan_compiled_programs_cover_interior_passes():
    """13 <= n <= 19 (partial-row layout B) and n = 16: every pass but the first
    and last runs a compiled straight-line program in both directions."""
    for n in (13, 14, 15, 16, 17, 18, 19, 20):
        d = _describe(n, 20, 10)
        assert d["passes"] == 21, n
        assert d["compiled_forward"] >= d["passes"] - 2, (n, d)
        assert d["compiled_backward"] >= d["passes"] - 3, (n, d)  # stage-0 Z passes excluded


def test_plan_resident_and_errors():
    from paper_2603_02804_b200 import capi
    d = _describe(12, 100, 10, batch=1024)
    assert d["resident"] == 1 and d["stages"] == 100 and d["slots"] == 9
    assert d["bytes_per_sample"] == (8 << 12) * (1 + 2 * 9)
    import pytest
    with pytest.raises(capi.QfInvalidArgument):
        _describe(12, 100, 7)  # CheckpointPlan::uniform: 7 does not divide 100
