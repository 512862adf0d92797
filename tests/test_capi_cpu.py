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
