"""ctypes binding of the C-ABI (include/qfuse_b200.h).

The product path is the in-tree ``libqfuse_b200.so`` (CUDA sm_100a). There is
no CPU fallback: if the library is missing, or no B200 is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .circuits import GATE_DTYPE

HERE = os.path.dirname(os.path.abspath(__file__))
# QFUSE_B200_LIB: alternative build of the same library (ablation experiments)
LIB_PATH = os.environ.get("QFUSE_B200_LIB") or os.path.join(HERE, "libqfuse_b200.so")

QF_OK, QF_EINVAL, QF_ECAPACITY, QF_EDEVICE = 0, 2, 3, 4

# exported symbols, in include/qfuse_b200.h order
SYMBOLS = (
    "qf_last_error", "qf_version", "qf_ctx_create", "qf_ctx_destroy", "qf_ctx_set_hbm_limit",
    "qf_ctx_set_plan_cache",
    "qf_gradient_c64", "qf_gradient_c64_ex", "qf_gradient_pergate_c64", "qf_forward_c64",
    "qf_gradient_c128",
    "qf_gradient_pergate_c128",
    "qf_plan_create",
    "qf_plan_create_ex", "qf_plan_destroy", "qf_plan_describe",
    "qf_plan_upload_psi0", "qf_plan_set_psi0_device", "qf_plan_gradient",
    "qf_plan_gradient_device", "qf_plan_gradient_pergate", "qf_plan_forward_state",
    "qf_plan_stream", "qf_plan_synchronize", "qf_plan_traffic", "qf_plan_random_psi0", "qf_plan_download_psi0",
    "qf_plan_set_profiling", "qf_plan_profile", "qf_plan_last_stats",
    "qf_group_create", "qf_group_destroy", "qf_group_size", "qf_group_plan_create",
    "qf_group_plan_destroy", "qf_group_plan_upload_psi0", "qf_group_plan_random_psi0",
    "qf_group_plan_gradient", "qf_gradient_c64_multi",
)

PROFILE_KINDS = ("forward_pass", "backward_pass", "observable", "resident", "prep_reduce",
                 "pergate", "slot_convert")
# qfuse::StorageMode (engine.hpp:30)
QF_STORAGE_FULL, QF_STORAGE_MEMSAVE = 0, 1
STORAGE = {"full": QF_STORAGE_FULL, "memsave": QF_STORAGE_MEMSAVE}


class QfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"qfuse-b200 error {code}: {msg}")
        self.code = code


class QfInvalidArgument(QfError, ValueError):
    pass


class QfCapacityError(QfError, MemoryError):
    pass


class QfStats(C.Structure):
    _fields_ = [
        ("forward_passes", C.c_uint64), ("backward_passes", C.c_uint64),
        ("observable_passes", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("hbm_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
        ("passes_per_layer", C.c_uint32), ("ckpt_layers", C.c_uint32),
        ("resident", C.c_uint32), ("stages", C.c_uint32), ("device_ms", C.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class QfPlanInfo(C.Structure):
    _fields_ = [(f, C.c_uint32) for f in (
        "stages", "resident", "layouts", "passes", "slots", "ckpt_passes", "balanced",
        "wide_forward", "compiled_forward", "compiled_backward")] + [("bytes_per_sample", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class QfProfile(C.Structure):
    _fields_ = [("launches", C.c_uint64 * 8), ("ms", C.c_double * 8), ("bytes", C.c_double * 8)]


_P = C.c_void_p
_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library; raises loudly when it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    L.qf_last_error.restype = C.c_char_p
    L.qf_version.restype = C.c_char_p
    L.qf_ctx_create.argtypes = [C.c_int, C.POINTER(_P)]
    L.qf_ctx_destroy.argtypes = [_P]
    L.qf_ctx_set_hbm_limit.argtypes = [_P, C.c_uint64]
    L.qf_ctx_set_plan_cache.argtypes = [_P, C.c_int]
    grad_args = [_P, _P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _P,
                 C.c_uint32, _P, C.c_uint64, C.c_uint64, C.POINTER(C.c_double), _P, _P,
                 C.POINTER(QfStats)]
    L.qf_gradient_c64.argtypes = grad_args
    L.qf_gradient_pergate_c64.argtypes = grad_args
    L.qf_gradient_c64_ex.argtypes = grad_args[:7] + [C.c_uint32] + grad_args[7:]
    L.qf_forward_c64.argtypes = [_P, _P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, _P,
                                 C.c_uint32, _P, _P, C.POINTER(QfStats)]
    L.qf_gradient_c128.argtypes = grad_args
    L.qf_gradient_pergate_c128.argtypes = grad_args
    L.qf_plan_create.argtypes = [_P, _P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(_P)]
    L.qf_plan_create_ex.argtypes = L.qf_plan_create.argtypes[:-1] + [C.c_uint32, C.POINTER(_P)]
    L.qf_plan_destroy.argtypes = [_P]
    L.qf_plan_upload_psi0.argtypes = [_P, _P]
    L.qf_plan_set_psi0_device.argtypes = [_P, _P]
    L.qf_plan_gradient.argtypes = [_P, _P, C.POINTER(C.c_double), _P, _P, C.POINTER(QfStats)]
    L.qf_plan_gradient_pergate.argtypes = L.qf_plan_gradient.argtypes
    L.qf_plan_gradient_device.argtypes = [_P, _P, _P]
    L.qf_plan_forward_state.argtypes = [_P, _P, _P]
    L.qf_plan_stream.argtypes = [_P]
    L.qf_plan_stream.restype = _P
    L.qf_plan_synchronize.argtypes = [_P]
    L.qf_plan_traffic.argtypes = [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64)]
    L.qf_plan_random_psi0.argtypes = [_P, C.c_uint64, C.c_uint64]
    L.qf_plan_describe.argtypes = [_P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_uint64, C.c_uint64, _P]
    L.qf_plan_download_psi0.argtypes = [_P, _P]
    L.qf_plan_set_profiling.argtypes = [_P, C.c_int]
    L.qf_plan_profile.argtypes = [_P, C.POINTER(QfProfile), C.c_int]
    L.qf_plan_last_stats.argtypes = [_P, C.POINTER(QfStats)]
    L.qf_group_create.argtypes = [C.c_int, _P, C.POINTER(_P)]
    L.qf_group_destroy.argtypes = [_P]
    L.qf_group_size.argtypes = [_P]
    L.qf_group_plan_create.argtypes = [_P, _P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                       C.c_uint32, C.POINTER(_P)]
    L.qf_group_plan_destroy.argtypes = [_P]
    L.qf_group_plan_upload_psi0.argtypes = [_P, _P]
    L.qf_group_plan_random_psi0.argtypes = [_P, C.c_uint64]
    L.qf_group_plan_gradient.argtypes = L.qf_plan_gradient.argtypes
    L.qf_gradient_c64_multi.argtypes = ([C.c_int, _P] + grad_args[1:7] + [C.c_uint32]
                                        + grad_args[7:])
    _lib = L
    return L


def _check(rc: int):
    if rc == QF_OK:
        return
    msg = _lib.qf_last_error().decode()
    if rc == QF_EINVAL:
        raise QfInvalidArgument(rc, msg)
    if rc == QF_ECAPACITY:
        raise QfCapacityError(rc, msg)
    raise QfError(rc, msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _psi0_batch(a, n_qubits: int) -> int:
    """Batch size of a psi0 array ((batch, 2^n, 2) or flat batch*2^(n+1)); the C
    side reads exactly batch * 2^(n+1) values, so a mismatch is rejected here."""
    per = 2 << n_qubits
    batch = a.shape[0] if a.ndim >= 2 else a.size // per
    if batch <= 0 or a.size != batch * per:
        raise QfInvalidArgument(QF_EINVAL, f"psi0 has {a.size} values, not batch * 2^(n+1) "
                                           f"for n = {n_qubits}")
    return batch


def _theta(theta, n_params: int):
    th = np.ascontiguousarray(theta, np.float64)
    if th.size != n_params:
        raise QfInvalidArgument(QF_EINVAL, "gradient: theta length mismatch")
    return th


def _gates(gates):
    g = np.ascontiguousarray(gates)
    if g.dtype != GATE_DTYPE:
        raise TypeError("gates must use circuits.GATE_DTYPE")
    return g


class Context:
    def __init__(self, device: int = 0):
        L = load()
        h = _P()
        _check(L.qf_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def set_hbm_limit(self, nbytes: int):
        _check(_lib.qf_ctx_set_hbm_limit(self.h, nbytes))

    def set_plan_cache(self, enable: bool):
        """One-shot calls reuse their plan while the circuit/shape repeats (default on)."""
        _check(_lib.qf_ctx_set_plan_cache(self.h, 1 if enable else 0))

    def close(self):
        if self.h:
            _lib.qf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GradientResult:
    """Mirror of qfuse::GradientResult (engine.hpp:65-69)."""
    loss: float
    gradient: np.ndarray
    expect: np.ndarray
    stats: dict


class Plan:
    """A planned circuit with its batch store resident in HBM."""

    def __init__(self, ctx: Context, gates, n_qubits: int, n_params: int, layers: int,
                 ckpt_layers: int, batch: int, pauli, storage: str = "full"):
        g = _gates(gates)
        self._gates = g
        self.ctx = ctx
        self.n, self.n_params, self.batch = n_qubits, n_params, batch
        h = _P()
        _check(_lib.qf_plan_create_ex(ctx.h, _ptr(g), len(g), n_qubits, n_params, layers,
                                      ckpt_layers, batch, pauli[0], pauli[1], STORAGE[storage],
                                      C.byref(h)))
        self.h = h

    def upload_psi0(self, psi0):
        a = np.ascontiguousarray(psi0, np.float32)
        if a.size != self.batch * (2 << self.n):
            raise ValueError("psi0 shape does not match the plan")
        _check(_lib.qf_plan_upload_psi0(self.h, _ptr(a)))
        self.synchronize()

    def upload_psi0_ptr(self, host_ptr: int):
        _check(_lib.qf_plan_upload_psi0(self.h, C.c_void_p(host_ptr)))

    def set_psi0_device(self, dev_ptr: int):
        _check(_lib.qf_plan_set_psi0_device(self.h, C.c_void_p(dev_ptr)))

    def gradient(self, theta, pergate: bool = False) -> GradientResult:
        th = np.ascontiguousarray(theta, np.float64)
        if th.size != self.n_params:
            raise QfInvalidArgument(QF_EINVAL, "gradient: theta length mismatch")
        grad = np.empty(self.n_params, np.float64)
        exp = np.empty(self.batch, np.float64)
        loss = C.c_double()
        st = QfStats()
        fn = _lib.qf_plan_gradient_pergate if pergate else _lib.qf_plan_gradient
        _check(fn(self.h, _ptr(th), C.byref(loss), _ptr(grad), _ptr(exp), C.byref(st)))
        return GradientResult(loss.value, grad, exp, st.as_dict())

    def gradient_device(self, theta_dev_ptr: int, out_dev_ptr: int):
        _check(_lib.qf_plan_gradient_device(self.h, C.c_void_p(theta_dev_ptr),
                                            C.c_void_p(out_dev_ptr)))

    def forward_state(self, theta):
        th = np.ascontiguousarray(theta, np.float64)
        out = np.empty((self.batch, 1 << self.n, 2), np.float32)
        _check(_lib.qf_plan_forward_state(self.h, _ptr(th), _ptr(out)))
        return out

    def random_psi0(self, seed: int, first_sample: int = 0):
        """new_random_state<float>(n, batch, seed) generated on the device."""
        _check(_lib.qf_plan_random_psi0(self.h, seed, first_sample))

    def download_psi0_ptr(self, host_ptr: int):
        _check(_lib.qf_plan_download_psi0(self.h, C.c_void_p(host_ptr)))

    def set_profiling(self, enable: bool):
        _check(_lib.qf_plan_set_profiling(self.h, 1 if enable else 0))

    def profile(self, reset: bool = True) -> dict:
        pr = QfProfile()
        _check(_lib.qf_plan_profile(self.h, C.byref(pr), 1 if reset else 0))
        return {k: {"launches": pr.launches[i], "ms": pr.ms[i], "bytes": pr.bytes[i]}
                for i, k in enumerate(PROFILE_KINDS)}

    def stream(self) -> int:
        return _lib.qf_plan_stream(self.h) or 0

    def synchronize(self):
        _check(_lib.qf_plan_synchronize(self.h))

    def traffic(self):
        t, p, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.qf_plan_traffic(self.h, C.byref(t), C.byref(p), C.byref(n)))
        return t.value, p.value, n.value

    def close(self):
        if getattr(self, "h", None):
            _lib.qf_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def describe_plan(gates, n_qubits, n_params, layers, ckpt_layers, batch, pauli) -> dict:
    """qf_plan_describe: the schedule qf_plan_create would build (host only, no device)."""
    load()
    g = _gates(gates)
    info = QfPlanInfo()
    _check(_lib.qf_plan_describe(_ptr(g), len(g), n_qubits, n_params, layers, ckpt_layers, batch,
                                 pauli[0], pauli[1], C.byref(info)))
    return info.as_dict()


def gradient_c64(ctx: Context, gates, n_qubits, n_params, layers, ckpt_layers, psi0, theta,
                 pauli, pergate: bool = False, storage: str = "full") -> GradientResult:
    """One-shot qf_gradient_c64 (the reference's gradient<float>/run_checkpointed<float>);
    storage "memsave" = StorageMode::MemSave (qf_gradient_c64_ex)."""
    g = _gates(gates)
    a = np.ascontiguousarray(psi0, np.float32)
    batch = _psi0_batch(a, n_qubits)
    th = _theta(theta, n_params)
    grad = np.empty(n_params, np.float64)
    exp = np.empty(batch, np.float64)
    loss = C.c_double()
    st = QfStats()
    if storage != "full" and not pergate:
        _check(_lib.qf_gradient_c64_ex(ctx.h, _ptr(g), len(g), n_qubits, n_params, layers,
                                       ckpt_layers, STORAGE[storage], _ptr(a), batch, _ptr(th),
                                       pauli[0], pauli[1], C.byref(loss), _ptr(grad), _ptr(exp),
                                       C.byref(st)))
        return GradientResult(loss.value, grad, exp, st.as_dict())
    fn = _lib.qf_gradient_pergate_c64 if pergate else _lib.qf_gradient_c64
    _check(fn(ctx.h, _ptr(g), len(g), n_qubits, n_params, layers, ckpt_layers, _ptr(a), batch,
              _ptr(th), pauli[0], pauli[1], C.byref(loss), _ptr(grad), _ptr(exp),
              C.byref(st)))
    return GradientResult(loss.value, grad, exp, st.as_dict())


def forward_c64(ctx: Context, gates, n_qubits, n_params, layers, psi0, theta) -> np.ndarray:
    """One-shot qf_forward_c64 (the reference's forward<float>): final state
    (batch, 2^n, 2) float32, global phase included."""
    g = _gates(gates)
    a = np.ascontiguousarray(psi0, np.float32)
    batch = _psi0_batch(a, n_qubits)
    th = _theta(theta, n_params)
    out = np.empty((batch, 1 << n_qubits, 2), np.float32)
    st = QfStats()
    _check(_lib.qf_forward_c64(ctx.h, _ptr(g), len(g), n_qubits, n_params, layers, _ptr(a), batch,
                               _ptr(th), _ptr(out), C.byref(st)))
    return out


def gradient_c128(ctx: Context, gates, n_qubits, n_params, layers, ckpt_layers, psi0, theta,
                  pauli, pergate: bool = False) -> GradientResult:
    """qf_gradient_c128: the reference's gradient<double> (complex128 state, fp64 compute,
    fused segments); pergate=True: qf_gradient_pergate_c128 (naive_gradient<double>)."""
    g = _gates(gates)
    a = np.ascontiguousarray(psi0, np.float64)
    batch = _psi0_batch(a, n_qubits)
    th = _theta(theta, n_params)
    grad = np.empty(n_params, np.float64)
    exp = np.empty(batch, np.float64)
    loss = C.c_double()
    st = QfStats()
    fn = _lib.qf_gradient_pergate_c128 if pergate else _lib.qf_gradient_c128
    _check(fn(ctx.h, _ptr(g), len(g), n_qubits, n_params, layers, ckpt_layers, _ptr(a), batch,
              _ptr(th), pauli[0], pauli[1], C.byref(loss), _ptr(grad), _ptr(exp), C.byref(st)))
    return GradientResult(loss.value, grad, exp, st.as_dict())


def _devices(devices):
    if devices is None:
        return None, None
    arr = (C.c_int * len(devices))(*devices)
    return arr, C.cast(arr, C.c_void_p)


class Group:
    """qf_group: one process driving several devices of the box, one NCCL
    all-reduce of [grad | loss] per gradient (include/qfuse_b200.h)."""

    def __init__(self, n_gpus: int, devices=None):
        L = load()
        keep, dp = _devices(devices)
        h = _P()
        _check(L.qf_group_create(n_gpus, dp, C.byref(h)))
        self.h = h
        self.size = L.qf_group_size(h)

    def close(self):
        if getattr(self, "h", None):
            _lib.qf_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GroupPlan:
    """qf_group_plan: a planned circuit over a group, the batch sharded in order."""

    def __init__(self, group: Group, gates, n_qubits: int, n_params: int, layers: int,
                 ckpt_layers: int, batch: int, pauli, storage: str = "full"):
        g = _gates(gates)
        self.group = group
        self.n, self.n_params, self.batch = n_qubits, n_params, batch
        h = _P()
        _check(_lib.qf_group_plan_create(group.h, _ptr(g), len(g), n_qubits, n_params, layers,
                                         ckpt_layers, batch, pauli[0], pauli[1], STORAGE[storage],
                                         C.byref(h)))
        self.h = h

    def upload_psi0(self, psi0):
        a = np.ascontiguousarray(psi0, np.float32)
        if a.size != self.batch * (2 << self.n):
            raise ValueError("psi0 shape does not match the plan")
        _check(_lib.qf_group_plan_upload_psi0(self.h, _ptr(a)))

    def random_psi0(self, seed: int):
        _check(_lib.qf_group_plan_random_psi0(self.h, seed))

    def gradient(self, theta) -> GradientResult:
        th = np.ascontiguousarray(theta, np.float64)
        if th.size != self.n_params:
            raise QfInvalidArgument(QF_EINVAL, "gradient: theta length mismatch")
        grad = np.empty(self.n_params, np.float64)
        exp = np.empty(self.batch, np.float64)
        loss = C.c_double()
        st = QfStats()
        _check(_lib.qf_group_plan_gradient(self.h, _ptr(th), C.byref(loss), _ptr(grad), _ptr(exp),
                                           C.byref(st)))
        return GradientResult(loss.value, grad, exp, st.as_dict())

    def close(self):
        if getattr(self, "h", None):
            _lib.qf_group_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gradient_c64_multi(n_gpus: int, gates, n_qubits, n_params, layers, ckpt_layers, psi0, theta,
                       pauli, devices=None, storage: str = "full") -> GradientResult:
    """One-shot qf_gradient_c64_multi: the batch sharded over n_gpus devices."""
    load()
    g = _gates(gates)
    a = np.ascontiguousarray(psi0, np.float32)
    batch = _psi0_batch(a, n_qubits)
    th = _theta(theta, n_params)
    grad = np.empty(n_params, np.float64)
    exp = np.empty(batch, np.float64)
    loss = C.c_double()
    st = QfStats()
    keep, dp = _devices(devices)
    _check(_lib.qf_gradient_c64_multi(n_gpus, dp, _ptr(g), len(g), n_qubits, n_params, layers,
                                      ckpt_layers, STORAGE[storage], _ptr(a), batch, _ptr(th),
                                      pauli[0], pauli[1], C.byref(loss), _ptr(grad), _ptr(exp),
                                      C.byref(st)))
    return GradientResult(loss.value, grad, exp, st.as_dict())
