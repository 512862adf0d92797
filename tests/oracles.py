"""ctypes wrappers for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/liboracle.so, the plain-C restatement (qf_oracle.c).
* ``RefLib``  -> oracle/_ref/libqfuse_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src plus the extern "C" shim ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libqfuse_ref.so")

GATE_DTYPE = np.dtype(
    [("kind", np.uint8), ("axis", np.uint8), ("pad", np.uint16), ("q0", np.uint32),
     ("q1", np.uint32), ("param", np.uint32)], align=True)
assert GATE_DTYPE.itemsize == 16

_P = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        L.qfo_random_state.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _P]
        L.qfo_random_parameters.argtypes = [C.c_uint64, C.c_uint64, _P]
        L.qfo_build_hea.argtypes = [C.c_uint32, C.c_uint32, _P, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.qfo_repeated_ixyz.argtypes = [C.c_uint32, C.c_char_p]
        L.qfo_parse_pauli.argtypes = [C.c_char_p, C.c_uint32, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.qfo_forward.argtypes = [_P, C.c_uint64, C.c_uint32, _P, C.c_uint32, _P]
        L.qfo_expectation.argtypes = [_P, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                      C.c_uint32, _P]
        L.qfo_gradient.argtypes = [_P, C.c_uint64, C.c_uint32, C.c_uint32, _P, C.c_uint32, _P,
                                   C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(C.c_double),
                                   _P, _P]
        L.qfo_gradient_f32in.argtypes = L.qfo_gradient.argtypes

    def random_state(self, n, batch, seed):
        out = np.empty((batch, 1 << n, 2), np.float64)
        self.lib.qfo_random_state(n, batch, seed, _ptr(out))
        return out

    def random_parameters(self, count, seed):
        out = np.empty(count, np.float64)
        self.lib.qfo_random_parameters(count, seed, _ptr(out))
        return out

    def build_hea(self, n, layers):
        ng, npar = C.c_uint64(), C.c_uint32()
        rc = self.lib.qfo_build_hea(n, layers, None, 0, C.byref(ng), C.byref(npar))
        if rc:
            raise ValueError("build_hea: bad arguments")
        g = np.zeros(ng.value, GATE_DTYPE)
        self.lib.qfo_build_hea(n, layers, _ptr(g), ng.value, C.byref(ng), C.byref(npar))
        return g, npar.value

    def repeated_ixyz(self, n):
        buf = C.create_string_buffer(n + 1)
        self.lib.qfo_repeated_ixyz(n, buf)
        return buf.value.decode()

    def parse_pauli(self, label, n=0):
        x, z, y = C.c_uint64(), C.c_uint64(), C.c_uint32()
        if self.lib.qfo_parse_pauli(label.encode(), n, C.byref(x), C.byref(z), C.byref(y)):
            raise ValueError(f"bad pauli label {label!r}")
        return x.value, z.value, y.value

    def forward(self, gates, n, psi0, theta):
        psi = np.array(psi0, np.float64, copy=True, order="C")
        batch = psi.shape[0]
        if self.lib.qfo_forward(_ptr(gates), len(gates), n, _ptr(psi), batch, _ptr(theta)):
            raise ValueError("forward: bad arguments")
        return psi

    def expectation(self, psi, n, pauli):
        psi = np.ascontiguousarray(psi, np.float64)
        out = np.empty(psi.shape[0], np.float64)
        self.lib.qfo_expectation(_ptr(psi), n, psi.shape[0], *pauli, _ptr(out))
        return out

    def gradient(self, gates, n, n_params, psi0, theta, pauli):
        psi0 = np.ascontiguousarray(psi0)
        batch = psi0.shape[0]
        grad = np.empty(n_params, np.float64)
        exp = np.empty(batch, np.float64)
        loss = C.c_double()
        fn = self.lib.qfo_gradient_f32in if psi0.dtype == np.float32 else self.lib.qfo_gradient
        if psi0.dtype not in (np.float32, np.float64):
            raise TypeError(psi0.dtype)
        rc = fn(_ptr(gates), len(gates), n, n_params, _ptr(psi0), batch,
                _ptr(np.ascontiguousarray(theta, np.float64)), *pauli, C.byref(loss),
                _ptr(grad), _ptr(exp))
        if rc:
            raise ValueError(f"oracle gradient failed rc={rc}")
        return loss.value, grad, exp


class RefLib:
    """The reference implementation itself (qfuse, CPU, OpenMP)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_max_threads.restype = C.c_int
        L.ref_set_alloc_limit.argtypes = [C.c_uint64]
        L.ref_random_state_f64.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _P]
        L.ref_random_state_f32.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _P]
        L.ref_random_parameters.argtypes = [C.c_uint64, C.c_uint64, _P]
        L.ref_build_hea.argtypes = [C.c_uint32, C.c_uint32, _P, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.ref_parse_pauli.argtypes = [C.c_char_p, C.c_uint32, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.ref_gradient.argtypes = [_P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_uint32, C.c_int, C.c_int, _P, C.c_uint32, _P,
                                   C.c_uint64, C.c_uint64, C.POINTER(C.c_double), _P, _P]
        L.ref_forward_f64.argtypes = [_P, C.c_uint64, C.c_uint32, C.c_uint32, _P, C.c_uint32,
                                      _P, _P]
        L.ref_parameter_shift.argtypes = [_P, C.c_uint64, C.c_uint32, C.c_uint32, _P,
                                          C.c_uint32, _P, C.c_uint64, C.c_uint64, _P]
        L.ref_set_alloc_limit(1 << 40)

    def _check(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.lib.ref_last_error().decode()}")

    def set_threads(self, t):
        self.lib.ref_set_threads(t)

    def max_threads(self):
        return self.lib.ref_max_threads()

    def random_state(self, n, batch, seed, dtype=np.float32):
        out = np.empty((batch, 1 << n, 2), dtype)
        fn = self.lib.ref_random_state_f32 if dtype == np.float32 else self.lib.ref_random_state_f64
        self._check(fn(n, batch, seed, _ptr(out)))
        return out

    def random_parameters(self, count, seed):
        out = np.empty(count, np.float64)
        self._check(self.lib.ref_random_parameters(count, seed, _ptr(out)))
        return out

    def build_hea(self, n, layers):
        ng, npar = C.c_uint64(), C.c_uint32()
        self._check(self.lib.ref_build_hea(n, layers, None, 0, C.byref(ng), C.byref(npar)))
        g = np.zeros(ng.value, GATE_DTYPE)
        self._check(self.lib.ref_build_hea(n, layers, _ptr(g), ng.value, C.byref(ng),
                                           C.byref(npar)))
        return g, npar.value

    def parse_pauli(self, label, n=0):
        x, z, y = C.c_uint64(), C.c_uint64(), C.c_uint32()
        self._check(self.lib.ref_parse_pauli(label.encode(), n, C.byref(x), C.byref(z),
                                             C.byref(y)))
        return x.value, z.value, y.value

    def gradient(self, gates, n, n_params, psi0, theta, pauli, layers=1, block_layers=0,
                 mode="fused", expect=False):
        psi0 = np.ascontiguousarray(psi0)
        prec = 0 if psi0.dtype == np.float32 else 1
        batch = psi0.shape[0]
        grad = np.empty(n_params, np.float64)
        exp = np.empty(batch, np.float64) if expect else None
        loss = C.c_double()
        m = {"fused": 0, "naive": 1, "mem_save": 2}[mode]
        self._check(self.lib.ref_gradient(
            _ptr(gates), len(gates), n, n_params, layers, block_layers, prec, m, _ptr(psi0),
            batch, _ptr(np.ascontiguousarray(theta, np.float64)), pauli[0], pauli[1],
            C.byref(loss), _ptr(grad), _ptr(exp)))
        return (loss.value, grad, exp) if expect else (loss.value, grad)

    def forward(self, gates, n, n_params, psi0, theta):
        psi0 = np.ascontiguousarray(psi0, np.float64)
        out = np.empty_like(psi0)
        self._check(self.lib.ref_forward_f64(_ptr(gates), len(gates), n, n_params, _ptr(psi0),
                                             psi0.shape[0], _ptr(theta), _ptr(out)))
        return out

    def parameter_shift(self, gates, n, n_params, psi0, theta, pauli):
        psi0 = np.ascontiguousarray(psi0, np.float64)
        grad = np.empty(n_params, np.float64)
        self._check(self.lib.ref_parameter_shift(_ptr(gates), len(gates), n, n_params,
                                                 _ptr(psi0), psi0.shape[0], _ptr(theta),
                                                 pauli[0], pauli[1], _ptr(grad)))
        return grad


def rel_diff(got, want):
    """Max-norm relative difference — tests/acceptance.cpp:63-73."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = np.max(np.abs(want)) if want.size else 0.0
    diff = np.max(np.abs(got - want)) if want.size else 0.0
    return diff / scale if scale > 0 else diff
