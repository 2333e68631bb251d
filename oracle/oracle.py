"""ctypes view of oracle/liboracle.so — TEST INFRASTRUCTURE ONLY.

The CPU fp64 restatement of the reference engine (see adpsgd_oracle.cpp header for
the file:line map). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
/ --impl reference legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None


class ModelDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("layers", "hidden", "bidirectional", "input_dim", "proj", "classes", "unroll")]


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        u64, i64, i32 = C.c_uint64, C.c_int64, C.c_int32
        P = C.POINTER
        L.or_mix_seed.restype = u64; L.or_mix_seed.argtypes = [u64]
        L.or_derive_seed.restype = u64; L.or_derive_seed.argtypes = [u64, u64]
        L.or_derive_seed3.restype = u64; L.or_derive_seed3.argtypes = [u64, u64, u64]
        L.or_mt_first.restype = u64; L.or_mt_first.argtypes = [u64]
        L.or_random_permutation.argtypes = [u64, C.c_int, P(i32)]
        L.or_permutation_for_iteration.argtypes = [u64, C.c_int, i64, P(i32)]
        L.or_ring_neighbors.argtypes = [C.c_int, u64, C.c_int, i64, C.c_int, P(i32), P(i32)]
        L.or_mixing_matrix.argtypes = [C.c_int, C.c_int, P(i32), P(C.c_double)]
        L.or_lr_at.restype = C.c_double
        L.or_lr_at.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int]
        L.or_param_count.restype = i64; L.or_param_count.argtypes = [P(ModelDesc)]
        L.or_param_offsets.argtypes = [P(ModelDesc), P(i64), C.c_int]
        L.or_init_w0.argtypes = [u64, i64, P(C.c_double)]
        L.or_learner_batches.argtypes = [u64, C.c_int, C.c_int, C.c_int, C.c_int, P(i32)]
        L.or_lstm_loss_grad.restype = C.c_double
        L.or_lstm_loss_grad.argtypes = [P(ModelDesc), P(C.c_double), P(C.c_float), P(i32), P(i32),
                                        C.c_int, P(C.c_double), C.c_int]
        L.or_engine_create.restype = C.c_void_p
        L.or_engine_create.argtypes = [P(ModelDesc), C.c_int, C.c_int, u64, P(C.c_float), P(i32),
                                       C.c_int, C.c_int, C.c_int, C.c_int]
        L.or_engine_destroy.argtypes = [C.c_void_p]
        L.or_engine_dim.restype = i64; L.or_engine_dim.argtypes = [C.c_void_p]
        L.or_engine_get_model.argtypes = [C.c_void_p, C.c_int, P(C.c_double)]
        L.or_engine_set_model.argtypes = [C.c_void_p, C.c_int, P(C.c_double)]
        L.or_engine_last_loss.restype = C.c_double
        L.or_engine_last_loss.argtypes = [C.c_void_p, C.c_int]
        L.or_engine_step.argtypes = [C.c_void_p, C.c_int, C.c_double, i64, C.c_int, P(i32)]
        L.or_coupled_async.restype = i64
        L.or_coupled_async.argtypes = [C.c_void_p, C.c_int, P(C.c_double), i64, C.c_int, P(C.c_double), C.c_int,
                                       P(i32), P(C.c_double)]
        L.or_engine_step_injected.argtypes = [C.c_void_p, C.c_int, C.c_double, i64, C.c_int, P(i32),
                                              P(C.c_double)]
        _LIB = L
    return _LIB


def ref_lib():
    """oracle/_ref/libref_rng.so (reference rng.hpp compiled in place) or None."""
    global _REF
    if _REF is None:
        path = os.path.join(_HERE, "_ref", "libref_rng.so")
        if not os.path.exists(path):
            return None
        R = C.CDLL(path)
        u64, i64, i32 = C.c_uint64, C.c_int64, C.c_int32
        R.ref_derive_seed.restype = u64; R.ref_derive_seed.argtypes = [u64, u64]
        R.ref_derive_seed3.restype = u64; R.ref_derive_seed3.argtypes = [u64, u64, u64]
        R.ref_mt_first.restype = u64; R.ref_mt_first.argtypes = [u64]
        R.ref_permutation_for_iteration.argtypes = [u64, C.c_int, i64, C.POINTER(i32)]
        R.ref_init_w0.argtypes = [u64, i64, C.POINTER(C.c_double)]
        R.ref_learner_batches.argtypes = [u64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(i32)]
        _REF = R
    return _REF


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def desc(layers, hidden, bidirectional, input_dim, proj, classes, unroll=21) -> ModelDesc:
    return ModelDesc(layers, hidden, int(bidirectional), input_dim, proj, classes, unroll)


def param_count(d: ModelDesc) -> int:
    return int(lib().or_param_count(C.byref(d)))


def param_offsets(d: ModelDesc) -> np.ndarray:
    out = np.zeros(256, dtype=np.int64)
    n = lib().or_param_offsets(C.byref(d), _p(out, C.c_int64), 256)
    return out[:n].copy()


def permutation_for_iteration(seed: int, L: int, k: int) -> np.ndarray:
    out = np.zeros(L, dtype=np.int32)
    rc = lib().or_permutation_for_iteration(seed, L, k, _p(out, C.c_int32))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return out


def ring_neighbors(strategy: int, seed: int, L: int, k: int, l: int):
    a, b = C.c_int32(), C.c_int32()
    rc = lib().or_ring_neighbors(strategy, seed, L, k, l, C.byref(a), C.byref(b))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return a.value, b.value


def mixing_matrix(kind: int, L: int, mapping=None) -> np.ndarray:
    out = np.zeros((L, L), dtype=np.float64)
    m = np.asarray(mapping if mapping is not None else np.arange(L), dtype=np.int32)
    rc = lib().or_mixing_matrix(kind, L, _p(m, C.c_int32), _p(out, C.c_double))
    if rc:
        raise ValueError(f"oracle error {rc}")
    return out


def init_w0(seed: int, D: int) -> np.ndarray:
    out = np.zeros(D, dtype=np.float64)
    lib().or_init_w0(seed, D, _p(out, C.c_double))
    return out


def learner_batches(seed: int, learner: int, n_steps: int, M: int, train_count: int) -> np.ndarray:
    out = np.zeros((n_steps, M), dtype=np.int32)
    lib().or_learner_batches(seed, learner, n_steps, M, train_count, _p(out, C.c_int32))
    return out


def lstm_loss_grad(d: ModelDesc, w: np.ndarray, feats: np.ndarray, labels: np.ndarray,
                   idx: np.ndarray, want_grad: bool = True, threads: int = 1):
    w = np.ascontiguousarray(w, dtype=np.float64)
    feats = np.ascontiguousarray(feats, dtype=np.float32)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    g = np.zeros_like(w) if want_grad else None
    loss = lib().or_lstm_loss_grad(C.byref(d), _p(w, C.c_double), _p(feats, C.c_float),
                                   _p(labels, C.c_int32), _p(idx, C.c_int32), len(idx),
                                   _p(g, C.c_double) if want_grad else None, threads)
    return (loss, g) if want_grad else loss


class OracleEngine:
    """fp64 restatement of engine::run_training's per-iteration state (engine.cpp:99-204)."""

    def __init__(self, d: ModelDesc, L: int, M: int, seed: int, feats, labels, train_count: int,
                 history_depth: int = 2, threads: int = 1):
        self._feats = np.ascontiguousarray(feats, dtype=np.float32)
        self._labels = np.ascontiguousarray(labels, dtype=np.int32)
        self.d, self.L, self.M = d, L, M
        self._h = lib().or_engine_create(C.byref(d), L, M, seed, _p(self._feats, C.c_float),
                                         _p(self._labels, C.c_int32), self._feats.shape[0],
                                         train_count, history_depth, threads)
        self.D = int(lib().or_engine_dim(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_engine_destroy(self._h)
            self._h = None

    def model(self, l: int) -> np.ndarray:
        out = np.zeros(self.D, dtype=np.float64)
        lib().or_engine_get_model(self._h, l, _p(out, C.c_double))
        return out

    def set_model(self, l: int, w) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        lib().or_engine_set_model(self._h, l, _p(w, C.c_double))

    def last_loss(self, l: int) -> float:
        return float(lib().or_engine_last_loss(self._h, l))

    def step(self, strategy: int, lr: float, k: int, generic_mix: int = 2, taus=None) -> int:
        t = None if taus is None else np.ascontiguousarray(taus, dtype=np.int32)
        return lib().or_engine_step(self._h, strategy, lr, k, generic_mix,
                                    _p(t, C.c_int32) if t is not None else None)

    def coupled_async(self, strategy: int, durations, target: int, ipe: int, lr_per_epoch):
        """chronos::coupled_async (chronos.cpp:178-299); returns (event learners, event times)."""
        d = np.ascontiguousarray(durations, dtype=np.float64)
        lrs = np.ascontiguousarray(lr_per_epoch, dtype=np.float64)
        ev = np.zeros(target, dtype=np.int32)
        et = np.zeros(target, dtype=np.float64)
        n = lib().or_coupled_async(self._h, strategy, _p(d, C.c_double), target, ipe, _p(lrs, C.c_double),
                                   len(lrs), _p(ev, C.c_int32), _p(et, C.c_double))
        if n < 0:
            raise ValueError(f"coupled_async failed with status {-n} (lr table shorter than the rounds run?)")
        return ev[:n], et[:n]

    def step_injected(self, strategy: int, lr: float, k: int, grads, generic_mix: int = 2,
                      taus=None) -> int:
        g = np.ascontiguousarray(grads, dtype=np.float64)
        t = None if taus is None else np.ascontiguousarray(taus, dtype=np.int32)
        return lib().or_engine_step_injected(self._h, strategy, lr, k, generic_mix,
                                             _p(t, C.c_int32) if t is not None else None,
                                             _p(g, C.c_double))
