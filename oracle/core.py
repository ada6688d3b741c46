"""ctypes wrapper over liblouiskv_oracle.so — TEST INFRASTRUCTURE ONLY.

Each wrapper only marshals numpy arrays; every arithmetic step is in
``louiskv_oracle.c`` and cites the passage it follows there.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "louiskv_oracle.c")
_LIB = os.path.join(_HERE, "liblouiskv_oracle.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_oracle())
        L.lko_bf16_round.restype = ctypes.c_float
        L.lko_bf16_round.argtypes = [ctypes.c_float]
        L.lko_cosine_r1.restype = ctypes.c_double
        L.lko_cosine_r1.argtypes = [_f32p, _f32p, ctypes.c_int]
        L.lko_trigger_r1.restype = ctypes.c_int
        L.lko_trigger_r1.argtypes = [_f32p, _f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
        L.lko_e4m3_round_n.restype = None
        L.lko_e4m3_round_n.argtypes = [_f32p, _f32p, ctypes.c_longlong]
        L.lko_bf16_round_n.restype = None
        L.lko_bf16_round_n.argtypes = [_f32p, _f32p, ctypes.c_longlong]
        L.lko_exp_r3_n.restype = None
        L.lko_exp_r3_n.argtypes = [_f32p, _f32p, ctypes.c_longlong]
        L.lko_exp_r3.restype = ctypes.c_float
        L.lko_exp_r3.argtypes = [ctypes.c_float]
        L.lko_group_scores_r2.restype = ctypes.c_int
        L.lko_group_scores_r2.argtypes = [_f32p, ctypes.c_int, _f32p, ctypes.c_int, ctypes.c_int, _f32p]
        L.lko_group_scores_f64.restype = ctypes.c_int
        L.lko_group_scores_f64.argtypes = [_f32p, ctypes.c_int, _f32p, ctypes.c_int, ctypes.c_int, _f64p]
        L.lko_select_greedy.restype = ctypes.c_int
        L.lko_select_greedy.argtypes = [_f32p, _i32p, ctypes.c_int, ctypes.c_longlong, _i32p]
        L.lko_kmeans.restype = ctypes.c_int
        L.lko_kmeans.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 _i32p, _f32p, _i32p, _f64p, _f32p]
        L.lko_centroids_of.restype = ctypes.c_int
        L.lko_centroids_of.argtypes = [_f32p, _i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _f32p]
        L.lko_segment_centroid.restype = None
        L.lko_segment_centroid.argtypes = [_f32p, ctypes.c_int, ctypes.c_int, _f32p]
        L.lko_attention_f64.restype = ctypes.c_int
        L.lko_attention_f64.argtypes = [_f32p, ctypes.c_int, _f32p, _f32p, ctypes.c_int, ctypes.c_int, _f64p]
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def bf16_round(x) -> np.ndarray:
    """Round fp32 values to bf16 (RNE), returned as fp32 (reading R-AMB18)."""
    a = _f32(x)
    out = np.empty_like(a)
    lib().lko_bf16_round_n(a.reshape(-1), out.reshape(-1), a.size)
    return out


def e4m3_round(x) -> np.ndarray:
    """E4M3 value (RNE, saturating at +-448) of every element, as fp32 (reading R-FP8)."""
    a = _f32(x)
    out = np.empty_like(a)
    lib().lko_e4m3_round_n(a.reshape(-1), out.reshape(-1), a.size)
    return out


def cosine_r1(a, b) -> float:
    a, b = _f32(a).reshape(-1), _f32(b).reshape(-1)
    return lib().lko_cosine_r1(a, b, a.size)


def trigger_r1(q_ref, q_cur, t: int, tau: float):
    """q_ref, q_cur: [H, d]. Returns (flag, r)."""
    q_ref, q_cur = _f32(q_ref), _f32(q_cur)
    H, d = q_cur.shape
    r = ctypes.c_double(0.0)
    flag = lib().lko_trigger_r1(q_ref, q_cur, H, d, int(t), float(tau), ctypes.byref(r))
    return int(flag), r.value


def exp_r3(x) -> np.ndarray:
    a = _f32(x)
    out = np.empty_like(a)
    lib().lko_exp_r3_n(a.reshape(-1), out.reshape(-1), a.size)
    return out


def group_scores_r2(q, C) -> np.ndarray:
    """q: [g, d]; C: [n, d] (bf16 values). Returns A fp32 [n] (recipe R2)."""
    q, C = _f32(q), _f32(C)
    g, d = q.shape
    n = C.shape[0]
    A = np.empty(n, dtype=np.float32)
    if lib().lko_group_scores_r2(q, g, C, n, d, A) != 0:
        raise ValueError("group_scores_r2: empty input")
    return A


def group_scores_f64(q, C) -> np.ndarray:
    q, C = _f32(q), _f32(C)
    g, d = q.shape
    n = C.shape[0]
    A = np.empty(n, dtype=np.float64)
    if lib().lko_group_scores_f64(q, g, C, n, d, A) != 0:
        raise ValueError("group_scores_f64: empty input")
    return A


def select_greedy(A, sizes, B: int) -> np.ndarray:
    """Selected unit ids (ascending) under budget B (greedy skip-and-continue)."""
    A = _f32(A)
    sizes = np.ascontiguousarray(np.asarray(sizes, dtype=np.int32))
    n = A.size
    out = np.empty(max(n, 1), dtype=np.int32)
    cnt = lib().lko_select_greedy(A, sizes, n, int(B), out)
    if cnt < 0:
        raise MemoryError("select_greedy")
    return out[:cnt].copy()


def kmeans(X, k: int, iters: int, mode: int = 1):
    """Returns (assign[N], C[k,d] fp32, counts[k], J[iters] fp64, dmin[N])."""
    X = _f32(X)
    N, d = X.shape
    assign = np.empty(N, dtype=np.int32)
    C = np.empty((k, d), dtype=np.float32)
    counts = np.empty(k, dtype=np.int32)
    J = np.empty(max(iters, 1), dtype=np.float64)
    dmin = np.empty(N, dtype=np.float32)
    rc = lib().lko_kmeans(X, N, d, k, iters, mode, assign, C, counts, J, dmin)
    if rc != 0:
        raise ValueError(f"kmeans: invalid arguments (rc={rc})")
    return assign, C, counts, J[:iters], dmin


def centroids_of(X, assign, k: int) -> np.ndarray:
    """fp32 centroids (fp64 means) of a given clustering; raises on an empty cluster."""
    X = _f32(X)
    assign = np.ascontiguousarray(assign, dtype=np.int32)
    N, d = X.shape
    C = np.zeros((k, d), np.float32)
    rc = lib().lko_centroids_of(X, assign, N, d, k, C)
    if rc != 0:
        raise ValueError("centroids_of: empty cluster")
    return C


def segment_centroid(keys) -> np.ndarray:
    keys = _f32(keys)
    n, d = keys.shape
    out = np.empty(d, dtype=np.float32)
    lib().lko_segment_centroid(keys, n, d, out)
    return out


def attention_f64(q, K, V) -> np.ndarray:
    """q: [g, d]; K, V: [n, d]. Returns fp64 [g, d]."""
    q, K, V = _f32(q), _f32(K), _f32(V)
    g, d = q.shape
    n = K.shape[0]
    out = np.empty((g, d), dtype=np.float64)
    if lib().lko_attention_f64(q, g, K, V, n, d, out) != 0:
        raise ValueError("attention_f64: empty key set")
    return out
