"""ctypes bindings for the oracle (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (the C restatement, dnd_oracle.c) and
`Reference` wraps oracle/_ref/libdndref.so (the unmodified reference library
plus ref_shim.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module; the product package
paper_2007_13552_b200 never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdndref.so")

_i64, _u64, _i32, _f64 = C.c_int64, C.c_uint64, C.c_int, C.c_double
_P = C.c_void_p


def build(force: bool = False) -> None:
    """Build liboracle.so (and _ref when /root/reference is present)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "dnd_oracle.c"))
    ):
        subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True, capture_output=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


class Oracle:
    """The C restatement; every method mirrors a dno_* function."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.dno_splitmix64.restype = _u64
        L.dno_splitmix64.argtypes = [_u64]
        L.dno_uniform01.restype = _f64
        L.dno_uniform01.argtypes = [_u64, _u64]
        L.dno_fill_uniform_f32.argtypes = [_u64, _i64, _i64, _i64, _P]
        L.dno_fill_uniform_f64.argtypes = [_u64, _i64, _i64, _i64, _P]
        L.dno_chunk_map.argtypes = [_i64, _i32, _P, _P]
        L.dno_row_norms.argtypes = [_P, _i64, _i64, _P]
        L.dno_cdist.argtypes = [_P, _i64, _i64, _i32, _P, _P]
        L.dno_cdist_xy.argtypes = [_P, _i64, _P, _i64, _i64, _P]
        L.dno_kmeans_init_indices.argtypes = [_i64, _i32, _u64, _P]
        L.dno_kmeans_fit.argtypes = [_P, _i64, _i64, _i32, _i32, _i32, _f64, _u64, _P, _P, _P]
        L.dno_kmeans_lloyd.argtypes = [_P, _i64, _i64, _i32, _i32, _i32, _f64, _P, _P, _P]
        L.dno_kmeans_predict.argtypes = [_P, _i64, _i64, _P, _i32, _P]
        L.dno_moments_axis0.argtypes = [_P, _i64, _i64, _i32, _i64, _P, _P]
        L.dno_local_moments_axis0.argtypes = [_P, _i64, _i64, _P, _P, _P]
        L.dno_welford_axis0_f32_continue.argtypes = [_P, _i64, _i64, _P, _P, _P]
        L.dno_kmeanspp_indices_f32.argtypes = [_P, _i64, _i64, _i32, _i32, _u64, _P]
        L.dno_kmeanspp_indices_f64.argtypes = [_P, _i64, _i64, _i32, _i32, _u64, _P]
        L.dno_lasso_fit.argtypes = [_P, _P, _i64, _i64, _i32, _f64, _i32, _f64, _P, _P, _P]
        L.dno_soft_threshold.argtypes = [_f64, _f64]
        L.dno_soft_threshold.restype = _f64

    def uniform_f32(self, rows, m, seed, row0=0):
        out = np.empty((rows, m), np.float32)
        self.lib.dno_fill_uniform_f32(seed, row0, rows, m, _ptr(out))
        return out

    def uniform_f64(self, rows, m, seed, row0=0):
        out = np.empty((rows, m), np.float64)
        self.lib.dno_fill_uniform_f64(seed, row0, rows, m, _ptr(out))
        return out

    def chunk_map(self, n, p):
        off = np.empty(p, np.int64)
        ext = np.empty(p, np.int64)
        if self.lib.dno_chunk_map(n, p, _ptr(off), _ptr(ext)) != 0:
            raise ValueError("chunk_map: invalid arguments")
        return off, ext

    def row_norms(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.shape[0], np.float64)
        self.lib.dno_row_norms(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
        return out

    def cdist(self, x, p=1):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        out = np.empty((n, n), np.float64)
        sr = np.zeros(1, np.int64)
        if self.lib.dno_cdist(_ptr(x), n, m, p, _ptr(out), _ptr(sr)) != 0:
            raise ValueError("cdist: input has no rows")
        return out

    def cdist_xy(self, x, y):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        if x.shape[1] != y.shape[1]:
            raise ValueError("cdist_xy: feature counts do not match")
        out = np.empty((x.shape[0], y.shape[0]), np.float64)
        self.lib.dno_cdist_xy(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], _ptr(out))
        return out

    def kmeans_init_indices(self, n, k, seed):
        out = np.empty(k, np.int64)
        if self.lib.dno_kmeans_init_indices(n, k, seed, _ptr(out)) != 0:
            raise ValueError("kmeans_init_indices: k out of range")
        return out

    def kmeans_fit(self, x, k, max_iter, tol=0.0, seed=42, p=1):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        cent = np.empty((k, m), np.float64)
        trace = np.zeros(max_iter, np.float64)
        it = np.zeros(1, np.int32)
        rc = self.lib.dno_kmeans_fit(_ptr(x), n, m, p, k, max_iter, tol, seed, _ptr(cent),
                                     _ptr(trace), _ptr(it))
        if rc != 0:
            raise ValueError("kmeans_fit: invalid arguments" if rc == -1 else
                             "kmeans_fit: input contains non-finite values")
        return cent, trace[: it[0]].copy(), int(it[0])

    def kmeans_lloyd(self, x, centroids, max_iter, tol=0.0, p=1):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        cent = np.array(centroids, np.float64, copy=True, order="C")
        k = cent.shape[0]
        trace = np.zeros(max_iter, np.float64)
        it = np.zeros(1, np.int32)
        if self.lib.dno_kmeans_lloyd(_ptr(x), n, m, p, k, max_iter, tol, _ptr(cent), _ptr(trace),
                                     _ptr(it)) != 0:
            raise ValueError("kmeans_lloyd: invalid arguments")
        return cent, trace[: it[0]].copy(), int(it[0])

    def kmeans_predict(self, x, centroids):
        x = np.ascontiguousarray(x, np.float64)
        c = np.ascontiguousarray(centroids, np.float64)
        out = np.empty(x.shape[0], np.int32)
        self.lib.dno_kmeans_predict(_ptr(x), x.shape[0], x.shape[1], _ptr(c), c.shape[0], _ptr(out))
        return out

    def moments_axis0(self, x, p=1, ddof=0):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        mean = np.empty(m, np.float64)
        var = np.empty(m, np.float64)
        if self.lib.dno_moments_axis0(_ptr(x), n, m, p, ddof, _ptr(mean), _ptr(var)) != 0:
            raise ValueError("var_axis: need more than ddof samples")
        return mean, var

    def local_moments_axis0(self, x):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        c = np.zeros(1, np.int64)
        mean = np.empty(m, np.float64)
        m2 = np.empty(m, np.float64)
        self.lib.dno_local_moments_axis0(_ptr(x), n, m, _ptr(c), _ptr(mean), _ptr(m2))
        return int(c[0]), mean, m2

    def welford_stream(self, blocks, m):
        """The reference's single-rank Welford (moments.cpp:100-114) over an
        iterable of fp32 [rows x m] blocks, in order; returns (count, mean, m2)."""
        cnt = np.zeros(1, np.int64)
        mean = np.zeros(m, np.float64)
        m2 = np.zeros(m, np.float64)
        for b in blocks:
            b = np.ascontiguousarray(b, np.float32)
            self.lib.dno_welford_axis0_f32_continue(_ptr(b), b.shape[0], m, _ptr(cnt), _ptr(mean), _ptr(m2))
        return int(cnt[0]), mean, m2

    def kmeanspp_indices(self, x, k, seed, p=1):
        """float64 input runs the same definition on the doubles; anything else as float32."""
        f64 = np.asarray(x).dtype == np.float64
        x = np.ascontiguousarray(x, np.float64 if f64 else np.float32)
        out = np.empty(k, np.int64)
        fn = self.lib.dno_kmeanspp_indices_f64 if f64 else self.lib.dno_kmeanspp_indices_f32
        if fn(_ptr(x), x.shape[0], x.shape[1], p, k, seed, _ptr(out)) != 0:
            raise ValueError("kmeanspp: k out of range")
        return out


def _oracle_lasso(self, x, y, lam, sweeps, tol=0.0, p=1):
    rc, w, trace, run = _lasso_call(self.lib.dno_lasso_fit, x, y, lam, sweeps, tol, p)
    if rc == -1:
        raise ValueError("lasso_fit: invalid arguments")
    if rc == -2:
        raise ValueError("lasso_fit: column 0 must be the all-ones bias column")
    return w, trace, run


def _lasso_call(fn, x, y, lam, sweeps, tol, p):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64).reshape(-1)
    n, m = x.shape
    w = np.zeros(m, np.float64)
    trace = np.zeros(sweeps, np.float64)
    run = np.zeros(1, np.int32)
    rc = fn(_ptr(x), _ptr(y), n, m, p, lam, sweeps, tol, _ptr(w), _ptr(trace), _ptr(run))
    return rc, w, trace[: run[0]].copy(), int(run[0])


class ReferenceError_(RuntimeError):
    pass


class Reference:
    """The unmodified reference library (oracle/_ref/libdndref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_chunk_map.argtypes = [_i64, _i32, _P, _P]
        L.ref_fill_uniform_f32.argtypes = [_i64, _i64, _u64, _i32, _P]
        L.ref_row_norms.argtypes = [_P, _i64, _i64, _P]
        L.ref_cdist.argtypes = [_P, _i64, _i64, _i32, _P, _P]
        L.ref_cdist_xy.argtypes = [_P, _i64, _P, _i64, _i64, _i32, _P]
        L.ref_kmeans_init_indices.argtypes = [_i64, _i32, _u64, _P]
        L.ref_kmeans_fit.argtypes = [_P, _i64, _i64, _i32, _i32, _i32, _f64, _u64, _P, _P, _P]
        L.ref_kmeans_fit_synthetic.argtypes = [_i64, _i64, _u64, _i32, _i32, _i32, _f64, _u64,
                                               _P, _P, _P]
        L.ref_kmeans_predict.argtypes = [_P, _i64, _i64, _i32, _P, _i32, _P]
        L.ref_moments_axis0.argtypes = [_P, _i64, _i64, _i32, _i64, _P, _P]
        L.ref_bench.argtypes = [_i32, _i64, _i64, _i32, _i32, _u64, _i32, _i32, _i32, _P, _P]
        L.ref_lasso_fit.argtypes = [_P, _P, _i64, _i64, _i32, _f64, _i32, _f64, _P, _P, _P]

    def _check(self, rc):
        if rc == -1:
            raise ValueError(self.lib.ref_last_error().decode())
        if rc != 0:
            raise ReferenceError_(self.lib.ref_last_error().decode())

    def chunk_map(self, n, p):
        off = np.empty(p, np.int64)
        ext = np.empty(p, np.int64)
        self._check(self.lib.ref_chunk_map(n, p, _ptr(off), _ptr(ext)))
        return off, ext

    def uniform_f32(self, n, m, seed, p=1):
        out = np.empty((n, m), np.float32)
        self._check(self.lib.ref_fill_uniform_f32(n, m, seed, p, _ptr(out)))
        return out

    def row_norms(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.shape[0], np.float64)
        self._check(self.lib.ref_row_norms(_ptr(x), x.shape[0], x.shape[1], _ptr(out)))
        return out

    def cdist(self, x, p=1):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        out = np.empty((n, n), np.float64)
        sr = np.zeros(1, np.uint64)
        self._check(self.lib.ref_cdist(_ptr(x), n, m, p, _ptr(out), _ptr(sr)))
        return out, int(sr[0])

    def cdist_xy(self, x, y, p=1):
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty((x.shape[0], y.shape[0]), np.float64)
        self._check(self.lib.ref_cdist_xy(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], p,
                                          _ptr(out)))
        return out

    def kmeans_init_indices(self, n, k, seed):
        out = np.empty(k, np.int64)
        self._check(self.lib.ref_kmeans_init_indices(n, k, seed, _ptr(out)))
        return out

    def kmeans_fit(self, x, k, max_iter, tol=0.0, seed=42, p=1):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        cent = np.empty((k, m), np.float64)
        trace = np.zeros(max_iter, np.float64)
        it = np.zeros(1, np.int32)
        self._check(self.lib.ref_kmeans_fit(_ptr(x), n, m, p, k, max_iter, tol, seed, _ptr(cent),
                                            _ptr(trace), _ptr(it)))
        return cent, trace[: it[0]].copy(), int(it[0])

    def kmeans_fit_synthetic(self, n, m, data_seed, k, max_iter, tol=0.0, seed=42, p=1):
        cent = np.empty((k, m), np.float64)
        trace = np.zeros(max_iter, np.float64)
        it = np.zeros(1, np.int32)
        self._check(self.lib.ref_kmeans_fit_synthetic(n, m, data_seed, p, k, max_iter, tol, seed,
                                                      _ptr(cent), _ptr(trace), _ptr(it)))
        return cent, trace[: it[0]].copy(), int(it[0])

    def kmeans_predict(self, x, centroids, p=1):
        x = np.ascontiguousarray(x, np.float64)
        c = np.ascontiguousarray(centroids, np.float64)
        out = np.empty(x.shape[0], np.int32)
        self._check(self.lib.ref_kmeans_predict(_ptr(x), x.shape[0], x.shape[1], p, _ptr(c),
                                                c.shape[0], _ptr(out)))
        return out

    def moments_axis0(self, x, p=1, ddof=0):
        x = np.ascontiguousarray(x, np.float64)
        n, m = x.shape
        mean = np.empty(m, np.float64)
        var = np.empty(m, np.float64)
        self._check(self.lib.ref_moments_axis0(_ptr(x), n, m, p, ddof, _ptr(mean), _ptr(var)))
        return mean, var

    def bench(self, algo, n, m, k, iters, seed, p, warmup, runs):
        """tools/bench.cpp protocol; algo 0 kmeans, 1 cdist, 2 moments."""
        secs = np.zeros(max(runs, 1), np.float64)
        chk = np.zeros(1, np.float64)
        self._check(self.lib.ref_bench(algo, n, m, k, iters, seed, p, warmup, runs, _ptr(secs),
                                       _ptr(chk)))
        return secs[:runs], float(chk[0])


Oracle.lasso_fit = _oracle_lasso


def _reference_lasso(self, x, y, lam, sweeps, tol=0.0, p=1):
    rc, w, trace, run = _lasso_call(self.lib.ref_lasso_fit, x, y, lam, sweeps, tol, p)
    self._check(rc)
    return w, trace, run


Reference.lasso_fit = _reference_lasso
