"""ctypes binding of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY).

The C source (oracle/sro_oracle.c) is the oracle: plain fp64 loops written
step by step from /root/reference/PAPER.md, compiled with -O2
-ffp-contract=off. This file only marshals arguments.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

__all__ = [
    "build_oracle", "Oracle", "OrOptions", "OrResult", "TRACE_DTYPE",
    "FW", "BCFW", "BCAFW", "BCPFW", "BATCHED", "DEC", "ELS", "U", "P", "GA",
    "COST_DENSE", "COST_SQEUCLID", "COST_EUCLID", "COST_HASH",
    "chunk_tree_sum", "rng_u64", "uniform53", "permutation", "fenwick_draw", "fenwick_updates", "splitmix64_mix",
    "OracleError",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "sro_oracle.c")

FW, BCFW, BCAFW, BCPFW, BATCHED = 0, 1, 2, 3, 4
DEC, ELS = 0, 1
U, P, GA = 0, 1, 2
COST_DENSE, COST_SQEUCLID, COST_EUCLID, COST_HASH = 0, 1, 2, 3
OK, NOT_CONVERGED = 0, 1


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2 -ffp-contract=off, single thread)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11",
                               "-o", LIB, SRC, "-lm"])
    return LIB


class OrOptions(ct.Structure):
    _fields_ = [("step_rule", ct.c_int32), ("sampling", ct.c_int32), ("epsilon", ct.c_double),
                ("gap_period", ct.c_int32), ("ga_M", ct.c_int32), ("ga_inner", ct.c_int32),
                ("ga_post_update", ct.c_int32), ("block_size", ct.c_int32), ("nranks", ct.c_int32)]


class OrResult(ct.Structure):
    _fields_ = [("iters_done", ct.c_int64), ("k", ct.c_int64), ("gap", ct.c_double), ("objective", ct.c_double),
                ("converged", ct.c_int32), ("gap_checks", ct.c_int32), ("entries_scanned", ct.c_int64)]


TRACE_DTYPE = np.dtype([("k", np.int64), ("i", np.int32), ("j", np.int32), ("v", np.int32), ("dir", np.int32),
                        ("gamma", np.float64), ("num", np.float64), ("den", np.float64), ("minval", np.float64)])

_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build_oracle())
        d, i32, i64, u64, vp = ct.c_double, ct.c_int32, ct.c_int64, ct.c_uint64, ct.c_void_p
        _lib.or_create.restype = vp
        _lib.or_create.argtypes = [i32, i32, d, vp, vp, i32, vp, i64, vp, vp, u64, i32, ct.POINTER(ct.c_int)]
        _lib.or_destroy.argtypes = [vp]
        _lib.or_reset.argtypes = [vp]
        _lib.or_solve.argtypes = [vp, i32, ct.POINTER(OrOptions), i64, u64, vp, ct.POINTER(OrResult), vp]
        _lib.or_gap.argtypes = [vp, ct.POINTER(d), vp, vp, vp]
        _lib.or_gap_thm2.argtypes = [vp, ct.POINTER(d)]
        _lib.or_lagrangian_dual.argtypes = [vp, ct.POINTER(d)]
        _lib.or_objective.argtypes = [vp, ct.POINTER(d)]
        _lib.or_barycentric.argtypes = [vp, vp, vp, vp]
        _lib.or_metrics.argtypes = [vp, ct.POINTER(d), ct.POINTER(d), ct.POINTER(d)]
        _lib.or_lp_metrics.argtypes = [vp, vp, vp, vp, i64, ct.POINTER(d), ct.POINTER(d)]
        _lib.or_get_plan_dense.argtypes = [vp, vp]
        _lib.or_get_plan_coo.argtypes = [vp, vp, vp, vp, i64, ct.POINTER(i64)]
        _lib.or_get_r.argtypes = [vp, vp]
        _lib.or_set_plan_dense.argtypes = [vp, vp]
        _lib.or_get_k.argtypes = [vp]
        _lib.or_get_k.restype = i64
        _lib.or_cost.argtypes = [vp, i32, i32]
        _lib.or_cost.restype = d
        _lib.or_lmo_column.argtypes = [vp, i32, ct.POINTER(i32), ct.POINTER(d)]
        _lib.or_max_cost.argtypes = [vp, ct.POINTER(d)]
        _lib.or_chunk_tree_sum.argtypes = [vp, i64, i32]
        _lib.or_chunk_tree_sum.restype = d
        _lib.or_splitmix64_mix.argtypes = [u64]
        _lib.or_splitmix64_mix.restype = u64
        _lib.or_rng_u64.argtypes = [u64, ct.c_uint32, u64]
        _lib.or_rng_u64.restype = u64
        _lib.or_uniform53.argtypes = [u64]
        _lib.or_uniform53.restype = d
        _lib.or_permutation.argtypes = [u64, i64, i32, vp]
        _lib.or_fenwick_draw.argtypes = [vp, i32, d, ct.POINTER(i32)]
        _lib.or_get_ga.argtypes = [vp, vp, vp]
        _lib.or_fenwick_updates.argtypes = [vp, i32, vp, vp, i32, vp, vp, i32, vp]
    return _lib


def _p(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def chunk_tree_sum(x, W: int) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return _L().or_chunk_tree_sum(_p(x), len(x), W)


def splitmix64_mix(z: int) -> int:
    return _L().or_splitmix64_mix(z)


def rng_u64(seed: int, stream: int, t: int) -> int:
    return _L().or_rng_u64(seed, stream, t)


def uniform53(x: int) -> float:
    return _L().or_uniform53(x)


def permutation(seed: int, epoch: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    _L().or_permutation(seed, epoch, n, _p(out))
    return out


def fenwick_draw(w, u53: float) -> int:
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = ct.c_int32()
    _L().or_fenwick_draw(_p(w), len(w), u53, ct.byref(out))
    return out.value


def fenwick_updates(w0, idx, newval, u53s):
    """Tree over w0, point updates column idx[u] := newval[u] (GA inner-refresh rule), then
    (prefix sums as the tree holds them, one draw per u53)."""
    w0 = np.ascontiguousarray(w0, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    newval = np.ascontiguousarray(newval, dtype=np.float64)
    u53s = np.ascontiguousarray(u53s, dtype=np.float64)
    prefix = np.empty(len(w0))
    draws = np.empty(len(u53s), dtype=np.int32)
    _L().or_fenwick_updates(_p(w0), len(w0), _p(idx), _p(newval), len(idx), _p(prefix), _p(u53s), len(u53s),
                            _p(draws))
    return prefix, draws


def make_options(step=ELS, sampling=U, epsilon=1e-6, gap_period=1, ga_M=1, ga_inner=1, ga_post_update=1,
                 block_size=1, nranks=1) -> OrOptions:
    return OrOptions(step, sampling, epsilon, gap_period, ga_M, ga_inner, ga_post_update, block_size, nranks)


class Oracle:
    """One oracle instance (problem + plan state)."""

    def __init__(self, a, b, lam, *, C=None, X=None, Y=None, cost="dense", prec="f64", hash_seed=0, cap=64):
        L = _L()
        self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        self.m, self.n = len(self.a), len(self.b)
        self.lam = float(lam)
        self.cap = cap
        kind = {"dense": COST_DENSE, "sqeuclid": COST_SQEUCLID, "euclid": COST_EUCLID, "hash": COST_HASH}[cost]
        if prec == "f32" and kind in (COST_SQEUCLID, COST_EUCLID):
            kind += 3            # colours evaluated in binary32 (OR_COST_*_F32)
            X = np.asarray(X, dtype=np.float32).astype(np.float64)
            Y = np.asarray(Y, dtype=np.float32).astype(np.float64)
        elif prec == "f32" and kind == COST_DENSE:
            C = np.asarray(C, dtype=np.float32).astype(np.float64)
        Cc = Xc = Yc = None
        ld = self.m
        if kind == COST_DENSE:
            # C given as m x n (row k, column i); store column-major: column i contiguous
            Cc = np.asfortranarray(np.asarray(C, dtype=np.float64))
            assert Cc.shape == (self.m, self.n)
            Cc = Cc.T.copy()  # n x m C-order == column-major m x n
        elif kind != COST_HASH:
            Xc = np.ascontiguousarray(X, dtype=np.float64)
            Yc = np.ascontiguousarray(Y, dtype=np.float64)
        st = ct.c_int(0)
        self.h = L.or_create(self.m, self.n, self.lam, _p(self.a), _p(self.b), kind, _p(Cc), ld, _p(Xc), _p(Yc),
                             hash_seed, cap, ct.byref(st))
        if not self.h:
            raise OracleError(st.value, "create")

    def __del__(self):
        if getattr(self, "h", None):
            _L().or_destroy(self.h)
            self.h = None

    def reset(self):
        _L().or_reset(self.h)

    def solve(self, variant, iters, seed=0, visit=None, trace=False, **opt):
        o = make_options(**opt)
        res = OrResult()
        tr = np.zeros(max(iters, 1), dtype=TRACE_DTYPE) if trace else None
        vis = None
        if visit is not None:
            vis = np.ascontiguousarray(visit, dtype=np.int32)
            assert len(vis) >= iters
        st = _L().or_solve(self.h, variant, ct.byref(o), iters, seed, _p(vis), ct.byref(res), _p(tr))
        if st not in (OK, NOT_CONVERGED):
            raise OracleError(st, "solve")
        out = {f: getattr(res, f) for f, _ in OrResult._fields_}
        out["status"] = st
        if trace:
            out["trace"] = tr[: res.iters_done]
        return out

    def gap(self):
        tot = ct.c_double()
        g = np.empty(self.n)
        j = np.empty(self.n, dtype=np.int32)
        mv = np.empty(self.n)
        st = _L().or_gap(self.h, ct.byref(tot), _p(g), _p(j), _p(mv))
        if st:
            raise OracleError(st, "gap")
        return tot.value, g, j, mv

    def gap_thm2(self):
        g = ct.c_double()
        st = _L().or_gap_thm2(self.h, ct.byref(g))
        if st:
            raise OracleError(st)
        return g.value

    def lagrangian_dual(self):
        w = ct.c_double()
        st = _L().or_lagrangian_dual(self.h, ct.byref(w))
        if st:
            raise OracleError(st)
        return w.value

    def objective(self):
        f = ct.c_double()
        _L().or_objective(self.h, ct.byref(f))
        return f.value

    def barycentric(self, X, Y):
        """Eq. 15: new source colours (m x 3); rows without mass keep X."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        out = np.empty((self.m, 3))
        st = _L().or_barycentric(self.h, _p(X), _p(Y), _p(out))
        if st:
            raise OracleError(st, "barycentric")
        return out

    def metrics(self):
        """(e_c, sparsity, <T, C>) — metrics (iii), (iv) and the <T,C> of (vi)."""
        e, sp, lin = ct.c_double(), ct.c_double(), ct.c_double()
        st = _L().or_metrics(self.h, ct.byref(e), ct.byref(sp), ct.byref(lin))
        if st:
            raise OracleError(st, "metrics")
        return e.value, sp.value, lin.value

    def lp_metrics(self, rows, cols, vals):
        """(e_m, e_v) — metrics (v) and (vi) against T* in COO sorted by (column, row)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        em, ev = ct.c_double(), ct.c_double()
        st = _L().or_lp_metrics(self.h, _p(rows), _p(cols), _p(vals), len(vals), ct.byref(em), ct.byref(ev))
        if st:
            raise OracleError(st, "lp_metrics")
        return em.value, ev.value

    def plan(self):
        T = np.empty(self.m * self.n)
        _L().or_get_plan_dense(self.h, _p(T))
        return T.reshape(self.n, self.m).T.copy()  # m x n

    def plan_coo(self, cap=None):
        cap = cap or self.n * self.cap
        r = np.empty(cap, dtype=np.int32)
        c = np.empty(cap, dtype=np.int32)
        v = np.empty(cap)
        nnz = ct.c_int64()
        st = _L().or_get_plan_coo(self.h, _p(r), _p(c), _p(v), cap, ct.byref(nnz))
        if st:
            raise OracleError(st)
        k = nnz.value
        return r[:k], c[:k], v[:k]

    def r(self):
        r = np.empty(self.m)
        _L().or_get_r(self.h, _p(r))
        return r

    def set_plan(self, T):
        Tc = np.ascontiguousarray(np.asarray(T, dtype=np.float64).T)  # column-major
        st = _L().or_set_plan_dense(self.h, _p(Tc))
        if st:
            raise OracleError(st, "set_plan")

    @property
    def k(self):
        return _L().or_get_k(self.h)

    def cost(self, k, i):
        return _L().or_cost(self.h, k, i)

    def lmo(self, i):
        j = ct.c_int32()
        v = ct.c_double()
        st = _L().or_lmo_column(self.h, i, ct.byref(j), ct.byref(v))
        if st:
            raise OracleError(st)
        return j.value, v.value

    def ga_state(self):
        """(stored gaps G, prefix sums of the GA tree) after a GA solve."""
        G = np.empty(self.n)
        pre = np.empty(self.n)
        st = _L().or_get_ga(self.h, _p(G), _p(pre))
        if st:
            raise OracleError(st, "ga_state")
        return G, pre

    def max_cost(self):
        v = ct.c_double()
        _L().or_max_cost(self.h, ct.byref(v))
        return v.value
