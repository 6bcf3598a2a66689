"""Thin ctypes binding of libsro.so (include/sro.h). Argument marshalling only:
every step of the method runs in the CUDA kernels behind the C-ABI. There is
no CPU fallback: if the library cannot be loaded, or no CUDA device is
present, every call raises.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

__all__ = [
    "load_library", "Solver", "SroError", "SRO_FW", "SRO_BCFW", "SRO_BCAFW", "SRO_BCPFW", "SRO_BATCHED",
    "STEP_DEC", "STEP_ELS", "SAMPLE_U", "SAMPLE_P", "SAMPLE_GA", "TRACE_DTYPE", "EXPORTED_SYMBOLS",
    "nccl_unique_id", "kmeans_quantize", "kmeanspp_init", "kmeans_features", "recolour", "colour_transfer",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SRO_LIB", os.path.join(HERE, "libsro.so"))


def _default_nccl_lib():
    """The libnccl.so.2 of the nvidia-nccl wheel torch is built against (the library dlopens NCCL
    for sharded handles; an older system copy loaded first would break a later `import torch`)."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


if "SRO_NCCL_LIB" not in os.environ:
    _nccl = _default_nccl_lib()
    if _nccl:
        os.environ["SRO_NCCL_LIB"] = _nccl

SRO_FW, SRO_BCFW, SRO_BCAFW, SRO_BCPFW, SRO_BATCHED = 0, 1, 2, 3, 4
STEP_DEC, STEP_ELS = 0, 1
SAMPLE_U, SAMPLE_P, SAMPLE_GA = 0, 1, 2
COST_KINDS = {"dense": 0, "sqeuclid": 1, "euclid": 2, "hash": 3}
PRECS = {"f64": 0, "f32": 1}
OK, NOT_CONVERGED = 0, 1
EXPORTED_SYMBOLS = ("sro_create", "sro_solve", "sro_gap", "sro_objective", "sro_get_plan", "sro_get_rowsums",
                    "sro_reset", "sro_destroy", "sro_last_error", "sro_version", "sro_get_stats", "sro_set_timing",
                    "sro_held_columns", "sro_nccl_unique_id", "sro_barycentric", "sro_metrics",
                    "sro_kmeans", "sro_recolour", "sro_kmeans_error", "sro_lp_metrics", "sro_kmeans_features",
                    "sro_kmeanspp")

_STATUS = {0: "OK", 1: "NOT_CONVERGED", 2: "ERR_INVALID_ARG", 3: "ERR_DIMENSION", 4: "ERR_MARGINALS",
           5: "ERR_NONFINITE", 6: "ERR_CAPACITY", 7: "ERR_CUDA", 8: "ERR_NCCL", 9: "ERR_OOM", 10: "ERR_STATE"}


class SroError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"sro status {status} ({_STATUS.get(status, '?')}): {msg}")
        self.status = status


class SroCost(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("prec", ct.c_int32), ("data", ct.c_void_p), ("ld", ct.c_int64),
                ("x", ct.c_void_p), ("y", ct.c_void_p), ("hash_seed", ct.c_uint64), ("data_on_device", ct.c_int32)]


# sro_exchange_fn: int32 (*)(void* user, double* buf, int64 count, int32 nranks, int32 rank)
EXCHANGE_FN = ct.CFUNCTYPE(ct.c_int32, ct.c_void_p, ct.POINTER(ct.c_double), ct.c_int64, ct.c_int32, ct.c_int32)


class SroParams(ct.Structure):
    _fields_ = [("m", ct.c_int32), ("n", ct.c_int32), ("lambda_", ct.c_double), ("slab_cap", ct.c_int32),
                ("device", ct.c_int32), ("cuda_stream", ct.c_void_p), ("shards", ct.c_int32),
                ("shard_block", ct.c_int32), ("nranks", ct.c_int32), ("rank", ct.c_int32), ("nccl_id", ct.c_void_p),
                ("max_sms", ct.c_int32), ("exchange", EXCHANGE_FN), ("exchange_user", ct.c_void_p)]


class SroTraceRec(ct.Structure):
    _fields_ = [("k", ct.c_int64), ("i", ct.c_int32), ("j", ct.c_int32), ("v", ct.c_int32), ("dir", ct.c_int32),
                ("gamma", ct.c_double), ("num", ct.c_double), ("den", ct.c_double), ("minval", ct.c_double)]


TRACE_DTYPE = np.dtype([("k", np.int64), ("i", np.int32), ("j", np.int32), ("v", np.int32), ("dir", np.int32),
                        ("gamma", np.float64), ("num", np.float64), ("den", np.float64), ("minval", np.float64)])
assert TRACE_DTYPE.itemsize == ct.sizeof(SroTraceRec)


class SroOptions(ct.Structure):
    _fields_ = [("step", ct.c_int32), ("sampling", ct.c_int32), ("epsilon", ct.c_double),
                ("gap_period", ct.c_int32), ("ga_M", ct.c_int32), ("ga_inner", ct.c_int32),
                ("ga_post_update", ct.c_int32), ("block_size", ct.c_int32), ("visit", ct.c_void_p),
                ("trace", ct.c_void_p)]


class SroResult(ct.Structure):
    _fields_ = [("iters_done", ct.c_int64), ("k", ct.c_int64), ("gap", ct.c_double), ("objective", ct.c_double),
                ("converged", ct.c_int32), ("gap_checks", ct.c_int32), ("entries_scanned", ct.c_int64),
                ("device_ms", ct.c_double), ("entries_read", ct.c_int64)]


class SroStats(ct.Structure):
    _fields_ = [("kernel_launches", ct.c_int64), ("bcfw_launches", ct.c_int64), ("bcfw_steps", ct.c_int64),
                ("bcfw_ms", ct.c_double), ("sweep_launches", ct.c_int64), ("sweep_columns", ct.c_int64),
                ("sweep_ms", ct.c_double), ("block_steps", ct.c_int64), ("block_ms", ct.c_double)]


_lib = None


def load_library():
    """Load libsro.so (built by paper_2103_05857_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SroError(-1, f"{LIB_PATH} missing: run `python -m paper_2103_05857_b200.build`")
        L = ct.CDLL(LIB_PATH)
        vp, i32, i64, u64, d = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint64, ct.c_double
        L.sro_create.argtypes = [vp, vp, ct.POINTER(SroCost), ct.POINTER(SroParams), ct.POINTER(vp)]
        L.sro_create.restype = ct.c_int
        L.sro_solve.argtypes = [vp, i32, ct.POINTER(SroOptions), i64, u64, ct.POINTER(SroResult)]
        L.sro_solve.restype = ct.c_int
        L.sro_gap.argtypes = [vp, ct.POINTER(d), vp, vp]
        L.sro_gap.restype = ct.c_int
        L.sro_objective.argtypes = [vp, ct.POINTER(d)]
        L.sro_objective.restype = ct.c_int
        L.sro_get_plan.argtypes = [vp, vp, vp, vp, vp, i64, ct.POINTER(i64)]
        L.sro_get_plan.restype = ct.c_int
        L.sro_get_rowsums.argtypes = [vp, vp]
        L.sro_get_rowsums.restype = ct.c_int
        L.sro_reset.argtypes = [vp]
        L.sro_reset.restype = ct.c_int
        L.sro_destroy.argtypes = [vp]
        L.sro_destroy.restype = None
        L.sro_last_error.argtypes = [vp]
        L.sro_last_error.restype = ct.c_char_p
        L.sro_get_stats.argtypes = [vp, ct.POINTER(SroStats), i32]
        L.sro_get_stats.restype = ct.c_int
        L.sro_set_timing.argtypes = [vp, i32]
        L.sro_set_timing.restype = ct.c_int
        L.sro_version.argtypes = []
        L.sro_version.restype = ct.c_char_p
        L.sro_held_columns.argtypes = [vp, vp, ct.POINTER(i32)]
        L.sro_held_columns.restype = ct.c_int
        L.sro_nccl_unique_id.argtypes = [vp]
        L.sro_nccl_unique_id.restype = ct.c_int
        L.sro_barycentric.argtypes = [vp, vp, vp, vp]
        L.sro_barycentric.restype = ct.c_int
        L.sro_metrics.argtypes = [vp, ct.POINTER(d), ct.POINTER(d), ct.POINTER(d)]
        L.sro_metrics.restype = ct.c_int
        L.sro_kmeans.argtypes = [vp, i64, i32, vp, i32, i32, vp, vp, vp, vp, ct.POINTER(i32), ct.POINTER(i32)]
        L.sro_kmeans.restype = ct.c_int
        L.sro_kmeanspp.argtypes = [vp, i64, i32, vp, i32, vp, vp]
        L.sro_kmeanspp.restype = ct.c_int
        L.sro_recolour.argtypes = [vp, i64, vp, i32, vp, vp]
        L.sro_recolour.restype = ct.c_int
        L.sro_lp_metrics.argtypes = [vp, vp, vp, vp, i64, ct.POINTER(d), ct.POINTER(d)]
        L.sro_lp_metrics.restype = ct.c_int
        L.sro_kmeans_features.argtypes = [vp, vp, i32, vp, vp]
        L.sro_kmeans_features.restype = ct.c_int
        L.sro_kmeans_error.argtypes = []
        L.sro_kmeans_error.restype = ct.c_char_p
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):          # torch tensor (device or host)
        return ct.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ct.c_void_p)


def _is_cuda(t):
    return hasattr(t, "is_cuda") and t.is_cuda


class Solver:
    """One solver handle: problem (a, b, cost, lambda) + plan state on the GPU.

    cost='dense': C is m x n (rows = source bins); numpy arrays are copied,
    CUDA torch tensors are borrowed (pass C.T-contiguous, i.e. column-major).
    cost='sqeuclid' / 'euclid': X (m x 3) and Y (n x 3) colours.
    cost='hash': iid uniform C generated on the device from hash_seed.
    prec='f64' | 'f32' is the storage / evaluation precision of the cost.
    max_sms > 0 sizes the handle's device-wide kernels for that many SMs (sro_params.max_sms).
    """

    def __init__(self, a, b, lam, *, C=None, X=None, Y=None, cost="dense", prec="f64", hash_seed=0, slab_cap=31,
                 device=0, stream=None, ld=None, shards=1, shard_block=0, nranks=1, rank=0, nccl_id=None,
                 max_sms=0, exchange=None):
        L = load_library()
        self._L = L
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        self.m, self.n = len(a), len(b)
        self.lam = float(lam)
        kind = COST_KINDS[cost]
        pr = PRECS[prec]
        dt = np.float32 if prec == "f32" else np.float64
        keep = []
        c = SroCost(kind=kind, prec=pr, data=None, ld=0, x=None, y=None, hash_seed=hash_seed, data_on_device=0)
        if kind == 0:
            if _is_cuda(C):
                # device tensor, column-major storage: shape (n, ld) row-major
                c.data, c.data_on_device = _ptr(C), 1
                c.ld = ld if ld is not None else C.shape[1]
            else:
                Cm = np.asarray(C, dtype=dt)
                assert Cm.shape[0] == self.m
                Ccm = np.ascontiguousarray(Cm.T)        # column i contiguous
                keep.append(Ccm)
                c.data, c.ld = _ptr(Ccm), self.m
        elif kind in (1, 2):
            if _is_cuda(X):
                c.x, c.y, c.data_on_device = _ptr(X), _ptr(Y), 1
            else:
                Xc = np.ascontiguousarray(X, dtype=dt)
                Yc = np.ascontiguousarray(Y, dtype=dt)
                keep += [Xc, Yc]
                c.x, c.y = _ptr(Xc), _ptr(Yc)
        idbuf = None
        if nccl_id is not None:
            idbuf = ct.create_string_buffer(bytes(nccl_id), 128)
        # exchange: a Python all-gather f(buf, rank) over an (nranks, count) float64 host array whose
        # row `rank` is filled (sro_exchange_fn); the ctypes thunk lives as long as the handle
        self._xfn = None
        if exchange is not None:
            def _thunk(user, buf, count, nr, rk, _f=exchange):
                try:
                    _f(np.ctypeslib.as_array(buf, shape=(nr * count,)).reshape(nr, count), rk)
                    return 0
                except Exception:  # noqa: BLE001 — reported to the library as a failed exchange
                    return 1
            self._xfn = EXCHANGE_FN(_thunk)
        p = SroParams(m=self.m, n=self.n, lambda_=self.lam, slab_cap=slab_cap, device=device,
                      cuda_stream=ct.c_void_p(stream) if stream else None, shards=shards, shard_block=shard_block,
                      nranks=nranks, rank=rank, nccl_id=ct.cast(idbuf, ct.c_void_p) if idbuf is not None else None,
                      max_sms=max_sms, exchange=self._xfn if self._xfn is not None else EXCHANGE_FN(),
                      exchange_user=None)
        h = ct.c_void_p()
        st = L.sro_create(_ptr(a), _ptr(b), ct.byref(c), ct.byref(p), ct.byref(h))
        if st != OK:
            raise SroError(st, L.sro_last_error(None).decode())
        self.h = h
        self.cap = slab_cap
        # borrowed device tensors must outlive the handle (sro.h): held until close()
        self._borrowed = tuple(t for t in (C, X, Y) if _is_cuda(t))
        nh = ct.c_int32()
        self._check(L.sro_held_columns(h, None, ct.byref(nh)))
        self.held = np.empty(nh.value, dtype=np.int32)
        self._check(L.sro_held_columns(h, _ptr(self.held), ct.byref(nh)))
        self.n_held = nh.value

    def _check(self, st, allow=(OK,)):
        if st not in allow:
            raise SroError(st, self._L.sro_last_error(self.h).decode())
        return st

    def close(self):
        if getattr(self, "h", None):
            self._L.sro_destroy(self.h)
            self.h = None
        self._borrowed = ()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, variant, iters, seed=0, *, step=STEP_ELS, sampling=SAMPLE_U, epsilon=1e-6, gap_period=1, ga_M=1,
              ga_inner=1, ga_post_update=1, block_size=1, visit=None, trace=False):
        vis = None
        if visit is not None:
            vis = np.ascontiguousarray(visit, dtype=np.int32)
            assert len(vis) >= iters
        tr = np.zeros(max(iters, 1), dtype=TRACE_DTYPE) if trace else None
        o = SroOptions(step=step, sampling=sampling, epsilon=epsilon, gap_period=gap_period, ga_M=ga_M,
                       ga_inner=ga_inner, ga_post_update=ga_post_update, block_size=block_size,
                       visit=_ptr(vis), trace=_ptr(tr))
        r = SroResult()
        st = self._L.sro_solve(self.h, variant, ct.byref(o), iters, seed, ct.byref(r))
        self._check(st, (OK, NOT_CONVERGED))
        out = {f: getattr(r, f) for f, _ in SroResult._fields_}
        out["status"] = st
        if trace:
            out["trace"] = tr[: r.iters_done]
        return out

    def gap(self):
        tot = ct.c_double()
        g = np.empty(self.n_held)
        j = np.empty(self.n_held, dtype=np.int32)
        self._check(self._L.sro_gap(self.h, ct.byref(tot), _ptr(g), _ptr(j)))
        return tot.value, g, j

    def objective(self):
        f = ct.c_double()
        self._check(self._L.sro_objective(self.h, ct.byref(f)))
        return f.value

    def plan(self):
        T = np.empty(self.m * self.n_held)
        nnz = ct.c_int64()
        self._check(self._L.sro_get_plan(self.h, _ptr(T), None, None, None, 0, ct.byref(nnz)))
        return T.reshape(self.n_held, self.m).T.copy()

    def plan_coo(self):
        nnz = ct.c_int64()
        self._check(self._L.sro_get_plan(self.h, None, None, None, None, 0, ct.byref(nnz)))
        k = nnz.value
        r = np.empty(k, dtype=np.int32)
        c = np.empty(k, dtype=np.int32)
        v = np.empty(k)
        self._check(self._L.sro_get_plan(self.h, None, _ptr(r), _ptr(c), _ptr(v), k, ct.byref(nnz)))
        return r, c, v

    def barycentric(self, X, Y):
        """Eq. 15: new source colours (m x 3); rows without mass keep X."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        assert X.shape == (self.m, 3) and Y.shape == (self.n, 3)
        out = np.empty((self.m, 3))
        self._check(self._L.sro_barycentric(self.h, _ptr(X), _ptr(Y), _ptr(out)))
        return out

    def metrics(self):
        """(e_c, sparsity, <T, C>): metrics (iii), (iv) and the plan value of (vi)."""
        e, sp, lin = ct.c_double(), ct.c_double(), ct.c_double()
        self._check(self._L.sro_metrics(self.h, ct.byref(e), ct.byref(sp), ct.byref(lin)))
        return e.value, sp.value, lin.value

    def lp_metrics(self, rows, cols, vals):
        """(e_m, e_v): metrics (v) and (vi) of P:419-421 against a reference plan T* (e.g. T*_LP)
        given as COO sorted by column, then row (sro_lp_metrics)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        em, ev = ct.c_double(), ct.c_double()
        self._check(self._L.sro_lp_metrics(self.h, _ptr(rows), _ptr(cols), _ptr(vals), len(vals), ct.byref(em),
                                           ct.byref(ev)))
        return em.value, ev.value

    def rowsums(self):
        r = np.empty(self.m)
        self._check(self._L.sro_get_rowsums(self.h, _ptr(r)))
        return r

    def reset(self):
        self._check(self._L.sro_reset(self.h))

    def set_timing(self, on=True):
        self._check(self._L.sro_set_timing(self.h, 1 if on else 0))

    def stats(self, reset=False):
        s = SroStats()
        self._check(self._L.sro_get_stats(self.h, ct.byref(s), 1 if reset else 0))
        return {f: getattr(s, f) for f, _ in SroStats._fields_}


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (create on rank 0, share with the other ranks)."""
    L = load_library()
    buf = ct.create_string_buffer(128)
    st = L.sro_nccl_unique_id(ct.cast(buf, ct.c_void_p))
    if st != OK:
        raise SroError(st, L.sro_last_error(None).decode())
    return buf.raw


# --------------------------------------------------------------------------- colour-transfer front end
def kmeans_quantize(pixels, k: int, init_idx, max_iters: int = 100, stream=None):
    """sro_kmeans: k-means quantisation of npix x 3 uint8 pixels (numpy, or a CUDA uint8 tensor,
    borrowed). Returns (centroids fp64 k x 3 in 0..255 units, labels int32, counts int64,
    iterations, converged)."""
    L = load_library()
    on_dev = 1 if _is_cuda(pixels) else 0
    if not on_dev:
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
    npix = int(pixels.shape[0])
    init = np.ascontiguousarray(init_idx, dtype=np.int32)
    cen = np.empty((k, 3), dtype=np.float64)
    lab = np.empty(npix, dtype=np.int32)
    cnt = np.empty(k, dtype=np.int64)
    it, conv = ct.c_int32(0), ct.c_int32(0)
    st = L.sro_kmeans(_ptr(pixels), npix, int(k), _ptr(init), int(max_iters), on_dev,
                      ct.c_void_p(stream) if stream else None, _ptr(cen), _ptr(lab), _ptr(cnt), ct.byref(it),
                      ct.byref(conv))
    if st != OK:
        raise SroError(st, L.sro_kmeans_error().decode())
    return cen, lab, cnt, int(it.value), bool(conv.value)


def kmeanspp_init(pixels, k: int, u, stream=None):
    """sro_kmeanspp: k-means++ seeding (R34) of k distinct pixel indices from the caller's k uniforms
    u in [0, 1) (numpy pixels, or a CUDA uint8 tensor, borrowed). Returns int32[k]."""
    L = load_library()
    on_dev = 1 if _is_cuda(pixels) else 0
    if not on_dev:
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
    npix = int(pixels.shape[0])
    uu = np.ascontiguousarray(u, dtype=np.float64)
    k = int(k)
    if uu.shape[0] < max(k, 0):
        raise SroError(2, "u needs k uniforms")
    out = np.empty(max(k, 0), dtype=np.int32)
    st = L.sro_kmeanspp(_ptr(pixels), npix, k, _ptr(uu), on_dev, ct.c_void_p(stream) if stream else None, _ptr(out))
    if st != OK:
        raise SroError(st, L.sro_kmeans_error().decode())
    return out


def kmeans_features(centroids, counts):
    """sro_kmeans_features: (colours k x 3 = centroid / 255, histogram counts / N), R29."""
    L = load_library()
    cen = np.ascontiguousarray(centroids, dtype=np.float64)
    cnt = np.ascontiguousarray(counts, dtype=np.int64)
    k = len(cnt)
    x = np.empty((k, 3))
    w = np.empty(k)
    st = L.sro_kmeans_features(_ptr(cen), _ptr(cnt), k, _ptr(x), _ptr(w))
    if st != OK:
        raise SroError(st, L.sro_kmeans_error().decode())
    return x, w


def recolour(labels, xhat, stream=None):
    """sro_recolour: npix x 3 uint8 pixels, each its class's colour rint(255 x_hat)."""
    L = load_library()
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    xh = np.ascontiguousarray(xhat, dtype=np.float64)
    out = np.empty((len(lab), 3), dtype=np.uint8)
    st = L.sro_recolour(_ptr(lab), len(lab), _ptr(xh), int(xh.shape[0]), ct.c_void_p(stream) if stream else None,
                        _ptr(out))
    if st != OK:
        raise SroError(st, L.sro_kmeans_error().decode())
    return out


def colour_transfer(src_pixels, ref_pixels, m: int, n: int, init_src, init_ref, lam: float = 1.0,
                    variant: int = SRO_BCFW, iters: int | None = None, epsilon: float = 1e-6, cost: str = "euclid",
                    prec: str = "f64", kmeans_iters: int = 100, seed: int = 0, **solve_opts):
    """The paper's colour-transfer pipeline on the GPU: quantise the source into m
    colours x with histogram a and the reference into n colours y with b (sro_kmeans),
    solve the semi-relaxed problem with C = ||x_k - y_i||_2 (or its square), project the
    source colours (Eq. 15, sro_barycentric) and recolour the source pixels (sro_recolour).
    init_src / init_ref: m / n distinct pixel indices (k-means++ seeds from kmeanspp_init, or any
    caller's draw). Returns (recoloured pixels, solve result dict, (x, a, y, b, xhat))."""
    cx, lx, ax_cnt, _, _ = kmeans_quantize(src_pixels, m, init_src, kmeans_iters)
    cy, _, by_cnt, _, _ = kmeans_quantize(ref_pixels, n, init_ref, kmeans_iters)
    x, a = kmeans_features(cx, ax_cnt)
    y, b = kmeans_features(cy, by_cnt)
    s = Solver(a, b, lam, X=x, Y=y, cost=cost, prec=prec)
    try:
        res = s.solve(variant, iters if iters is not None else 1000 * n, seed=seed, epsilon=epsilon, **solve_opts)
        xhat = s.barycentric(x, y)
    finally:
        s.close()
    return recolour(lx, xhat), res, (x, a, y, b, xhat)
