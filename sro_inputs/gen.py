"""Input recipes for the five BASELINE.json configs.

The paper's workloads are k-means-quantised colour histograms of real photo
pairs (P:422, P:425-427 of /root/reference/PAPER.md); those photos are not
available, so seeded synthetic colour sets with the same structure stand in:
Gaussian-mixture colours in [0,1]^3 with density-shaped histogram weights, and
for config [3] an iid-uniform dense cost defined by a random-access hash.

Random numbers come from a counter-based SplitMix64 stream implemented here
in numpy uint64 arithmetic, so every array is reproducible bit-for-bit on any
host. Nothing here computes anything the solver computes.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "GOLDEN", "splitmix64_mix", "rng_u64", "uniform53", "normals",
    "uniform_colours", "mixture_colours", "density_weights", "uniform_weights",
    "sqeuclid_cost", "hash_uniform_cost", "instance", "CONFIGS",
    "synthetic_image", "kmeans_init", "kmeanspp_uniforms",
]

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_mix(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def rng_u64(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Values offset..offset+count-1 of the SplitMix64 sequence seeded by `seed`."""
    t = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (t + np.uint64(1)) * GOLDEN
    return splitmix64_mix(z)


def uniform53(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normals(seed: int, count: int) -> np.ndarray:
    """Box-Muller standard normals from the seed's uniform stream."""
    half = (count + 1) // 2
    u = uniform53(rng_u64(seed, 2 * half))
    u1 = 1.0 - u[0::2]          # (0, 1]
    u2 = u[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    z = np.concatenate([rad * np.cos(2 * np.pi * u2), rad * np.sin(2 * np.pi * u2)])
    return z[:count]


def uniform_colours(count: int, seed: int) -> np.ndarray:
    """count x 3 colours iid uniform in [0,1]^3 (BASELINE config [0])."""
    return uniform53(rng_u64(seed, 3 * count)).reshape(count, 3)


def mixture_colours(count: int, K: int, sigma: float, seed: int, quantise: bool = False):
    """Colours from a K-component Gaussian mixture in [0,1]^3 (configs [1],[2],[4]).

    Means ~ U[0,1]^3, weights ~ Dirichlet(1) (normalised Exp(1)), point
    x = clip(mu_z + sigma N(0, I3), 0, 1); `quantise` rounds to the 1/255 grid,
    which produces exact duplicate colours (exact cost ties).
    Returns (X, means, pis).
    """
    means = uniform53(rng_u64(seed * 7919 + 1, 3 * K)).reshape(K, 3)
    e = -np.log(1.0 - uniform53(rng_u64(seed * 7919 + 2, K)))
    pis = e / e.sum()
    u = uniform53(rng_u64(seed * 7919 + 3, count))
    z = np.searchsorted(np.cumsum(pis), u, side="right")
    z = np.minimum(z, K - 1)
    X = means[z] + sigma * normals(seed * 7919 + 4, 3 * count).reshape(count, 3)
    X = np.clip(X, 0.0, 1.0)
    if quantise:
        X = np.round(255.0 * X) / 255.0
    return X, means, pis


def density_weights(X: np.ndarray, means: np.ndarray, pis: np.ndarray, sigma: float) -> np.ndarray:
    """'Mixture-histogram weights': a_k proportional to the mixture density at x_k, normalised to 1."""
    d2 = ((X[:, None, :] - means[None, :, :]) ** 2).sum(-1)
    w = (pis[None, :] * np.exp(-d2 / (2 * sigma * sigma))).sum(-1)
    w = np.maximum(w, 1e-300)
    a = w / w.sum()
    return a


def uniform_weights(count: int) -> np.ndarray:
    return np.full(count, 1.0 / count)


def sqeuclid_cost(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Column-major view helper: returns C with C[k, i] = ||x_k - y_i||^2 in fp64,
    evaluated as ((dx*dx + dy*dy) + dz*dz) in that order (m x n, C order)."""
    dx = X[:, None, 0] - Y[None, :, 0]
    dy = X[:, None, 1] - Y[None, :, 1]
    dz = X[:, None, 2] - Y[None, :, 2]
    return (dx * dx + dy * dy) + dz * dz


def hash_uniform_cost(seed: int, m: int, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Config [3] cost: C_ki = (splitmix64(seed, i*m + k) >> 40) * 2^-24 (exact in fp32)."""
    idx = cols.astype(np.uint64) * np.uint64(m) + rows.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx + np.uint64(1)) * GOLDEN
    return (splitmix64_mix(z) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


CONFIGS = {
    0: dict(name="tiny-bcfw-fp64", m=256, n=256, lam=1.0, cost="dense", dtype="f64"),
    1: dict(name="colour-4096", m=4096, n=4096, lam=1.0, cost="dense", dtype="f32"),
    2: dict(name="quantised-16384-batched", m=16384, n=16384, lam=1.0, cost="sqeuclid", dtype="f32", B=256),
    3: dict(name="dense-uniform-65536-fw", m=65536, n=65536, lam=1.0, cost="hash", dtype="f32"),
    4: dict(name="rect-4096x262144-batched", m=4096, n=262144, lam=1.0, cost="sqeuclid", dtype="f32", B=1024),
}


def instance(cfg: int, m: int | None = None, n: int | None = None, seed: int = 0):
    """Problem inputs for BASELINE config `cfg`, optionally at a reduced size.

    Returns a dict: m, n, lam, a, b (fp64), X, Y (fp64 colours, or None),
    C64 (m x n fp64, C order, for dense configs at sizes that fit), C32
    (float32 version), cost ('dense' | 'sqeuclid' | 'hash'), hash_seed.
    """
    c = CONFIGS[cfg]
    m = c["m"] if m is None else m
    n = c["n"] if n is None else n
    out = dict(cfg=cfg, m=m, n=n, lam=c["lam"], cost=c["cost"], dtype=c["dtype"], X=None, Y=None,
               C64=None, C32=None, hash_seed=None, B=c.get("B"))
    if cfg == 0:
        X = uniform_colours(m, seed)
        Y = uniform_colours(n, seed + 1_000_003)
        out.update(X=X, Y=Y, a=uniform_weights(m), b=uniform_weights(n))
        out["C64"] = sqeuclid_cost(X, Y)
    elif cfg in (1, 2, 4):
        K = 16 if cfg == 2 else 8
        X, mx, px = mixture_colours(m, K, 0.05, 2 * seed + 1, quantise=(cfg == 2))
        Y, my, py = mixture_colours(n, K, 0.05, 2 * seed + 2, quantise=(cfg == 2))
        out.update(X=X, Y=Y, a=density_weights(X, mx, px, 0.05), b=density_weights(Y, my, py, 0.05))
        if cfg == 1:
            C64 = sqeuclid_cost(X, Y)
            out["C32"] = C64.astype(np.float32)
            out["C64"] = out["C32"].astype(np.float64)
    elif cfg == 3:
        out.update(a=uniform_weights(m), b=uniform_weights(n), hash_seed=0x5EED0003 + seed)
    return out


# --------------------------------------------------------------------------- colour-transfer front end
def synthetic_image(height: int, width: int, K: int = 8, sigma: float = 0.05, seed: int = 0) -> np.ndarray:
    """An 8-bit RGB image (height*width x 3, row-major pixels) standing in for the paper's photos
    (P:422): K smooth regions (nearest of K random seed points), each region's pixels
    drawn from its own Gaussian colour (mean ~ U[0,1]^3, sd sigma), clipped and rounded to
    0..255. Exact duplicate pixel colours occur, as in real 8-bit images."""
    N = height * width
    pts = uniform53(rng_u64(seed * 104729 + 11, 2 * K)).reshape(K, 2)
    means = uniform53(rng_u64(seed * 104729 + 12, 3 * K)).reshape(K, 3)
    yy, xx = np.meshgrid((np.arange(height) + 0.5) / height, (np.arange(width) + 0.5) / width, indexing="ij")
    d = (yy.reshape(-1, 1) - pts[None, :, 0]) ** 2 + (xx.reshape(-1, 1) - pts[None, :, 1]) ** 2
    z = np.argmin(d, axis=1)
    X = means[z] + sigma * normals(seed * 104729 + 13, 3 * N).reshape(N, 3)
    return np.round(255.0 * np.clip(X, 0.0, 1.0)).astype(np.uint8)


def kmeans_init(npix: int, k: int, seed: int) -> np.ndarray:
    """k distinct pixel indices (the k-means initial centres, drawn by sampling without
    replacement: a partial Fisher-Yates shuffle on the seed's uniform stream). This is the
    random draw of the k-means front end, passed as an input to both the oracle and the GPU."""
    if not 1 <= k <= npix:
        raise ValueError("need 1 <= k <= number of pixels")
    u = uniform53(rng_u64(seed * 1000003 + 17, k))
    perm = {}
    out = np.empty(k, dtype=np.int32)
    for t in range(k):
        r = t + int(u[t] * (npix - t))
        r = min(r, npix - 1)
        vt, vr = perm.get(t, t), perm.get(r, r)
        perm[t], perm[r] = vr, vt
        out[t] = vr
    return out


def kmeanspp_uniforms(k: int, seed: int) -> np.ndarray:
    """The k uniforms in [0, 1) that k-means++ seeding consumes (one per centre), passed as an
    input to both the oracle and the GPU (the draw itself is the method's; R34)."""
    if k < 1:
        raise ValueError("need k >= 1")
    return uniform53(rng_u64(seed * 1000003 + 29, k))
