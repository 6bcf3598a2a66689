"""Oracle for the colour-transfer front end: k-means quantisation of an
8-bit RGB image into m colours x_k with histogram a (TEST INFRASTRUCTURE ONLY: imported by
tests/, __graft_entry__.smoke() and bench.py's baseline legs, never by the product path).

PAPER.md P:425-426: "The algorithm of the feature extraction uses the k-means algorithm for
image quantization ... After executing k-means with a predefined number of classes, all the
pixels in the image are assigned into each class. Averaging all the pixel values assigned in
each class yields ... centroids ... we obtain a color histogram a by counting of the assigned
pixels". The paper's litekmeans internals are not given; readings R28-R30 fix
them: Lloyd iterations from k given distinct pixels, squared Euclidean RGB distance
((d0^2 + d1^2) + d2^2) in fp64 with the first (lowest-index) minimum, centroids = exact integer
channel sums / count, stop when an assignment repeats the previous one and the previous
update moved no pixel; an empty cluster takes the pixel farthest from its own centroid (SPEC
S:400), clusters in ascending order.
Plain numpy, fp64, written out step by step.
"""
from __future__ import annotations

import numpy as np

__all__ = ["kmeans_quantize", "kmeanspp_init", "sqdist", "colour_features", "recolour"]


def sqdist(P: np.ndarray, C: np.ndarray) -> np.ndarray:
    """||p - c||^2 evaluated as ((d0*d0 + d1*d1) + d2*d2) in fp64; P: N x 3, C: K x 3 -> N x K."""
    d0 = P[:, None, 0] - C[None, :, 0]
    d1 = P[:, None, 1] - C[None, :, 1]
    d2 = P[:, None, 2] - C[None, :, 2]
    return (d0 * d0 + d1 * d1) + d2 * d2


def _assign(P, cen, chunk=4096):
    lab = np.empty(len(P), dtype=np.int32)
    for s in range(0, len(P), chunk):
        lab[s:s + chunk] = np.argmin(sqdist(P[s:s + chunk], cen), axis=1)   # first minimum
    return lab


def kmeans_quantize(pixels: np.ndarray, k: int, init_idx: np.ndarray, max_iters: int):
    """pixels: N x 3 uint8; init_idx: k distinct pixel indices. Returns (centroids N.B. in
    0..255 units, fp64 k x 3; labels int32 N; counts int64 k; iterations; converged)."""
    P = np.asarray(pixels, dtype=np.uint8).astype(np.float64)
    N = len(P)
    cen = P[np.asarray(init_idx)].copy()
    labels = None
    counts = np.zeros(k, dtype=np.int64)
    it = 0
    converged = False
    repaired = False
    while it < max_iters:
        it += 1
        new = _assign(P, cen)
        if labels is not None and not repaired and np.array_equal(new, labels):
            converged = True
            break
        labels = new
        repaired = False
        counts = np.bincount(labels, minlength=k).astype(np.int64)
        for c in range(3):   # exact: integer sums below 2^53
            s = np.bincount(labels, weights=P[:, c], minlength=k)
            nz = counts > 0
            cen[nz, c] = s[nz] / counts[nz]
        for c in np.nonzero(counts == 0)[0]:
            own = cen[labels]
            d = (((P[:, 0] - own[:, 0]) * (P[:, 0] - own[:, 0]) + (P[:, 1] - own[:, 1]) * (P[:, 1] - own[:, 1]))
                 + (P[:, 2] - own[:, 2]) * (P[:, 2] - own[:, 2]))
            d[counts[labels] <= 1] = -1.0          # never empty another cluster
            p = int(np.argmax(d))                  # first maximum
            if d[p] < 0.0:
                continue
            cen[c] = P[p]
            counts[labels[p]] -= 1
            labels[p] = c
            counts[c] = 1
            repaired = True
    return cen, labels, counts, it, converged


def kmeanspp_init(pixels: np.ndarray, k: int, u: np.ndarray) -> np.ndarray:
    """k-means++ seeding (reading R34 in DESIGN.md) of the k initial centres as pixel
    indices, from k uniforms u in [0, 1) drawn by the caller:
      c_0 = min(floor(u_0 N), N - 1);
      D2(p) = min over the chosen centres c of ||P_p - P_c||^2 (8-bit pixels: exact integers);
      c_t = the first p whose inclusive prefix sum of D2 (pixel order) exceeds
            min(floor(u_t * total), total - 1), total = sum_p D2(p) (a D2-weighted draw);
            if total == 0 (every pixel repeats a chosen colour) c_t = the lowest index not chosen.
    Integer sums, so no summation order enters."""
    P = np.asarray(pixels, dtype=np.uint8).astype(np.int64)
    N = len(P)
    u = np.asarray(u, dtype=np.float64)
    out = np.empty(k, dtype=np.int32)
    chosen = np.zeros(N, dtype=bool)
    c = min(int(np.float64(u[0]) * np.float64(N)), N - 1)
    D2 = None
    for t in range(k):
        if t > 0:
            total = int(D2.sum())
            if total == 0:
                c = int(np.nonzero(~chosen)[0][0])
            else:
                target = int(np.float64(u[t]) * np.float64(total))   # one rounded product, then floor
                target = min(target, total - 1)
                prefix = np.cumsum(D2)
                c = int(np.searchsorted(prefix, target, side="right"))   # first prefix > target
        out[t] = c
        chosen[c] = True
        d = P - P[c]
        dist = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
        D2 = dist if D2 is None else np.minimum(D2, dist)
    return out


def colour_features(cen: np.ndarray, counts: np.ndarray, npix: int):
    """(x, a) of P:426: colours in [0,1]^3 (centroid / 255) and the histogram counts / N."""
    return cen / 255.0, counts.astype(np.float64) / float(npix)


def recolour(labels: np.ndarray, xhat: np.ndarray) -> np.ndarray:
    """each pixel takes its class's projected colour x_hat (Eq. 15), back to 8 bits:
    round-half-even of 255 * x_hat, clipped to [0, 255]."""
    v = np.rint(255.0 * xhat[labels])
    return np.clip(v, 0.0, 255.0).astype(np.uint8)
