"""Colour-transfer front end: k-means quantisation.

CPU: the oracle (oracle/kmeans.py) pinned by closed forms (k distinct colours, k = 1), the
Lloyd fixed-point conditions checked by brute force, and the empty-cluster rule on a worked
example. GPU: sro_kmeans bit-exact against the oracle (centroids, labels, counts, iterations).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from oracle.kmeans import colour_features, kmeans_quantize, kmeanspp_init, recolour
from sro_inputs import kmeans_init, kmeanspp_uniforms, synthetic_image


def test_k_distinct_colours_are_recovered_exactly():
    rng = np.random.default_rng(0)
    k = 7
    cols = rng.integers(0, 256, size=(k, 3)).astype(np.uint8)
    mult = rng.integers(1, 20, size=k)
    pix = np.repeat(cols, mult, axis=0)
    order = rng.permutation(len(pix))
    pix = pix[order]
    first = np.array([int(np.nonzero((pix == c).all(1))[0][0]) for c in cols], dtype=np.int32)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, k, first, 50)
    assert conv and it == 2
    assert np.array_equal(cen, cols.astype(np.float64))
    assert np.array_equal(cnt, mult)
    assert np.array_equal(cols[lab], pix)


def test_single_class_is_the_exact_mean():
    pix = synthetic_image(10, 13, seed=3)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, 1, np.array([5], dtype=np.int32), 10)
    assert conv and cnt[0] == len(pix) and np.all(lab == 0)
    for c in range(3):   # the correctly rounded quotient of the exact integer sum
        assert cen[0, c] == float(int(pix[:, c].astype(np.int64).sum())) / len(pix)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_converged_point_satisfies_lloyd_conditions(seed):
    """Brute force on a small image: every pixel's class is its nearest centroid (first
    minimum, exact rational distances) and every centroid is its members' mean."""
    pix = synthetic_image(12, 15, K=4, seed=seed)
    k = 6
    cen, lab, cnt, it, conv = kmeans_quantize(pix, k, kmeans_init(len(pix), k, seed), 200)
    assert conv
    P = [[Fraction(int(v)) for v in p] for p in pix]
    C = [[Fraction(float(v)) for v in c] for c in cen]
    for q in range(len(pix)):
        d = [sum((P[q][t] - C[c][t]) ** 2 for t in range(3)) for c in range(k)]
        best = min(d)
        # exact-rational nearest; ties / 1-ulp fp64 differences resolved to the lowest index
        assert d[lab[q]] == best or abs(float(d[lab[q]] - best)) <= 1e-9 * float(best + 1)
    for c in range(k):
        mem = pix[lab == c].astype(np.int64)
        assert len(mem) == cnt[c]
        if len(mem):
            for t in range(3):
                assert cen[c, t] == float(int(mem[:, t].sum())) / len(mem)


def test_empty_cluster_takes_the_farthest_pixel():
    """Worked example: both initial centres black -> the second class is empty after the
    first assignment; the update puts class 0 at the mean (53, 53, 53) and the repair gives
    class 1 the farthest pixel (white); the next update moves class 0 to the mean of the rest."""
    pix = np.array([[0, 0, 0], [0, 0, 0], [0, 0, 0], [255, 255, 255], [10, 10, 10]], dtype=np.uint8)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, 2, np.array([0, 1], dtype=np.int32), 20)
    assert conv and it == 3
    assert np.array_equal(lab, [0, 0, 0, 1, 0])
    assert np.array_equal(cnt, [4, 1])
    assert np.array_equal(cen, [[2.5, 2.5, 2.5], [255.0, 255.0, 255.0]])


def test_features_and_recolour():
    cen = np.array([[0.0, 127.5, 255.0], [10.2, 20.7, 30.5]])
    x, a = colour_features(cen, np.array([3, 1]), 4)
    assert np.array_equal(a, [0.75, 0.25]) and np.array_equal(x[0], [0.0, 0.5, 1.0])
    out = recolour(np.array([0, 1, 1]), np.array([[0.5, 1.2, -0.1], [0.002, 0.998, 0.5]]))
    assert out.tolist() == [[128, 255, 0], [1, 254, 128], [1, 254, 128]]


# --------------------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("h,w,k,seed", [(16, 16, 5, 0), (64, 48, 32, 1), (128, 128, 256, 2), (97, 101, 300, 3),
                                          (256, 256, 1024, 4)])
def test_gpu_kmeans_bitexact(h, w, k, seed):
    sro = pytest.importorskip("paper_2103_05857_b200")
    pix = synthetic_image(h, w, seed=seed)
    init = kmeans_init(len(pix), k, seed + 7)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, k, init, 60)
    gc, gl, gn, git, gconv = sro.kmeans_quantize(pix, k, init, 60)
    assert git == it and gconv == conv
    assert np.array_equal(gl, lab) and np.array_equal(gn, cnt) and np.array_equal(gc, cen)


@pytest.mark.gpu
def test_gpu_kmeans_empty_cluster_repair_bitexact():
    sro = pytest.importorskip("paper_2103_05857_b200")
    pix = synthetic_image(40, 40, K=3, seed=9)
    # initial centres with repeated colours force empty classes (and repairs) in the first pass
    _, first, inv = np.unique(pix, axis=0, return_index=True, return_inverse=True)
    rep = np.nonzero(np.bincount(inv.ravel()) >= 2)[0][:4]
    pairs = [np.nonzero(inv.ravel() == r)[0][:2] for r in rep]
    init = np.unique(np.concatenate([np.concatenate(pairs), kmeans_init(len(pix), 12, 3)])).astype(np.int32)
    k = len(init)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, k, init, 60)
    gc, gl, gn, git, gconv = sro.kmeans_quantize(pix, k, init, 60)
    assert git == it and np.array_equal(gl, lab) and np.array_equal(gn, cnt) and np.array_equal(gc, cen)
    # the worked example as well
    pix2 = np.array([[0, 0, 0], [0, 0, 0], [0, 0, 0], [255, 255, 255], [10, 10, 10]], dtype=np.uint8)
    gc, gl, gn, git, gconv = sro.kmeans_quantize(pix2, 2, np.array([0, 1], dtype=np.int32), 20)
    assert git == 3 and gl.tolist() == [0, 0, 0, 1, 0] and gn.tolist() == [4, 1]
    assert gc.tolist() == [[2.5, 2.5, 2.5], [255.0, 255.0, 255.0]]


@pytest.mark.gpu
@pytest.mark.parametrize("cost", ["euclid", "sqeuclid"])
def test_gpu_colour_transfer_pipeline_bitexact(cost):
    """The whole pipeline of P:424-432 on a small image pair: k-means (m, n colours), BCFW-P-ELS
    to g <= 1e-8, Eq. 15 projection and recolouring; the GPU's recoloured pixels, plan and
    colours equal the oracle chain's bit for bit."""
    sro = pytest.importorskip("paper_2103_05857_b200")
    from oracle import BCFW, ELS, P, Oracle
    src, ref = synthetic_image(48, 40, seed=21), synthetic_image(40, 56, seed=22)
    m, n = 24, 20
    init_s, init_r = kmeans_init(len(src), m, 1), kmeans_init(len(ref), n, 2)
    out, res, (x, a, y, b, xhat) = sro.colour_transfer(src, ref, m, n, init_s, init_r, lam=1.0, variant=sro.SRO_BCFW,
                                                       iters=400 * n, epsilon=1e-8, cost=cost, step=sro.STEP_ELS,
                                                       sampling=sro.SAMPLE_P, seed=3)
    cx, lx, cnx, _, _ = kmeans_quantize(src, m, init_s, 100)
    cy, _, cny, _, _ = kmeans_quantize(ref, n, init_r, 100)
    ox, oa = colour_features(cx, cnx, len(src))
    oy, ob = colour_features(cy, cny, len(ref))
    assert np.array_equal(ox, x) and np.array_equal(oa, a) and np.array_equal(oy, y) and np.array_equal(ob, b)
    o = Oracle(oa, ob, 1.0, X=ox, Y=oy, cost=cost, prec="f64", cap=31)
    r = o.solve(BCFW, 400 * n, seed=3, step=ELS, sampling=P, epsilon=1e-8)
    assert r["iters_done"] == res["iters_done"] and r["gap"] == res["gap"]
    oxh = o.barycentric(ox, oy)
    assert np.array_equal(oxh, xhat)
    assert np.array_equal(recolour(lx, oxh), out)


@pytest.mark.gpu
def test_gpu_kmeans_errors_and_k_equals_npix():
    sro = pytest.importorskip("paper_2103_05857_b200")
    pix = synthetic_image(6, 5, seed=4)
    with pytest.raises(sro.SroError):
        sro.kmeans_quantize(pix, 3, np.array([1, 1, 2], dtype=np.int32), 10)     # repeated initial centre
    with pytest.raises(sro.SroError):
        sro.kmeans_quantize(pix, 31, np.arange(31, dtype=np.int32), 10)          # k > number of pixels
    with pytest.raises(sro.SroError):
        sro.kmeans_quantize(pix, 2, np.array([0, 30], dtype=np.int32), 10)       # index out of range
    # k = npix: every pixel its own class unless colours repeat (repairs keep classes non-empty)
    init = np.arange(len(pix), dtype=np.int32)
    cen, lab, cnt, it, conv = kmeans_quantize(pix, len(pix), init, 20)
    gc, gl, gn, git, gconv = sro.kmeans_quantize(pix, len(pix), init, 20)
    assert git == it and np.array_equal(gc, cen) and np.array_equal(gl, lab) and np.array_equal(gn, cnt)


@pytest.mark.gpu
def test_gpu_kmeans_features_match_oracle_and_reject_bad_input():
    """sro_kmeans_features (R29 behind the C-ABI): colours = centroid / 255 and histogram = count / N
    bit-equal to the oracle's colour_features; negative counts, all-zero counts and k < 1 raise."""
    sro = pytest.importorskip("paper_2103_05857_b200")
    from oracle.kmeans import colour_features
    rng = np.random.default_rng(3)
    cen = rng.random((17, 3)) * 255.0
    cnt = rng.integers(0, 50, size=17).astype(np.int64)
    cnt[4] = 0
    x, a = sro.kmeans_features(cen, cnt)
    xo, ao = colour_features(cen, cnt, int(cnt.sum()))
    assert np.array_equal(x, xo) and np.array_equal(a, ao)
    for bad in (np.array([3, -1, 2]), np.zeros(3, dtype=np.int64)):
        with pytest.raises(sro.SroError):
            sro.kmeans_features(np.ones((3, 3)), bad)


# ---- k-means++ seeding (R34) ----------------------------------------

def _brute_d2(P, centres):
    """min over the centres of the squared RGB distance, python integers (independent of the oracle)."""
    out = []
    for p in P:
        out.append(min(sum((int(p[q]) - int(P[c][q])) ** 2 for q in range(3)) for c in centres))
    return out


def test_kmeanspp_oracle_draw_is_d2_weighted():
    """Pin: the second centre is drawn with probability D2(p) / sum D2 — over a uniform grid of G values
    of u_1 each pixel is chosen G * D2(p) / total times up to one per boundary."""
    P = np.array([[0, 0, 0], [10, 0, 0], [0, 20, 0], [3, 4, 12], [255, 255, 255], [0, 0, 0], [7, 7, 7]], np.uint8)
    u0 = 0.0   # first centre: pixel 0
    d2 = _brute_d2(P, [0])
    total = sum(d2)
    G = 20000
    counts = np.zeros(len(P), dtype=np.int64)
    for g in range(G):
        c = kmeanspp_init(P, 2, np.array([u0, (g + 0.5) / G]))
        assert c[0] == 0
        counts[c[1]] += 1
    for p in range(len(P)):
        assert abs(counts[p] - G * d2[p] / total) <= 1.0 + 1e-9, (p, counts[p], G * d2[p] / total)
    assert counts[0] == 0 and counts[5] == 0   # D2 = 0: never drawn


def test_kmeanspp_oracle_first_centre_and_edges():
    P = synthetic_image(9, 11, seed=4).reshape(-1, 3)
    N = len(P)
    for u0 in (0.0, 0.3, 0.999999999):
        c = kmeanspp_init(P, 1, np.array([u0]))
        assert c[0] == min(int(u0 * N), N - 1)
    # u_t = 0: the first pixel with D2 > 0 (the target 0 is exceeded by the first nonzero prefix)
    c = kmeanspp_init(P, 3, np.array([0.5, 0.0, 0.0]))
    d2 = _brute_d2(P, [c[0]])
    assert c[1] == next(p for p in range(N) if d2[p] > 0)
    d2 = _brute_d2(P, [c[0], c[1]])
    assert c[2] == next(p for p in range(N) if d2[p] > 0)
    # every centre is a pixel index, all distinct, and each later centre had D2 > 0 when drawn
    u = kmeanspp_uniforms(12, 2)
    c = kmeanspp_init(P, 12, u)
    assert len(set(c.tolist())) == 12
    for t in range(1, 12):
        assert _brute_d2(P, c[:t].tolist())[c[t]] > 0


def test_kmeanspp_oracle_fewer_colours_than_centres():
    """Every pixel repeats one of three colours, k = 6: three centres of distinct colours, then (total D2
    = 0) the lowest indices not yet chosen."""
    base = np.array([[1, 2, 3], [200, 100, 0], [50, 50, 50]], np.uint8)
    P = base[np.array([0, 1, 0, 2, 1, 1, 0, 2])]
    c = kmeanspp_init(P, 6, np.array([0.4, 0.9, 0.1, 0.5, 0.5, 0.5]))
    assert len({tuple(P[i]) for i in c[:3]}) == 3
    rest = [p for p in range(len(P)) if p not in set(c[:3].tolist())][:3]
    assert c[3:].tolist() == rest


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,k,seed", [(1, 1, 1, 0), (7, 13, 5, 1), (100, 100, 64, 2), (333, 517, 257, 3),
                                        (1000, 1000, 128, 4)])
def test_gpu_kmeanspp_bitexact(h, w, k, seed):
    """k-means++ seeding on the GPU (sro_kmeanspp) equals the oracle's centre for centre."""
    import paper_2103_05857_b200 as sro
    img = synthetic_image(h, w, seed=seed).reshape(-1, 3)
    k = min(k, len(img))
    u = kmeanspp_uniforms(k, seed)
    ref = kmeanspp_init(img, k, u)
    got = sro.kmeanspp_init(img, k, u)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
def test_gpu_kmeanspp_degenerate_and_errors():
    import paper_2103_05857_b200 as sro
    base = np.array([[1, 2, 3], [200, 100, 0], [50, 50, 50]], np.uint8)
    rng = np.random.default_rng(5)
    P = base[rng.integers(0, 3, size=5000)]
    u = kmeanspp_uniforms(9, 7)
    assert np.array_equal(sro.kmeanspp_init(P, 9, u), kmeanspp_init(P, 9, u))
    with pytest.raises(sro.SroError):
        sro.kmeanspp_init(P, 0, u)
    with pytest.raises(sro.SroError):
        sro.kmeanspp_init(P[:4], 9, u)
    with pytest.raises(sro.SroError):
        sro.kmeanspp_init(P, 2, np.array([0.5, 1.0]))


@pytest.mark.gpu
def test_gpu_kmeans_from_kmeanspp_seeds_bitexact():
    """Lloyd from k-means++ seeds: the GPU chain (sro_kmeanspp -> sro_kmeans) equals the oracle chain."""
    import paper_2103_05857_b200 as sro
    img = synthetic_image(120, 160, seed=6).reshape(-1, 3)
    u = kmeanspp_uniforms(32, 6)
    init = kmeanspp_init(img, 32, u)
    ref = kmeans_quantize(img, 32, init, 50)
    g_init = sro.kmeanspp_init(img, 32, u)
    got = sro.kmeans_quantize(img, 32, g_init, 50)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])
