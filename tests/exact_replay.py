"""Exact-rational replay of the paper's algorithms (a pin for the fp64 oracle).

An independent, deliberately naive implementation in Python `fractions`:
dense T, exact arithmetic, written straight from PAPER.md —
  * gradient  grad_i f = c_i + (T 1_n - a)/lambda
  * LMO       s_i = b_i e_j, j = argmin_k grad_ki (lowest k) (Eq. 9)
  * BCFW      gamma = 2n/(k+2n) or Eq. 10 line search       (Alg. 1)
  * FW        gamma = 2/(k+2) or Eq. A.1                    (Alg. A.1)
  * BCAFW / BCPFW with Eq. 14                              (Alg. A.2/A.3)
Exact arithmetic has no summation-order or rounding choices, so agreement
with the fp64 oracle (argmins exact, values to ~1e-13) pins the oracle's
indices, signs and operand order independently of its fp64 code.
"""
from __future__ import annotations

from fractions import Fraction as Fr


class ExactState:
    def __init__(self, C, a, b, lam):
        self.m, self.n = len(a), len(b)
        self.C = [[Fr(C[k][i]) for i in range(self.n)] for k in range(self.m)]
        self.a = [Fr(x) for x in a]
        self.b = [Fr(x) for x in b]
        self.lam = Fr(lam)
        # T^(0) = (b_1 e_1, ..., b_n e_1)
        self.T = [[self.b[i] if k == 0 else Fr(0) for i in range(self.n)] for k in range(self.m)]
        self.k = 0

    def r(self):
        return [sum(self.T[k]) for k in range(self.m)]

    def grad(self, i):
        r = self.r()
        return [self.C[k][i] + (r[k] - self.a[k]) / self.lam for k in range(self.m)]

    def lmo(self, i):
        g = self.grad(i)
        j = min(range(self.m), key=lambda k: (g[k], k))
        return j, g

    def lmo_tied(self, i):
        """True if the exact minimum of grad_i f is attained by more than one row: an
        exact tie (created structurally by exact line searches) that fp64
        breaks by rounding, so exact and fp64 replays may legitimately part there."""
        g = self.grad(i)
        mn = min(g)
        return sum(1 for x in g if x == mn) > 1

    def f(self):
        r = self.r()
        lin = sum(self.T[k][i] * self.C[k][i] for k in range(self.m) for i in range(self.n))
        return lin + sum((r[k] - self.a[k]) ** 2 for k in range(self.m)) / (2 * self.lam)

    def gap(self):
        tot = Fr(0)
        for i in range(self.n):
            j, g = self.lmo(i)
            tot += sum(self.T[k][i] * g[k] for k in range(self.m)) - self.b[i] * g[j]
        return tot

    def col(self, i):
        return [self.T[k][i] for k in range(self.m)]

    def set_col(self, i, t):
        for k in range(self.m):
            self.T[k][i] = t[k]

    def bcfw_step(self, i, rule):
        j, g = self.lmo(i)
        t = self.col(i)
        s = [self.b[i] if k == j else Fr(0) for k in range(self.m)]
        if rule == "dec":
            gamma = Fr(2 * self.n, self.k + 2 * self.n)
        else:
            r = self.r()
            num = self.lam * sum((t[k] - s[k]) * self.C[k][i] for k in range(self.m)) + \
                sum((t[k] - s[k]) * (r[k] - self.a[k]) for k in range(self.m))      # Eq. 10 numerator
            den = sum((t[k] - s[k]) ** 2 for k in range(self.m))
            gamma = Fr(0) if (num <= 0 or den == 0) else min(num / den, Fr(1))
        self.set_col(i, [(1 - gamma) * t[k] + gamma * s[k] for k in range(self.m)])
        self.k += 1
        return j, gamma

    def fw_step(self, rule):
        S = [self.lmo(i)[0] for i in range(self.n)]
        r = self.r()
        S1 = [sum(self.b[i] for i in range(self.n) if S[i] == k) for k in range(self.m)]
        if rule == "dec":
            gamma = Fr(2, self.k + 2)
        else:
            tc = sum(self.T[k][i] * self.C[k][i] for k in range(self.m) for i in range(self.n))
            sc = sum(self.b[i] * self.C[S[i]][i] for i in range(self.n))
            num = self.lam * (tc - sc) + sum((r[k] - S1[k]) * (r[k] - self.a[k]) for k in range(self.m))  # Eq. A.1
            den = sum((r[k] - S1[k]) ** 2 for k in range(self.m))
            gamma = Fr(0) if (num <= 0 or den == 0) else min(num / den, Fr(1))
        for i in range(self.n):
            for k in range(self.m):
                self.T[k][i] = (1 - gamma) * self.T[k][i] + (gamma * self.b[i] if k == S[i] else 0)
        self.k += 1
        return S, gamma

    def away_or_pair_step(self, i, pairwise):
        """Alg. A.2 (away) / Alg. A.3 (pairwise) with the Eq. 14 line search."""
        j, g = self.lmo(i)
        t = self.col(i)
        supp = [k for k in range(self.m) if t[k] != 0]
        v = max(supp, key=lambda k: (g[k], -k))          # argmax over the active set, lowest k on ties
        bi = self.b[i]
        s = [bi if k == j else Fr(0) for k in range(self.m)]
        vv = [bi if k == v else Fr(0) for k in range(self.m)]
        alpha = t[v] / bi
        if pairwise:
            if v == j:
                self.k += 1
                return j, v, Fr(0), "noop"
            d = [s[k] - vv[k] for k in range(self.m)]
            gmax, kind = alpha, "pair"
        else:
            dfw = [s[k] - t[k] for k in range(self.m)]
            daw = [t[k] - vv[k] for k in range(self.m)]
            lin_fw = -sum(g[k] * dfw[k] for k in range(self.m))
            lin_aw = -sum(g[k] * daw[k] for k in range(self.m))
            if len(supp) == 1 or lin_fw >= lin_aw:
                d, gmax, kind = dfw, Fr(1), "fw"
            else:
                d, gmax, kind = daw, alpha / (1 - alpha), "away"
        r = self.r()
        num = -(self.lam * sum(d[k] * self.C[k][i] for k in range(self.m)) +
                sum(d[k] * (r[k] - self.a[k]) for k in range(self.m)))                  # Eq. 14
        den = sum(x * x for x in d)
        gamma = Fr(0) if (num <= 0 or den == 0) else min(num / den, gmax)
        self.set_col(i, [t[k] + gamma * d[k] for k in range(self.m)])
        self.k += 1
        return j, v, gamma, kind


# --------------------------------------------------------------------------- Alg. A.4 (BCFW-GA)
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z):
    """SplitMix64 finaliser (public-domain constants), plain Python integers."""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def u53_exact(seed, stream, t):
    """R21's counter-based draw as an exact rational in [0, 1): value t of stream s is
    mix(mix(seed ^ 0x5851F42D4C957F2D (s+1)) + (t+1) golden), top 53 bits / 2^53."""
    key = _mix((seed ^ ((0x5851F42D4C957F2D * (stream + 1)) & M64)) & M64)
    x = _mix((key + (t + 1) * GOLDEN) & M64)
    return Fr(x >> 11, 1 << 53)


def column_gap(ex, i):
    """g_i(T) = <t_i - s_i, grad_i f> = sum_k t_ki grad_ki - b_i min_k grad_ki (Eq. 11)."""
    j, g = ex.lmo(i)
    return sum(ex.T[k][i] * g[k] for k in range(ex.m)) - ex.b[i] * g[j]


def ga_replay(ex, variant, steps, seed, M, inner, post, cinit, rule="els"):
    """Alg. A.4 exactly as the paper states it, in exact arithmetic:
      line 1   stored gaps G_i = C, "a large constant" (R14: cinit = max C + 2/lambda)
      line 2   draw i with probability max(G_i, 0) / sum_l max(G_l, 0) through the O(n)
               cumulative sum of P:407: the smallest i with w_1 + ... + w_i > u W, where
               u is draw k of stream 1 (R21)
      line 3-5 the block step on column i (Alg. 1 with Eq. 10 or the decay rule; away /
               pairwise with Eq. 14)
      line 6   G_i = g_i(T^{k+1}) after the update ("after update of t_i"; R15),
               or g_i(T^k) with post = False
      global   every M n steps all G_i = g_i(T) (R16: after step k when
               (k+1) mod (M n) == 0). GAS is inner = False with M = 1.
    Returns one record per step, stopping before a step whose draw lies within 1e-9 W of a
    cumulative boundary or whose LMO has an exact tie: there fp64 rounding, not the
    algorithm, decides."""
    n = ex.n
    G = [Fr(cinit)] * n
    out = []
    for k in range(steps):
        w = [x if x > 0 else Fr(0) for x in G]
        W = sum(w)
        u = u53_exact(seed, 1, k)
        if W == 0:
            i = int(u * n)                                      # all-zero weights: uniform (R17)
        else:
            uw, cum, i, margin = u * W, Fr(0), None, None
            for q in range(n):
                cum += w[q]
                d = abs(float((cum - uw) / W))
                margin = d if margin is None else min(margin, d)
                if i is None and cum > uw:
                    i = q
            if margin < 1e-9:
                break
        if ex.lmo_tied(i):
            break
        gpre = column_gap(ex, i)
        if variant == "plain":
            j, gamma = ex.bcfw_step(i, rule)
            v, kind = -1, "fw"
        else:
            j, v, gamma, kind = ex.away_or_pair_step(i, pairwise=(variant == "pair"))
        if inner:
            G[i] = column_gap(ex, i) if post else gpre
        if (k + 1) % (M * n) == 0:
            G = [column_gap(ex, q) for q in range(n)]
        out.append(dict(k=k, i=i, j=j, v=v, gamma=gamma, kind=kind, G=list(G)))
    return out
