"""Encrypted layer workloads on the CKKS core (BASELINE.json configs 4 and 5).

Both are compositions of the reference's operators (rotations, plaintext and ciphertext
products, rescales, additions) written against the same backend interface as the bootstrap
(bootstrap.CkksCircuit), so the product runs on the B200 kernels (GpuBackend: fused hoisted
BSGS `k_bsgs_ext`, fused relinearisation + double rescale) and the CPU oracle backend
reproduces every output residue for the parity tests.

* C4 — ResNet-20 basic block (`ResNetBlock`): conv3x3 -> polynomial ReLU -> conv3x3 ->
  + shortcut -> polynomial ReLU on a C x H x W activation packed channel-major in the slots
  (slot c*H*W + y*W + x, replicated).  A 3x3 convolution is the rotate-and-sum of the
  reference's BSGS mat-vec emitter (bsgs.py:45-123) over the C*9 diagonals
  d = r*H*W + dy*W + dx (output channel c reads input channel (c + r) mod C; out-of-image taps
  are zero in the diagonal), evaluated with hoisted baby rotations and giant steps.
* C5 — transformer block (`TransformerBlock`): T tokens x d features packed row-major; Q, K, V
  and output projections and the two FFN matrices as BSGS mat-vecs of I_T (x) W; attention
  scores as ciphertext-ciphertext products with rotate-and-sum over the features; softmax as
  a Chebyshev exp approximation normalised by a Chebyshev 1/x approximation of the row sum;
  GELU as the reference's least-squares polynomial fit (bench.py:216-220).

Scale discipline (as in the bootstrap): activations live at one working scale S, linear maps
use diagonals encoded at q_l q_(l-1) and two rescales (scale-preserving), ciphertext products
use the fused relinearisation + double rescale, and polynomial outputs are brought back to S
exactly (`_match`).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from .bootstrap import BootConfig, CkksCircuit, CtBatch, ListBatch, bsgs_apply_plain, bsgs_plan, cheb_interp

# ---------------------------------------------------------------------------------------
# slot-domain models (host, float64)
# ---------------------------------------------------------------------------------------


def conv3x3_diagonals(w: np.ndarray, C: int, H: int, W: int, n: int) -> dict:
    """Diagonal form {offset: vector} of a padded 3x3 convolution with weights w[c_out, c_in,
    ky, kx] on the packing slot = c*H*W + y*W + x (replicated n / (C*H*W) times)."""
    HW, CHW = H * W, C * H * W
    assert n % CHW == 0, "the activation must tile the slots"
    s = np.arange(n)
    p = s % CHW
    co, y, x = p // HW, (p % HW) // W, p % W
    M = {}
    for r in range(C):
        ci = (co + r) % C
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = (y + dy >= 0) & (y + dy < H) & (x + dx >= 0) & (x + dx < W)
                v = np.where(ok, w[co, ci, dy + 1, dx + 1], 0.0)
                d = (r * HW + dy * W + dx) % n
                M[d] = M.get(d, 0.0) + v
    return M


def conv3x3_plain(act: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Reference model: act (C, H, W), zero padding 1, stride 1."""
    C, H, W = act.shape
    a = np.pad(act, ((0, 0), (1, 1), (1, 1)))
    out = np.zeros_like(act)
    for co in range(C):
        for ci in range(C):
            for ky in range(3):
                for kx in range(3):
                    out[co] += w[co, ci, ky, kx] * a[ci, ky: ky + H, kx: kx + W]
    return out


def blockdiag_diagonals(Wm: np.ndarray, T: int, n: int) -> dict:
    """Diagonal form of I_T (x) Wm^T acting on a row-major (T x d) packing (slot t*d + j,
    replicated): out[t, i] = sum_j Wm[i, j] x[t, j]."""
    d = Wm.shape[0]
    TD = T * d
    assert n % TD == 0
    s = np.arange(n)
    i = s % d
    M = {}
    for delta in range(-(d - 1), d):
        j = i + delta
        ok = (j >= 0) & (j < d)
        v = np.where(ok, Wm[i, np.clip(j, 0, d - 1)], 0.0)
        if np.any(v):
            M[delta % n] = v
    return M


def gelu_lsq(degree: int = 7, lo: float = -4.0, hi: float = 4.0) -> np.ndarray:
    """Least-squares power-basis fit of GELU on [lo, hi] — the reference's
    gelu_coefficients (bench.py:216-220) restated."""
    from math import erf, sqrt
    x = np.linspace(lo, hi, 512)
    y = np.array([0.5 * v * (1 + erf(v / sqrt(2))) for v in x])
    return np.polynomial.polynomial.polyfit(x, y, degree)


# ---------------------------------------------------------------------------------------
# the layers
# ---------------------------------------------------------------------------------------

class _Layers(CkksCircuit):
    """Shared helpers: BSGS linear maps and Chebyshev activations at the working scale."""

    def __init__(self, backend, cfg: BootConfig):
        super().__init__(backend, cfg)

    def linear(self, x, plan, tag, const: float = 1.0):
        """sum_d diag_d * rot(x, d) (bsgs_plan of a DiagMat): scale preserved, 2 primes."""
        l = x.level
        return self._linear(x, plan, tag, const, Fraction(self.q[l]) * self.q[l - 1], 2)

    def activation(self, x, coeffs: np.ndarray, scale):
        """sum_k c_k T_k(x) (x already in [-1, 1]) brought back exactly to `scale`."""
        deg = len(coeffs) - 1
        T = self._cheb_powers(x, deg)
        t = T[1].level - 2
        while t >= 0 and not self._feasible(coeffs, T, t):
            t -= 1
        if t < 2:
            raise ValueError("not enough levels for the activation")
        y = self._cheb_eval(coeffs, T, t, Fraction(self.q[t + 1]) * self.q[t + 2])
        return self._match(y, t - 2, scale)


class ResNetBlock(_Layers):
    """One ResNet-20 basic block on a C x H x W activation (C4): relu(conv2(relu(conv1(x))) + x)
    with a Chebyshev ReLU of degree `relu_degree` on [-1, 1]."""

    def __init__(self, backend, w1, w2, shape, relu_degree: int = 15, cfg: BootConfig = BootConfig(),
                 plan_ratio: int = 64):
        super().__init__(backend, cfg)
        self.C, self.H, self.W = shape
        self.w1, self.w2 = np.asarray(w1, float), np.asarray(w2, float)
        self.M1 = conv3x3_diagonals(self.w1, *shape, self.n)
        self.M2 = conv3x3_diagonals(self.w2, *shape, self.n)
        self.p1 = bsgs_plan(self.M1, self.n, plan_ratio)
        self.p2 = bsgs_plan(self.M2, self.n, plan_ratio)
        self.relu_c = cheb_interp(lambda u: np.maximum(u, 0.0), relu_degree)

    def required_rotations(self) -> list:
        return sorted(self.p1.rotations() | self.p2.rotations())

    def forward(self, x):
        be, S = self.be, Fraction(x.scale)
        y = self.linear(x, self.p1, "conv1")
        y = self.activation(y, self.relu_c, S)
        y = self.linear(y, self.p2, "conv2")
        z = be.add(y, be.drop_to_level(x, y.level))
        return self.activation(z, self.relu_c, S)

    # models ----------------------------------------------------------------------------
    def relu_model(self, v):
        from numpy.polynomial import chebyshev as Ch
        return Ch.chebval(v, self.relu_c)

    def plain(self, slots: np.ndarray) -> np.ndarray:
        """Exact slot model of forward() (the same diagonals, the same polynomial)."""
        y = self.relu_model(bsgs_apply_plain(self.p1, slots).real)
        y = bsgs_apply_plain(self.p2, y).real + slots
        return self.relu_model(y)

    def reference(self, act: np.ndarray) -> np.ndarray:
        """The network itself (true ReLU, direct convolution) on a (C, H, W) activation."""
        y = np.maximum(conv3x3_plain(act, self.w1), 0)
        return np.maximum(conv3x3_plain(y, self.w2) + act, 0)

    def pack(self, act: np.ndarray) -> np.ndarray:
        return np.tile(act.reshape(-1), self.n // act.size)


class TransformerBlock(_Layers):
    """One single-head transformer block (C5) on T tokens x d features, packed row-major:
        q, k, v = X Wq^T, X Wk^T, X Wv^T
        a[t, u] = softmax_u(<q_t, k_u> / sqrt(d))      (exp and 1/sum as Chebyshev polynomials)
        h = X + (a v) Wo^T
        out = h + W2 gelu(W1 h)                         (GELU: reference least-squares fit)
    Scores <q_t, k_u> for a fixed offset delta = u - t come from ONE ciphertext product
    q * rot(k, delta d) and a rotate-and-sum over the d features; a v accumulates
    a_delta * rot(v, delta d) over the T offsets."""

    def __init__(self, backend, Wq, Wk, Wv, Wo, W1, W2, T: int, d: int, exp_degree: int = 7,
                 inv_degree: int = 7, gelu_degree: int = 7, cfg: BootConfig = BootConfig(),
                 score_bound: float = 1.0, gelu_bound: float = 1.0):
        super().__init__(backend, cfg)
        self.T, self.d = T, d
        assert self.n % (T * d) == 0
        self.mats = {k: np.asarray(v, float) for k, v in
                     dict(q=Wq, k=Wk, v=Wv, o=Wo, f1=W1, f2=W2).items()}
        self.plans = {k: bsgs_plan(blockdiag_diagonals(m, T, self.n), self.n, 4) for k, m in self.mats.items()}
        self.sb = score_bound                 # |<q_t, k_u>| / sqrt(d) <= sb on the inputs used
        self.gb = gelu_bound                  # |W1 h| <= gb
        # exp(sb * x) on [-1, 1]; 1/y for the row sum y in [T e^-sb, T e^sb] mapped to [-1, 1]
        self.exp_c = cheb_interp(lambda x: np.exp(self.sb * x), exp_degree)
        self.lo, self.hi = T * np.exp(-self.sb), T * np.exp(self.sb)
        mid, half = (self.hi + self.lo) / 2, (self.hi - self.lo) / 2
        self.inv_c = cheb_interp(lambda x: 1.0 / (mid + half * x), inv_degree)
        self.inv_map = (1.0 / half, -mid / half)
        g = gelu_lsq(gelu_degree, -gelu_bound, gelu_bound)
        self.gelu_c = np.polynomial.chebyshev.poly2cheb(
            [c * gelu_bound ** i for i, c in enumerate(g)])   # gelu(gb x), x in [-1, 1]

    def required_rotations(self) -> list:
        r = set()
        for p in self.plans.values():
            r |= p.rotations()
        n, d, T = self.n, self.d, self.T
        for delta in range(T):
            if (delta * d) % n:
                r.add((delta * d) % n)
        s = 1
        while s < d:
            r.add(s % n)                   # rotate-and-sum over the features
            r.add((-s) % n)                # broadcast of each row's sum
            s *= 2
        return sorted(r)

    def _rot(self, x, s):
        if s % self.n == 0:
            return x
        if isinstance(x, (CtBatch, ListBatch)):
            return self.be.rotate_same(x, s % self.n)
        return self.be.rotate_hoisted(x, [s % self.n])[0]

    def _rot_sum(self, x, width):
        """sum over the `width` slots starting at each slot's row (rotate-and-sum, log2 width)."""
        s = 1
        while s < width:
            x = self.be.add(x, self._rot(x, s))
            s *= 2
        return x

    def _mask(self, x, vec, tag):
        """x * plaintext(vec) at the working scale (two primes)."""
        l = x.level
        pt = self._pt(tag, vec, l, Fraction(self.q[l]) * self.q[l - 1])
        if isinstance(x, (CtBatch, ListBatch)):
            return self.be.rescale2(self.be.mul_plain_batch(x, pt))
        return self.be.rescale2(self.be.mul_plain_sum([(x, pt)]))

    def _row_sum_broadcast(self, x):
        """Each token's value at feature 0 broadcast over its d features."""
        m = np.zeros(self.n)
        m[:: self.d] = 1.0
        y = self._mask(x, m, "m0")
        s = 1
        while s < self.d:
            y = self.be.add(y, self._rot(y, -s))
            s *= 2
        return y

    def forward(self, X):
        """The T score offsets run as ONE batch of T ciphertexts through every kernel: the T
        rotations of k (and of v) are one hoisted batch, q is broadcast over the batch (an
        instance stride of 0), the rotate-and-sums, the mask, the exp polynomial and the
        products are batched launches, and the softmax denominator and the attention output
        are batch sums.  Residue for residue the same circuit as one offset at a time."""
        be, T, d = self.be, self.T, self.d
        S = Fraction(X.scale)
        q = self.linear(X, self.plans["q"], "wq", 1.0 / (np.sqrt(d) * self.sb))
        k = self.linear(X, self.plans["k"], "wk")
        v = self.linear(X, self.plans["v"], "wv")
        steps = [(delta * d) % self.n for delta in range(T)]
        # scores for every offset delta: s_delta[t] = <q_t, k_(t+delta)>/(sqrt(d) sb), in [-1, 1]
        prod = self._mulr2(be.broadcast(q, T), be.rot_batch(k, steps))
        prod = self._match(prod, prod.level - 2, S)
        sdl = self._row_sum_broadcast(self._rot_sum(prod, d))
        E = self.activation(sdl, self.exp_c, S)            # exp(sb * s), batch of T
        sc = be.batch_sum(E)
        # 1/sum through the affine map onto [-1, 1]
        a_, b_ = self.inv_map
        lv = E.level
        u = be.add_const(self._scale_const(sc, a_), b_)
        inv = self.activation(u, self.inv_c, S)
        # attention output: (sum_delta e_delta * rot(v, delta d)) / sum — the T products run at
        # the exp level, one product by 1/sum at the end
        acc = be.batch_sum(self._mulr2(E, be.rot_batch(be.drop_to_level(v, lv), steps)))
        acc = self._match(acc, acc.level - 2, S)
        lo = min(acc.level, inv.level)
        acc = self._mulr2(be.drop_to_level(acc, lo), be.drop_to_level(inv, lo))
        acc = self._match(acc, acc.level - 2, S)
        h = self.linear(acc, self.plans["o"], "wo")
        h = be.add(h, be.drop_to_level(X, h.level))
        f = self.linear(h, self.plans["f1"], "w1", 1.0 / self.gb)
        f = self.activation(f, self.gelu_c, S)
        f = self.linear(f, self.plans["f2"], "w2")
        return be.add(f, be.drop_to_level(h, f.level))

    def _scale_const(self, x, c):
        """x * c with c encoded at q_l q_(l-1) and two rescales (scale preserved)."""
        l = x.level
        return self.be.rescale2(self.be.mul_const(x, c, Fraction(self.q[l]) * self.q[l - 1]))

    # models ----------------------------------------------------------------------------
    def reference(self, Xm: np.ndarray) -> np.ndarray:
        """The block in float64 (true softmax and GELU)."""
        from math import erf, sqrt
        M = self.mats
        Q, K, V = Xm @ M["q"].T, Xm @ M["k"].T, Xm @ M["v"].T
        A = Q @ K.T / np.sqrt(self.d)
        A = np.exp(A - 0)
        A /= A.sum(axis=1, keepdims=True)
        H = Xm + (A @ V) @ M["o"].T
        F = H @ M["f1"].T
        G = np.vectorize(lambda z: 0.5 * z * (1 + erf(z / sqrt(2))))(F)
        return H + G @ M["f2"].T

    def pack(self, Xm: np.ndarray) -> np.ndarray:
        return np.tile(Xm.reshape(-1), self.n // Xm.size)
