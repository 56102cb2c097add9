"""CKKS bootstrapping built from the fused operator API.

The reference has no bootstrap.  This module composes the
reference's own primitives — hom_rotate (hoisted), mul_plain, hom_add/sub, hom_mul, rescale,
plus conjugation (a Galois key with g = 2N-1 through keys.py:129-136) — into the standard
pipeline, so that every primitive call is bit-exact against the reference primitive on the
same inputs and the whole composition is bit-exact against the CPU oracle composing the
same calls (tests/test_bootstrap.py).  The algorithm is written once, against a small backend
interface; `GpuBackend` below is the product (sm_100a kernels through the C ABI), the oracle
backend lives in oracle/boot_backend.py and is test infrastructure.

Pipeline (input: ciphertext at level 0, modulus q0, any scale Delta_in):

1. ModRaise.  INTT the q0 rows, lift each coefficient centred to (-q0/2, q0/2], reduce into
   every main prime, NTT (kernel `lf_modraise`).  Decrypts to t = m + e + q0*I with small I
   (sparse ternary secret, h = 64).
2. CoeffToSlot.  z = Embed(t)/Delta_in; w = U^-1 z with U_jk = zeta^(5^j k) (the canonical
   embedding of encoding.py:23-61).  U = F_n ... F_2 BR (radix-2 "special FFT"), so
   BR U^-1 = F_2^-1 ... F_n^-1: `cts_levels` groups the inverse butterfly stages into
   `cfg.cts_levels` sparse matrices (<= 2^(r+1)-1 diagonals each) applied with baby-step /
   giant-step rotations.  Output (bit-reversed order): y_k = c (t_k + i t_{k+n}) / q0.
   Plaintext diagonals are encoded at the product of the next two primes (q_l q_{l-1}) and
   the level rescales twice: the input slots are dominated by q0*I, so the diagonals need
   ~2^-40 relative precision, which a single 26-bit prime cannot give.
3. Real / imaginary split with one conjugation: re = y + conj(y), im = (y - conj(y)) * (-i)
   (multiplication by -i is the monomial -X^(N/2), exact).
4. EvalMod on both parts: u = alpha x + beta maps x = t/q0 in [-K, K] to [-1, 1]; a
   Chebyshev interpolant of cos(2 pi (x - 1/4) / 2^r) (degree `cheb_degree`, evaluated by
   recursive Chebyshev division over the powers T_1..T_7, T_8, T_16) followed by r double
   angles c <- c^2 - s gives sin(2 pi x) / (2 pi) ~= m/q0.  EvalMod runs at scale ~2^52 (two
   primes per multiplicative level): its absolute noise must stay far below m/q0 ~ 2^-11.
   Scales are tracked exactly (Fraction) as in the reference; additions of terms that reach
   a level by different paths are aligned by a multiplication with the constant 1 encoded at
   the exact compensating scale.
5. Recombine re + i*im, SlotToCoeff: v = U (bit-reversed input), `cfg.stc_levels` levels,
   single-prime diagonals, then one final rescale back to a ~2^26 scale.

Precision: see `DESIGN.md` §6 and `bench.py --workload bootstrap` (reported in bits).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from math import pi

import numpy as np

from .encoding import embed_inverse

# ---------------------------------------------------------------------------------------
# slot-domain linear algebra (host, complex128)
#
# A slot-linear map is stored in diagonal form {offset: vec}: (M z)[p] = sum_d vec_d[p] *
# z[(p + d) mod n]; rotating a ciphertext by d slots (hom_rotate, "left rotation",
# ckks.py:197-217) realises z -> z[(p + d) mod n].
# ---------------------------------------------------------------------------------------

DiagMat = dict


def dm_apply(M: DiagMat, z: np.ndarray) -> np.ndarray:
    out = np.zeros_like(z, dtype=np.complex128)
    for d, v in M.items():
        out += v * np.roll(z, -d)
    return out


def dm_compose(A: DiagMat, B: DiagMat, n: int, tol: float = 0.0) -> DiagMat:
    """A after B: sum_{a,b} diag(alpha_a * rot(beta_b, a)) R^(a+b)."""
    out = {}
    for a, va in A.items():
        for b, vb in B.items():
            d = (a + b) % n
            t = va * np.roll(vb, -a)
            out[d] = out[d] + t if d in out else t
    return {d: v for d, v in out.items() if np.abs(v).max() > tol}


def dm_scale(A: DiagMat, c) -> DiagMat:
    return {d: v * c for d, v in A.items()}


@lru_cache(maxsize=None)
def _rot_group(N: int):
    return tuple(pow(5, j, 2 * N) for j in range(N // 2))


def _stage(N: int, L: int, inverse: bool) -> DiagMat:
    """Butterfly stage of block length L of the special FFT (U = F_n ... F_2 BR):
    (u, v) -> (u + xi v, u - xi v), xi = exp(2 pi i (5^j mod 4L) / 4L) for position j of the
    half block.  The inverse maps (a, b) -> ((a + b)/2, (a - b)/(2 xi))."""
    n = N // 2
    h = L // 2
    rg = _rot_group(N)
    p = np.arange(n)
    j = p % L
    first = j < h
    jj = np.where(first, j, j - h)
    xi = np.exp(2j * np.pi * (np.array(rg, dtype=np.int64)[jj] % (4 * L)) / (4 * L))
    d0 = np.zeros(n, np.complex128)
    dp = np.zeros(n, np.complex128)      # offset +h (first half reads p + h)
    dm = np.zeros(n, np.complex128)      # offset -h (second half reads p - h)
    if not inverse:
        d0[first] = 1.0
        dp[first] = xi[first]
        dm[~first] = 1.0
        d0[~first] = -xi[~first]
    else:
        # a = out[i+j] (first half), b = out[i+j+h]: u = (a + b)/2 at first, v = (a - b)/(2 xi)
        d0[first] = 0.5
        dp[first] = 0.5
        dm[~first] = 0.5 / xi[~first]
        d0[~first] = -0.5 / xi[~first]
    M = {}

    def put(d, v):
        d %= n
        M[d] = M[d] + v if d in M else v

    put(0, d0)
    put(h, dp)
    put(-h, dm)
    return M


def _groups(nstages: int, nlev: int):
    """Split nstages consecutive stages into nlev groups, larger groups first."""
    base, extra = divmod(nstages, nlev)
    sizes = [base + (1 if i < extra else 0) for i in range(nlev)]
    return sizes


def stc_matrices(N: int, nlev: int) -> list:
    """SlotToCoeff factors in application order: F_2..F_n grouped into nlev matrices."""
    n = N // 2
    logn = n.bit_length() - 1
    sizes = _groups(logn, nlev)
    mats, s = [], 1
    for sz in sizes:
        M = None
        for k in range(s, s + sz):
            F = _stage(N, 1 << k, inverse=False)
            M = F if M is None else dm_compose(F, M, n)
        mats.append(M)
        s += sz
    return mats


def cts_matrices(N: int, nlev: int) -> list:
    """CoeffToSlot factors in application order: F_n^-1 .. F_2^-1 grouped into nlev
    matrices (the product equals BR U^-1)."""
    n = N // 2
    logn = n.bit_length() - 1
    sizes = _groups(logn, nlev)
    mats, s = [], logn
    for sz in sizes:
        M = None
        for k in range(s, s - sz, -1):
            F = _stage(N, 1 << k, inverse=True)
            M = F if M is None else dm_compose(F, M, n)
        mats.append(M)
        s -= sz
    return mats


def bit_reverse_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    r = np.zeros(n, dtype=np.int64)
    for i in range(n):
        r[i] = int(format(i, f"0{bits}b")[::-1], 2) if bits else 0
    return r


# ---------------------------------------------------------------------------------------
# baby-step / giant-step plan of one diagonal matrix
# ---------------------------------------------------------------------------------------

@dataclass
class BsgsPlan:
    unit: int                    # all offsets are multiples of `unit`
    g: int                       # baby-step span
    baby: list                   # baby rotation amounts (slots), 0 first
    giants: dict                 # k -> {b: diag pre-rotated by -k*g*unit}
    n: int

    def rotations(self) -> set:
        r = {b % self.n for b in self.baby if b % self.n}
        r |= {(k * self.g * self.unit) % self.n for k in self.giants if (k * self.g * self.unit) % self.n}
        return r


def bsgs_plan(M: DiagMat, n: int, ratio: int = 1) -> BsgsPlan:
    """Baby-step span g: the smallest power of two with g^2 >= span * ratio.  ratio > 1 favours
    baby steps, right when a giant step costs `ratio` baby steps (hoisted ModDown: baby steps
    skip ModDown, giant steps pay a ModDown plus a full rotation)."""
    offs = sorted(M)
    signed = [d if d <= n // 2 else d - n for d in offs]
    nz = [abs(s) for s in signed if s]
    unit = 1
    if nz:
        from math import gcd
        unit = 0
        for s in nz:
            unit = gcd(unit, s)
    ms = [s // unit for s in signed]
    span = max(ms) - min(ms) + 1
    g = 1
    while g * g < span * ratio:
        g *= 2
    giants = {}
    babies = set()
    for d, m in zip(offs, ms):
        b = m % g
        k = (m - b) // g
        babies.add(b)
        shift = k * g * unit
        giants.setdefault(k, {})[b] = np.roll(M[d], shift)
    baby = sorted(babies)
    return BsgsPlan(unit=unit, g=g, baby=[b * unit for b in baby], giants=giants, n=n)


def bsgs_apply_plain(plan: BsgsPlan, z: np.ndarray) -> np.ndarray:
    """Plaintext model of the homomorphic BSGS evaluation (for tests)."""
    out = np.zeros_like(z, dtype=np.complex128)
    for k, terms in plan.giants.items():
        inner = np.zeros_like(z, dtype=np.complex128)
        for b in plan.baby:
            if b // plan.unit in terms:
                inner += terms[b // plan.unit] * np.roll(z, -b)
        out += np.roll(inner, -k * plan.g * plan.unit)
    return out


# ---------------------------------------------------------------------------------------
# EvalMod polynomial (Chebyshev basis)
# ---------------------------------------------------------------------------------------

def cheb_interp(f, deg: int) -> np.ndarray:
    """Chebyshev coefficients of the degree-`deg` interpolant of f on [-1, 1]."""
    from numpy.polynomial import chebyshev as C
    k = np.arange(deg + 1)
    x = np.cos(np.pi * (k + 0.5) / (deg + 1))
    return C.chebfit(x, f(x), deg)


def cheb_divmod(c: np.ndarray, G: int):
    """p = q T_G + r in the Chebyshev basis (T_{G+j} = 2 T_G T_j - T_{G-j}); deg p < 2G."""
    c = np.array(c, dtype=np.float64)
    deg = len(c) - 1
    q = np.zeros(max(deg - G + 1, 1))
    r = np.array(c[:G], dtype=np.float64) if deg >= G else c.copy()
    if deg < G:
        return np.zeros(1), r
    for j in range(deg - G, -1, -1):
        a = c[G + j]
        if j == 0:
            q[0] += a
        else:
            q[j] += 2 * a
            r[G - j] -= a
    return q, r


EARLY_RESCALE_MIN_SCALE = 2 ** 40   # BSGS giants rescaled before their rotations only above this scale
TWICE_MIN_SCALE = 2 ** 20      # lowest declared scale the free Chebyshev doubling may leave (default
                               # degree 31: T_16 at ~2^37, untouched)


@dataclass(frozen=True)
class BootConfig:
    cts_levels: int = 4
    stc_levels: int = 3
    K: int = 16                  # |t/q0| <= K (I bound + margin for h = 64)
    r: int = 3                   # double angles
    cheb_degree: int = 31
    baby: int = 8                # Chebyshev baby steps T_0..T_7
    lazy_moddown: bool = True    # BSGS: one ModDown per giant step instead of per rotation
    bsgs_ratio: int = 8          # giant/baby cost ratio used to size the baby steps (swept: DESIGN §6)


def evalmod_constants(cfg: BootConfig):
    """alpha, beta (u = alpha x + beta), Chebyshev coefficients of s0 cos(2 pi Y u), and the
    double-angle offsets s_1..s_r with c_{k+1} = c_k^2 - s_{k+1} giving sin(2 pi x)/(2 pi)."""
    Y = (cfg.K + 0.25) / 2 ** cfg.r
    alpha = 1.0 / (cfg.K + 0.25)
    beta = -0.25 / (cfg.K + 0.25)
    s = [1.0 / (2 * pi)]
    for _ in range(cfg.r):
        s.append(float(np.sqrt(2 * s[-1])))
    s = s[::-1]                  # s[0] = s0, s[r] = 1/(2 pi)
    coeffs = cheb_interp(lambda u: s[0] * np.cos(2 * pi * Y * u), cfg.cheb_degree)
    return alpha, beta, coeffs, s[1:]


def evalmod_plain(x: np.ndarray, cfg: BootConfig) -> np.ndarray:
    from numpy.polynomial import chebyshev as C
    alpha, beta, coeffs, s = evalmod_constants(cfg)
    c = C.chebval(alpha * x + beta, coeffs)
    for sk in s:
        c = c * c - sk
    return c


# ---------------------------------------------------------------------------------------
# the algorithm over a backend
# ---------------------------------------------------------------------------------------

class _ChebPowers(dict):
    """T_k by k, plus the odd powers stored as T_k + T_1 (`folded`)."""

    def __init__(self, *a):
        super().__init__(*a)
        self.folded = set()


class CkksCircuit:
    """Scale / level bookkeeping and the homomorphic building blocks shared by the bootstrap
    and the encrypted layer workloads (workloads.py): BSGS linear maps with hoisted rotations
    (`_linear`), exact scale matching (`_match`), relinearised products with the double-prime
    rescale (`_mul2`), and Chebyshev-basis polynomial evaluation (`_cheb_powers`,
    `_cheb_eval`).  Everything is written against a backend (GpuBackend for the product, the
    oracle backend in tests), so each composition is checked residue for residue."""

    def __init__(self, backend, cfg):
        self.be = backend
        self.cfg = cfg
        self.N = backend.N
        self.n = self.N // 2
        self.q = list(backend.main_primes)
        self.L = len(self.q) - 1
        self.q0 = self.q[0]
        self.out_scale = Fraction(getattr(backend, "default_scale", 1 << 26))
        self._pt_cache = {}

    # -- helpers ---------------------------------------------------------------------
    def _pt(self, key, vec, level, scale, ext=False):
        k = (key, level, scale, ext)
        pt = self._pt_cache.get(k)
        if pt is None:
            pt = self.be.encode_slots(vec, level, scale, ext=ext)
            self._pt_cache[k] = pt
        return pt

    def _linear(self, ct, plan: BsgsPlan, tag, const, S_p, nres: int):
        """sum_d diag_d * rot(ct, d) with BSGS: diagonals (times `const`) encoded at the
        plaintext scale S_p, then `nres` rescales.

        Hoisted ModDown (cfg.lazy_moddown): the baby-step rotations share one ModUp and stop
        before ModDown, (P sigma_b(b) + acc_b, acc_a) over the extended basis Q_l P
        (keyswitch_inner_product, ckks.py:120-131); the identity step is P*ct.  Each giant
        step multiplies them by its extended-basis diagonals, sums, and runs ONE mod_down
        (poly.py:251-281) — instead of one per baby rotation.  The composition only uses
        reference primitives, so the oracle backend reproduces it residue for residue."""
        be = self.be
        l = ct.level
        S_p = Fraction(S_p)
        lazy = self.cfg.lazy_moddown and hasattr(be, "rotate_hoisted_ext")
        # The giants' rescale can run before their rotations (fused into the giants' ModDown)
        # only while the rescaled scale stays large: a rotation's keyswitch noise is absolute,
        # so rotating at a ~2^26 scale would cost precision (SlotToCoeff keeps the old order).
        s_out = Fraction(ct.scale) * S_p
        for i in range(nres):
            s_out /= self.q[l - i]
        early = nres if s_out >= EARLY_RESCALE_MIN_SCALE else 0

        def finish(acc):
            if early:
                return acc
            return be.rescale2(acc) if nres == 2 else be.rescale(acc)
        if lazy and hasattr(be, "bsgs_fused_ext"):
            # the backend fuses the baby rotations with the giant-step plaintext sums
            groups = []
            for k in sorted(plan.giants, key=lambda k: (k != 0, k)):
                terms = plan.giants[k]
                pairs = [(b, self._pt((tag, k, b // plan.unit, True), terms[b // plan.unit] * const, l,
                                      S_p, ext=True))
                         for b in plan.baby if b // plan.unit in terms]
                groups.append(((k * plan.g * plan.unit) % self.n, pairs))
            acc = be.bsgs_fused_ext(ct, groups, early)
            if acc is not None:
                return finish(acc)
        if lazy:
            nz = [b for b in plan.baby if b % self.n]
            ext = dict(zip(nz, be.rotate_hoisted_ext(ct, nz))) if nz else {}
            if any(b % self.n == 0 for b in plan.baby):
                ext.update({b: be.extend(ct) for b in plan.baby if b % self.n == 0})
        else:
            rmap = dict(zip(plan.baby, be.rotate_hoisted(ct, plan.baby)))
        groups = []
        for k in sorted(plan.giants, key=lambda k: (k != 0, k)):   # the unrotated giant first
            terms = plan.giants[k]
            pairs = []
            for b in plan.baby:
                bu = b // plan.unit
                if bu in terms:
                    pt = self._pt((tag, k, bu, lazy), terms[bu] * const, l, S_p, ext=lazy)
                    pairs.append(((ext if lazy else rmap)[b], pt))
            groups.append(((k * plan.g * plan.unit) % self.n, pairs))
        if lazy:
            return finish(be.bsgs_combine_ext(groups, early))
        acc = be.bsgs_combine(groups)
        return be.rescale2(acc) if nres == 2 else be.rescale(acc)

    def _match(self, ct, level, scale):
        """ct (level >= level+1) -> (level, scale) via multiplication by the constant 1
        encoded at the exact compensating scale (two primes: precision ~2^-52)."""
        be = self.be
        assert ct.level >= level + 2, (ct.level, level)
        ct = be.drop_to_level(ct, level + 2)
        S_p = Fraction(scale) * self.q[level + 2] * self.q[level + 1] / Fraction(ct.scale)
        out = be.rescale2(be.mul_const(ct, 1.0, S_p))
        assert out.level == level and out.scale == scale
        return out

    def _mul2(self, a, b):
        """a * b, relinearised, then two rescales (double-prime level)."""
        be = self.be
        lv = min(a.level, b.level)
        a, b = be.drop_to_level(a, lv), be.drop_to_level(b, lv)
        return self._mulr2(a, b)

    def _mulr2(self, a, b):
        be = self.be
        if hasattr(be, "mul_rescale2"):
            return be.mul_rescale2(a, b)
        return be.rescale2(be.hom_mul(a, b))

    def _fused_consts(self):
        return hasattr(self.be, "mul_rescale2_many")

    def _mulr2_many(self, ops, addk=None):
        """[_mulr2(a, b) (+ addk[i] on b) for a, b in ops]; one batched pipeline per level when
        the backend has one (operand lists, no gathering copies, the integer addk[i] added in
        the product's epilogue).  addk is only given when _fused_consts()."""
        be = self.be
        addk = addk or [None] * len(ops)
        if hasattr(be, "mul_rescale2_many"):
            out = [None] * len(ops)
            levels = sorted({a.level for a, _ in ops})
            for lv in levels:
                idx = [i for i, (a, _) in enumerate(ops) if a.level == lv]
                for i, r in zip(idx, be.mul_rescale2_many([ops[i] for i in idx], [addk[i] for i in idx])):
                    out[i] = r
            return out
        assert not any(k is not None for k in addk)
        return [self._mulr2(a, b) for a, b in ops]

    def _prod_scale(self, a, b):
        lv = min(a.level, b.level)
        return Fraction(a.scale) * Fraction(b.scale) / self.q[lv] / self.q[lv - 1]

    def _cheb_powers(self, u, degree=None):
        """T_1..T_(baby-1) and the giant powers T_baby, T_2baby, ... up to `degree`.

        T_3 = T_1 (2 T_2 - 1) (one product, no subtraction).  An odd power T_2k+1 (k >= 2)
        that no later product reads is kept as 2 T_k T_k+1 = T_2k+1 + T_1: its -T_1 moves into
        the T_1 coefficient of the leaf combinations (`_leaf`), which saves the exact scale
        match of T_1 (a constant product and a double rescale) per such power."""
        be = self.be
        T = _ChebPowers({1: u})
        g = self.cfg.baby
        degree = self.cfg.cheb_degree if degree is None else degree
        read = {m // 2 for m in range(2, g)} | {m // 2 + 1 for m in range(3, g, 2)}
        G = g
        while G <= degree:
            read.add(G // 2)
            G *= 2

        def twice(x):
            # 2x: the same residues at half the declared scale (free) while the scale stays
            # >= 2^20 (advisor budget: 2^k - 1 < log2 s - 20); past that (high cheb_degree: T_2^k sits at
            # s / 2^(2^k - 1)) an exact addition keeps the scale
            if Fraction(x.scale) / 2 >= TWICE_MIN_SCALE:
                return be.with_scale(x, Fraction(x.scale) / 2)
            return be.add(x, x)

        # every power is one relinearised product: T_2k = 2 T_k^2 - 1, T_2k+1 = 2 T_k T_k+1 - T_1,
        # T_3 = T_1 (2 T_2 - 1).  Products whose operands exist form a dependency wave and run
        # as one batch (mul_rescale2_many); the post-processing is per power.
        plan = {m: m // 2 for m in range(2, g)}
        G = g
        while G <= degree:
            plan[G] = G // 2
            G *= 2

        def deps(m):
            k = plan[m]
            return (k,) if m % 2 == 0 else ((1, 2) if k == 1 else (k, k + 1))

        pending = sorted(plan)
        while pending:
            wave = [m for m in pending if all(dp in T for dp in deps(m))]
            ops, addk = [], []
            for m in wave:
                k = plan[m]
                if m % 2 == 0:
                    a, b = T[k], T[k]
                elif k == 1:
                    a, b = T[1], be.add_const(twice(T[2]), -1.0)
                else:
                    a, b = T[k], T[k + 1]
                lv = min(a.level, b.level)
                ops.append((be.drop_to_level(a, lv), be.drop_to_level(b, lv)))
                # 2 x - 1 of a double: the halved declared scale is free and the -1 (encoded at
                # that scale) is added by the product's epilogue when the backend can
                half = self._prod_scale(a, b) / 2
                addk.append(round(-half) if m % 2 == 0 and self._fused_consts() and half >= TWICE_MIN_SCALE
                            else None)
            for m, x, kk in zip(wave, self._mulr2_many(ops, addk), addk):
                k = plan[m]
                if m % 2 == 0 and kk is not None:
                    T[m] = be.with_scale(x, Fraction(x.scale) / 2)
                elif m % 2 == 0:
                    T[m] = be.add_const(twice(x), -1.0)
                elif k == 1:
                    T[m] = x
                else:
                    x = twice(x)
                    if m not in read:
                        T.folded.add(m)
                        T[m] = x
                    else:
                        T[m] = be.sub(x, self._match(T[1], x.level, x.scale))
            pending = [m for m in pending if m not in wave]
        return T

    def _leaf(self, c, T, level, scale):
        """sum_i c_i T_i (i < baby) at exactly (level, scale): every term is dropped to
        level + 2 and multiplied by c_i encoded at the scale that makes all products share
        scale * q_{level+2} q_{level+1}; one linear combination, one double rescale.  Powers
        stored as T_m + T_1 (`_cheb_powers`) take their -T_1 through the T_1 coefficient."""
        be = self.be
        c = np.array(c, dtype=np.float64)
        for m in getattr(T, "folded", ()):
            if m < len(c) and c[m] != 0.0:
                c[1] -= c[m]
        terms = []
        for i in range(1, len(c)):
            if c[i] == 0.0:
                continue
            t = T[i]
            assert t.level >= level + 2, (i, t.level, level)
            t = be.drop_to_level(t, level + 2)
            S_p = Fraction(scale) * self.q[level + 2] * self.q[level + 1] / Fraction(t.scale)
            terms.append((t, float(c[i]), S_p))
        assert terms
        # the constant term joins the linear combination (before the double rescale)
        acc = be.rescale2(be.lincomb(terms, const=float(c[0])))
        assert acc.level == level and acc.scale == scale
        return acc

    def _feasible(self, c, T, t):
        g = self.cfg.baby
        if len(c) <= g:
            need = min(T[i].level for i in range(1, len(c)) if c[i] != 0.0)
            return t + 2 <= need
        G = self._giant_for(len(c) - 1)
        q, r = cheb_divmod(c, G)
        return (t + 2 <= T[G].level and self._feasible(q, T, t + 2)
                and self._feasible(r, T, t))

    def _giant_for(self, deg):
        G = self.cfg.baby
        while 2 * G <= deg:
            G *= 2
        return G

    def _cheb_eval(self, c, T, level, scale):
        """sum_k c_k T_k at exactly (level, scale) by Chebyshev division: c = q T_G + r with
        the q-part one level-pair higher, multiplied by T_G.  When the remainder r is itself
        split (r = q' T_G' + r'), its product q'·T_G' sits at the same level as q·T_G and both
        run as ONE batched relinearised product (`_mulr2_many`)."""
        be = self.be
        g = self.cfg.baby
        c = np.trim_zeros(np.asarray(c, dtype=np.float64), "b")
        if len(c) <= g:
            return self._leaf(c, T, level, scale)
        m = level + 2

        def split(cc):
            G = self._giant_for(len(cc) - 1)
            q, r = cheb_divmod(cc, G)
            TG = be.drop_to_level(T[G], m)
            q_scale = Fraction(scale) * self.q[m] * self.q[m - 1] / Fraction(TG.scale)
            return self._cheb_eval(q, T, m, q_scale), TG, r

        qc, TG, r = split(c)
        r = np.trim_zeros(np.asarray(r, dtype=np.float64), "b")
        if len(r) > g:
            qc2, TG2, r2 = split(r)
            prod, prod2 = self._mulr2_many([(qc, TG), (qc2, TG2)])
            assert prod.level == prod2.level == level and prod.scale == prod2.scale == scale
            return be.add(prod, be.add(prod2, self._cheb_eval(r2, T, level, scale)))
        prod = self._mulr2(qc, TG)
        assert prod.level == level and prod.scale == scale
        return be.add(prod, self._cheb_eval(r, T, level, scale))


class Bootstrapper(CkksCircuit):
    """Precomputes the plaintext diagonals of CoeffToSlot / SlotToCoeff for `params` and runs
    the pipeline over `backend` (GpuBackend for the product)."""

    def __init__(self, backend, cfg: BootConfig = BootConfig()):
        super().__init__(backend, cfg)
        self.alpha, self.beta, self.cheb, self.dbl = evalmod_constants(cfg)
        self._build_linear()

    # -- planning --------------------------------------------------------------------
    def _build_linear(self):
        cfg, n = self.cfg, self.n
        cts = cts_matrices(self.N, cfg.cts_levels)
        stc = stc_matrices(self.N, cfg.stc_levels)
        # fold alpha * (q-relative) constants: CtS output y = alpha/2 * (t_k + i t_{k+n}) / q0
        # given input slots z = Embed(t)/Delta_in; Delta_in varies, so the factor Delta_in/q0
        # is applied through the declared scale (see bootstrap()).  Balance the magnitude over
        # the levels so every diagonal is O(1) (plaintext precision).
        ratio = cfg.bsgs_ratio if cfg.lazy_moddown else 1
        self.cts_plans = [bsgs_plan(M, n, ratio) for M in cts]
        self.stc_plans = [bsgs_plan(M, n, ratio) for M in stc]
        self.cts_const = self.alpha / 2
        self.rotations = set()
        for pl in self.cts_plans + self.stc_plans:
            self.rotations |= pl.rotations()
        # level schedule
        l = self.L
        self.cts_at = []
        for i in range(cfg.cts_levels):
            self.cts_at.append(l)
            l -= 2
        self.evalmod_in = l
        self._pt_cache = {}

    def required_rotations(self) -> list:
        return sorted(self.rotations)

    def levels_used(self) -> dict:
        return {"cts": self.cts_at, "evalmod_in": self.evalmod_in}

    def _evalmod(self, x):
        """x: slots in [-K, K] (already u = alpha x + beta) -> sin(2 pi x)/(2 pi)."""
        be = self.be
        T = self._cheb_powers(x)
        c = self.cheb
        t = T[1].level - 2
        while t >= 0 and not self._feasible(c, T, t):
            t -= 1
        if t < 0:
            raise ValueError("not enough levels for EvalMod")
        scale = Fraction(self.q[t + 1]) * self.q[t + 2]
        y = self._cheb_eval(c, T, t, scale)
        for sk in self.dbl:                 # c <- c^2 - s_k (the constant in the epilogue when fused)
            if self._fused_consts():
                y = self._mulr2_many([(y, y)], [round(Fraction(-sk) * self._prod_scale(y, y))])[0]
            else:
                y = be.add_const(self._mul2(y, y), -sk)
        return y

    # -- the pipeline ----------------------------------------------------------------
    def _mark(self, name):
        if getattr(self, "marks", None) is not None:
            import torch
            # external events become event-record nodes when the pipeline is being captured
            e = torch.cuda.Event(enable_timing=True,
                                 external=torch.cuda.is_current_stream_capturing())
            e.record()
            self.marks.append((name, e))

    def bootstrap(self, ct, out_scale=None):
        """Refresh a level-0 ciphertext; returns a ciphertext at level
        L - (2 cts_levels - 1) - 2 (EvalMod depth) - (stc_levels + 1) with scale `out_scale`
        (default: the parameter set's scale)."""
        be = self.be
        if ct.level != 0:
            ct = be.drop_to_level(ct, 0)
        delta_in = Fraction(ct.scale)
        q = self.q
        self._mark("start")
        x = be.mod_raise(ct)                                  # level L, scale Delta_in
        self._mark("modraise")
        # Lift the integers to a ~2^52 scale with an exact integer multiplication (no level):
        # the keyswitch and rescale noise of CoeffToSlot is absolute, the slots are dominated
        # by q0*I, and m/q0 must survive at ~2^-40 relative precision.
        lift = 1 << max(0, 52 - int(delta_in).bit_length())
        if lift > 1:
            x = be.mul_const(x, 1.0, lift)
        # CoeffToSlot: plaintext diagonals at q_l q_{l-1} (~2^52) and two rescales per level;
        # the last level folds alpha/2 * Delta_in/q0 and lands exactly on the EvalMod working
        # scale q_l' q_{l'-1} (l' = its output level).
        c0 = self.cts_const * float(delta_in) / self.q0
        nc = len(self.cts_plans)
        for i, plan in enumerate(self.cts_plans):
            l = x.level
            if i < nc - 1:
                x = self._linear(x, plan, ("cts", i), 1.0, Fraction(q[l]) * q[l - 1], 2)
            else:
                lo = l - 2
                S_p = Fraction(q[lo]) * q[lo - 1] * q[l] * q[l - 1] / Fraction(x.scale)
                x = self._linear(x, plan, ("cts", i, float(delta_in)), c0, S_p, 2)
        self._mark("coeff_to_slot")
        # conjugation split (both EvalMod inputs carry the same level and scale)
        xc = be.conjugate(x)
        re = be.add(x, xc)
        im = be.mul_monomial(be.sub(x, xc), 3 * self.N // 2)   # * (-i) = * X^(3N/2)
        if hasattr(be, "batch_buffer"):                       # both parts written into one batch
            buf = be.batch_buffer(2, re.level)
            be.add_const(re, self.beta, out=buf.data[0])
            be.add_const(im, self.beta, out=buf.data[1])
            batch = CtBatch(buf.data, re.scale, re.level)
        else:
            batch = be.stack([be.add_const(re, self.beta), be.add_const(im, self.beta)])
        self._mark("conj_split")
        re, im = be.unstack(self._evalmod(batch))             # both parts in one batch
        self._mark("evalmod")
        y = be.add(re, be.mul_monomial(im, self.N // 2))       # re + i im
        # SlotToCoeff: the first level folds q0/Delta_in, the last lands on out_scale
        out_scale = Fraction(self.out_scale if out_scale is None else out_scale)
        c1 = self.q0 / float(delta_in)
        ns = len(self.stc_plans)
        for i, plan in enumerate(self.stc_plans):
            l = y.level
            const = c1 if i == 0 else 1.0
            tag = ("stc", i, float(delta_in)) if i == 0 else ("stc", i)
            if i < ns - 1:
                y = self._linear(y, plan, tag, const, Fraction(q[l]), 1)
            else:
                S_p = out_scale * q[l] * q[l - 1] / Fraction(y.scale)
                y = self._linear(y, plan, tag, const, S_p, 2)
        self._mark("slot_to_coeff")
        return y


class ListBatch:
    """A batch of ciphertexts with one level and scale, executed one by one (backends without
    batched kernels, e.g. the test oracle)."""

    def __init__(self, cts):
        self.cts = list(cts)
        assert all(c.level == self.cts[0].level and c.scale == self.cts[0].scale for c in self.cts)
        self.level, self.scale = self.cts[0].level, self.cts[0].scale


class ExtCt:
    """A ciphertext over the extended basis Q_l P (eval domain) before mod_down: data (2, ext, N)."""

    def __init__(self, data, scale, level):
        self.data, self.scale, self.level = data, Fraction(scale), level


class CtBatch:
    """B ciphertexts at one level and scale in one (B, 2, level+1, N) device tensor; the GPU
    backend runs every operation on all of them in one batched launch.  `data` may be a
    row-prefix view of a higher-level batch (drop_to_level does not copy); `dense()` gives a
    contiguous batch for the calls whose C-ABI takes one instance stride."""

    def __init__(self, data, scale, level):
        self.data, self.scale, self.level = data, Fraction(scale), level

    def dense(self):
        return self if self.data.is_contiguous() else CtBatch(self.data.contiguous(), self.scale, self.level)

    def pitched(self):
        """(instance stride, rows per polynomial) when `data` is a row-prefix view of a
        contiguous (B, 2, P, N) block (the pitched kernels take it in place), else None."""
        d = self.data
        N = d.shape[-1]
        st = d.stride()
        if st[3] == 1 and st[2] == N and st[1] % N == 0 and (st[0] == 2 * st[1] or st[0] == 0):
            return st[0], st[1] // N           # stride 0: one ciphertext broadcast over the batch
        return None


def map_batch(fn, *args):
    """Apply a single-ciphertext op element-wise when the first argument is a ListBatch."""
    if isinstance(args[0], ListBatch):
        return ListBatch([fn(*[a.cts[i] if isinstance(a, ListBatch) else a for a in args])
                          for i in range(len(args[0].cts))])
    return None


# ---------------------------------------------------------------------------------------
# GPU backend (the product): every operation is a kernel of libcerium_b200.so
# ---------------------------------------------------------------------------------------

def encode_ints(values, N: int, scale) -> np.ndarray:
    """Integer coefficients round(embed_inverse(values) * scale) of a (complex) slot vector,
    the reference's encode arithmetic (encoding.py:82-105) without the range check."""
    r = np.rint(embed_inverse(np.asarray(values, dtype=np.complex128), N) * float(scale))
    if np.abs(r).max(initial=0.0) >= 2.0 ** 62:
        raise OverflowError("plaintext coefficients exceed int64")
    return r.astype(np.int64)


def monomial_ints(N: int, e: int) -> np.ndarray:
    """Coefficients of X^e in Z[X]/(X^N + 1)."""
    c = np.zeros(N, dtype=np.int64)
    e %= 2 * N
    c[e % N] = -1 if e >= N else 1
    return c


class GpuBackend:
    """Bootstrap backend over the B200 operator API (ckks.py / fused.py kernels)."""

    def __init__(self, params, relin_key, conj_key, rot_keys: dict):
        from . import ckks as C
        self.C = C
        self.params = params
        self.N = params.N
        self.main_primes = tuple(params.rns_basis)
        self.default_scale = params.scale
        self.rlk = relin_key
        self.ck = conj_key
        self.rk = rot_keys
        self._mono = {}
        self.permuted_keys = True       # rotations through the *_pk entry points (see _pkey)
        self._pk = {}

    def _pkey(self, steps: int):
        """Rotation key for `steps` in permuted form (fused.permute_rotation_key), made once and
        kept resident next to the reference-form key."""
        from types import SimpleNamespace
        s = steps % self.params.n
        k = self._pk.get(s)
        if k is None:
            from . import fused
            k = SimpleNamespace(data=fused.permute_rotation_key(self.params, self.rk[s],
                                                                galois_element_of(self.N, s)))
            self._pk[s] = k
        return k

    def _rot_keys(self, steps):
        if self.permuted_keys:
            return [self._pkey(s) for s in steps]
        return [self.rk[s % self.params.n] for s in steps]

    # batches (the two EvalMod evaluations run as one batch of 2 in every kernel)
    def stack(self, cts):
        import torch
        return CtBatch(torch.stack([torch.stack([c.b.limbs, c.a.limbs]) for c in cts]),
                       cts[0].scale, cts[0].level)

    # batches built from / reduced to single ciphertexts (the layer workloads, workloads.py)
    def rot_batch(self, x, steps):
        """The rotations of ONE ciphertext by every step (hoisted: one ModUp), as a batch in
        the order of `steps`; identity steps first."""
        import torch
        from . import fused
        from .fused import ct_block
        n = self.params.n
        nid = 0
        while nid < len(steps) and steps[nid] % n == 0:
            nid += 1
        assert all(st % n for st in steps[nid:]), "identity steps must come first"
        out = torch.empty((len(steps), 2, x.level + 1, self.N), dtype=torch.int32, device="cuda")
        blk = ct_block(x)
        for i in range(nid):
            out[i].copy_(blk)
        if nid < len(steps):
            gs = [galois_element_of(self.N, st) for st in steps[nid:]]
            keys = [self.rk[st % n] for st in steps[nid:]]
            fused.rotate_hoisted(self.params, x, gs, keys, out=out[nid:])
        return CtBatch(out, x.scale, x.level)

    def broadcast(self, x, B: int):
        """One ciphertext as a batch of B (an instance stride of 0: no copies)."""
        from .fused import ct_block
        blk = ct_block(x)
        return CtBatch(blk.unsqueeze(0).expand(B, *blk.shape), x.scale, x.level)

    def batch_sum(self, x):
        """The sum of a batch's ciphertexts (pairwise halving adds)."""
        from .poly import LF_OP_ADD
        x = x.dense()
        while x.data.shape[0] > 1:
            B = x.data.shape[0]
            h = B // 2
            s = self._b_ewise(LF_OP_ADD, CtBatch(x.data[:h], x.scale, x.level), CtBatch(x.data[h: 2 * h], x.scale, x.level))
            if B % 2:
                s = CtBatch(__import__("torch").cat([s.data, x.data[2 * h:]]), x.scale, x.level)
            x = s
        return self.unstack(x)[0]

    def rotate_same(self, x, steps: int):
        """Every instance of a batch rotated by the same step (one batched pipeline)."""
        from . import fused
        if steps % self.params.n == 0:
            return x
        x = x.dense()
        B = x.data.shape[0]
        g = galois_element_of(self.N, steps)
        keys = self._rot_keys([steps] * B)
        r = fused.rotate_batch(self.params, x.level, x.data, [g] * B, keys, permuted=self.permuted_keys)
        return CtBatch(r, x.scale, x.level)

    def mul_plain_batch(self, x, pt):
        """Every instance times one plaintext (no rescale)."""
        import torch
        out = torch.empty((x.data.shape[0], 2, x.level + 1, self.N), dtype=torch.int32, device="cuda")
        for i, c in enumerate(self.unstack(x)):
            self.mul_plain_sum([(c, pt)], out=out[i])
        return CtBatch(out, Fraction(x.scale) * Fraction(pt.scale), x.level)

    def batch_buffer(self, B: int, level: int):
        import torch
        return CtBatch(torch.empty((B, 2, level + 1, self.N), dtype=torch.int32, device="cuda"), 1, level)

    def unstack(self, x):
        from .poly import Domain, RnsPolynomial, main_ids
        ids = main_ids(x.level)
        return [self.C.Ciphertext(RnsPolynomial(x.data[i, 0], Domain.EVAL, ids),
                                  RnsPolynomial(x.data[i, 1], Domain.EVAL, ids), x.scale, x.level)
                for i in range(x.data.shape[0])]

    def _rows_pidx(self, x):
        return tuple(range(x.level + 1)) * (2 * x.data.shape[0])

    # ciphertext plumbing
    def drop_to_level(self, ct, level):
        C = self.C
        if ct.level == level:
            return ct
        if isinstance(ct, CtBatch):
            return CtBatch(ct.data[:, :, : level + 1], ct.scale, level)       # a view
        assert level < ct.level
        from .poly import RnsPolynomial, main_ids
        ids = main_ids(level)
        return C.Ciphertext(RnsPolynomial(ct.b.limbs[: level + 1], ct.b.domain, ids),
                            RnsPolynomial(ct.a.limbs[: level + 1], ct.a.domain, ids),
                            ct.scale, level)

    def mod_raise(self, ct):
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .poly import Domain, RnsPolynomial, main_ids, ntt_rows
        p = self.params
        L = p.max_level
        rows = torch.stack([ct.b.limbs[0], ct.a.limbs[0]])
        ntt_rows(p, rows, (0, 0), inverse=True)
        out = torch.empty((2, L + 1, p.N), dtype=torch.int32, device=rows.device)
        ctx = get_context(p)
        _native.check(_native.lib().lf_modraise(ctx.handle, dptr(out), dptr(rows), 2, L + 1,
                                                stream_handle()), "lf_modraise")
        ids = main_ids(L)
        ntt_rows(p, out.view(2 * (L + 1), p.N), ids + ids)
        return self.C.Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids),
                                 RnsPolynomial(out[1], Domain.EVAL, ids), ct.scale, L)

    def encode_slots(self, values, level, scale, ext=False):
        from .encoding import Plaintext, signed_to_eval
        from .poly import extended_ids, main_ids
        ints = encode_ints(values, self.params.N, scale)
        if ext:                      # extended basis (main 0..level + specials): hoisted ModDown
            pt = Plaintext.__new__(Plaintext)
            pt.poly = signed_to_eval(ints, self.params, extended_ids(self.params, level))
            pt.scale, pt.level, pt.compression = Fraction(scale), level, "ext"
            return pt
        return Plaintext(signed_to_eval(ints, self.params, main_ids(level)), Fraction(scale), level)

    # hoisted-ModDown BSGS (extended-basis ciphertexts: ExtCt with data (2, ext, N))
    def extend(self, ct):
        """P * ct over the extended basis (special rows zero): its mod_down is exactly ct."""
        import torch
        from .poly import LF_OP_SCALAR_MUL, ewise, main_ids
        l1 = ct.level + 1
        ext = l1 + self.params.num_special
        data = torch.zeros((2, ext, self.params.N), dtype=torch.int32, device=ct.b.limbs.device)
        P = self.params.special_product()
        sc = [P % q for q in self.params.rns_basis[:l1]]
        ewise(self.params, LF_OP_SCALAR_MUL, data[0, :l1], ct.b.limbs, main_ids(ct.level), scalars=sc)
        ewise(self.params, LF_OP_SCALAR_MUL, data[1, :l1], ct.a.limbs, main_ids(ct.level), scalars=sc)
        return ExtCt(data, ct.scale, ct.level)

    def rotate_hoisted_ext(self, ct, steps):
        import ctypes
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .fused import ct_block
        ctx = get_context(self.params)
        n = len(steps)
        lib = _native.lib()
        level = ct.level
        ext = level + 1 + self.params.num_special
        ws = torch.empty(lib.lf_rotate_hoisted_workspace_bytes(ctx.handle, level, n) // 4,
                         dtype=torch.int32, device="cuda")
        out = torch.empty((n, 2, ext, self.params.N), dtype=torch.int32, device="cuda")
        gs = [galois_element_of(self.params.N, s) for s in steps]
        keys = self._rot_keys(steps)
        karr = (ctypes.c_void_p * n)(*[ctx.check_evk(k).data_ptr() for k in keys])
        c = ct_block(ct)
        fn = lib.lf_rotate_hoisted_ext_pk if self.permuted_keys else lib.lf_rotate_hoisted_ext
        _native.check(fn(ctx.handle, level, dptr(c), n, _native.u32_array(gs), karr,
                         dptr(out), out[0].numel(), dptr(ws), stream_handle()),
                      "lf_rotate_hoisted_ext")
        return [ExtCt(out[i], ct.scale, level) for i in range(n)]

    def bsgs_fused_ext(self, ct, groups, nres=0):
        """groups: [(giant shift, [(baby step, extended plaintext)])].  All baby rotations and
        every giant step's plaintext sum in one lf_bsgs_ext pipeline, then one batched
        mod_down and the giant rotations (rotate_and_sum).  None when the plan exceeds the
        kernel's limits (the caller then composes the unfused primitives)."""
        import torch
        n = self.params.n
        rot = sorted({b for _, pairs in groups for b, _ in pairs if b % n})
        G = len(groups)
        if not rot or len(rot) > 32 or not self.permuted_keys:
            return None
        if G > 4:
            # more giant steps than one k_bsgs_ext holds: chunks of 4 giants (each chunk reruns
            # the hoisted ModUp and its baby rotations), then ONE batched mod_down of all giants
            chunks = [groups[i: i + 4] for i in range(0, G, 4)]
            if any(not any(b % n for _, prs in c for b, _ in prs) for c in chunks):
                return None
            inner = [self._bsgs_inner(ct, c) for c in chunks]
            pt0 = groups[0][1][0][1]
            return self._moddown_and_sum(torch.cat(inner), [st for st, _ in groups], ct.scale * pt0.scale,
                                         ct.level, nres)
        inner = self._bsgs_inner(ct, groups)
        pt0 = next(pt for _, pairs in groups for _, pt in pairs)
        return self._moddown_and_sum(inner, [st for st, _ in groups], ct.scale * pt0.scale, ct.level, nres)

    def _bsgs_inner(self, ct, groups):
        """lf_bsgs_ext for <= 4 giant groups: (G, 2, ext, N) extended-basis giant sums."""
        import ctypes
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .fused import ct_block
        n = self.params.n
        rot = sorted({b for _, pairs in groups for b, _ in pairs if b % n})
        G = len(groups)
        slot = {b: 1 + i for i, b in enumerate(rot)}
        ctx = get_context(self.params)
        lib = _native.lib()
        level = ct.level
        ext = level + 1 + self.params.num_special
        N = self.params.N
        ptrs = [None] * (G * (len(rot) + 1))
        pt0 = None
        for k, (_, pairs) in enumerate(groups):
            for b, pt in pairs:
                ptrs[k * (len(rot) + 1) + (slot[b] if b % n else 0)] = pt.poly.limbs.data_ptr()
                pt0 = pt
        parr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        keys = self._rot_keys(rot)
        karr = (ctypes.c_void_p * len(rot))(*[ctx.check_evk(k).data_ptr() for k in keys])
        gs = [galois_element_of(N, b) for b in rot]
        ws = torch.empty(lib.lf_rotate_hoisted_workspace_bytes(ctx.handle, level, 1) // 4,
                         dtype=torch.int32, device="cuda")
        inner = torch.empty((G, 2, ext, N), dtype=torch.int32, device="cuda")
        _native.check(lib.lf_bsgs_ext(ctx.handle, level, dptr(ct_block(ct)), len(rot), _native.u32_array(gs),
                                      karr, G, parr, dptr(inner), dptr(ws), stream_handle()), "lf_bsgs_ext")
        return inner

    def _moddown_and_sum(self, inner, shifts, scale, level, nres=0):
        """ONE batched mod_down of the giant steps' extended sums (lf_moddown_ext; with nres
        rescales fused into the same division, lf_moddown_ext_rescale), then the giant
        rotations and the final sum (rotate_and_sum)."""
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .poly import Domain, RnsPolynomial, main_ids
        ctx = get_context(self.params)
        lib = _native.lib()
        G = inner.shape[0]
        N = self.params.N
        ws = torch.empty(lib.lf_moddown_workspace_bytes(ctx.handle, level, G) // 4, dtype=torch.int32,
                         device="cuda")
        if nres:
            q = self.params.rns_basis
            out = torch.empty((G, 2, level + 1 - nres, N), dtype=torch.int32, device="cuda")
            _native.check(lib.lf_moddown_ext_rescale(ctx.handle, level, nres, dptr(inner), inner[0].numel(),
                                                     dptr(out), out[0].numel(), G, dptr(ws), stream_handle()),
                          "lf_moddown_ext_rescale")
            for i in range(nres):
                scale = Fraction(scale) / q[level - i]
            level -= nres
        else:
            out = torch.empty((G, 2, level + 1, N), dtype=torch.int32, device="cuda")
            _native.check(lib.lf_moddown_ext(ctx.handle, level, dptr(inner), inner[0].numel(), dptr(out),
                                             out[0].numel(), G, dptr(ws), stream_handle()), "lf_moddown_ext")
        ids = main_ids(level)
        cts = [self.C.Ciphertext(RnsPolynomial(out[i, 0], Domain.EVAL, ids),
                                 RnsPolynomial(out[i, 1], Domain.EVAL, ids), scale, level) for i in range(G)]
        return self.rotate_and_sum(list(zip(shifts, cts)), batch=out)

    def bsgs_combine_ext(self, groups, nres=0):
        """Per giant step: sum_b ext_b * pt_{k,b} over the extended basis (lf_ptmac_rows) into one
        batch, ONE batched mod_down of all giant steps (lf_moddown_ext; + nres rescales in the
        same division), then the batched giant rotations and the final sum (rotate_and_sum)."""
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .poly import Domain, RnsPolynomial, extended_ids, main_ids
        ctx = get_context(self.params)
        lib = _native.lib()
        x0 = groups[0][1][0][0]
        level = x0.level
        ext_ids = extended_ids(self.params, level)
        ext = len(ext_ids)
        N = self.params.N
        G = len(groups)
        inner = torch.empty((G, 2, ext, N), dtype=torch.int32, device="cuda")
        pidx = ctx.pidx_array(ext_ids)
        for i, (_, pairs) in enumerate(groups):
            assert len(pairs) <= 32
            n = len(pairs)
            bp = (ctypes_void_p * n)(*[x.data[0].data_ptr() for x, _ in pairs])
            ap = (ctypes_void_p * n)(*[x.data[1].data_ptr() for x, _ in pairs])
            pp = (ctypes_void_p * n)(*[pt.poly.limbs.data_ptr() for _, pt in pairs])
            _native.check(lib.lf_ptmac_rows(ctx.handle, ctypes_void_p(inner[i].data_ptr()), ext, pidx, n,
                                            bp, ap, pp, stream_handle()), "lf_ptmac_rows")
        scale = x0.scale * groups[0][1][0][1].scale
        return self._moddown_and_sum(inner, [st for st, _ in groups], scale, level, nres)

    def rotate_and_sum(self, items, batch=None):
        """sum_k rot_{s_k}(ct_k): the rotated ones in one lf_rotate_batch pipeline (they must be
        contiguous in `batch` when given), the sum in one linear-combination launch."""
        import torch
        from . import fused
        from .poly import Domain, RnsPolynomial, main_ids
        ct0 = items[0][1]
        level, scale = ct0.level, ct0.scale
        parts = [c for st, c in items if st % self.params.n == 0]
        rot = [(i, st) for i, (st, _) in enumerate(items) if st % self.params.n]
        if rot:
            lo, hi = rot[0][0], rot[-1][0] + 1
            assert [i for i, _ in rot] == list(range(lo, hi)), "rotated giants must be contiguous"
            src = batch[lo:hi] if batch is not None else torch.stack(
                [torch.stack([c.b.limbs, c.a.limbs]) for _, c in items[lo:hi]])
            gs = [galois_element_of(self.params.N, st) for _, st in rot]
            keys = self._rot_keys([st for _, st in rot])
            r = fused.rotate_batch(self.params, level, src, gs, keys, permuted=self.permuted_keys)
            ids = main_ids(level)
            parts.extend(self.C.Ciphertext(RnsPolynomial(r[j, 0], Domain.EVAL, ids),
                                           RnsPolynomial(r[j, 1], Domain.EVAL, ids), scale, level)
                         for j in range(hi - lo))
        if len(parts) == 1:
            return parts[0]
        acc = self.lincomb([(c, 1.0, Fraction(1)) for c in parts])
        return self.C.Ciphertext(acc.b, acc.a, scale, level)

    # arithmetic
    def with_scale(self, x, scale):
        """The same residues declared at another scale (exact: value = residues / scale)."""
        if isinstance(x, CtBatch):
            return CtBatch(x.data, scale, x.level)
        return self.C.Ciphertext(x.b, x.a, Fraction(scale), x.level)

    def _b_ewise(self, op, x, y):
        import torch
        from .poly import ewise
        assert x.level == y.level and x.scale == y.scale and x.data.shape == y.data.shape
        out = torch.empty(x.data.shape, dtype=x.data.dtype, device=x.data.device)
        if x.data.is_contiguous() and y.data.is_contiguous():
            n = x.data.shape[0] * 2 * (x.level + 1)
            ewise(self.params, op, out.view(n, -1), x.data.view(n, -1), self._rows_pidx(x), b=y.data.view(n, -1))
        else:
            # level-dropped views: one launch per polynomial (its rows are contiguous) instead
            # of a copy of the whole batch
            ids = tuple(range(x.level + 1))
            for i in range(x.data.shape[0]):
                for k in range(2):
                    ewise(self.params, op, out[i, k], x.data[i, k], ids, b=y.data[i, k])
        return CtBatch(out, x.scale, x.level)

    def add(self, x, y):
        if isinstance(x, CtBatch):
            from .poly import LF_OP_ADD
            return self._b_ewise(LF_OP_ADD, x, y)
        return self.C.hom_add(x, y, self.params)

    def sub(self, x, y):
        if isinstance(x, CtBatch):
            from .poly import LF_OP_SUB
            return self._b_ewise(LF_OP_SUB, x, y)
        return self.C.hom_sub(x, y, self.params)

    def rescale(self, x):
        return self.C.rescale(x, self.params)

    def rescale2(self, x):
        """Two successive rescales (ckks.py:220-225) fused into one pass (lf_rescale_multi)."""
        from . import fused
        if x.level < 2:
            raise ValueError("double rescale below level 2")
        q = self.params.rns_basis
        if isinstance(x, CtBatch):
            import torch
            from . import _native
            from .context import dptr, get_context, stream_handle
            ctx = get_context(self.params)
            pv = x.pitched()
            if pv is None:
                x = x.dense()
                pv = (x.data[0].numel(), x.level + 1)
            B = x.data.shape[0]
            ws = ctx.rescale_workspace(x.level, B)
            out = torch.empty((B, 2, x.level - 1, self.params.N), dtype=torch.int32, device=x.data.device)
            _native.check(_native.lib().lf_rescale_multi_p(ctx.handle, x.level, 2, dptr(x.data, strided=True), pv[0],
                                                           pv[1], dptr(out), out[0].numel(), B, dptr(ws),
                                                           stream_handle()), "lf_rescale_multi_p")
            return CtBatch(out, x.scale / q[x.level] / q[x.level - 1], x.level - 2)
        b, a = fused.rescale_multi(self.params, x, 2)
        q = self.params.rns_basis
        return self.C.Ciphertext(b, a, x.scale / q[x.level] / q[x.level - 1], x.level - 2)

    def mul_rescale2_many(self, pairs, addk=None):
        """[mul_rescale2(x, y) for x, y in pairs] as ONE batch over an operand list
        (lf_hom_mul_rescale_list): all pairs at one level, all CtBatch or all single."""
        import ctypes
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        from .fused import ct_block
        lv = pairs[0][0].level
        assert all(x.level == lv and y.level == lv for x, y in pairs)
        q = self.params.rns_basis
        bases1, bases2, p1, p2, sizes, scales = [], [], [], [], [], []

        def inst(x):
            if isinstance(x, CtBatch):
                pv = x.pitched()
                if pv is None:
                    x = x.dense()
                    pv = (x.data[0].numel(), x.level + 1)
                return [x.data[i] for i in range(x.data.shape[0])], pv[1], x
            blk = ct_block(x)
            return [blk], x.level + 1, x

        keep = []
        for x, y in pairs:
            ix, px, x = inst(x)
            iy, py, y = inst(y)
            assert len(ix) == len(iy)
            keep += [x, y] + ix + iy              # operand blocks stay alive until the launch
            bases1 += [t.data_ptr() for t in ix]
            bases2 += [t.data_ptr() for t in iy]
            p1 += [px] * len(ix)
            p2 += [py] * len(iy)
            sizes.append(len(ix))
            scales.append(x.scale * y.scale / q[lv] / q[lv - 1])
        B = len(bases1)
        kb = None
        if addk and any(k is not None for k in addk):
            ks = []
            for n, k in zip(sizes, addk):
                ks += [int(k or 0)] * n
            kb = (ctypes.c_int64 * B)(*ks)
        ctx = get_context(self.params)
        ws = ctx.ks_workspace(lv, min(B, 64))
        out = torch.empty((B, 2, lv - 1, self.N), dtype=torch.int32, device="cuda")
        c1 = (ctypes.c_void_p * B)(*bases1)
        c2 = (ctypes.c_void_p * B)(*bases2)
        a1 = (ctypes.c_int * B)(*p1)
        a2 = (ctypes.c_int * B)(*p2)
        _native.check(_native.lib().lf_hom_mul_rescale_list(ctx.handle, lv, 2, c1, a1, c2, a2, kb,
                                                            dptr(self.rlk.data), dptr(out), out[0].numel(), B,
                                                            dptr(ws), stream_handle()), "lf_hom_mul_rescale_list")
        res, o = [], 0
        for (x, _), n, sc in zip(pairs, sizes, scales):
            blk = CtBatch(out[o: o + n], sc, lv - 2)
            res.append(blk if isinstance(x, CtBatch) else self.unstack(blk)[0])
            o += n
        return res

    def mul_rescale2(self, x, y):
        """rescale2(hom_mul(x, y)) in one pipeline (lf_hom_mul_rescale, ndrop 2)."""
        import torch
        from . import _native
        from .context import dptr, get_context, stream_handle
        assert x.level == y.level and x.level >= 2
        q = self.params.rns_basis
        scale = x.scale * y.scale / q[x.level] / q[x.level - 1]
        ctx = get_context(self.params)
        if isinstance(x, CtBatch):
            assert x.data.shape == y.data.shape
            px, py = x.pitched(), y.pitched()
            if px is None:
                x = x.dense()
                px = (x.data[0].numel(), x.level + 1)
            if py is None:
                y = y.dense()
                py = (y.data[0].numel(), y.level + 1)
            B = x.data.shape[0]
            c1, c2 = x.data, y.data
        else:
            from .fused import ct_block
            B = 1
            c1, c2 = ct_block(x), ct_block(y)
            px, py = (c1.numel(), x.level + 1), (c2.numel(), y.level + 1)
        ws = ctx.ks_workspace(x.level, B)
        out = torch.empty((B, 2, x.level - 1, self.N), dtype=torch.int32, device=c1.device)
        _native.check(_native.lib().lf_hom_mul_rescale_p(ctx.handle, x.level, 2, dptr(c1, strided=True), px[0], px[1],
                                                         dptr(c2, strided=True), py[0], py[1], dptr(self.rlk.data),
                                                         dptr(out), out[0].numel(), B, dptr(ws), stream_handle()),
                      "lf_hom_mul_rescale_p")
        if isinstance(x, CtBatch):
            return CtBatch(out, scale, x.level - 2)
        from .poly import Domain, RnsPolynomial, main_ids
        ids = main_ids(x.level - 2)
        return self.C.Ciphertext(RnsPolynomial(out[0, 0], Domain.EVAL, ids),
                                 RnsPolynomial(out[0, 1], Domain.EVAL, ids), scale, x.level - 2)

    def hom_mul(self, x, y):
        if isinstance(x, CtBatch):
            import torch
            from . import _native
            from .context import dptr, get_context, stream_handle
            assert x.level == y.level and x.data.shape == y.data.shape and x.level >= 1
            x, y = x.dense(), y.dense()
            ctx = get_context(self.params)
            B = x.data.shape[0]
            ws = ctx.ks_workspace(x.level, B)
            out = torch.empty_like(x.data)
            _native.check(_native.lib().lf_hom_mul(ctx.handle, x.level, dptr(x.data), dptr(y.data), x.data[0].numel(),
                                                   dptr(self.rlk.data), dptr(out), out[0].numel(), B, dptr(ws),
                                                   stream_handle()), "lf_hom_mul")
            return CtBatch(out, x.scale * y.scale, x.level)
        return self.C.hom_mul(x, y, self.rlk, self.params)

    def conjugate(self, x):
        return self.C.hom_conjugate(x, self.ck, self.params)

    def lincomb(self, terms, out=None, const=None):
        """sum_i round(c_i S_i) * ct_i, all ct_i at one level with equal ct_i.scale * S_i;
        `const` adds round(const * scale) to b in the same pass (lf_lincomb_c)."""
        import torch
        if isinstance(terms[0][0], CtBatch):
            t0 = terms[0][0]
            B = t0.data.shape[0]
            out = torch.empty((B, 2, t0.level + 1, self.N), dtype=torch.int32, device=t0.data.device)
            for i in range(B):       # per instance, straight into the batch (views, no copies)
                self.lincomb([(self.unstack(t)[i], c, S) for t, c, S in terms], out=out[i], const=const)
            return CtBatch(out, Fraction(t0.scale) * Fraction(terms[0][2]), t0.level)
        from . import _native
        from .context import get_context, stream_handle
        from .poly import Domain, RnsPolynomial, main_ids
        ct0 = terms[0][0]
        level = ct0.level
        scale = Fraction(ct0.scale) * Fraction(terms[0][2])
        nrows = level + 1
        qs = self.params.rns_basis[:nrows]
        dst, out = out, None
        ctx = get_context(self.params)
        for i0 in range(0, len(terms), 8):
            chunk = terms[i0: i0 + 8]
            n = len(chunk)
            ks = []
            for ct, c, S in chunk:
                assert ct.level == level and Fraction(ct.scale) * Fraction(S) == scale
                k = round(Fraction(c) * Fraction(S))
                ks.extend(k % q for q in qs)
            tgt = dst if (i0 == 0 and dst is not None) else \
                torch.empty((2, nrows, self.params.N), dtype=torch.int32, device=ct0.b.limbs.device)
            bp = (ctypes_void_p * n)(*[ct.b.limbs.data_ptr() for ct, _, _ in chunk])
            ap = (ctypes_void_p * n)(*[ct.a.limbs.data_ptr() for ct, _, _ in chunk])
            from . import _native as nat
            if const is not None and i0 == 0:
                kc = round(Fraction(const) * scale)
                _native.check(nat.lib().lf_lincomb_c(ctx.handle, ctypes_void_p(tgt.data_ptr()), nrows, n, bp, ap,
                                                     nat.u32_array(ks), nat.u32_array([kc % q for q in qs]),
                                                     stream_handle()), "lf_lincomb_c")
            else:
                _native.check(nat.lib().lf_lincomb(ctx.handle, ctypes_void_p(tgt.data_ptr()), nrows, n, bp, ap,
                                                   nat.u32_array(ks), stream_handle()), "lf_lincomb")
            if out is None:
                out = tgt
            else:
                from .poly import LF_OP_ADD, ewise
                for p in range(2):
                    ewise(self.params, LF_OP_ADD, out[p], out[p], main_ids(level), b=tgt[p])
        ids = main_ids(level)
        return self.C.Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids),
                                 RnsPolynomial(out[1], Domain.EVAL, ids), scale, level)

    def rotate_hoisted(self, x, steps):
        return self.C.hom_rotate_hoisted(x, list(steps), self.rk, self.params)

    def rotate_many(self, xs, steps):
        return [x if s % self.params.n == 0 else
                self.C.hom_rotate(x, s, self.rk[s % self.params.n], self.params)
                for x, s in zip(xs, steps)]

    def bsgs_combine(self, groups):
        """sum_k rot_{s_k}(sum_b ct_b * pt_{k,b}): the plaintext sums of all giant steps land in
        one batch tensor, the rotated ones go through one batched rotation pipeline
        (lf_rotate_batch), and the results are added in one linear-combination launch."""
        import torch
        from . import fused
        from .poly import Domain, RnsPolynomial, main_ids
        ct0 = groups[0][1][0][0]
        level = ct0.level
        N = self.params.N
        n = len(groups)
        inner = torch.empty((n, 2, level + 1, N), dtype=torch.int32, device=ct0.b.limbs.device)
        for i, (_, pairs) in enumerate(groups):
            self.mul_plain_sum(pairs, out=inner[i])
        scale = ct0.scale * groups[0][1][0][1].scale
        ids = main_ids(level)
        rot_idx = [i for i, (st, _) in enumerate(groups) if st % self.params.n]
        parts = [inner[i] for i, (st, _) in enumerate(groups) if st % self.params.n == 0]
        if rot_idx:
            lo, hi = rot_idx[0], rot_idx[-1] + 1
            assert rot_idx == list(range(lo, hi)), "rotated giants must be contiguous"
            gs = [galois_element_of(N, groups[i][0]) for i in rot_idx]
            keys = self._rot_keys([groups[i][0] for i in rot_idx])
            rot = fused.rotate_batch(self.params, level, inner[lo:hi], gs, keys, permuted=self.permuted_keys)
            parts.extend(rot[j] for j in range(hi - lo))
        cts = [self.C.Ciphertext(RnsPolynomial(p[0], Domain.EVAL, ids), RnsPolynomial(p[1], Domain.EVAL, ids),
                                 scale, level) for p in parts]
        acc = cts[0]
        if len(cts) > 1:
            acc = self.lincomb([(c, 1.0, Fraction(1)) for c in cts])
            acc = self.C.Ciphertext(acc.b, acc.a, scale, level)
        return acc

    def mul_plain_sum(self, pairs, out=None):
        import torch
        from . import _native
        from .context import get_context, stream_handle
        from .poly import Domain, RnsPolynomial, main_ids
        ct0, pt0 = pairs[0]
        level = ct0.level
        N = self.params.N
        if out is None:
            out = torch.empty((2, level + 1, N), dtype=torch.int32, device=ct0.b.limbs.device)
        ctx = get_context(self.params)
        lib = _native.lib()
        for i in range(0, len(pairs), 32):
            chunk = pairs[i: i + 32]
            n = len(chunk)
            bp = (ctypes_void_p * n)(*[c.b.limbs.data_ptr() for c, _ in chunk])
            ap = (ctypes_void_p * n)(*[c.a.limbs.data_ptr() for c, _ in chunk])
            pp = (ctypes_void_p * n)(*[pt.poly.limbs.data_ptr() for _, pt in chunk])
            assert all(c.level == level and pt.level == level for c, pt in chunk)
            tgt = out if i == 0 else torch.empty_like(out)
            _native.check(lib.lf_ptmac(ctx.handle, ctypes_void_p(tgt.data_ptr()), level + 1, n,
                                       bp, ap, pp, stream_handle()), "lf_ptmac")
            if i:
                out.copy_(torch.stack([self._addrows(out[0], tgt[0], level), self._addrows(out[1], tgt[1], level)]))
        ids = main_ids(level)
        scale = ct0.scale * pt0.scale
        return self.C.Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids),
                                 RnsPolynomial(out[1], Domain.EVAL, ids), scale, level)

    def _addrows(self, x, y, level):
        from .poly import LF_OP_ADD, ewise, main_ids
        o = x.clone()
        ewise(self.params, LF_OP_ADD, o, x, main_ids(level), b=y)
        return o

    def _scalar_rows(self, ct, k: int):
        return [k % q for q in self.params.rns_basis[: ct.level + 1]]

    def mul_const(self, ct, c: float, S_p):
        """ct * round(c * S_p) with the declared plaintext scale S_p (no rescale)."""
        import torch
        from .poly import LF_OP_SCALAR_MUL, Domain, RnsPolynomial, ewise, main_ids
        k = round(Fraction(c) * Fraction(S_p))
        ids = main_ids(ct.level)
        sc = self._scalar_rows(ct, k)
        if isinstance(ct, CtBatch):
            B = ct.data.shape[0]
            out = torch.empty((B, 2, ct.level + 1, self.N), dtype=torch.int32, device=ct.data.device)
            if ct.data.is_contiguous():
                n = B * 2 * (ct.level + 1)
                ewise(self.params, LF_OP_SCALAR_MUL, out.view(n, -1), ct.data.view(n, -1),
                      self._rows_pidx(ct), scalars=sc * (2 * B))
            else:                    # a dropped view: per polynomial, its rows are contiguous
                for i in range(B):
                    for p in range(2):
                        ewise(self.params, LF_OP_SCALAR_MUL, out[i, p], ct.data[i, p], ids, scalars=sc)
            return CtBatch(out, ct.scale * Fraction(S_p), ct.level)
        out = torch.empty((2, ct.level + 1, self.params.N), dtype=torch.int32, device=ct.b.limbs.device)
        ewise(self.params, LF_OP_SCALAR_MUL, out[0], ct.b.limbs, ids, scalars=sc)
        ewise(self.params, LF_OP_SCALAR_MUL, out[1], ct.a.limbs, ids, scalars=sc)
        return self.C.Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids),
                                 RnsPolynomial(out[1], Domain.EVAL, ids), ct.scale * Fraction(S_p), ct.level)

    def add_const(self, ct, c: float, out=None):
        """ct + c (the constant encoded at the ciphertext's own scale; b only).  `out`: a
        (2, level + 1, N) slot to write into (e.g. one instance of a batch being assembled)."""
        import torch
        from .poly import LF_OP_ADD_SCALAR, Domain, RnsPolynomial, ewise, main_ids
        k = round(Fraction(c) * Fraction(ct.scale))
        ids = main_ids(ct.level)
        if isinstance(ct, CtBatch):
            B = ct.data.shape[0]
            out = torch.empty(ct.data.shape, dtype=ct.data.dtype, device=ct.data.device)
            if ct.data.is_contiguous():
                n = B * 2 * (ct.level + 1)
                sc = (self._scalar_rows(ct, k) + [0] * (ct.level + 1)) * B       # b rows only
                ewise(self.params, LF_OP_ADD_SCALAR, out.view(n, -1), ct.data.view(n, -1), self._rows_pidx(ct),
                      scalars=sc)
            else:                              # a level-dropped view: per polynomial, no copy
                rows = tuple(range(ct.level + 1))
                for i in range(B):
                    ewise(self.params, LF_OP_ADD_SCALAR, out[i, 0], ct.data[i, 0], rows,
                          scalars=self._scalar_rows(ct, k))
                    ewise(self.params, LF_OP_ADD_SCALAR, out[i, 1], ct.data[i, 1], rows,
                          scalars=[0] * len(rows))
            return CtBatch(out, ct.scale, ct.level)
        if out is None:
            out = torch.empty((2, ct.level + 1, self.params.N), dtype=torch.int32, device=ct.b.limbs.device)
        ewise(self.params, LF_OP_ADD_SCALAR, out[0], ct.b.limbs, ids, scalars=self._scalar_rows(ct, k))
        ewise(self.params, LF_OP_ADD_SCALAR, out[1], ct.a.limbs, ids, scalars=[0] * len(ids))
        return self.C.Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids),
                                 RnsPolynomial(out[1], Domain.EVAL, ids), ct.scale, ct.level)

    def mul_monomial(self, ct, e: int):
        """ct * X^e (exact: slots times zeta^(e 5^j); X^(N/2) multiplies every slot by i)."""
        from .encoding import Plaintext, signed_to_eval
        from .poly import main_ids
        key = (e, ct.level)
        pt = self._mono.get(key)
        if pt is None:
            pt = Plaintext(signed_to_eval(monomial_ints(self.params.N, e), self.params,
                                          main_ids(ct.level)), Fraction(1), ct.level)
            self._mono[key] = pt
        return self.C.mul_plain(ct, pt, self.params)


from ctypes import c_void_p as ctypes_void_p  # noqa: E402


def galois_element_of(N: int, steps: int) -> int:
    from .ntt_host import galois_element
    return galois_element(N, steps % (N // 2))


def make_bootstrap_keys(params, sk, rotations, seed: int = 99):
    """Conjugation key and the rotation keys a Bootstrapper needs (host RNG in the reference's
    draw order per key, keys.py:129-159)."""
    from .keys import make_conjugation_key, make_rotation_key
    rng = np.random.default_rng(seed)
    ck = make_conjugation_key(params, sk, rng)
    rk = {}
    for s in sorted(rotations):
        rk[s] = make_rotation_key(params, sk, s, rng)
    return ck, rk


class GraphedCircuit:
    """A circuit `fn(ct) -> ct` over a GpuBackend captured once as a CUDA graph (the paper's
    runtime also replays CUDA graphs).  Every kernel, with its workspace and the
    resident plaintexts and keys, is recorded on the first call; later calls copy the input
    ciphertext into the captured input buffers and replay.  Inputs must arrive at the captured
    level and scale (plaintext constants are encoded against them)."""

    def __init__(self, backend, fn, example_ct, level=None):
        import torch
        from .ckks import Ciphertext
        from .poly import RnsPolynomial
        self.be, self.fn = backend, fn
        self.level = example_ct.level if level is None else level
        ct0 = backend.drop_to_level(example_ct, self.level)
        self.scale = ct0.scale
        self._in = torch.stack([ct0.b.limbs.clone(), ct0.a.limbs.clone()])
        ids = ct0.b.basis_ids
        self._ct = Ciphertext(RnsPolynomial(self._in[0], ct0.b.domain, ids),
                              RnsPolynomial(self._in[1], ct0.a.domain, ids), ct0.scale, self.level)
        fn(self._ct)                                     # encode / cache every plaintext
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn(self._ct)                                 # warm the allocator pool
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._out = fn(self._ct)

    def __call__(self, ct):
        from .ckks import Ciphertext
        from .poly import RnsPolynomial
        ct0 = self.be.drop_to_level(ct, self.level)
        if ct0.scale != self.scale:
            raise ValueError(f"{type(self).__name__}: input scale differs from the captured one")
        self._in[0].copy_(ct0.b.limbs)
        self._in[1].copy_(ct0.a.limbs)
        self.graph.replay()
        o = self._out
        return Ciphertext(RnsPolynomial(o.b.limbs.clone(), o.b.domain, o.b.basis_ids),
                          RnsPolynomial(o.a.limbs.clone(), o.a.domain, o.a.basis_ids), o.scale, o.level)


class GraphedBootstrap(GraphedCircuit):
    """A Bootstrapper captured once as a CUDA graph; inputs must share the captured
    ciphertext's level-0 scale (the diagonals fold Delta_in in)."""

    def __init__(self, bootstrapper: Bootstrapper, example_ct):
        self.bt = bootstrapper
        super().__init__(bootstrapper.be, bootstrapper.bootstrap, example_ct, level=0)
