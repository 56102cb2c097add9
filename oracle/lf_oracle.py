"""CPU oracle for the CKKS hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/Python integers, the algorithm of the
reference package `limbforge` (paths below are relative to
/root/reference/pkg/src/limbforge/) for every function on the hot path:
parameter synthesis, NTT tables, negacyclic NTT, automorphism, exact RNS base
conversion, mod-down, the hybrid keyswitch (ModUp / inner product / ModDown),
the homomorphic operators, encoding and key generation.

It is the CHECKER, never the product: only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s CPU-baseline / `--impl reference` leg may import it.  The
product package `paper_2512_11269_b200` must never import this file.

Parity status: PINNED.  `tests/golden/make_golden.py` generated the fixtures
in `tests/golden/` by importing the real reference from /root/reference; the
CPU tests (`tests/test_oracle_golden.py`) check this oracle against them
bit-for-bit (residues) and within the reference tolerances (decoded slots).

Representation: a polynomial is `Poly(rows, ids, is_eval)` with `rows` a
(len(ids), N) uint64 array of canonical residues, `ids` the basis ids
(main primes 0..L, special primes SPECIAL_BASE + j).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache
from math import ceil

import numpy as np

U64 = np.uint64
SPECIAL_BASE = 1 << 16          # poly.py:20
PRIME_CAP = 1 << 28             # params.py:14-15
DEFAULT_SCALE = 1 << 20         # params.py:18
DEFAULT_H = 64                  # params.py:19
DEFAULT_SIGMA = 3.2             # params.py:20


# ----------------------------------------------------------------------------
# modular arithmetic (modmath.py)
# ----------------------------------------------------------------------------

def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin with the first 12 prime bases (modmath.py:6-30)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _distinct_prime_factors(n: int) -> list:
    out, f = [], 2
    while f * f <= n:
        if n % f == 0:
            out.append(f)
            while n % f == 0:
                n //= f
        f += 1
    if n > 1:
        out.append(n)
    return out


def smallest_generator(q: int) -> int:
    """Smallest generator of (Z/q)^* (modmath.py:37-44)."""
    fs = _distinct_prime_factors(q - 1)
    g = 2
    while any(pow(g, (q - 1) // f, q) == 1 for f in fs):
        g += 1
    return g


def root_2n(N: int, q: int) -> int:
    """psi = g^((q-1)/2N) for the smallest generator g (modmath.py:61-68)."""
    return pow(smallest_generator(q), (q - 1) // (2 * N), q)


def bitrev(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    i = np.arange(n, dtype=np.int64)
    r = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        r |= ((i >> b) & 1) << (bits - 1 - b)
    return r


def crt_centered(rows, primes) -> list:
    """Exact centred CRT lift (modmath.py:82-99)."""
    primes = [int(p) for p in primes]
    Q = 1
    for p in primes:
        Q *= p
    acc = [0] * len(rows[0])
    for row, p in zip(rows, primes):
        h = Q // p
        f = h * pow(h % p, -1, p)
        for k, r in enumerate(row):
            acc[k] += int(r) * f
    half = Q // 2
    out = []
    for c in acc:
        c %= Q
        out.append(c - Q if c > half else c)
    return out


# ----------------------------------------------------------------------------
# parameters (params.py)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class Params:
    N: int
    main: tuple          # rns_basis
    special: tuple       # special_basis
    scale: Fraction
    h: int
    d: int
    seed: int = 0
    sigma: float = DEFAULT_SIGMA

    @property
    def n(self):
        return self.N // 2

    @property
    def L(self):
        return len(self.main) - 1

    @property
    def alpha(self):
        return len(self.special)

    def prime(self, bid: int) -> int:
        return self.special[bid - SPECIAL_BASE] if bid >= SPECIAL_BASE else self.main[bid]

    def main_ids(self, level):
        return tuple(range(level + 1))

    def special_ids(self):
        return tuple(SPECIAL_BASE + j for j in range(self.alpha))

    def ext_ids(self, level):
        return self.main_ids(level) + self.special_ids()

    def digits(self, level):
        """Round-robin digit groups, limb i -> digit i % d (params.py:23-41)."""
        g = [[i for i in range(level + 1) if i % self.d == j] for j in range(self.d)]
        return [x for x in g if x]


def gen_params(N, num_levels, d=3, seed=0, scale=DEFAULT_SCALE, hamming_weight=DEFAULT_H) -> Params:
    """Prime synthesis of params.py:124-171: q0 = largest NTT prime < 2^28, specials the
    next-largest (sorted ascending), remaining main primes the smallest above `scale`."""
    if N < 16 or N & (N - 1):
        raise ValueError("N must be a power of two, at least 16")
    if d < 1:
        raise ValueError("digit count must be >= 1")
    step = 2 * N
    n_main = num_levels + 1
    n_sp = ceil(n_main / d)
    top, p = [], PRIME_CAP - 1 - (PRIME_CAP - 2) % step
    while p > step and len(top) < 1 + n_sp:
        if is_prime(p):
            top.append(p)
        p -= step
    if len(top) < 1 + n_sp:
        raise ValueError("not enough primes")
    s = int(Fraction(scale))
    lows, p = [], s + step - (s % step) + 1
    if p <= s:
        p += step
    excl = set(top)
    while p < PRIME_CAP and len(lows) < num_levels:
        if p not in excl and is_prime(p):
            lows.append(p)
        p += step
    if len(lows) < num_levels:
        raise ValueError("not enough primes above the scale")
    return Params(N, (top[0], *lows), tuple(sorted(top[1:])), Fraction(scale), hamming_weight, d, seed)


# ----------------------------------------------------------------------------
# NTT (ntt.py)
# ----------------------------------------------------------------------------

@lru_cache(maxsize=None)
def twiddles(N: int, q: int):
    """(psi_brv, ipsi_brv, n_inv): psi_brv[i] = psi^brv(i) (ntt.py:22-67)."""
    psi = root_2n(N, q)
    ipsi = pow(psi, -1, q)
    fw = np.empty(N, dtype=object)
    iv = np.empty(N, dtype=object)
    a = b = 1
    for i in range(N):
        fw[i], iv[i] = a, b
        a, b = a * psi % q, b * ipsi % q
    r = bitrev(N)
    return fw[r].astype(U64), iv[r].astype(U64), pow(N, -1, q)


def ntt_fwd(x: np.ndarray, q: int) -> np.ndarray:
    """Cooley-Tukey, natural coefficients -> bit-reversed evaluations (ntt.py:70-86)."""
    N = x.shape[-1]
    w_all, _, _ = twiddles(N, q)
    Q = U64(q)
    a = np.array(x, dtype=U64, copy=True)
    lead = a.shape[:-1]
    t, m = 1, N >> 1
    while m:
        v = a.reshape(*lead, t, 2, m)
        w = w_all[t:2 * t][:, None]
        lo = v[..., 0, :].copy()
        hi = v[..., 1, :] * w % Q
        v[..., 0, :] = (lo + hi) % Q
        v[..., 1, :] = (lo + Q - hi) % Q
        t, m = t << 1, m >> 1
    return a


def ntt_inv(x: np.ndarray, q: int) -> np.ndarray:
    """Gentleman-Sande then *N^-1; exact inverse of ntt_fwd (ntt.py:89-105)."""
    N = x.shape[-1]
    _, w_all, ninv = twiddles(N, q)
    Q = U64(q)
    a = np.array(x, dtype=U64, copy=True)
    lead = a.shape[:-1]
    t, m = N >> 1, 1
    while m < N:
        v = a.reshape(*lead, t, 2, m)
        w = w_all[t:2 * t][:, None]
        lo = v[..., 0, :].copy()
        hi = v[..., 1, :].copy()
        v[..., 0, :] = (lo + hi) % Q
        v[..., 1, :] = (lo + Q - hi) % Q * w % Q
        t, m = t >> 1, m << 1
    return a * U64(ninv) % Q


def galois_element(N: int, steps: int) -> int:
    return pow(5, steps % (N // 2), 2 * N)          # ntt.py:129-132


@lru_cache(maxsize=None)
def automorphism_perm(N: int, g: int) -> np.ndarray:
    """perm[i] = brv(((2 brv(i) + 1) g mod 2N - 1) / 2) (ntt.py:108-121)."""
    if g % 2 == 0:
        raise ValueError("automorphism index must be odd")
    r = bitrev(N)
    e = (2 * r + 1) * g % (2 * N)
    return r[(e - 1) // 2]


# ----------------------------------------------------------------------------
# RNS polynomials and row primitives (poly.py)
# ----------------------------------------------------------------------------

@dataclass
class Poly:
    rows: np.ndarray          # (len(ids), N) uint64
    ids: tuple
    is_eval: bool = True

    def row(self, bid):
        return self.rows[self.ids.index(bid)]

    def sub(self, ids):
        return Poly(np.stack([self.row(b) for b in ids]), tuple(ids), self.is_eval)


def _qcol(P: Params, ids):
    return np.array([P.prime(b) for b in ids], dtype=U64)[:, None]


def p_add(P, x: Poly, y: Poly) -> Poly:
    assert x.ids == y.ids and x.is_eval == y.is_eval
    return Poly((x.rows + y.rows) % _qcol(P, x.ids), x.ids, x.is_eval)


def p_sub(P, x: Poly, y: Poly) -> Poly:
    assert x.ids == y.ids and x.is_eval == y.is_eval
    q = _qcol(P, x.ids)
    return Poly((x.rows + q - y.rows) % q, x.ids, x.is_eval)


def p_mul(P, x: Poly, y: Poly) -> Poly:
    assert x.ids == y.ids and x.is_eval == y.is_eval
    return Poly(x.rows * y.rows % _qcol(P, x.ids), x.ids, x.is_eval)


def p_scale(P, x: Poly, scalars: dict) -> Poly:
    q = _qcol(P, x.ids)
    s = np.array([scalars[b] % P.prime(b) for b in x.ids], dtype=U64)[:, None]
    return Poly(x.rows * s % q, x.ids, x.is_eval)


def p_ntt(P, x: Poly) -> Poly:
    assert not x.is_eval
    return Poly(np.stack([ntt_fwd(r, P.prime(b)) for r, b in zip(x.rows, x.ids)]), x.ids, True)


def p_intt(P, x: Poly) -> Poly:
    assert x.is_eval
    return Poly(np.stack([ntt_inv(r, P.prime(b)) for r, b in zip(x.rows, x.ids)]), x.ids, False)


def p_automorph(P, x: Poly, g: int) -> Poly:
    assert x.is_eval
    return Poly(x.rows[:, automorphism_perm(P.N, g)], x.ids, True)


@lru_cache(maxsize=None)
def bconv_consts(src: tuple, dst: int):
    S = 1
    for s in src:
        S *= s
    inv = np.array([pow(S // s, -1, s) for s in src], dtype=U64)
    wts = np.array([(S // s) % dst for s in src], dtype=U64)
    return inv, wts, S % dst, S


def bconv_row(rows: np.ndarray, src: tuple, dst: int) -> np.ndarray:
    """Exact CRT lift of the value held by `rows` over primes `src`, reduced mod `dst`
    (poly.py:150-178): y_i = r_i (S/s_i)^-1 mod s_i; u = floor(sum y_i/s_i) via float64
    with an exact big-integer decision for |v - rint(v)| < 2^-40; out = sum y_i (S/s_i)
    - u S  (mod dst)."""
    src = tuple(int(s) for s in src)
    inv, wts, S_mod, S = bconv_consts(src, int(dst))
    sv = np.array(src, dtype=U64)[:, None]
    y = rows * inv[:, None] % sv
    acc = (y * wts[:, None]).sum(axis=0, dtype=U64) % U64(dst)
    v = (y / np.array(src, dtype=np.float64)[:, None]).sum(axis=0)
    u = np.floor(v)
    for k in np.nonzero(np.abs(v - np.rint(v)) < 2.0 ** -40)[0]:
        u[k] = sum(int(yy) * (S // s) for yy, s in zip(y[:, k], src)) // S
    sub = u.astype(U64) * U64(S_mod) % U64(dst)
    return (acc + U64(dst) - sub) % U64(dst)


def base_convert(P, x: Poly, targets) -> Poly:
    """poly.py:234-248: targets already in the source pass through unchanged."""
    assert not x.is_eval
    src = tuple(P.prime(b) for b in x.ids)
    out = np.empty((len(targets), P.N), dtype=U64)
    for k, b in enumerate(targets):
        out[k] = x.row(b) if b in x.ids else bconv_row(x.rows, src, P.prime(b))
    return Poly(out, tuple(targets), False)


def mod_down(P, x: Poly, targets) -> Poly:
    """poly.py:251-281: floor-divide by the product of dropped primes."""
    drop = tuple(b for b in x.ids if b not in targets)
    assert drop
    dp = tuple(P.prime(b) for b in drop)
    prod = 1
    for q in dp:
        prod *= q
    dr = np.stack([x.row(b) for b in drop])
    if x.is_eval:
        dr = np.stack([ntt_inv(r, q) for r, q in zip(dr, dp)])
    out = np.empty((len(targets), P.N), dtype=U64)
    for k, b in enumerate(targets):
        q = P.prime(b)
        c = bconv_row(dr, dp, q)
        if x.is_eval:
            c = ntt_fwd(c, q)
        Q = U64(q)
        out[k] = (x.row(b) + Q - c) % Q * U64(pow(prod, -1, q)) % Q
    return Poly(out, tuple(targets), x.is_eval)


def rescale_poly(P, x: Poly) -> Poly:
    assert x.ids == P.main_ids(len(x.ids) - 1)
    return mod_down(P, x, x.ids[:-1])


# ----------------------------------------------------------------------------
# encoding (encoding.py)
# ----------------------------------------------------------------------------

@lru_cache(maxsize=None)
def _slot_bins(N: int):
    n, two = N // 2, 2 * N
    pos, neg, t = np.empty(n, np.int64), np.empty(n, np.int64), 1
    for j in range(n):
        pos[j] = (t - 1) // 2
        neg[j] = (two - t - 1) // 2
        t = t * 5 % two
    return pos, neg


def embed_inverse(slots, N):
    pos, neg = _slot_bins(N)
    z = np.zeros(N // 2, dtype=np.complex128)
    z[:len(slots)] = slots
    ev = np.zeros(N, dtype=np.complex128)
    ev[pos] = z
    ev[neg] = np.conj(z)
    return (np.fft.fft(ev) * np.exp(-1j * np.pi * np.arange(N) / N) / N).real


def embed_forward(coeffs, N):
    pos, _ = _slot_bins(N)
    ev = np.fft.ifft(coeffs * np.exp(1j * np.pi * np.arange(N) / N)) * N
    return ev[pos]


@dataclass
class Plain:
    poly: Poly
    scale: Fraction
    level: int


def encode(values, P: Params, level=None, scale=None) -> Plain:
    level = P.L if level is None else level
    scale = Fraction(P.scale if scale is None else scale)
    values = np.asarray(values, dtype=np.float64)
    if values.ndim != 1 or len(values) > P.n:
        raise ValueError("bad slot vector")
    r = np.rint(embed_inverse(values, P.N) * float(scale))
    Qp = 1
    for q in P.main[:level + 1]:
        Qp *= q
    if int(np.abs(r).max(initial=0.0)) >= Qp // 4:     # exact: Qp can exceed the float range
        raise OverflowError("ScaleOverflow")
    ints = r.astype(np.int64)
    rows = np.stack([ntt_fwd(np.mod(ints, q).astype(U64), q) for q in P.main[:level + 1]])
    return Plain(Poly(rows, P.main_ids(level), True), scale, level)


def decode(poly: Poly, P: Params, scale) -> np.ndarray:
    c = p_intt(P, poly) if poly.is_eval else poly
    cen = crt_centered(c.rows, [P.prime(b) for b in c.ids])
    sc = Fraction(scale)
    f = np.array([float(Fraction(v) / sc) for v in cen])
    return embed_forward(f, P.N).real


# ----------------------------------------------------------------------------
# keys (keys.py) — same RNG draw order as the reference
# ----------------------------------------------------------------------------

def sample_ternary(rng, N, h):
    c = np.zeros(N, dtype=np.int8)
    sup = rng.choice(N, size=h, replace=False)
    c[sup] = rng.integers(0, 2, size=h, dtype=np.int8) * 2 - 1
    return c


def sample_gaussian(rng, N, sigma):
    return np.rint(rng.normal(0.0, sigma, size=N)).astype(np.int64)


def signed_to_eval(P, ints, ids) -> Poly:
    rows = np.stack([ntt_fwd(np.mod(ints, P.prime(b)).astype(U64), P.prime(b)) for b in ids])
    return Poly(rows, tuple(ids), True)


def sample_uniform(P, rng, ids) -> Poly:
    rows = np.empty((len(ids), P.N), dtype=U64)
    for k, b in enumerate(ids):
        rows[k] = rng.integers(0, P.prime(b), size=P.N, dtype=np.uint64)
    return Poly(rows, tuple(ids), True)


def digit_hat(P, j):
    f = 1
    for i, q in enumerate(P.main):
        if i % P.d != j:
            f *= q
    return f


def special_product(P):
    f = 1
    for q in P.special:
        f *= q
    return f


@dataclass
class Keys:
    s_coeffs: np.ndarray
    s_eval: Poly                # over ext ids at max level
    pk: tuple                   # (b, a) over main ids
    rlk: "EvalKeyO"


@dataclass
class EvalKeyO:
    purpose: object
    digits: list                # [(b Poly, a Poly)] over ext ids(L)


def _key_pair(P, rng, s_eval: Poly, target: Poly | None, factor: int, ids):
    a = sample_uniform(P, rng, ids)
    e = signed_to_eval(P, sample_gaussian(rng, P.N, P.sigma), ids)
    q = _qcol(P, ids)
    s = s_eval.sub(ids).rows
    b = (q - a.rows * s % q + e.rows) % q
    if target is not None:
        f = np.array([factor % P.prime(bb) for bb in ids], dtype=U64)[:, None]
        b = (b + target.sub(ids).rows * f % q) % q
    return Poly(b, tuple(ids), True), a


def _evalkey(P, rng, s_eval, target, purpose):
    ids = P.ext_ids(P.L)
    sp = special_product(P)
    digs = []
    for j in range(P.d):
        digs.append(_key_pair(P, rng, s_eval, target, sp * digit_hat(P, j), ids))
    return EvalKeyO(purpose, digs)


def keygen(P: Params, seed=None) -> Keys:
    rng = np.random.default_rng(P.seed if seed is None else seed)
    sc = sample_ternary(rng, P.N, P.h)
    s_eval = signed_to_eval(P, sc.astype(np.int64), P.ext_ids(P.L))
    pk = _key_pair(P, rng, s_eval, None, 0, P.main_ids(P.L))
    q = _qcol(P, s_eval.ids)
    s2 = Poly(s_eval.rows * s_eval.rows % q, s_eval.ids, True)
    rlk = _evalkey(P, rng, s_eval, s2, "relin")
    return Keys(sc, s_eval, pk, rlk)


def rotation_key(P: Params, keys: Keys, steps: int, rng) -> EvalKeyO:
    steps %= P.n
    if steps == 0:
        raise ValueError("identity rotation needs no key")
    g = galois_element(P.N, steps)
    rot = Poly(keys.s_eval.rows[:, automorphism_perm(P.N, g)], keys.s_eval.ids, True)
    return _evalkey(P, rng, keys.s_eval, rot, ("rot", g))


def conj_key(P: Params, keys: Keys, rng) -> EvalKeyO:
    """Conjugation key g = 2N-1 through the same evalkey construction (keys.py:129-136)."""
    g = 2 * P.N - 1
    rot = Poly(keys.s_eval.rows[:, automorphism_perm(P.N, g)], keys.s_eval.ids, True)
    return _evalkey(P, rng, keys.s_eval, rot, ("rot", g))


# ----------------------------------------------------------------------------
# CKKS operators (ckks.py)
# ----------------------------------------------------------------------------

@dataclass
class Ct:
    b: Poly
    a: Poly
    scale: Fraction
    level: int


def encrypt(pt: Plain, keys: Keys, P: Params, rng=None) -> Ct:
    rng = rng or np.random.default_rng(P.seed + 1)
    ids = P.main_ids(pt.level)
    u = signed_to_eval(P, sample_ternary(rng, P.N, P.h).astype(np.int64), ids)
    e0 = signed_to_eval(P, sample_gaussian(rng, P.N, P.sigma), ids)
    e1 = signed_to_eval(P, sample_gaussian(rng, P.N, P.sigma), ids)
    pkb, pka = keys.pk[0].sub(ids), keys.pk[1].sub(ids)
    b = p_add(P, p_add(P, p_mul(P, pkb, u), e0), pt.poly)
    a = p_add(P, p_mul(P, pka, u), e1)
    return Ct(b, a, pt.scale, pt.level)


def decrypt(ct: Ct, keys: Keys, P: Params) -> np.ndarray:
    s = keys.s_eval.sub(ct.b.ids)
    m = p_add(P, ct.b, p_mul(P, ct.a, s))
    return decode(m, P, ct.scale)


def decomposition_scalars(P, j, limbs):
    f = digit_hat(P, j)
    return {i: pow(f % P.main[i], -1, P.main[i]) for i in limbs}


def ks_decompose(P, x: Poly):
    """ModUp (ckks.py:95-117): per digit, scale, INTT, exact BConv to the rest of the
    extended basis, NTT; own rows keep the scaled eval residues."""
    level = len(x.ids) - 1
    ext = P.ext_ids(level)
    pieces = []
    for grp in P.digits(level):
        j = grp[0] % P.d
        own = p_scale(P, x.sub(grp), decomposition_scalars(P, j, grp))
        others = tuple(b for b in ext if b not in grp)
        conv = p_ntt(P, base_convert(P, p_intt(P, own), others))
        rows = np.stack([own.row(b) if b in grp else conv.row(b) for b in ext])
        pieces.append((j, Poly(rows, ext, True)))
    return pieces


def ks_inner(P, pieces, evk: EvalKeyO):
    ext = pieces[0][1].ids
    q = _qcol(P, ext)
    acc_b = np.zeros((len(ext), P.N), dtype=U64)
    acc_a = np.zeros((len(ext), P.N), dtype=U64)
    for j, d in pieces:
        kb, ka = evk.digits[j]
        acc_b = (acc_b + d.rows * kb.sub(ext).rows) % q
        acc_a = (acc_a + d.rows * ka.sub(ext).rows) % q
    return Poly(acc_b, ext, True), Poly(acc_a, ext, True)


def keyswitch(P, x: Poly, evk: EvalKeyO):
    level = len(x.ids) - 1
    ab, aa = ks_inner(P, ks_decompose(P, x), evk)
    ids = P.main_ids(level)
    return mod_down(P, ab, ids), mod_down(P, aa, ids)


def hom_add(P, c1: Ct, c2: Ct) -> Ct:
    return Ct(p_add(P, c1.b, c2.b), p_add(P, c1.a, c2.a), c1.scale, c1.level)


def hom_sub(P, c1: Ct, c2: Ct) -> Ct:
    return Ct(p_sub(P, c1.b, c2.b), p_sub(P, c1.a, c2.a), c1.scale, c1.level)


def add_plain(P, c: Ct, pt: Plain) -> Ct:
    return Ct(p_add(P, c.b, pt.poly), c.a, c.scale, c.level)


def mul_plain(P, c: Ct, pt: Plain) -> Ct:
    return Ct(p_mul(P, c.b, pt.poly), p_mul(P, c.a, pt.poly), c.scale * pt.scale, c.level)


def hom_mul(P, c1: Ct, c2: Ct, rlk: EvalKeyO) -> Ct:
    """ckks.py:182-194: tensor, relinearise d2, no rescale."""
    d0 = p_mul(P, c1.b, c2.b)
    d1 = p_add(P, p_mul(P, c1.b, c2.a), p_mul(P, c1.a, c2.b))
    d2 = p_mul(P, c1.a, c2.a)
    kb, ka = keyswitch(P, d2, rlk)
    return Ct(p_add(P, d0, kb), p_add(P, d1, ka), c1.scale * c2.scale, c1.level)


def hom_rotate(P, c: Ct, steps: int, rk: EvalKeyO) -> Ct:
    """ckks.py:197-217: decompose-then-permute."""
    steps %= P.n
    if steps == 0:
        return c
    g = galois_element(P.N, steps)
    return apply_galois(P, c, g, rk)


def apply_galois(P, c: Ct, g: int, rk: EvalKeyO) -> Ct:
    pieces = [(j, p_automorph(P, d, g)) for j, d in ks_decompose(P, c.a)]
    ab, aa = ks_inner(P, pieces, rk)
    ids = P.main_ids(c.level)
    b = p_add(P, p_automorph(P, c.b, g), mod_down(P, ab, ids))
    return Ct(b, mod_down(P, aa, ids), c.scale, c.level)


def rescale(P, c: Ct) -> Ct:
    return Ct(rescale_poly(P, c.b), rescale_poly(P, c.a), c.scale / P.main[c.level], c.level - 1)
