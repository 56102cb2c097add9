"""CPU oracle backend of the bootstrap composition — TEST INFRASTRUCTURE ONLY.

`paper_2512_11269_b200.bootstrap.Bootstrapper` is written against a small backend interface.
This backend implements it with the oracle restatement of the reference primitives
(oracle/lf_oracle.py: hom_rotate ckks.py:197-217, mul_plain/hom_add/hom_sub ckks.py:152-179,
hom_mul ckks.py:182-194, rescale ckks.py:220-225, p_scale poly.py:204-209) plus the two
bootstrap-only helpers restated in numpy (ModRaise, constant add), so that the GPU bootstrap
can be checked residue for residue against the same composition on the CPU.
Only tests/ may import this module.
"""

from fractions import Fraction

import numpy as np

from paper_2512_11269_b200.bootstrap import ListBatch, map_batch

from . import lf_oracle as O

U64 = np.uint64


def encode_ints(values, N, scale):
    r = np.rint(O.embed_inverse(np.asarray(values, dtype=np.complex128), N) * float(scale))
    return r.astype(np.int64)


def monomial_ints(N, e):
    c = np.zeros(N, dtype=np.int64)
    e %= 2 * N
    c[e % N] = -1 if e >= N else 1
    return c


class OracleBackend:
    def __init__(self, P: O.Params, rlk, ck, rk: dict):
        self.P = P
        self.N = P.N
        self.main_primes = tuple(P.main)
        self.default_scale = P.scale
        self.rlk, self.ck, self.rk = rlk, ck, rk
        self.calls = []

    def _ids(self, level):
        return self.P.main_ids(level)

    def drop_to_level(self, ct, level):
        r = map_batch(self.drop_to_level, ct, level)
        if r is not None:
            return r
        if ct.level == level:
            return ct
        ids = self._ids(level)
        return O.Ct(O.Poly(ct.b.rows[: level + 1].copy(), ids), O.Poly(ct.a.rows[: level + 1].copy(), ids),
                    ct.scale, level)

    def mod_raise(self, ct):
        P = self.P
        q0 = P.main[0]
        L = P.L
        ids = self._ids(L)
        out = []
        for poly in (ct.b, ct.a):
            c = O.ntt_inv(poly.rows[0].copy(), q0).astype(np.int64)
            c = np.where(c > q0 // 2, c - q0, c)
            rows = np.stack([O.ntt_fwd(np.mod(c, q).astype(U64), q) for q in P.main])
            out.append(O.Poly(rows, ids))
        return O.Ct(out[0], out[1], ct.scale, L)

    def encode_slots(self, values, level, scale, ext=False):
        ints = encode_ints(values, self.N, scale)
        ids = self.P.ext_ids(level) if ext else self._ids(level)
        return O.Plain(O.signed_to_eval(self.P, ints, ids), Fraction(scale), level)

    # hoisted ModDown: extended-basis ciphertexts as O.Ct over ext ids
    def extend(self, ct):
        P = self.P
        ext = P.ext_ids(ct.level)
        Pp = O.special_product(P)
        q = np.array([P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
        s = np.array([Pp % P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
        z = np.zeros((P.alpha, P.N), dtype=U64)
        b = O.Poly(np.concatenate([ct.b.rows * s % q, z]), ext)
        a = O.Poly(np.concatenate([ct.a.rows * s % q, z]), ext)
        return O.Ct(b, a, ct.scale, ct.level)

    def rotate_hoisted_ext(self, ct, steps):
        """keyswitch_decompose -> automorph -> keyswitch_inner_product (ckks.py:95-131), and
        P * sigma_g(b) on the main rows: hom_rotate (ckks.py:197-217) before its mod_down."""
        P = self.P
        ext = P.ext_ids(ct.level)
        Pp = O.special_product(P)
        pieces = O.ks_decompose(P, ct.a)
        out = []
        for st in steps:
            g = O.galois_element(P.N, st % P.n)
            ab, aa = O.ks_inner(P, [(j, O.p_automorph(P, d, g)) for j, d in pieces], self.rk[st % P.n])
            sb = O.p_automorph(P, ct.b, g)
            q = np.array([P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
            s = np.array([Pp % P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
            main = ab.rows[: ct.level + 1]
            b = O.Poly(np.concatenate([(main + sb.rows * s % q) % q, ab.rows[ct.level + 1:]]), ext)
            out.append(O.Ct(b, aa, ct.scale, ct.level))
        return out

    def bsgs_combine_ext(self, groups, nres=0):
        """Per giant: sum over the extended basis, mod_down, then `nres` rescales BEFORE the
        giant rotation (the GPU backend fuses the three into one division), rotate, sum."""
        P = self.P
        acc = None
        for st, pairs in groups:
            s = None
            for x, pt in pairs:
                t = O.Ct(O.p_mul(P, x.b, pt.poly), O.p_mul(P, x.a, pt.poly), x.scale * pt.scale, x.level)
                s = t if s is None else O.hom_add(P, s, t)
            ids = P.main_ids(s.level)
            c = O.Ct(O.mod_down(P, s.b, ids), O.mod_down(P, s.a, ids), s.scale, s.level)
            for _ in range(nres):
                c = self.rescale(c)
            if st % P.n:
                c = O.hom_rotate(P, c, st, self.rk[st % P.n])
            acc = c if acc is None else O.hom_add(P, acc, c)
        return acc

    def with_scale(self, x, scale):
        r = map_batch(lambda c: self.with_scale(c, scale), x)
        if r is not None:
            return r
        import dataclasses
        from fractions import Fraction
        return dataclasses.replace(x, scale=Fraction(scale))

    def add(self, x, y):
        r = map_batch(self.add, x, y)
        if r is not None:
            return r
        assert x.level == y.level and x.scale == y.scale
        return O.hom_add(self.P, x, y)

    def sub(self, x, y):
        r = map_batch(self.sub, x, y)
        if r is not None:
            return r
        assert x.level == y.level and x.scale == y.scale
        return O.hom_sub(self.P, x, y)

    def rescale(self, x):
        r = map_batch(self.rescale, x)
        if r is not None:
            return r
        return O.rescale(self.P, x)

    def rescale2(self, x):
        r = map_batch(self.rescale2, x)
        if r is not None:
            return r
        return O.rescale(self.P, O.rescale(self.P, x))

    def stack(self, cts):
        return ListBatch(cts)

    # batches built from / reduced to single ciphertexts (workloads.py); same results as the
    # GPU backend's batched kernels, one ciphertext at a time
    def rot_batch(self, x, steps):
        return ListBatch(self.rotate_hoisted(x, steps))

    def broadcast(self, x, B):
        return ListBatch([x] * B)

    def batch_sum(self, x):
        acc = None
        for c in x.cts:
            acc = c if acc is None else O.hom_add(self.P, acc, c)
        return acc

    def rotate_same(self, x, steps):
        return ListBatch(self.rotate_many(x.cts, [steps] * len(x.cts)))

    def mul_plain_batch(self, x, pt):
        return ListBatch([self.mul_plain_sum([(c, pt)]) for c in x.cts])

    def unstack(self, x):
        return list(x.cts)

    def lincomb(self, terms, const=None):
        """sum_i round(c_i S_i) ct_i, then (const) + round(const * scale) on b."""
        if isinstance(terms[0][0], ListBatch):
            B = len(terms[0][0].cts)
            return ListBatch([self.lincomb([(t.cts[i], c, S) for t, c, S in terms], const) for i in range(B)])
        if const is not None:
            return self.add_const(self.lincomb(terms), const)
        acc = None
        for ct, c, S in terms:
            t = self.mul_const(ct, c, S)
            acc = t if acc is None else O.hom_add(self.P, acc, t)
        return acc

    def hom_mul(self, x, y):
        r = map_batch(self.hom_mul, x, y)
        if r is not None:
            return r
        return O.hom_mul(self.P, x, y, self.rlk)

    def conjugate(self, x):
        return O.apply_galois(self.P, x, 2 * self.N - 1, self.ck)

    def rotate_hoisted(self, x, steps):
        return [x if s % self.P.n == 0 else O.hom_rotate(self.P, x, s, self.rk[s % self.P.n]) for s in steps]

    def rotate_many(self, xs, steps):
        return [x if s % self.P.n == 0 else O.hom_rotate(self.P, x, s, self.rk[s % self.P.n])
                for x, s in zip(xs, steps)]

    def bsgs_combine(self, groups):
        acc = None
        for st, pairs in groups:
            c = self.mul_plain_sum(pairs)
            if st % self.P.n:
                c = O.hom_rotate(self.P, c, st, self.rk[st % self.P.n])
            acc = c if acc is None else O.hom_add(self.P, acc, c)
        return acc

    def mul_plain_sum(self, pairs):
        acc = None
        for c, pt in pairs:
            t = O.mul_plain(self.P, c, pt)
            acc = t if acc is None else O.hom_add(self.P, acc, t)
        return acc

    def mul_const(self, ct, c, S_p):
        r = map_batch(self.mul_const, ct, c, S_p)
        if r is not None:
            return r
        k = round(Fraction(c) * Fraction(S_p))
        sc = {b: k % self.P.prime(b) for b in ct.b.ids}
        return O.Ct(O.p_scale(self.P, ct.b, sc), O.p_scale(self.P, ct.a, sc), ct.scale * Fraction(S_p), ct.level)

    def add_const(self, ct, c):
        r = map_batch(self.add_const, ct, c)
        if r is not None:
            return r
        k = round(Fraction(c) * Fraction(ct.scale))
        q = np.array([self.P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
        kk = np.array([k % self.P.prime(b) for b in ct.b.ids], dtype=U64)[:, None]
        b = O.Poly((ct.b.rows + kk) % q, ct.b.ids)
        return O.Ct(b, ct.a, ct.scale, ct.level)

    def mul_monomial(self, ct, e):
        m = O.signed_to_eval(self.P, monomial_ints(self.N, e), ct.b.ids)
        return O.Ct(O.p_mul(self.P, ct.b, m), O.p_mul(self.P, ct.a, m), ct.scale, ct.level)
