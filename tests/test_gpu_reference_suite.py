"""The reference's own value-level tests (pkg/tests/test_ckks_ops.py:41-198 and
pkg/tests/test_ntt.py:17-108), restated against this package's GPU operator API with the same
fixtures (params_small = gen_params(256, 4, d=3, seed=3), keygen(seed=11), rng 77) and the
same tolerance TOL = 0.05.  The NTT checks use an independent schoolbook oracle."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu
TOL = 0.05


def naive_negacyclic_convolution(a, b, q):
    N = len(a)
    out = [0] * N
    for i in range(N):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(N):
            k = i + j
            term = ai * int(b[j])
            if k >= N:
                out[k - N] = (out[k - N] - term) % q
            else:
                out[k] = (out[k] + term) % q
    return np.array(out, dtype=np.uint64)


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    return B


@pytest.fixture(scope="module")
def ctx(B):
    p = B.gen_params(256, 4, d=3, seed=3)
    sk, pk, rlk = B.keygen(p, seed=11)
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct_v = B.encrypt(B.encode(v, p), pk, p, rng)
    ct_w = B.encrypt(B.encode(w, p), pk, p, rng)
    return p, sk, pk, rlk, v, w, ct_v, ct_w


def test_encrypt_decrypt(B, ctx):
    p, sk, _, _, v, _, ct_v, _ = ctx
    assert np.abs(B.decrypt(ct_v, sk, p) - v).max() < TOL


def test_add_zero_is_identity(B, ctx):
    p, sk, pk, _, v, _, ct_v, _ = ctx
    zero = B.encrypt(B.encode(np.zeros(p.n), p), pk, p, np.random.default_rng(3))
    assert np.abs(B.decrypt(B.hom_add(ct_v, zero, p), sk, p) - v).max() < TOL


def test_sub_self_is_zero(B, ctx):
    p, sk, _, _, _, _, ct_v, _ = ctx
    assert np.abs(B.decrypt(B.hom_sub(ct_v, ct_v, p), sk, p)).max() < TOL


def test_mul_plain_pointwise(B, ctx):
    p, sk, _, _, v, w, ct_v, _ = ctx
    out = B.mul_plain(ct_v, B.encode(w, p), p)
    assert out.scale == p.scale * p.scale
    assert np.abs(B.decrypt(out, sk, p) - v * w).max() < TOL


def test_hom_mul_then_rescale(B, ctx):
    p, sk, _, rlk, v, w, ct_v, ct_w = ctx
    out = B.rescale(B.hom_mul(ct_v, ct_w, rlk, p), p)
    assert out.level == ct_v.level - 1
    assert out.scale == p.scale * p.scale / p.rns_basis[ct_v.level]
    assert np.abs(B.decrypt(out, sk, p) - v * w).max() < TOL


def test_rotate_shifts_slots(B, ctx):
    p, sk, _, _, v, _, ct_v, _ = ctx
    rk = B.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    assert np.abs(B.decrypt(B.hom_rotate(ct_v, 1, rk, p), sk, p) - np.roll(v, -1)).max() < TOL


def test_rotate_group_inverse(B, ctx):
    p, sk, _, _, v, _, ct_v, _ = ctx
    rho = 3
    rk = B.make_rotation_key(p, sk, rho, np.random.default_rng(6))
    rk_inv = B.make_rotation_key(p, sk, p.n - rho, np.random.default_rng(7))
    back = B.hom_rotate(B.hom_rotate(ct_v, rho, rk, p), p.n - rho, rk_inv, p)
    assert np.abs(B.decrypt(back, sk, p) - v).max() < TOL


def test_conjugation(B, ctx):
    p, sk, _, _, v, _, ct_v, _ = ctx
    ck = B.make_conjugation_key(p, sk, np.random.default_rng(8))
    assert np.abs(B.decrypt(B.hom_conjugate(ct_v, ck, p), sk, p) - v).max() < TOL   # real slots


def test_keygen_and_encrypt_deterministic(B, ctx):
    p = ctx[0]
    a, b = B.keygen(p, seed=123), B.keygen(p, seed=123)
    assert np.array_equal(a[0].coeffs, b[0].coeffs)
    assert np.array_equal(a[1].b.numpy(), b[1].b.numpy())
    pt = B.encode(ctx[4], p)
    c1 = B.encrypt(pt, ctx[2], p, np.random.default_rng(9))
    c2 = B.encrypt(pt, ctx[2], p, np.random.default_rng(9))
    assert np.array_equal(c1.b.numpy(), c2.b.numpy()) and np.array_equal(c1.a.numpy(), c2.a.numpy())


def test_residues_below_primes_after_ops(B, ctx):
    p, sk, _, rlk, v, w, ct_v, ct_w = ctx
    for ct in (B.hom_add(ct_v, ct_w, p), B.hom_mul(ct_v, ct_w, rlk, p),
               B.rescale(B.hom_mul(ct_v, ct_w, rlk, p), p)):
        ct.b.validate(p)
        ct.a.validate(p)


def test_rescale_metadata(B, ctx):
    p, _, _, _, _, _, ct_v, _ = ctx
    out = B.rescale(ct_v, p)
    assert out.level == ct_v.level - 1 and out.scale == ct_v.scale / p.rns_basis[ct_v.level]


# ---- NTT (pkg/tests/test_ntt.py) -------------------------------------------------------

def _ntt(B, p, rows, q_idx, inverse=False):
    from paper_2512_11269_b200 import poly as P
    t = P.to_device(np.asarray(rows, dtype=np.uint64).reshape(1, -1))
    P.ntt_rows(p, t, (q_idx,), inverse=inverse)
    return P.to_host(t)[0]


def test_ntt_pointwise_product_matches_schoolbook(B):
    p = B.gen_params(16, 2, d=1, seed=7, hamming_weight=8)
    q = p.rns_basis[0]
    rng = np.random.default_rng(12345)
    x = rng.integers(0, q, 16, dtype=np.uint64)
    y = rng.integers(0, q, 16, dtype=np.uint64)
    ev = _ntt(B, p, x, 0) * _ntt(B, p, y, 0) % np.uint64(q)
    assert np.array_equal(_ntt(B, p, ev, 0, inverse=True), naive_negacyclic_convolution(x, y, q))
    z = np.zeros(16, dtype=np.uint64)
    assert np.array_equal(_ntt(B, p, z, 0), z)


@settings(max_examples=25, deadline=None)
@given(st.integers(0, 2 ** 32), st.sampled_from([16, 64, 256]))
def test_ntt_roundtrip_property(B, seed, N):
    p = B.gen_params(N, 1, d=1, seed=0, hamming_weight=min(64, N // 2))
    rng = np.random.default_rng(seed)
    for i, q in enumerate(p.rns_basis):
        x = rng.integers(0, q, N, dtype=np.uint64)
        assert np.array_equal(_ntt(B, p, _ntt(B, p, x, i), i, inverse=True), x)


def test_automorphism_coefficient_semantics(B):
    """sigma_g in the eval domain == X -> X^g on coefficients (with the negacyclic sign)."""
    from paper_2512_11269_b200 import poly as P
    p = B.gen_params(64, 1, d=1, seed=0, hamming_weight=16)
    q = p.rns_basis[0]
    N = p.N
    rng = np.random.default_rng(3)
    c = rng.integers(0, q, N, dtype=np.uint64)
    for g in (5, 25, 2 * N - 1):
        want = np.zeros(N, dtype=np.uint64)
        for i in range(N):
            e = i * g % (2 * N)
            if e < N:
                want[e] = (want[e] + c[i]) % q
            else:
                want[e - N] = (want[e - N] + q - c[i]) % q
        ev = P.to_device(_ntt(B, p, c, 0).reshape(1, -1))
        out = P.to_device(np.zeros((1, N), dtype=np.uint64))
        P.automorph_rows(p, out, ev, g)
        assert np.array_equal(_ntt(B, p, P.to_host(out)[0], 0, inverse=True), want)
    with pytest.raises(ValueError):
        P.poly_automorph(P.RnsPolynomial(np.zeros((1, N), dtype=np.uint64), P.Domain.EVAL, (0,)), 4, p)
