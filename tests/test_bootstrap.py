"""Bootstrap: the plaintext model of every stage (CPU), the oracle
composition's precision (CPU), and the GPU pipeline residue-for-residue against the oracle
composition on identical keys and inputs (GPU).  Decrypted precision is checked against the
input ciphertext's own decryption, so the encryption noise of the input does not count."""

import numpy as np
import pytest

from paper_2512_11269_b200 import bootstrap as BT

TOY = dict(N=256, num_levels=30, d=3, seed=0, scale=2 ** 26)
TOY_CFG = BT.BootConfig(cts_levels=3, stc_levels=3)


def _U(N):
    n, M = N // 2, 2 * N
    rg = [pow(5, j, M) for j in range(n)]
    zeta = np.exp(1j * np.pi / N)
    return np.array([[zeta ** (rg[j] * k) for k in range(n)] for j in range(n)])


@pytest.mark.parametrize("N,nlev", [(64, 2), (64, 4), (1024, 3), (1024, 4)])
def test_linear_factorisation(N, nlev):
    n = N // 2
    U = _U(N)
    br = BT.bit_reverse_perm(n)
    rng = np.random.default_rng(N + nlev)
    w = rng.normal(size=n) + 1j * rng.normal(size=n)
    z = U @ w
    v = z.copy()
    for M in BT.cts_matrices(N, nlev):
        v = BT.dm_apply(M, v)
    assert np.abs(v - w[br]).max() < 1e-9 * np.abs(w).max() * n
    v = w[br].copy()
    for M in BT.stc_matrices(N, nlev):
        v = BT.dm_apply(M, v)
    assert np.abs(v - z).max() < 1e-9 * np.abs(z).max() * n
    for M in BT.cts_matrices(N, nlev) + BT.stc_matrices(N, nlev):
        plan = BT.bsgs_plan(M, n)
        assert np.allclose(BT.bsgs_apply_plain(plan, z), BT.dm_apply(M, z), atol=1e-9 * np.abs(z).max())
        assert len(M) <= 2 ** (int(np.log2(n)) // nlev + 2) - 1


def test_chebyshev_division():
    from numpy.polynomial import chebyshev as C
    c = np.random.default_rng(1).normal(size=32)
    q, r = BT.cheb_divmod(c, 16)
    x = np.linspace(-1, 1, 101)
    assert np.allclose(C.chebval(x, q) * C.chebval(x, [0] * 16 + [1]) + C.chebval(x, r), C.chebval(x, c))


def test_evalmod_model():
    cfg = BT.BootConfig()
    x = np.concatenate([np.arange(-cfg.K, cfg.K + 1) + d for d in np.linspace(-0.02, 0.02, 9)])
    f = BT.evalmod_plain(x, cfg)
    assert np.abs(f - np.sin(2 * np.pi * x) / (2 * np.pi)).max() < 1e-8


def _oracle_setup(kw=TOY, cfg=TOY_CFG, in_scale=2 ** 22):
    from oracle import lf_oracle as O
    from oracle.boot_backend import OracleBackend

    P = O.gen_params(**kw)
    keys = O.keygen(P, seed=11)

    class _Plan:
        N = P.N
        main_primes = P.main
    rots = BT.Bootstrapper(_Plan, cfg).required_rotations()
    rng = np.random.default_rng(99)
    ck = O.conj_key(P, keys, rng)
    rk = {s: O.rotation_key(P, keys, s, rng) for s in rots}
    be = OracleBackend(P, keys.rlk, ck, rk)
    v = np.random.default_rng(77).uniform(-1, 1, P.n)
    ct = O.encrypt(O.encode(v, P, level=0, scale=in_scale), keys, P, np.random.default_rng(5))
    return O, P, keys, be, v, ct


def test_oracle_bootstrap_precision():
    O, P, keys, be, v, ct = _oracle_setup()
    out = BT.Bootstrapper(be, TOY_CFG).bootstrap(ct)
    din = O.decrypt(ct, keys, P)[: P.n]
    dout = O.decrypt(out, keys, P)[: P.n]
    assert out.level >= 1 and out.scale == P.scale
    err = np.abs(dout - din).max()
    assert err < 2 ** -12, err
    assert np.abs(dout - v).max() < 0.05                    # reference TOL (test_ckks_ops.py:27)


@pytest.mark.gpu
def test_gpu_bootstrap_bit_exact_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    O, P, keys, be, v, ct_o = _oracle_setup()
    want = BT.Bootstrapper(be, TOY_CFG).bootstrap(ct_o)

    p = B.gen_params(**TOY)
    sk, pk, rlk = B.keygen(p, seed=11)
    planner = BT.Bootstrapper(type("P", (), {"N": p.N, "main_primes": p.rns_basis}), TOY_CFG)
    ck, rk = BT.make_bootstrap_keys(p, sk, planner.required_rotations(), seed=99)
    ct = B.encrypt(B.encode(v, p, level=0, scale=2 ** 22), pk, p, np.random.default_rng(5))
    assert np.array_equal(ct.b.numpy(), ct_o.b.rows) and np.array_equal(ct.a.numpy(), ct_o.a.rows)
    bt = BT.Bootstrapper(BT.GpuBackend(p, rlk, ck, rk), TOY_CFG)
    got = bt.bootstrap(ct)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(got.b.numpy(), want.b.rows)
    assert np.array_equal(got.a.numpy(), want.a.rows)
    # the CUDA-graph replay of the same pipeline gives the same residues, also for a new input
    g = BT.GraphedBootstrap(bt, ct)
    assert np.array_equal(g(ct).b.numpy(), want.b.rows)
    ct2 = B.encrypt(B.encode(-v, p, level=0, scale=2 ** 22), pk, p, np.random.default_rng(6))
    assert np.array_equal(g(ct2).a.numpy(), bt.bootstrap(ct2).a.numpy())


@pytest.mark.gpu
def test_gpu_bootstrap_c3_precision():
    """N=2^16 full-slot bootstrap (C3 variant: 48 main primes) — decrypted precision."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    p = B.gen_params(65536, 47, d=4, seed=0, scale=2 ** 26)
    sk, pk, rlk = B.keygen(p, seed=11)
    planner = BT.Bootstrapper(type("P", (), {"N": p.N, "main_primes": p.rns_basis}), BT.BootConfig())
    ck, rk = BT.make_bootstrap_keys(p, sk, planner.required_rotations(), seed=99)
    v = np.random.default_rng(77).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p, level=0, scale=2 ** 26), pk, p, np.random.default_rng(5))
    out = BT.Bootstrapper(BT.GpuBackend(p, rlk, ck, rk)).bootstrap(ct)
    din = B.decrypt(ct, sk, p)
    dout = B.decrypt(out, sk, p)
    assert out.level >= 10
    assert np.abs(dout - din).max() < 2 ** -8
    assert np.abs(dout - v).max() < 0.05
