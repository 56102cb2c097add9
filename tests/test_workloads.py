"""Encrypted layer workloads (BASELINE configs 4-5, paper_2512_11269_b200/workloads.py).

CPU: the slot models (conv diagonals == direct convolution, block-diagonal matmul == X W^T),
the oracle composition of a ResNet-20 basic block and of a transformer block against their
plaintext models.  GPU: the B200 composition equals the oracle composition residue for residue
on identical keys and inputs (the bootstrap's pattern, tests/test_bootstrap.py)."""

from fractions import Fraction

import numpy as np
import pytest

from paper_2512_11269_b200 import bootstrap as BT
from paper_2512_11269_b200 import workloads as WL

TOY = dict(N=256, num_levels=30, d=3, seed=0, scale=2 ** 26)
TOY_T = dict(N=256, num_levels=52, d=3, seed=0, scale=2 ** 26)
RN_SHAPE = (2, 4, 4)           # C, H, W: 32 values, replicated 4x in n = 128 slots
TF_SHAPE = (4, 8)              # T tokens, d features


def _resnet_weights(C, seed=3):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C), rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C)


def _tf_weights(d, seed=4):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, (d, d)) / d for _ in range(6)]


def test_conv_diagonals_match_direct_convolution():
    C, H, W = 3, 4, 4
    n = 2 * C * H * W
    w = np.random.default_rng(1).normal(size=(C, C, 3, 3))
    act = np.random.default_rng(2).normal(size=(C, H, W))
    M = WL.conv3x3_diagonals(w, C, H, W, n)
    z = np.tile(act.reshape(-1), 2)
    got = BT.dm_apply(M, z).real
    want = WL.conv3x3_plain(act, w).reshape(-1)
    assert np.allclose(got[: C * H * W], want) and np.allclose(got[C * H * W:], want)
    plan = BT.bsgs_plan(M, n, 64)
    assert np.allclose(BT.bsgs_apply_plain(plan, z).real, got)


def test_blockdiag_is_row_matmul():
    T, d = 4, 8
    Wm = np.random.default_rng(1).normal(size=(d, d))
    X = np.random.default_rng(2).normal(size=(T, d))
    n = 4 * T * d
    got = BT.dm_apply(WL.blockdiag_diagonals(Wm, T, n), np.tile(X.reshape(-1), 4)).real
    assert np.allclose(got[: T * d], (X @ Wm.T).reshape(-1))


def _oracle_env(kw, rotations, seed=99):
    from oracle import lf_oracle as O
    from oracle.boot_backend import OracleBackend
    P = O.gen_params(**kw)
    keys = O.keygen(P, seed=11)
    rng = np.random.default_rng(seed)
    ck = O.conj_key(P, keys, rng)
    rk = {s: O.rotation_key(P, keys, s, rng) for s in sorted(rotations)}
    return O, P, keys, OracleBackend(P, keys.rlk, ck, rk)


def _planner(kw):
    class _P:
        N = kw["N"]
        main_primes = None
    from paper_2512_11269_b200.params import gen_params
    p = gen_params(**kw)
    _P.main_primes = p.rns_basis
    return _P


def _working_scale(kw, level):
    from paper_2512_11269_b200.params import gen_params
    q = gen_params(**kw).rns_basis
    return Fraction(q[level]) * q[level - 1]


def _run_resnet(be, O, P, keys, enc):
    C, H, W = RN_SHAPE
    w1, w2 = _resnet_weights(C)
    blk = WL.ResNetBlock(be, w1, w2, RN_SHAPE)
    act = np.random.default_rng(7).uniform(-1, 1, RN_SHAPE) * 0.5
    ct = enc(blk.pack(act))
    return blk, act, blk.forward(ct)


def test_oracle_resnet_block_matches_models():
    C, H, W = RN_SHAPE
    w1, w2 = _resnet_weights(C)
    rots = WL.ResNetBlock(_planner(TOY), w1, w2, RN_SHAPE).required_rotations()
    O, P, keys, be = _oracle_env(TOY, rots)
    S = _working_scale(TOY, P.L)

    def enc(v):
        return O.encrypt(O.encode(v, P, level=P.L, scale=S), keys, P, np.random.default_rng(5))
    blk, act, out = _run_resnet(be, O, P, keys, enc)
    got = O.decrypt(out, keys, P)[: P.n].real
    model = blk.plain(blk.pack(act))
    assert np.abs(got - model).max() < 1e-3                  # CKKS noise on top of the exact model
    true = blk.reference(act).reshape(-1)
    assert np.abs(got[: C * H * W] - true).max() < 0.05      # degree-15 Chebyshev ReLU on [-1, 1]


@pytest.mark.gpu
def test_gpu_resnet_block_bit_exact_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    C, H, W = RN_SHAPE
    w1, w2 = _resnet_weights(C)
    rots = WL.ResNetBlock(_planner(TOY), w1, w2, RN_SHAPE).required_rotations()
    O, P, keys, bo = _oracle_env(TOY, rots)
    S = _working_scale(TOY, P.L)
    _, act, want = _run_resnet(bo, O, P, keys, lambda v: O.encrypt(O.encode(v, P, level=P.L, scale=S), keys, P,
                                                                   np.random.default_rng(5)))
    p = B.gen_params(**TOY)
    sk, pk, rlk = B.keygen(p, seed=11)
    ck, rk = BT.make_bootstrap_keys(p, sk, rots, seed=99)
    bg = BT.GpuBackend(p, rlk, ck, rk)
    _, _, got = _run_resnet(bg, None, None, None, lambda v: B.encrypt(B.encode(v, p, level=p.max_level, scale=S),
                                                                      pk, p, np.random.default_rng(5)))
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(got.b.numpy(), want.b.rows) and np.array_equal(got.a.numpy(), want.a.rows)


def _run_tf(be, enc):
    T, d = TF_SHAPE
    Ws = _tf_weights(d)
    blk = WL.TransformerBlock(be, *Ws, T=T, d=d, score_bound=1.0, gelu_bound=2.0)
    X = np.random.default_rng(8).uniform(-1, 1, (T, d)) * 0.5
    return blk, X, blk.forward(enc(blk.pack(X)))


def test_oracle_transformer_block_matches_reference():
    T, d = TF_SHAPE
    Ws = _tf_weights(d)
    rots = WL.TransformerBlock(_planner(TOY_T), *Ws, T=T, d=d).required_rotations()
    O, P, keys, be = _oracle_env(TOY_T, rots)
    S = _working_scale(TOY_T, P.L)
    blk, X, out = _run_tf(be, lambda v: O.encrypt(O.encode(v, P, level=P.L, scale=S), keys, P,
                                                   np.random.default_rng(6)))
    got = O.decrypt(out, keys, P)[: T * d].real.reshape(T, d)
    assert np.abs(got - blk.reference(X)).max() < 0.05


@pytest.mark.gpu
def test_gpu_transformer_block_bit_exact_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    T, d = TF_SHAPE
    Ws = _tf_weights(d)
    rots = WL.TransformerBlock(_planner(TOY_T), *Ws, T=T, d=d).required_rotations()
    O, P, keys, bo = _oracle_env(TOY_T, rots)
    S = _working_scale(TOY_T, P.L)
    _, X, want = _run_tf(bo, lambda v: O.encrypt(O.encode(v, P, level=P.L, scale=S), keys, P, np.random.default_rng(6)))
    p = B.gen_params(**TOY_T)
    sk, pk, rlk = B.keygen(p, seed=11)
    ck, rk = BT.make_bootstrap_keys(p, sk, rots, seed=99)
    bg = BT.GpuBackend(p, rlk, ck, rk)
    _, _, got = _run_tf(bg, lambda v: B.encrypt(B.encode(v, p, level=p.max_level, scale=S), pk, p,
                                                 np.random.default_rng(6)))
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(got.b.numpy(), want.b.rows) and np.array_equal(got.a.numpy(), want.a.rows)
