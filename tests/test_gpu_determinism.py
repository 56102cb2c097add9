"""Repeatability of the tensor-core base conversion under a realistic launch history.

A round-2 variant of k_bconv_tc that let the last warp to finish reading a round's TMEM
accumulators issue the next round's MMAs (an acq_rel shared counter instead of a CTA barrier)
produced wrong accumulators in a few CTAs of the FIRST large rescale after another workload
had run in the process (found by bench.py's graph-vs-eager check on the C5 unit).  This test
replays that history: a ResNet-20 block at the C3 parameters, then batch-128 double rescales
at the C5 parameters, which must agree bit for bit."""

from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bconv_tc_repeatable_after_other_workload():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import bootstrap as BT
    from paper_2512_11269_b200 import workloads as WL
    # launch history: a ResNet-20 basic block (C3 parameters, 16 x 32 x 32)
    kw = dict(N=65536, num_levels=47, d=4, seed=0, scale=2 ** 26)
    p = B.gen_params(**kw)
    rng = np.random.default_rng(5)
    C, shape = 16, (16, 32, 32)
    w1, w2 = rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C), rng.uniform(-1, 1, (C, C, 3, 3)) / (9 * C)

    class P:
        N = p.N
        main_primes = p.rns_basis
    rots = WL.ResNetBlock(P, w1, w2, shape).required_rotations()
    sk, pk, rlk = B.keygen(p, seed=11)
    ck, rk = BT.make_bootstrap_keys(p, sk, rots, seed=99)
    be = BT.GpuBackend(p, rlk, ck, rk)
    blk = WL.ResNetBlock(be, w1, w2, shape)
    S = Fraction(p.rns_basis[p.max_level]) * p.rns_basis[p.max_level - 1]
    vec = blk.pack(np.random.default_rng(7).uniform(-1, 1, shape) * 0.5)
    blk.forward(B.encrypt(B.encode(vec, p, level=p.max_level, scale=S), pk, p, np.random.default_rng(5)))
    torch.cuda.synchronize()
    del be, blk, rk, ck
    # then large batched double rescales at the C5 parameters
    p5 = B.gen_params(65536, 52, d=4, seed=0, scale=2 ** 26)
    sk5, pk5, rlk5 = B.keygen(p5, seed=11)
    be5 = BT.GpuBackend(p5, rlk5, None, {})
    lv = 44
    q = torch.tensor(p5.rns_basis[: lv + 1], dtype=torch.int64, device="cuda")[:, None]
    x = (torch.randint(0, 2 ** 62, (128, 2, lv + 1, p5.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
    X = BT.CtBatch(x, 1, lv)
    outs = [be5.rescale2(X).data.clone() for _ in range(4)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])
