"""Parity at the production shapes of the bootstrap (C3: N=2^16, 48 main + 12 special primes,
d=4, i.e. 12-source base conversions on the tensor-core BConv with 64-byte operand rows) and of
the C2 hoisted rotations.

Every fused kernel is checked residue for residue against either the CPU oracle (the
restatement of the reference, pinned by tests/golden) or the unfused GPU composition of
golden-pinned primitives, and the two base-conversion engines (tcgen05 tensor cores and
IMAD.WIDE) against each other.  The full bootstrap is checked against the digest of the oracle
composition on the same keys and input (tests/golden/make_c3_bootstrap.py)."""

import json
import os
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C3 = dict(N=65536, num_levels=47, d=4, seed=0, scale=2 ** 26)
C2 = dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26)
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def c3():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    p = B.gen_params(**C3)
    sk, pk, rlk = B.keygen(p, seed=11)
    return B, p, sk, pk, rlk


def _engine(e):
    from paper_2512_11269_b200 import _native
    _native.check(_native.lib().lf_set_bconv_engine(e), "lf_set_bconv_engine")


@pytest.fixture(autouse=True)
def _restore_engine():
    yield
    _engine(1)


def _rand_ct(B, p, level, seed):
    ids = tuple(range(level + 1))
    rng = np.random.default_rng(seed)
    rows = lambda: np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in ids])
    E = B.Domain.EVAL
    return B.Ciphertext(B.RnsPolynomial(rows(), E, ids), B.RnsPolynomial(rows(), E, ids), p.scale, level)


def _pack(ct):
    return np.stack([ct.b.numpy(), ct.a.numpy()])


@pytest.mark.parametrize("level", [47, 45])
def test_c3_keyswitch_vs_oracle_both_engines(c3, level):
    """12-source ModUp / ModDown conversions (64-byte A rows): GPU keyswitch == oracle, on both
    base-conversion engines."""
    from oracle import lf_oracle as O
    B, p, sk, pk, rlk = c3
    P = O.gen_params(**C3)
    ko = O.keygen(P, seed=11)
    ct = _rand_ct(B, p, level, 500 + level)
    x = O.Poly(ct.a.numpy(), P.main_ids(level), True)
    wb, wa = O.keyswitch(P, x, ko.rlk)
    for eng in (1, 0):
        _engine(eng)
        kb, ka = B.keyswitch(ct.a, rlk, p)
        assert np.array_equal(kb.numpy(), wb.rows), eng
        assert np.array_equal(ka.numpy(), wa.rows), eng


def test_c3_modraise_vs_oracle(c3):
    from oracle import lf_oracle as O
    from oracle.boot_backend import OracleBackend
    from paper_2512_11269_b200 import bootstrap as BT
    B, p, sk, pk, rlk = c3
    P = O.gen_params(**C3)
    ko = O.keygen(P, seed=11)
    v = np.random.default_rng(77).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p, level=0), pk, p, np.random.default_rng(5))
    cto = O.encrypt(O.encode(v, P, level=0), ko, P, np.random.default_rng(5))
    got = BT.GpuBackend(p, rlk, None, {}).mod_raise(ct)
    want = OracleBackend(P, ko.rlk, None, {}).mod_raise(cto)
    assert got.level == p.max_level == 47
    assert np.array_equal(got.b.numpy(), want.b.rows) and np.array_equal(got.a.numpy(), want.a.rows)


@pytest.mark.parametrize("level", [47, 30])
def test_c3_mul_rescale2_from_14_sources(c3, level):
    """lf_hom_mul_rescale ndrop=2: ModDown from alpha + 2 = 14 sources onto l - 1 targets ==
    hom_mul then two rescales; batched through the bootstrap backend; both engines."""
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.bootstrap import GpuBackend
    B, p, sk, pk, rlk = c3
    xs = [_rand_ct(B, p, level, 10 * level + i) for i in range(3)]
    ys = [_rand_ct(B, p, level, 10 * level + 5 + i) for i in range(3)]
    want = [B.rescale(B.rescale(B.hom_mul(x, y, rlk, p), p), p) for x, y in zip(xs, ys)]
    for eng in (1, 0):
        _engine(eng)
        b, a = fused.hom_mul_rescale(p, xs[0], ys[0], rlk, 2)
        assert np.array_equal(b.numpy(), want[0].b.numpy()) and np.array_equal(a.numpy(), want[0].a.numpy())
        be = GpuBackend(p, rlk, None, {})
        out = be.mul_rescale2(be.stack(xs), be.stack(ys))
        for i in range(3):
            assert np.array_equal(out.data[i, 0].cpu().numpy().astype(np.uint64), want[i].b.numpy()), (eng, i)
            assert np.array_equal(out.data[i, 1].cpu().numpy().astype(np.uint64), want[i].a.numpy()), (eng, i)


@pytest.fixture(scope="module")
def c3_rot(c3):
    B, p, sk, pk, rlk = c3
    steps = list(range(1, 32)) + [32, 64, 96]
    rng = np.random.default_rng(31)
    return {s: B.make_rotation_key(p, sk, s, rng) for s in steps}


@pytest.mark.parametrize("level,nrot,G", [(45, 15, 2), (45, 31, 3), (43, 15, 4), (43, 31, 2)])
def test_c3_bsgs_fused_equals_unfused(c3, c3_rot, level, nrot, G):
    """k_bsgs_ext (all baby rotations + G giant-step sums in one kernel, permuted keys) ==
    hoisted extended rotations + per-giant plaintext sums + batched ModDown + giant rotations."""
    import torch
    from paper_2512_11269_b200 import bootstrap as BT
    B, p, sk, pk, rlk = c3
    be = BT.GpuBackend(p, rlk, None, c3_rot)
    ct = B.encrypt(B.encode(np.random.default_rng(level).uniform(-1, 1, p.n), p, level=level), pk, p,
                   np.random.default_rng(level + 1))
    babies = list(range(nrot + 1))
    shifts = [0, 32, 64, 96][:G]
    rng = np.random.default_rng(nrot * G)
    S = Fraction(p.rns_basis[level])
    gspec = []
    for sh in shifts:
        pairs = []
        for b in babies:
            d = rng.uniform(-1, 1, p.n) + 1j * rng.uniform(-1, 1, p.n)
            pairs.append((b, be.encode_slots(d, level, S, ext=True)))
        gspec.append((sh, pairs))
    fused = be.bsgs_fused_ext(ct, gspec)
    assert fused is not None
    ext = {0: be.extend(ct), **dict(zip(babies[1:], be.rotate_hoisted_ext(ct, babies[1:])))}
    un = be.bsgs_combine_ext([(sh, [(ext[b], pt) for b, pt in prs]) for sh, prs in gspec])
    assert fused.scale == un.scale and fused.level == un.level == level
    assert torch.equal(fused.b.limbs, un.b.limbs) and torch.equal(fused.a.limbs, un.a.limbs)
    _engine(0)
    fz0 = be.bsgs_fused_ext(ct, gspec)
    assert torch.equal(fz0.b.limbs, fused.b.limbs) and torch.equal(fz0.a.limbs, fused.a.limbs)


def test_c3_moddown_ext_batch_and_lincomb(c3):
    """lf_moddown_ext on a batch of 3 P*ct extensions returns the ciphertexts exactly (mod_down
    of P*x is x), and lf_lincomb(_c) with a constant == mul_const + hom_add + add_const."""
    import torch
    from paper_2512_11269_b200 import _native, bootstrap as BT
    from paper_2512_11269_b200.context import dptr, get_context, stream_handle
    B, p, sk, pk, rlk = c3
    be = BT.GpuBackend(p, rlk, None, {})
    level = 44
    cts = [_rand_ct(B, p, level, 900 + i) for i in range(3)]
    ext = torch.stack([be.extend(c).data for c in cts])
    ctx = get_context(p)
    out = torch.empty((3, 2, level + 1, p.N), dtype=torch.int32, device="cuda")
    ws = torch.empty(_native.lib().lf_moddown_workspace_bytes(ctx.handle, level, 3) // 4, dtype=torch.int32,
                     device="cuda")
    for eng in (1, 0):
        _engine(eng)
        out.zero_()
        _native.check(_native.lib().lf_moddown_ext(ctx.handle, level, dptr(ext), ext[0].numel(), dptr(out),
                                                   out[0].numel(), 3, dptr(ws), stream_handle()), "moddown")
        for i, c in enumerate(cts):
            assert torch.equal(out[i, 0], c.b.limbs) and torch.equal(out[i, 1], c.a.limbs)
    terms = [(c, x, Fraction(2 ** 20)) for c, x in zip(cts, (0.5, -1.25, 3.0))]
    lc = be.lincomb(terms, const=0.375)
    acc = None
    for c, x, S in terms:
        m = be.mul_const(c, x, S)
        acc = m if acc is None else B.hom_add(acc, m, p)
    acc = be.add_const(acc, 0.375)
    assert lc.scale == acc.scale
    assert torch.equal(lc.b.limbs, acc.b.limbs) and torch.equal(lc.a.limbs, acc.a.limbs)


def test_c2_hoisted_rotations_equal_separate():
    """hom_rotate_hoisted at C2 (one ModUp, 5 keys incl. conjugation-free steps) == separate
    hom_rotate calls, at full level and a low level."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    p = B.gen_params(**C2)
    sk, pk, rlk = B.keygen(p, seed=3)
    steps = [1, 2, 5, p.n - 1, 0, 1000]
    keys = {s: B.make_rotation_key(p, sk, s, np.random.default_rng(10 + s)) for s in steps if s % p.n}
    v = np.random.default_rng(4).uniform(-1, 1, p.n)
    for level in (p.max_level, 3):
        ct = B.encrypt(B.encode(v, p, level=level), pk, p, np.random.default_rng(level))
        got = B.hom_rotate_hoisted(ct, steps, keys, p)
        for s, g in zip(steps, got):
            want = B.hom_rotate(ct, s, keys.get(s % p.n), p)
            assert np.array_equal(_pack(g), _pack(want)), (level, s)


def test_engines_agree_c2_batch():
    """C2 batch-8 keyswitch, rotation batch and hom_mul: tensor-core and IMAD base conversion
    give identical residues."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import fused
    p = B.gen_params(**C2)
    sk, pk, rlk = B.keygen(p, seed=3)
    l1 = p.max_level + 1
    q = torch.tensor(p.rns_basis, dtype=torch.int64, device="cuda")[:, None]
    xs = (torch.randint(0, 2 ** 62, (8, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
    outs = []
    for eng in (1, 0):
        _engine(eng)
        outs.append(fused.keyswitch_batch(p, p.max_level, xs, rlk).clone())
    assert torch.equal(outs[0], outs[1])


def test_c3_bootstrap_digest_vs_oracle(c3):
    """The whole C3 bootstrap (ModRaise, 4 CtS stages of fused BSGS, EvalMod with fused
    relinearisation + double rescale, 3 StC stages), eager and CUDA-graph replay, equals the
    oracle composition's output residue for residue (digest written by
    tests/golden/make_c3_bootstrap.py on the same keys and input)."""
    import hashlib
    path = os.path.join(GOLDEN, "c3_bootstrap.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c3_bootstrap.json not generated")
    from paper_2512_11269_b200 import bootstrap as BT
    B, p, sk, pk, rlk = c3
    meta = json.load(open(path))
    planner = BT.Bootstrapper(type("P", (), {"N": p.N, "main_primes": p.rns_basis}), BT.BootConfig())
    rots = planner.required_rotations()
    assert len(rots) == meta["rotations"]
    ck, rk = BT.make_bootstrap_keys(p, sk, rots, seed=99)
    v = np.random.default_rng(77).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p, level=0, scale=2 ** 26), pk, p, np.random.default_rng(5))

    def dig(c):
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(c.b.numpy().astype(np.uint32)).tobytes())
        h.update(np.ascontiguousarray(c.a.numpy().astype(np.uint32)).tobytes())
        return h.hexdigest()
    assert dig(ct) == meta["input_sha256"]
    bt = BT.Bootstrapper(BT.GpuBackend(p, rlk, ck, rk))
    out = bt.bootstrap(ct)
    assert out.level == meta["level"]
    assert out.scale == Fraction(*meta["scale"])
    assert dig(out) == meta["sha256"]
    g = BT.GraphedBootstrap(bt, ct)
    assert dig(g(ct)) == meta["sha256"]


def test_engines_agree_16_source_moddown():
    """gen_params(65536, 52, d=4) (the C5 parameters, alpha = 14): the relinearisation fused
    with a double rescale converts from alpha + 2 = 16 sources, which fill all 64 K-bytes of
    the tensor-core operand (the overflow term moves to the epilogue).  Tensor-core and IMAD
    base conversion give identical residues, batched and single."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import bootstrap as BT
    p = B.gen_params(65536, 52, d=4, seed=0, scale=2 ** 26)
    assert p.num_special + 2 == 16
    sk, pk, rlk = B.keygen(p, seed=3)
    be = BT.GpuBackend(p, rlk, None, {})
    rng = np.random.default_rng(2)
    cts = [B.encrypt(B.encode(rng.uniform(-1, 1, p.n), p), pk, p, np.random.default_rng(i)) for i in range(4)]
    x, y = be.stack(cts[:2]), be.stack(cts[2:])
    outs = []
    for eng in (1, 0):
        _engine(eng)
        outs.append((be.mul_rescale2(x, y).data.clone(), ckks_block(be.mul_rescale2(cts[0], cts[1]))))
    _engine(1)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def ckks_block(ct):
    import torch
    return torch.stack([ct.b.limbs, ct.a.limbs]).clone()
