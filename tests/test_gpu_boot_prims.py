"""Bootstrap building blocks on the GPU against the CPU oracle / unfused compositions at the
reference desk size (N=4096, 7 main + 3 special primes) and at C2 (N=2^16):
ModRaise, hoisted rotations stopped before ModDown + batched mod_down, the batched rotation
pipeline, plaintext / constant linear combinations."""

from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DESK = dict(N=4096, num_levels=6, d=3, seed=0)


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from oracle import lf_oracle as O
    p, P = B.gen_params(**DESK), O.gen_params(**DESK)
    sk, pk, rlk = B.keygen(p, seed=11)
    ko = O.keygen(P, seed=11)
    steps = [1, 3, 7]
    rng_b, rng_o = np.random.default_rng(9), np.random.default_rng(9)
    rk = {s: B.make_rotation_key(p, sk, s, rng_b) for s in steps}
    rko = {s: O.rotation_key(P, ko, s, rng_o) for s in steps}
    v = np.random.default_rng(77).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p), pk, p, np.random.default_rng(1))
    cto = O.encrypt(O.encode(v, P), ko, P, np.random.default_rng(1))
    return B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto


def _pack(ct):
    return np.stack([ct.b.numpy(), ct.a.numpy()])


def test_modraise_matches_oracle(env):
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    from oracle.boot_backend import OracleBackend
    from paper_2512_11269_b200 import bootstrap as BT
    be = BT.GpuBackend(p, rlk, None, rk)
    bo = OracleBackend(P, ko.rlk, None, rko)
    c0 = be.drop_to_level(ct, 0)
    o0 = bo.drop_to_level(cto, 0)
    got, want = be.mod_raise(c0), bo.mod_raise(o0)
    assert got.level == p.max_level
    assert np.array_equal(got.b.numpy(), want.b.rows) and np.array_equal(got.a.numpy(), want.a.rows)


def test_hoisted_ext_and_moddown_match_oracle(env):
    import torch
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    from oracle.boot_backend import OracleBackend
    from paper_2512_11269_b200 import bootstrap as BT
    be = BT.GpuBackend(p, rlk, None, rk)
    bo = OracleBackend(P, ko.rlk, None, rko)
    got = be.rotate_hoisted_ext(ct, steps)
    want = bo.rotate_hoisted_ext(cto, steps)
    be.permuted_keys = False                 # reference-form keys: the same residues
    for g, r in zip(got, be.rotate_hoisted_ext(ct, steps)):
        assert torch.equal(g.data, r.data)
    be.permuted_keys = True
    for g, w in zip(got, want):
        assert np.array_equal(g.data[0].cpu().numpy().view(np.uint32), w.b.rows.astype(np.uint32))
        assert np.array_equal(g.data[1].cpu().numpy().view(np.uint32), w.a.rows.astype(np.uint32))
    # extended diagonals, one ModDown per group, giant rotation: the BSGS composition
    rng = np.random.default_rng(4)
    diag = [rng.uniform(-1, 1, p.n) + 1j * rng.uniform(-1, 1, p.n) for _ in steps]
    S = Fraction(p.rns_basis[ct.level])
    pts = [be.encode_slots(d, ct.level, S, ext=True) for d in diag]
    pto = [bo.encode_slots(d, cto.level, S, ext=True) for d in diag]
    groups = [(0, list(zip(got[:2], pts[:2]))), (3, list(zip(got[2:], pts[2:])))]
    groups_o = [(0, list(zip(want[:2], pto[:2]))), (3, list(zip(want[2:], pto[2:])))]
    g = be.bsgs_combine_ext(groups)
    w = bo.bsgs_combine_ext(groups_o)
    assert g.scale == w.scale
    assert np.array_equal(g.b.numpy(), w.b.rows) and np.array_equal(g.a.numpy(), w.a.rows)
    # fused baby rotations + giant sums (lf_bsgs_ext) == hoisted_ext + ptmac_rows composition
    ext_map = {0: be.extend(ct), **dict(zip(steps, got))}
    gspec = [(0, [(0, pts[0]), (1, pts[1])]), (3, [(3, pts[1]), (7, pts[2]), (0, pts[2])])]
    fz = be.bsgs_fused_ext(ct, gspec)
    un = be.bsgs_combine_ext([(sh, [(ext_map[b], pt) for b, pt in prs]) for sh, prs in gspec])
    assert fz.scale == un.scale
    assert torch.equal(fz.b.limbs, un.b.limbs) and torch.equal(fz.a.limbs, un.a.limbs)
    # and P*ct extends exactly: mod_down(P*ct) == ct
    e = be.extend(ct)
    from paper_2512_11269_b200 import fused  # noqa: F401
    import torch
    from paper_2512_11269_b200 import _native
    from paper_2512_11269_b200.context import dptr, get_context, stream_handle
    ctx = get_context(p)
    out = torch.empty((1, 2, ct.level + 1, p.N), dtype=torch.int32, device="cuda")
    ws = torch.empty(_native.lib().lf_moddown_workspace_bytes(ctx.handle, ct.level, 1) // 4,
                     dtype=torch.int32, device="cuda")
    _native.check(_native.lib().lf_moddown_ext(ctx.handle, ct.level, dptr(e.data), e.data.numel(), dptr(out),
                                               out[0].numel(), 1, dptr(ws), stream_handle()), "moddown")
    assert torch.equal(out[0, 0], ct.b.limbs) and torch.equal(out[0, 1], ct.a.limbs)


@pytest.mark.parametrize("cfg", ["desk", "c2"])
def test_rotate_batch_equals_separate_rotations(env, cfg):
    B = env[0]
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.ntt_host import galois_element
    kw = DESK if cfg == "desk" else dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26)
    p = B.gen_params(**kw)
    sk, pk, rlk = B.keygen(p, seed=3)
    steps = [1, 5, 2]
    rk = {s: B.make_rotation_key(p, sk, s, np.random.default_rng(20 + s)) for s in steps}
    level = p.max_level - 1
    cts = [B.encrypt(B.encode(np.random.default_rng(i).uniform(-1, 1, p.n), p, level=level), pk, p,
                     np.random.default_rng(50 + i)) for i in range(3)]
    blk = torch.stack([torch.stack([c.b.limbs, c.a.limbs]) for c in cts])
    gs = [galois_element(p.N, s) for s in steps]
    out = fused.rotate_batch(p, level, blk, gs, [rk[s] for s in steps])
    for i, (c, s) in enumerate(zip(cts, steps)):
        want = B.hom_rotate(c, s, rk[s], p)
        assert torch.equal(out[i, 0], want.b.limbs) and torch.equal(out[i, 1], want.a.limbs)
    # permuted-key form (lf_rotate_batch_pk): bit-identical
    from types import SimpleNamespace
    pks = [SimpleNamespace(data=fused.permute_rotation_key(p, rk[s], g)) for s, g in zip(steps, gs)]
    assert torch.equal(fused.rotate_batch(p, level, blk, gs, pks, permuted=True), out)


def test_ptmac_and_lincomb_equal_unfused(env):
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    import torch
    from paper_2512_11269_b200 import bootstrap as BT
    be = BT.GpuBackend(p, rlk, None, rk)
    rng = np.random.default_rng(8)
    cts = [B.encrypt(B.encode(rng.uniform(-1, 1, p.n), p), B.keygen(p, seed=11)[1], p,
                     np.random.default_rng(60 + i)) for i in range(3)]
    pts = [B.encode(rng.uniform(-1, 1, p.n), p) for _ in range(3)]
    got = be.mul_plain_sum(list(zip(cts, pts)))
    want = B.mul_plain(cts[0], pts[0], p)
    for c, t in zip(cts[1:], pts[1:]):
        want = B.hom_add(want, B.mul_plain(c, t, p), p)
    assert torch.equal(got.b.limbs, want.b.limbs) and torch.equal(got.a.limbs, want.a.limbs)
    terms = [(c, float(x), Fraction(2 ** 20)) for c, x in zip(cts, (0.5, -1.25, 3.0))]
    lc = be.lincomb(terms)
    acc = None
    for c, x, S in terms:
        m = be.mul_const(c, x, S)
        acc = m if acc is None else B.hom_add(acc, m, p)
    assert lc.scale == acc.scale
    assert torch.equal(lc.b.limbs, acc.b.limbs) and torch.equal(lc.a.limbs, acc.a.limbs)


def test_pitched_views_equal_dense(env):
    """lf_hom_mul_rescale_p / lf_rescale_multi_p on level-dropped row-prefix views of a batch
    (no copy) give the residues of the same calls on contiguous copies."""
    import torch
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    from paper_2512_11269_b200 import bootstrap as BT
    be = BT.GpuBackend(p, rlk, None, rk)
    ct2 = B.encrypt(B.encode(np.random.default_rng(3).uniform(-1, 1, p.n), p), B.keygen(p, seed=11)[1], p,
                    np.random.default_rng(4))
    x = be.stack([ct, ct2])
    y = be.stack([ct2, ct])
    lv = p.max_level - 2
    xv, yv = be.drop_to_level(x, lv), be.drop_to_level(y, lv)
    assert not xv.data.is_contiguous() and xv.pitched() is not None
    xd, yd = BT.CtBatch(xv.data.contiguous(), xv.scale, lv), BT.CtBatch(yv.data.contiguous(), yv.scale, lv)
    got, want = be.mul_rescale2(xv, yv), be.mul_rescale2(xd, yd)
    assert torch.equal(got.data, want.data) and got.level == want.level == lv - 2
    got, want = be.rescale2(xv), be.rescale2(xd)
    assert torch.equal(got.data, want.data)
    # operands with different pitches (views of blocks at two levels)
    z = be.rescale2(y)                                   # level L - 2, pitch L - 1
    lw = z.level - 2
    xw, zw = be.drop_to_level(x, lw), be.drop_to_level(z, lw)
    assert xw.pitched()[1] != zw.pitched()[1]
    got = be.mul_rescale2(xw, zw)
    want = be.mul_rescale2(BT.CtBatch(xw.data.contiguous(), xw.scale, lw), BT.CtBatch(zw.data.contiguous(), zw.scale, lw))
    assert torch.equal(got.data, want.data)
    # a batch of single ciphertexts through the same pitched entry point equals the unbatched op
    one = be.mul_rescale2(be.drop_to_level(ct, lv), be.drop_to_level(ct2, lv))
    assert np.array_equal(one.b.numpy(), be.mul_rescale2(xd, yd).data[0, 0].cpu().numpy())


def test_mul_rescale_list_equals_pairs(env):
    """lf_hom_mul_rescale_list over operand pairs of different blocks, pitches and batch sizes
    (with and without an epilogue constant) equals the pairs one at a time (+ add_const)."""
    import torch
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    from fractions import Fraction
    from paper_2512_11269_b200 import bootstrap as BT
    be = BT.GpuBackend(p, rlk, None, rk)
    pk = B.keygen(p, seed=11)[1]
    cts = [B.encrypt(B.encode(np.random.default_rng(i).uniform(-1, 1, p.n), p), pk, p, np.random.default_rng(10 + i))
           for i in range(4)]
    hi = be.stack(cts[:2])                                # level L block
    lo = be.rescale2(be.stack(cts[2:]))                   # level L - 2 block, other pitch
    lv = lo.level - 1
    x1, y1 = be.drop_to_level(hi, lv), be.drop_to_level(lo, lv)
    x2, y2 = be.drop_to_level(lo, lv), be.drop_to_level(lo, lv)
    single = (be.drop_to_level(cts[0], lv), be.drop_to_level(cts[3], lv))
    pairs = [(x1, y1), (x2, y2)]
    K = -12345678901
    got = be.mul_rescale2_many(pairs, [None, K])
    want0 = be.mul_rescale2(x1, y1)
    want1 = be.add_const(be.mul_rescale2(x2, y2), Fraction(K) / Fraction(be.mul_rescale2(x2, y2).scale))
    assert torch.equal(got[0].data, want0.data) and torch.equal(got[1].data, want1.data)
    g1 = be.mul_rescale2_many([single])[0]
    w1 = be.mul_rescale2(*single)
    assert np.array_equal(g1.b.numpy(), w1.b.numpy()) and np.array_equal(g1.a.numpy(), w1.a.numpy())


def test_moddown_ext_rescale_equals_moddown_then_rescales(env):
    """lf_moddown_ext_rescale (ModDown and nd rescales as one division) equals lf_moddown_ext
    followed by nd rescales, residue for residue, on hoisted extended-basis rotations."""
    import torch
    B, O, p, P, sk, rlk, ko, rk, rko, steps, ct, cto = env
    from paper_2512_11269_b200 import _native
    from paper_2512_11269_b200 import bootstrap as BT
    from paper_2512_11269_b200.context import dptr, get_context, stream_handle
    be = BT.GpuBackend(p, rlk, None, rk)
    ext = be.rotate_hoisted_ext(ct, steps)                        # ExtCt, data (2, ext, N)
    inner = torch.stack([e.data for e in ext])
    G, level, N = inner.shape[0], ext[0].level, p.N
    ctx = get_context(p)
    lib = _native.lib()
    ws = torch.empty(lib.lf_moddown_workspace_bytes(ctx.handle, level, G) // 4, dtype=torch.int32, device="cuda")
    plain = torch.empty((G, 2, level + 1, N), dtype=torch.int32, device="cuda")
    _native.check(lib.lf_moddown_ext(ctx.handle, level, dptr(inner), inner[0].numel(), dptr(plain),
                                     plain[0].numel(), G, dptr(ws), stream_handle()), "lf_moddown_ext")
    for nd in (1, 2):
        fused = torch.empty((G, 2, level + 1 - nd, N), dtype=torch.int32, device="cuda")
        _native.check(lib.lf_moddown_ext_rescale(ctx.handle, level, nd, dptr(inner), inner[0].numel(), dptr(fused),
                                                 fused[0].numel(), G, dptr(ws), stream_handle()),
                      "lf_moddown_ext_rescale")
        want = BT.CtBatch(plain, 1, level)
        want = be.rescale2(want) if nd == 2 else BT.CtBatch(torch.stack(
            [torch.stack([c.b.limbs, c.a.limbs]) for c in (be.rescale(x) for x in be.unstack(want))]), 1, level - 1)
        assert torch.equal(fused, want.data)
