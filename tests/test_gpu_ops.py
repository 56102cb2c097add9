"""GPU parity of the operator API (fused sm_100a pipeline) against the reference golden
vectors (tests/golden/, produced by the real limbforge) and the CPU oracle."""

from fractions import Fraction

import numpy as np
import pytest

from conftest import digest, load_json, load_npz

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    return B


def _pack(ct):
    return np.stack([ct.b.numpy(), ct.a.numpy()])


def _ctx(B, p):
    from paper_2512_11269_b200 import keys as K
    sk, pk, rlk = B.keygen(p, seed=11)
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct_v = B.encrypt(B.encode(v, p), pk, p, rng)
    ct_w = B.encrypt(B.encode(w, p), pk, p, rng)
    rk1 = B.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    rk3 = B.make_rotation_key(p, sk, 3, np.random.default_rng(6))
    rkc = B.make_conjugation_key(p, sk, np.random.default_rng(8))
    return sk, pk, rlk, v, w, ct_v, ct_w, rk1, rk3, rkc


@pytest.mark.parametrize("name", ["small", "desk"])
def test_ops_match_reference(B, golden_params, name):
    p = B.gen_params(**golden_params[name]["kwargs"])
    meta = load_json(f"ops_{name}.json")
    z = load_npz(f"ops_{name}.npz")
    sk, pk, rlk, v, w, ct_v, ct_w, rk1, rk3, rkc = _ctx(B, p)
    kd = meta["keys"]
    assert digest(sk.s_eval.numpy()) == kd["sk_eval"]
    assert digest(pk.b.numpy()) == kd["pk_b"] and digest(pk.a.numpy()) == kd["pk_a"]
    assert [[digest(b.numpy()), digest(a.numpy())] for b, a in rlk.digits] == kd["rlk"]
    assert [[digest(b.numpy()), digest(a.numpy())] for b, a in rk1.digits] == meta["rk1"]
    assert [[digest(b.numpy()), digest(a.numpy())] for b, a in rkc.digits] == meta["rkc"]
    pt_w = B.encode(w, p)
    mul = B.hom_mul(ct_v, ct_w, rlk, p)
    low = B.encrypt(B.encode(v, p, level=2), pk, p, np.random.default_rng(2))
    res = {
        "ct_v": ct_v, "ct_w": ct_w,
        "add": B.hom_add(ct_v, ct_w, p), "sub": B.hom_sub(ct_v, ct_w, p),
        "mul_plain": B.mul_plain(ct_v, pt_w, p), "add_plain": B.add_plain(ct_v, pt_w, p),
        "mul": mul, "mul_rescale": B.rescale(mul, p),
        "rot1": B.hom_rotate(ct_v, 1, rk1, p), "rot3": B.hom_rotate(ct_v, 3, rk3, p),
        "rescale_v": B.rescale(ct_v, p), "conj": B.hom_conjugate(ct_v, rkc, p),
        "low": low, "low_mul_rescale": B.rescale(B.hom_mul(low, low, rlk, p), p),
        "low_rot1": B.hom_rotate(low, 1, rk1, p),
    }
    for k, ct in res.items():
        m = meta["cts"][k]
        assert ct.level == m["level"], k
        assert ct.scale == Fraction(*m["scale"]), k
        got = _pack(ct)
        if k in z.files:
            assert np.array_equal(got, z[k]), k
        assert digest(got) == m["digest"], k
    pieces = B.keyswitch_decompose(ct_v.a, p)
    assert [[j, digest(d.numpy())] for j, d in pieces] == meta["pieces"]
    kb, ka = B.keyswitch(ct_v.a, rlk, p)
    assert [digest(kb.numpy()), digest(ka.numpy())] == meta["ks"]
    dec = B.decrypt(res["mul_rescale"], sk, p)
    assert np.abs(dec - v * w).max() < 0.05
    assert np.abs(dec - z["dec_mul_rescale"]).max() < 1e-6
    dec = B.decrypt(res["rot1"], sk, p)
    assert np.abs(dec - np.roll(v, -1)).max() < 0.05


def test_fused_equals_unfused(B, golden_params):
    from paper_2512_11269_b200 import ckks as C
    p = B.gen_params(**golden_params["desk"]["kwargs"])
    sk, pk, rlk, v, w, ct_v, ct_w, rk1, rk3, rkc = _ctx(B, p)
    for level in (6, 4, 1):
        ct = B.encrypt(B.encode(v, p, level=level), pk, p, np.random.default_rng(level))
        fb, fa = B.keyswitch(ct.a, rlk, p)
        ub, ua = C.keyswitch_unfused(ct.a, rlk, p)
        assert np.array_equal(fb.numpy(), ub.numpy()) and np.array_equal(fa.numpy(), ua.numpy())
        r1 = B.hom_rotate(ct, 1, rk1, p)
        r2 = C.hom_rotate_unfused(ct, 1, rk1, p)
        assert np.array_equal(_pack(r1), _pack(r2)), level
        pf = B.keyswitch_decompose(ct.a, p)
        pu = C.keyswitch_decompose_unfused(ct.a, p)
        for (j1, d1), (j2, d2) in zip(pf, pu):
            assert j1 == j2 and np.array_equal(d1.numpy(), d2.numpy())


def test_small_rings_against_oracle(B, golden_params):
    """p16 (d=1, N=16) and n64 through every fused op, checked against the oracle."""
    from oracle import lf_oracle as O
    for name in ("p16", "n64", "n1024"):
        kw = dict(golden_params[name]["kwargs"])
        kw["hamming_weight"] = min(64, kw["N"] // 4)
        p, po = B.gen_params(**kw), O.gen_params(**kw)
        sk, pk, rlk = B.keygen(p, seed=5)
        ko = O.keygen(po, seed=5)
        assert np.array_equal(rlk.data[0, 0].cpu().numpy().view(np.uint32), ko.rlk.digits[0][0].rows)
        rng = np.random.default_rng(1)
        L = p.max_level
        ids = tuple(range(L + 1))
        qs = np.array(p.rns_basis, dtype=np.uint64)[:, None]
        b = rng.integers(0, 2**62, (L + 1, p.N), dtype=np.uint64) % qs
        a = rng.integers(0, 2**62, (L + 1, p.N), dtype=np.uint64) % qs
        ct = B.Ciphertext(B.RnsPolynomial(b, B.Domain.EVAL, ids), B.RnsPolynomial(a, B.Domain.EVAL, ids),
                          p.scale, L)
        cto = O.Ct(O.Poly(b, ids), O.Poly(a, ids), po.scale, L)
        m = B.hom_mul(ct, ct, rlk, p)
        mo = O.hom_mul(po, cto, cto, ko.rlk)
        assert np.array_equal(_pack(m), np.stack([mo.b.rows, mo.a.rows])), name
        r = B.rescale(ct, p)
        ro = O.rescale(po, cto)
        assert np.array_equal(_pack(r), np.stack([ro.b.rows, ro.a.rows])), name
        rk = B.make_rotation_key(p, sk, 1, np.random.default_rng(3))
        rko = O.rotation_key(po, ko, 1, np.random.default_rng(3))
        x = B.hom_rotate(ct, 1, rk, p)
        xo = O.hom_rotate(po, cto, 1, rko)
        assert np.array_equal(_pack(x), np.stack([xo.b.rows, xo.a.rows])), name


def test_error_paths(B, golden_params):
    from paper_2512_11269_b200 import errors as E
    p = B.gen_params(**golden_params["small"]["kwargs"])
    sk, pk, rlk = B.keygen(p, seed=11)
    v = np.random.default_rng(0).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p), pk, p, np.random.default_rng(1))
    low = B.encrypt(B.encode(v, p, level=1), pk, p, np.random.default_rng(2))
    with pytest.raises(E.LevelMismatch):
        B.hom_add(ct, low, p)
    other = B.encrypt(B.encode(v, p, scale=1 << 21), pk, p, np.random.default_rng(2))
    with pytest.raises(E.ScaleMismatch):
        B.hom_add(ct, other, p)
    ct0 = B.encrypt(B.encode(v, p, level=0), pk, p, np.random.default_rng(3))
    with pytest.raises(E.LevelExhausted):
        B.hom_mul(ct0, ct0, rlk, p)
    with pytest.raises(E.LevelExhausted):
        B.rescale(ct0, p)
    with pytest.raises(E.MissingEvalKey):
        B.hom_mul(ct, ct, None, p)
    with pytest.raises(E.MissingEvalKey):
        B.hom_rotate(ct, 1, rlk, p)
    with pytest.raises(ValueError):
        B.make_rotation_key(p, sk, 0, np.random.default_rng(0))
    assert B.hom_rotate(ct, p.n, None, p) is ct
    # C-ABI argument checks of the fused entry points fail loudly (no silent fallback)
    from paper_2512_11269_b200 import _native, fused
    with pytest.raises(_native.NativeError, match="lf_hom_mul_rescale"):
        fused.hom_mul_rescale(p, ct0, ct0, rlk, 1)           # level 0 cannot drop a prime
    with pytest.raises(_native.NativeError, match="lf_hom_mul_rescale"):
        fused.hom_mul_rescale(p, ct, ct, rlk, 3)             # ndrop outside {1, 2}
    lib = _native.lib()
    from paper_2512_11269_b200.context import get_context
    import ctypes
    rc = lib.lf_bsgs_ext(get_context(p).handle, ct.level, None, 0, None, None, 0, None, None, None, None)
    assert rc != 0 and b"lf_bsgs_ext" in lib.lf_last_error()


@pytest.mark.parametrize("level", [35, 20])
def test_c2_matches_reference(B, golden_params, level):
    """N=2^16, L=35, d=4 (C2) keyswitch / rotate / hom_mul / rescale digests."""
    p = B.gen_params(**golden_params["c2"]["kwargs"])
    meta = load_json("c2.json")
    sk, pk, rlk = B.keygen(p, seed=11)
    assert [[digest(b.numpy()), digest(a.numpy())] for b, a in rlk.digits] == meta["keys"]["rlk"]
    rk1 = B.make_rotation_key(p, sk, 1, np.random.default_rng(99))
    assert [[digest(b.numpy()), digest(a.numpy())] for b, a in rk1.digits] == meta["rk1"]
    ids = tuple(range(level + 1))

    def synth(seed):
        rng = np.random.default_rng(seed)
        return np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in ids])

    E = B.Domain.EVAL
    ct1 = B.Ciphertext(B.RnsPolynomial(synth(1000), E, ids), B.RnsPolynomial(synth(1001), E, ids), p.scale, level)
    ct2 = B.Ciphertext(B.RnsPolynomial(synth(1002), E, ids), B.RnsPolynomial(synth(1003), E, ids), p.scale, level)
    m = meta["levels"][str(level)]
    kb, ka = B.keyswitch(ct1.a, rlk, p)
    assert [digest(kb.numpy()), digest(ka.numpy())] == m["ks"]
    assert digest(_pack(B.hom_rotate(ct1, 1, rk1, p))) == m["rot1"]
    assert digest(_pack(B.hom_mul(ct1, ct2, rlk, p))) == m["mul"]
    assert digest(_pack(B.rescale(ct1, p))) == m["rescale"]


@pytest.mark.parametrize("name", ["desk", "n1024"])
def test_hoisted_rotations_bit_identical(B, golden_params, name):
    """One shared ModUp for several rotations == separate hom_rotate calls (the reference's
    hoisting contract, tests/test_polyir.py:257-265), including conjugation."""
    kw = dict(golden_params[name]["kwargs"])
    p = B.gen_params(**kw)
    sk, pk, rlk = B.keygen(p, seed=3)
    steps = [1, 2, 5, p.n - 1, 0, 7]
    keys = {s: B.make_rotation_key(p, sk, s, np.random.default_rng(10 + s)) for s in steps if s % p.n}
    v = np.random.default_rng(4).uniform(-1, 1, p.n)
    for level in (p.max_level, 2):
        ct = B.encrypt(B.encode(v, p, level=level), pk, p, np.random.default_rng(level))
        got = B.hom_rotate_hoisted(ct, steps, keys, p)
        for s, g in zip(steps, got):
            want = B.hom_rotate(ct, s, keys.get(s % p.n), p)
            assert np.array_equal(_pack(g), _pack(want)), (level, s)
    dec = B.decrypt(got[0], sk, p)
    assert np.abs(dec - np.roll(v, -1)).max() < 0.05


def test_batched_keyswitch_matches_single(B, golden_params):
    from paper_2512_11269_b200 import fused
    p = B.gen_params(**golden_params["desk"]["kwargs"])
    sk, pk, rlk = B.keygen(p, seed=3)
    import torch
    l1 = p.max_level + 1
    q = torch.tensor(p.rns_basis, dtype=torch.int64, device="cuda")[:, None]
    xs = (torch.randint(0, 2 ** 62, (70, l1, p.N), device="cuda", dtype=torch.int64) % q).to(torch.int32)
    out = fused.keyswitch_batch(p, p.max_level, xs, rlk)      # > LF_MAXB: chunked
    for i in (0, 37, 69):
        kb, ka = B.keyswitch(B.RnsPolynomial(xs[i], B.Domain.EVAL, tuple(range(l1))), rlk, p)
        assert np.array_equal(out[i, 0].cpu().numpy(), kb.limbs.cpu().numpy())
        assert np.array_equal(out[i, 1].cpu().numpy(), ka.limbs.cpu().numpy())


@pytest.mark.parametrize("name", ["desk", "c2"])
def test_double_rescale_equals_two_rescales(B, golden_params, name):
    """lf_rescale_multi(ndrop=2) == rescale(rescale(ct)) bit for bit (floor(floor(X/a)/b) =
    floor(X/ab)); used by the bootstrap's double-prime levels."""
    from paper_2512_11269_b200 import fused
    p = B.gen_params(**golden_params[name]["kwargs"])
    sk, pk, rlk = B.keygen(p, seed=3)
    for level in (p.max_level, 2):
        ids = tuple(range(level + 1))
        rng = np.random.default_rng(level)
        rows = lambda: np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in ids])
        E = B.Domain.EVAL
        ct = B.Ciphertext(B.RnsPolynomial(rows(), E, ids), B.RnsPolynomial(rows(), E, ids), p.scale, level)
        want = B.rescale(B.rescale(ct, p), p)
        b, a = fused.rescale_multi(p, ct, 2)
        assert np.array_equal(b.numpy(), want.b.numpy()) and np.array_equal(a.numpy(), want.a.numpy())


@pytest.mark.parametrize("name", ["small", "desk"])
def test_mul_rescale_fused_matches_reference(B, golden_params, name):
    """lf_hom_mul_rescale(ndrop=1) == the reference's rescale(hom_mul(.)) golden vectors."""
    from paper_2512_11269_b200 import fused
    p = B.gen_params(**golden_params[name]["kwargs"])
    meta = load_json(f"ops_{name}.json")
    sk, pk, rlk, v, w, ct_v, ct_w, rk1, rk3, rkc = _ctx(B, p)
    low = B.encrypt(B.encode(v, p, level=2), pk, p, np.random.default_rng(2))
    for key, (x, y) in {"mul_rescale": (ct_v, ct_w), "low_mul_rescale": (low, low)}.items():
        b, a = fused.hom_mul_rescale(p, x, y, rlk, 1)
        assert digest(np.stack([b.numpy(), a.numpy()])) == meta["cts"][key]["digest"], key


@pytest.mark.parametrize("name", ["desk", "c2"])
def test_mul_rescale_fused_equals_composition(B, golden_params, name):
    """ndrop 1 and 2 on full-range random ciphertexts (every residue, so the floor divisions'
    carries are exercised): equal to hom_mul then ndrop rescales, single and batched."""
    import torch
    from paper_2512_11269_b200 import fused
    from paper_2512_11269_b200.bootstrap import CtBatch, GpuBackend
    p = B.gen_params(**golden_params[name]["kwargs"])
    sk, pk, rlk = B.keygen(p, seed=3)
    E = B.Domain.EVAL
    for level in (p.max_level, 2):
        ids = tuple(range(level + 1))
        rng = np.random.default_rng(100 + level)
        rows = lambda: np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in ids])
        mk = lambda: B.Ciphertext(B.RnsPolynomial(rows(), E, ids), B.RnsPolynomial(rows(), E, ids),
                                  p.scale, level)
        x, y = mk(), mk()
        prod = B.hom_mul(x, y, rlk, p)
        for nd in (1, 2):
            want = prod
            for _ in range(nd):
                want = B.rescale(want, p)
            b, a = fused.hom_mul_rescale(p, x, y, rlk, nd)
            assert np.array_equal(b.numpy(), want.b.numpy()), (level, nd)
            assert np.array_equal(a.numpy(), want.a.numpy()), (level, nd)
        # batch of 3 through the bootstrap backend (one pipeline, shared relinearisation key)
        be = GpuBackend(p, rlk, None, {})
        xs, ys = [x, mk(), mk()], [y, mk(), mk()]
        out = be.mul_rescale2(be.stack(xs), be.stack(ys))
        for i in range(3):
            want = B.rescale(B.rescale(B.hom_mul(xs[i], ys[i], rlk, p), p), p)
            assert np.array_equal(out.data[i, 0].cpu().numpy().astype(np.uint64), want.b.numpy()), (level, i)
            assert np.array_equal(out.data[i, 1].cpu().numpy().astype(np.uint64), want.a.numpy()), (level, i)
        torch.cuda.synchronize()
