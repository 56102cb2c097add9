"""Pin the CPU oracle (oracle/lf_oracle.py) to the golden fixtures produced by the real
reference (tests/golden/make_golden.py).  CPU only."""

from fractions import Fraction

import numpy as np
import pytest

from conftest import digest, load_json, load_npz
from oracle import lf_oracle as O


def _params(golden_params, name):
    return O.gen_params(**golden_params[name]["kwargs"])


@pytest.mark.parametrize("name", ["p16", "small", "desk", "c2", "c2b", "n1024", "n64", "n32"])
def test_params_match_reference(golden_params, name):
    p = _params(golden_params, name)
    g = golden_params[name]["params"]
    assert list(p.main) == g["main"]
    assert list(p.special) == g["special"]
    assert p.d == g["d"]


@pytest.mark.parametrize("name", ["p16", "n32", "n64", "small", "n1024", "desk"])
def test_ntt_matches_reference(golden_params, name):
    z = load_npz("ntt.npz")
    p = _params(golden_params, name)
    for k, q in enumerate(p.main + p.special):
        x = z[f"{name}_{k}_x"].astype(np.uint64)
        assert int(z[f"{name}_{k}_psi"][0]) == O.root_2n(p.N, q)
        assert np.array_equal(O.ntt_fwd(x, q), z[f"{name}_{k}_fwd"])
        assert np.array_equal(O.ntt_inv(x, q), z[f"{name}_{k}_inv"])
        assert np.array_equal(O.ntt_inv(O.ntt_fwd(x, q), q), x)


def test_ntt_big_digests(golden_params):
    meta = load_json("ntt_big.json")
    p = _params(golden_params, "c2")
    allp = p.main + p.special
    for key, m in meta.items():
        k = int(key.split("_")[1])
        q = allp[k]
        assert q == m["q"] and O.root_2n(p.N, q) == m["psi"]
        x = np.random.default_rng(100 + k).integers(0, q, p.N, dtype=np.uint64)
        assert digest(O.ntt_fwd(x, q)) == m["fwd"]
        assert digest(O.ntt_inv(x, q)) == m["inv"]


def test_automorphism_perms():
    z = load_npz("ntt.npz")
    for N in (16, 256, 4096):
        for steps in (1, 3, 7):
            g = O.galois_element(N, steps)
            assert np.array_equal(O.automorphism_perm(N, g), z[f"perm_{N}_{steps}"])
        assert np.array_equal(O.automorphism_perm(N, 2 * N - 1), z[f"perm_{N}_conj"])


def test_bconv_cases(golden_params):
    z = load_npz("bconv.npz")
    p = _params(golden_params, "p16")
    for case in ("rand", "c42", "qm1", "zero"):
        src = O.Poly(z[f"{case}_in"].astype(np.uint64), p.main_ids(2), False)
        out = O.base_convert(p, src, p.special_ids())
        assert np.array_equal(out.rows, z[f"{case}_out"]), case
    ps = _params(golden_params, "small")
    src = O.Poly(z["small_in"].astype(np.uint64), (0, 3), False)
    out = O.base_convert(ps, src, (1, 2, 4) + ps.special_ids())
    assert np.array_equal(out.rows, z["small_out"])


def _ops_ctx(p):
    keys = O.keygen(p, seed=11)
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct_v = O.encrypt(O.encode(v, p), keys, p, rng)
    ct_w = O.encrypt(O.encode(w, p), keys, p, rng)
    rk1 = O.rotation_key(p, keys, 1, np.random.default_rng(5))
    rk3 = O.rotation_key(p, keys, 3, np.random.default_rng(6))
    rkc = O.conj_key(p, keys, np.random.default_rng(8))
    return keys, v, w, ct_v, ct_w, rk1, rk3, rkc


def _ops_results(p, keys, v, w, ct_v, ct_w, rk1, rk3, rkc):
    pt_w = O.encode(w, p)
    mul = O.hom_mul(p, ct_v, ct_w, keys.rlk)
    low = O.encrypt(O.encode(v, p, level=2), keys, p, np.random.default_rng(2))
    return {
        "ct_v": ct_v, "ct_w": ct_w,
        "add": O.hom_add(p, ct_v, ct_w), "sub": O.hom_sub(p, ct_v, ct_w),
        "mul_plain": O.mul_plain(p, ct_v, pt_w), "add_plain": O.add_plain(p, ct_v, pt_w),
        "mul": mul, "mul_rescale": O.rescale(p, mul),
        "rot1": O.hom_rotate(p, ct_v, 1, rk1), "rot3": O.hom_rotate(p, ct_v, 3, rk3),
        "rescale_v": O.rescale(p, ct_v),
        "conj": O.apply_galois(p, ct_v, 2 * p.N - 1, rkc),
        "low": low, "low_mul_rescale": O.rescale(p, O.hom_mul(p, low, low, keys.rlk)),
        "low_rot1": O.hom_rotate(p, low, 1, rk1),
    }


def _pack(ct):
    return np.stack([ct.b.rows, ct.a.rows])


@pytest.mark.parametrize("name", ["small", "desk"])
def test_ops_match_reference(golden_params, name):
    p = _params(golden_params, name)
    meta = load_json(f"ops_{name}.json")
    z = load_npz(f"ops_{name}.npz")
    keys, v, w, ct_v, ct_w, rk1, rk3, rkc = _ops_ctx(p)
    kd = meta["keys"]
    assert digest(keys.s_eval.rows) == kd["sk_eval"]
    assert digest(keys.pk[0].rows) == kd["pk_b"] and digest(keys.pk[1].rows) == kd["pk_a"]
    assert [[digest(b.rows), digest(a.rows)] for b, a in keys.rlk.digits] == kd["rlk"]
    assert [[digest(b.rows), digest(a.rows)] for b, a in rk1.digits] == meta["rk1"]
    assert [[digest(b.rows), digest(a.rows)] for b, a in rkc.digits] == meta["rkc"]
    assert np.array_equal(v, z["v"]) and np.array_equal(w, z["w"])
    res = _ops_results(p, keys, v, w, ct_v, ct_w, rk1, rk3, rkc)
    for k, ct in res.items():
        m = meta["cts"][k]
        assert ct.level == m["level"], k
        assert ct.scale == Fraction(*m["scale"]), k
        assert digest(_pack(ct)) == m["digest"], k
        if k in z.files:
            assert np.array_equal(_pack(ct), z[k]), k
    pieces = O.ks_decompose(p, ct_v.a)
    assert [[j, digest(d.rows)] for j, d in pieces] == meta["pieces"]
    kb, ka = O.keyswitch(p, ct_v.a, keys.rlk)
    assert [digest(kb.rows), digest(ka.rows)] == meta["ks"]
    # value level (reference TOL 0.05, test_ckks_ops.py:27)
    dec = O.decrypt(res["mul_rescale"], keys, p)
    assert np.abs(dec - z["dec_mul_rescale"]).max() < 1e-6
    assert np.abs(dec - v * w).max() < 0.05
    dec = O.decrypt(res["rot1"], keys, p)
    assert np.abs(dec - np.roll(v, -1)).max() < 0.05


@pytest.mark.slow
def test_c2_keyswitch_matches_reference(golden_params):
    """Full-level N=2^16 keyswitch (C2) against the reference digest."""
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, "c2.json")):
        pytest.skip("c2 fixture not generated")
    meta = load_json("c2.json")
    p = _params(golden_params, "c2")
    keys = O.keygen(p, seed=11)
    assert [[digest(b.rows), digest(a.rows)] for b, a in keys.rlk.digits] == meta["keys"]["rlk"]
    level = 35
    ids = p.main_ids(level)
    rng = np.random.default_rng(1001)
    a1 = np.stack([rng.integers(0, p.main[i], p.N, dtype=np.uint64) for i in ids])
    kb, ka = O.keyswitch(p, O.Poly(a1, ids, True), keys.rlk)
    assert [digest(kb.rows), digest(ka.rows)] == meta["levels"][str(level)]["ks"]
