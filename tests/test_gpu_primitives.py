"""GPU parity of the row primitives against the reference golden vectors and the oracle."""

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


def _params(B, golden_params, name):
    return B.gen_params(**golden_params[name]["kwargs"])


@pytest.mark.parametrize("name", ["p16", "n32", "n64", "small", "n1024", "desk"])
def test_ntt_fwd_inv_match_reference(B, golden_params, name):
    from paper_2512_11269_b200 import poly as P
    z = load_npz("ntt.npz")
    p = _params(B, golden_params, name)
    allp = p.rns_basis + p.special_basis
    ids = P.extended_ids(p, p.max_level)
    for k, bid in enumerate(ids):
        x = z[f"{name}_{k}_x"]
        for inv, key in ((False, "fwd"), (True, "inv")):
            t = P.to_device(x)
            P.ntt_rows(p, t, (bid, bid), inverse=inv)
            got = P.to_host(t)
            assert np.array_equal(got, z[f"{name}_{k}_{key}"]), (name, k, key)
    # batched: all primes at once, forward then inverse round trip
    rows = np.stack([z[f"{name}_{k}_x"][0] for k in range(len(allp))])
    t = P.to_device(rows)
    P.ntt_rows(p, t, ids)
    assert np.array_equal(P.to_host(t), np.stack([z[f"{name}_{k}_fwd"][0] for k in range(len(allp))]))
    P.ntt_rows(p, t, ids, inverse=True)
    assert np.array_equal(P.to_host(t), rows)


def test_ntt_big_digests(B, golden_params):
    from paper_2512_11269_b200 import poly as P
    meta = load_json("ntt_big.json")
    p = _params(B, golden_params, "c2")
    ids = P.extended_ids(p, p.max_level)
    for key, m in meta.items():
        k = int(key.split("_")[1])
        q = m["q"]
        x = np.random.default_rng(100 + k).integers(0, q, p.N, dtype=np.uint64)
        t = P.to_device(x[None])
        P.ntt_rows(p, t, (ids[k],))
        assert digest(P.to_host(t)) == m["fwd"], key
        t = P.to_device(x[None])
        P.ntt_rows(p, t, (ids[k],), inverse=True)
        assert digest(P.to_host(t)) == m["inv"], key


def test_ewise_ops_match_oracle(B, golden_params):
    from oracle import lf_oracle as O
    from paper_2512_11269_b200 import poly as P
    p = _params(B, golden_params, "desk")
    ids = P.extended_ids(p, p.max_level)
    qs = np.array([P.prime_for_id(p, b) for b in ids], dtype=np.uint64)[:, None]
    rng = np.random.default_rng(3)
    a = (rng.integers(0, 2**62, (len(ids), p.N), dtype=np.uint64) % qs)
    b = (rng.integers(0, 2**62, (len(ids), p.N), dtype=np.uint64) % qs)
    c = (rng.integers(0, 2**62, (len(ids), p.N), dtype=np.uint64) % qs)
    a[:, :4] = 0
    b[:, 4:8] = qs - 1
    da, db, dc = P.to_device(a), P.to_device(b), P.to_device(c)
    sc = [int(x) for x in rng.integers(0, 2**40, len(ids))]
    scq = np.array([s % int(q) for s, q in zip(sc, qs[:, 0])], dtype=np.uint64)[:, None]
    want = {
        P.LF_OP_ADD: (a + b) % qs, P.LF_OP_SUB: (a + qs - b) % qs, P.LF_OP_MUL: a * b % qs,
        P.LF_OP_NEG: (qs - a) % qs, P.LF_OP_SCALAR_MUL: a * scq % qs,
        P.LF_OP_MULACC: (c + a * b) % qs, P.LF_OP_MODSTEP: (a + qs - b) % qs * scq % qs,
        P.LF_OP_MUL_SCALAR_ADD: (a * scq % qs + b) % qs,
    }
    for op, w in want.items():
        out = da.clone()
        P.ewise(p, op, out, da, ids, b=db, c=dc, scalars=sc)
        assert np.array_equal(P.to_host(out), w), op


def test_automorph_matches_reference_perm(B, golden_params):
    from paper_2512_11269_b200 import poly as P
    z = load_npz("ntt.npz")
    for name, N in (("p16", 16), ("small", 256), ("desk", 4096)):
        p = _params(B, golden_params, name)
        x = np.random.default_rng(9).integers(0, p.rns_basis[0], (3, N), dtype=np.uint64)
        for key in ("1", "3", "7", "conj"):
            perm = z[f"perm_{N}_{key}"]
            g = 2 * N - 1 if key == "conj" else pow(5, int(key), 2 * N)
            out = P.to_device(np.zeros_like(x))
            P.automorph_rows(p, out, P.to_device(x), g)
            assert np.array_equal(P.to_host(out), x[:, perm]), (name, key)


def test_bconv_matches_reference(B, golden_params):
    from paper_2512_11269_b200 import poly as P
    z = load_npz("bconv.npz")
    p = _params(B, golden_params, "p16")
    for case in ("rand", "c42", "qm1", "zero"):
        src = P.RnsPolynomial(P.to_device(z[f"{case}_in"]), P.Domain.COEFF, P.main_ids(2))
        out = P.base_convert(src, P.special_ids(p), p)
        assert np.array_equal(out.numpy(), z[f"{case}_out"]), case
    ps = _params(B, golden_params, "small")
    src = P.RnsPolynomial(P.to_device(z["small_in"]), P.Domain.COEFF, (0, 3))
    out = P.base_convert(src, (1, 2, 4) + P.special_ids(ps), ps)
    assert np.array_equal(out.numpy(), z["small_out"])


def test_mod_down_matches_oracle(B, golden_params):
    from oracle import lf_oracle as O
    from paper_2512_11269_b200 import poly as P
    for name in ("small", "desk"):
        p = _params(B, golden_params, name)
        po = O.gen_params(**golden_params[name]["kwargs"])
        ids = P.extended_ids(p, 3)
        qs = np.array([P.prime_for_id(p, b) for b in ids], dtype=np.uint64)[:, None]
        x = np.random.default_rng(5).integers(0, 2**62, (len(ids), p.N), dtype=np.uint64) % qs
        want = O.mod_down(po, O.Poly(x, ids, True), P.main_ids(3))
        got = P.mod_down(P.RnsPolynomial(P.to_device(x), P.Domain.EVAL, ids), P.main_ids(3), p)
        assert np.array_equal(got.numpy(), want.rows), name
        # rescale of a main-basis poly
        xm = x[:4]
        want = O.rescale_poly(po, O.Poly(xm, P.main_ids(3), True))
        got = P.rescale_poly(P.RnsPolynomial(P.to_device(xm), P.Domain.EVAL, P.main_ids(3)), p)
        assert np.array_equal(got.numpy(), want.rows), name
