"""CPU tests of the product's host-side logic (parameter synthesis, number theory, embedding,
sampling order, BConv table construction) against the reference golden fixtures and the
oracle.  No GPU needed."""

from fractions import Fraction

import numpy as np
import pytest

from conftest import load_npz
from oracle import lf_oracle as O


@pytest.mark.parametrize("name", ["p16", "small", "desk", "c2", "c2b", "n1024", "n64", "n32"])
def test_gen_params_matches_reference(golden_params, name):
    from paper_2512_11269_b200.params import gen_params
    p = gen_params(**golden_params[name]["kwargs"])
    g = golden_params[name]["params"]
    assert list(p.rns_basis) == g["main"] and list(p.special_basis) == g["special"]
    assert p.scale == Fraction(*g["scale"]) and p.ks.d == g["d"] and p.hamming_weight == g["h"]


def test_params_validation():
    from paper_2512_11269_b200.params import gen_params
    with pytest.raises(ValueError):
        gen_params(100, 3)
    with pytest.raises(ValueError):
        gen_params(8, 3)
    p = gen_params(256, 6, d=3)
    groups = p.ks.digits_at_level(6)
    assert sorted(sum(groups, [])) == list(range(7))
    assert len(p.ks.digits_at_level(2)) == 3


def test_psi_matches_reference():
    from paper_2512_11269_b200.modmath import primitive_root_of_unity
    z = load_npz("ntt.npz")
    p = O.gen_params(4096, 6, d=3, seed=0)
    for k, q in enumerate(p.main + p.special):
        assert primitive_root_of_unity(2 * p.N, q) == int(z[f"desk_{k}_psi"][0])


def test_embedding_roundtrip_and_oracle_agreement():
    from paper_2512_11269_b200.encoding import embed_forward, embed_inverse
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, 128)
    c = embed_inverse(v, 256)
    assert np.abs(embed_forward(c, 256).real - v).max() < 1e-12
    assert np.array_equal(c, O.embed_inverse(v, 256))


def test_automorphism_table_matches_reference():
    from paper_2512_11269_b200.ntt_host import automorphism_permutation, galois_element
    z = load_npz("ntt.npz")
    for N in (16, 256, 4096):
        for s in (1, 3, 7):
            assert np.array_equal(automorphism_permutation(N, galois_element(N, s)), z[f"perm_{N}_{s}"])


def test_sampling_order_matches_oracle():
    from paper_2512_11269_b200 import keys as K
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    assert np.array_equal(K.sample_ternary(r1, 256, 64), O.sample_ternary(r2, 256, 64))
    assert np.array_equal(K.sample_gaussian(r1, 256, 3.2), O.sample_gaussian(r2, 256, 3.2))


def test_bconv_blob_emulates_exact_conversion():
    """Evaluate the host-built table with the device algorithm (float64 fast path + exact
    decision) in numpy and compare with the oracle's exact conversion."""
    from paper_2512_11269_b200.context import bconv_blob, bconv_words
    p = O.gen_params(256, 4, d=3, seed=3)
    src = [p.main[0], p.main[3]]
    tgt = [p.main[1], p.main[2], p.main[4]] + list(p.special)
    blob = bconv_blob(src, [0, 3], tgt, [1, 2, 4, 5, 6])
    k, m, W = len(src), len(tgt), bconv_words(src)
    inv_s = blob[: 2 * k].view(np.float64)
    c = blob[3 * k:4 * k].astype(np.uint64)
    negS = blob[5 * k + m:5 * k + 2 * m].astype(np.uint64)
    w = blob[5 * k + 2 * m:5 * k + 2 * m + k * m].astype(np.uint64).reshape(m, k)
    rows = np.stack([np.random.default_rng(i).integers(0, s, 256, dtype=np.uint64) for i, s in enumerate(src)])
    rows[:, :3] = 0
    S = src[0] * src[1]
    y = rows * c[:, None] % np.array(src, dtype=np.uint64)[:, None]
    v = (y.astype(np.float64) * inv_s[:, None]).sum(axis=0)
    u = np.floor(v).astype(np.uint64)
    for j in np.nonzero(np.abs(v - np.rint(v)) < 2.0 ** -40)[0]:
        u[j] = sum(int(y[i, j]) * (S // src[i]) for i in range(k)) // S
    for t in range(m):
        got = ((y * w[t][:, None]).sum(axis=0) + u * negS[t]) % np.uint64(tgt[t])
        assert np.array_equal(got, O.bconv_row(rows, tuple(src), tgt[t]))
