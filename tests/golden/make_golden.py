"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything is produced by the reference's own public functions
(limbforge.params/ntt/poly/keys/ckks/encoding) on seeded inputs, following the
seeds of the reference tests (pkg/tests/conftest.py:8-44, test_ckks_ops.py:27-40)
and of SURVEY.md §8(d).  Small configurations are stored as full uint32 arrays;
the N=4096 and N=2^16 configurations are stored as SHA-256 digests of the
little-endian uint32 residue rows (plus the seeds needed to rebuild the inputs).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

import limbforge  # noqa: F401  (from PYTHONPATH=/root/reference/pkg/src)
from limbforge import ckks, keys, ntt, poly
from limbforge.encoding import decode, encode
from limbforge.params import gen_params

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(rows) -> str:
    a = np.ascontiguousarray(np.asarray(rows, dtype=np.uint64).astype("<u4"))
    return hashlib.sha256(a.tobytes()).hexdigest()


def pdesc(p):
    return {"N": p.N, "main": list(p.rns_basis), "special": list(p.special_basis),
            "scale": [p.scale.numerator, p.scale.denominator], "h": p.hamming_weight,
            "d": p.ks.d, "seed": p.seed}


CONFIGS = {
    "p16": dict(N=16, num_levels=2, d=1, seed=7),
    "small": dict(N=256, num_levels=4, d=3, seed=3),
    "desk": dict(N=4096, num_levels=6, d=3, seed=0),
    "c2": dict(N=65536, num_levels=35, d=4, seed=0, scale=2 ** 26),
    "c2b": dict(N=65536, num_levels=24, d=3, seed=0, scale=2 ** 26),
    "n1024": dict(N=1024, num_levels=8, d=3, seed=0),
    "n64": dict(N=64, num_levels=2, d=3, seed=0),
    "n32": dict(N=32, num_levels=2, d=3, seed=0),
}


def params_fixture():
    out = {}
    for name, kw in CONFIGS.items():
        out[name] = {"kwargs": kw, "params": pdesc(gen_params(**kw))}
    with open(os.path.join(HERE, "params.json"), "w") as f:
        json.dump(out, f, indent=1)


def ntt_fixture():
    arrs = {}
    meta = {}
    for name in ("p16", "n32", "n64", "small", "n1024", "desk"):
        p = gen_params(**CONFIGS[name])
        for k, q in enumerate(p.rns_basis + p.special_basis):
            rng = np.random.default_rng(100 + k)
            x = rng.integers(0, q, (2, p.N), dtype=np.uint64)
            arrs[f"{name}_{k}_x"] = x.astype(np.uint32)
            arrs[f"{name}_{k}_fwd"] = ntt.ntt_forward(x, q).astype(np.uint32)
            arrs[f"{name}_{k}_inv"] = ntt.ntt_inverse(x, q).astype(np.uint32)
            arrs[f"{name}_{k}_psi"] = np.array([ntt.ntt_tables(p.N, q).psi], dtype=np.uint64)
    for name in ("c2",):
        p = gen_params(**CONFIGS[name])
        allp = p.rns_basis + p.special_basis
        for k in (0, 1, 35, 36, 44):
            q = allp[k]
            x = np.random.default_rng(100 + k).integers(0, q, p.N, dtype=np.uint64)
            meta[f"{name}_{k}"] = {"q": q, "psi": ntt.ntt_tables(p.N, q).psi,
                                   "fwd": digest(ntt.ntt_forward(x, q)),
                                   "inv": digest(ntt.ntt_inverse(x, q))}
    # automorphism permutations (bit-reversed eval order)
    for N in (16, 256, 4096):
        for steps in (1, 3, 7):
            g = ntt.galois_element(N, steps)
            arrs[f"perm_{N}_{steps}"] = ntt.automorphism_permutation(N, g).astype(np.int32)
        arrs[f"perm_{N}_conj"] = ntt.automorphism_permutation(N, 2 * N - 1).astype(np.int32)
    np.savez_compressed(os.path.join(HERE, "ntt.npz"), **arrs)
    with open(os.path.join(HERE, "ntt_big.json"), "w") as f:
        json.dump(meta, f, indent=1)


def bconv_fixture():
    arrs = {}
    p = gen_params(**CONFIGS["p16"])
    rng = np.random.default_rng(12345)
    rows = np.stack([rng.integers(0, q, 16, dtype=np.uint64) for q in p.rns_basis])
    cases = {
        "rand": rows,
        "c42": np.stack([np.full(16, 42, dtype=np.uint64)] * 3),
        "qm1": np.stack([np.full(16, q - 1, dtype=np.uint64) for q in p.rns_basis]),
        "zero": np.zeros((3, 16), dtype=np.uint64),
    }
    for name, r in cases.items():
        src = poly.RnsPolynomial(r, poly.Domain.COEFF, poly.main_ids(2))
        out = poly.base_convert(src, poly.special_ids(p), p)
        arrs[f"{name}_in"] = r.astype(np.uint32)
        arrs[f"{name}_out"] = out.limbs.astype(np.uint32)
    # ModUp-shaped conversion at N=256 (digit 0 -> rest), including mixed zero coeffs
    ps = gen_params(**CONFIGS["small"])
    rng = np.random.default_rng(4321)
    grp = [0, 3]
    r = np.stack([rng.integers(0, ps.rns_basis[i], 256, dtype=np.uint64) for i in grp])
    r[:, :8] = 0
    src = poly.RnsPolynomial(r, poly.Domain.COEFF, tuple(grp))
    tgt = (1, 2, 4) + poly.special_ids(ps)
    out = poly.base_convert(src, tgt, ps)
    arrs["small_in"] = r.astype(np.uint32)
    arrs["small_out"] = out.limbs.astype(np.uint32)
    np.savez_compressed(os.path.join(HERE, "bconv.npz"), **arrs)


def _keys_digest(sk, pk, rlk, p):
    ids = poly.extended_ids(p, p.max_level)
    return {
        "sk_coeffs": hashlib.sha256(sk.coeffs.astype(np.int8).tobytes()).hexdigest(),
        "sk_eval": digest(np.stack([sk.eval_rows[b] for b in ids])),
        "pk_b": digest(pk.b.limbs), "pk_a": digest(pk.a.limbs),
        "rlk": [[digest(b.limbs), digest(a.limbs)] for b, a in rlk.digits],
    }


def ct_pack(ct):
    return np.stack([ct.b.limbs, ct.a.limbs]).astype(np.uint32)


def ops_fixture(name, full: bool):
    """The reference test_ckks_ops.py ctx (seed 77 slot vectors, keygen seed 11)."""
    p = gen_params(**CONFIGS[name])
    t0 = time.time()
    sk, pk, rlk = keys.keygen(p, seed=11)
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct_v = ckks.encrypt(encode(v, p), pk, p, rng)
    ct_w = ckks.encrypt(encode(w, p), pk, p, rng)
    rk1 = keys.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    rk3 = keys.make_rotation_key(p, sk, 3, np.random.default_rng(6))
    rkc = keys._make_evalkey(p, sk, {b: sk.eval_rows[b][ntt.automorphism_permutation(p.N, 2 * p.N - 1)]
                                     for b in poly.extended_ids(p, p.max_level)},
                             ("rot", 2 * p.N - 1), np.random.default_rng(8))
    pt_w = encode(w, p)
    mul = ckks.hom_mul(ct_v, ct_w, rlk, p)
    res = {
        "ct_v": ct_v, "ct_w": ct_w,
        "add": ckks.hom_add(ct_v, ct_w, p),
        "sub": ckks.hom_sub(ct_v, ct_w, p),
        "mul_plain": ckks.mul_plain(ct_v, pt_w, p),
        "add_plain": ckks.add_plain(ct_v, pt_w, p),
        "mul": mul,
        "mul_rescale": ckks.rescale(mul, p),
        "rot1": ckks.hom_rotate(ct_v, 1, rk1, p),
        "rot3": ckks.hom_rotate(ct_v, 3, rk3, p),
        "rescale_v": ckks.rescale(ct_v, p),
    }
    # conjugation through the generic galois path (decompose-then-permute)
    g = 2 * p.N - 1
    pieces = ckks.keyswitch_decompose(ct_v.a, p)
    rot = [(j, poly.poly_automorph(d, g, p)) for j, d in pieces]
    ab, aa = ckks.keyswitch_inner_product(rot, rkc, p)
    ids = poly.main_ids(ct_v.level)
    res["conj"] = ckks.Ciphertext(
        poly.poly_add(poly.poly_automorph(ct_v.b, g, p), poly.mod_down(ab, ids, p), p),
        poly.mod_down(aa, ids, p), ct_v.scale, ct_v.level)
    # lower-level ops: encrypt at level 2 (seed 2), mul + rescale, rotate
    low = ckks.encrypt(encode(v, p, level=2), pk, p, np.random.default_rng(2))
    res["low"] = low
    res["low_mul_rescale"] = ckks.rescale(ckks.hom_mul(low, low, rlk, p), p)
    res["low_rot1"] = ckks.hom_rotate(low, 1, rk1, p)
    # keyswitch pieces of ct_v.a and the keyswitch output
    ksb, ksa = ckks.keyswitch(ct_v.a, rlk, p)

    arrs, meta = {}, {"keys": _keys_digest(sk, pk, rlk, p),
                      "rk1": [[digest(b.limbs), digest(a.limbs)] for b, a in rk1.digits],
                      "rkc": [[digest(b.limbs), digest(a.limbs)] for b, a in rkc.digits],
                      "cts": {}}
    for k, ct in res.items():
        meta["cts"][k] = {"level": ct.level, "scale": [ct.scale.numerator, ct.scale.denominator],
                          "digest": digest(ct_pack(ct))}
        if full:
            arrs[k] = ct_pack(ct)
    meta["pieces"] = [[j, digest(d.limbs)] for j, d in pieces]
    meta["ks"] = [digest(ksb.limbs), digest(ksa.limbs)]
    if full:
        for j, d in pieces:
            arrs[f"piece_{j}"] = d.limbs.astype(np.uint32)
        arrs["ks_b"] = ksb.limbs.astype(np.uint32)
        arrs["ks_a"] = ksa.limbs.astype(np.uint32)
    # decrypted values (value-level checks, TOL 0.05)
    arrs["v"] = v
    arrs["w"] = w
    arrs["dec_mul_rescale"] = ckks.decrypt(res["mul_rescale"], sk, p)
    arrs["dec_rot1"] = ckks.decrypt(res["rot1"], sk, p)
    np.savez_compressed(os.path.join(HERE, f"ops_{name}.npz"), **arrs)
    with open(os.path.join(HERE, f"ops_{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"ops_{name}: {time.time() - t0:.1f}s")


def c2_fixture(name="c2", levels=(35, 20)):
    """Full-level (and one lower-level) keyswitch / rotate / hom_mul / rescale at N=2^16 on
    synthetic ciphertexts: rows default_rng(1000+i).integers(0, q_r)."""
    p = gen_params(**CONFIGS[name])
    t0 = time.time()
    sk, pk, rlk = keys.keygen(p, seed=11)
    rk1 = keys.make_rotation_key(p, sk, 1, np.random.default_rng(99))
    print(f"{name} keygen {time.time() - t0:.1f}s")
    meta = {"keys": _keys_digest(sk, pk, rlk, p),
            "rk1": [[digest(b.limbs), digest(a.limbs)] for b, a in rk1.digits], "levels": {}}
    for level in levels:
        ids = poly.main_ids(level)

        def synth(seed):
            rng = np.random.default_rng(seed)
            return np.stack([rng.integers(0, p.rns_basis[i], p.N, dtype=np.uint64) for i in ids])

        b1, a1, b2, a2 = synth(1000), synth(1001), synth(1002), synth(1003)
        E = poly.Domain.EVAL
        ct1 = ckks.Ciphertext(poly.RnsPolynomial(b1, E, ids), poly.RnsPolynomial(a1, E, ids),
                              p.scale, level)
        ct2 = ckks.Ciphertext(poly.RnsPolynomial(b2, E, ids), poly.RnsPolynomial(a2, E, ids),
                              p.scale, level)
        t1 = time.time()
        ksb, ksa = ckks.keyswitch(ct1.a, rlk, p)
        t_ks = time.time() - t1
        rot = ckks.hom_rotate(ct1, 1, rk1, p)
        mul = ckks.hom_mul(ct1, ct2, rlk, p)
        rs = ckks.rescale(ct1, p)
        meta["levels"][str(level)] = {
            "ks": [digest(ksb.limbs), digest(ksa.limbs)],
            "rot1": digest(ct_pack(rot)), "mul": digest(ct_pack(mul)),
            "rescale": digest(ct_pack(rs)), "t_keyswitch_s": t_ks,
        }
        print(f"{name} level {level}: keyswitch {t_ks:.1f}s, total {time.time() - t1:.1f}s")
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["params", "ntt", "bconv", "small", "desk", "c2"]
    if "params" in which:
        params_fixture()
    if "ntt" in which:
        ntt_fixture()
    if "bconv" in which:
        bconv_fixture()
    if "small" in which:
        ops_fixture("small", full=True)
    if "desk" in which:
        ops_fixture("desk", full=False)
    if "c2" in which:
        c2_fixture("c2", levels=(35, 20))
