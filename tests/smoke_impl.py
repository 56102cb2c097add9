"""__graft_entry__.smoke(): one small fused hot-path invocation on cuda:0 (N=4096, 7 main +
3 special primes, d=3 — the reference desk config) checked bit-for-bit against the CPU oracle."""

import numpy as np


def run_smoke():
    import torch
    assert torch.cuda.is_available(), "smoke() needs a CUDA device"
    torch.cuda.set_device(0)
    import paper_2512_11269_b200 as B
    from oracle import lf_oracle as O

    kw = dict(N=4096, num_levels=6, d=3, seed=0)
    p, po = B.gen_params(**kw), O.gen_params(**kw)
    sk, pk, rlk = B.keygen(p, seed=11)
    ko = O.keygen(po, seed=11)
    rk = B.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    rko = O.rotation_key(po, ko, 1, np.random.default_rng(5))
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct_v = B.encrypt(B.encode(v, p), pk, p, np.random.default_rng(1))
    ct_w = B.encrypt(B.encode(w, p), pk, p, np.random.default_rng(2))
    co_v = O.encrypt(O.encode(v, po), ko, po, np.random.default_rng(1))
    co_w = O.encrypt(O.encode(w, po), ko, po, np.random.default_rng(2))

    got = B.rescale(B.hom_mul(ct_v, ct_w, rlk, p), p)
    want = O.rescale(po, O.hom_mul(po, co_v, co_w, ko.rlk))
    assert np.array_equal(got.b.numpy(), want.b.rows) and np.array_equal(got.a.numpy(), want.a.rows)
    rot = B.hom_rotate(ct_v, 1, rk, p)
    rwant = O.hom_rotate(po, co_v, 1, rko)
    assert np.array_equal(rot.b.numpy(), rwant.b.rows) and np.array_equal(rot.a.numpy(), rwant.a.rows)
    err = np.abs(B.decrypt(got, sk, p) - v * w).max()
    assert err < 0.05, err
    torch.cuda.synchronize()
    print(f"smoke ok: hom_mul+rescale and rotate bit-exact vs oracle at N=4096; max slot error {err:.2e}")
