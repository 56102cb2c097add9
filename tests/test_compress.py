"""Compressed plaintexts (reference compress.py): stored values vs golden output of the real
reference (tests/golden/make_compress.py, CPU), and the GPU multiply bit-equal to dense
mul_plain / expansion equal to dense encode (GPU)."""

import numpy as np
import pytest

from conftest import load_npz
from paper_2512_11269_b200 import compress as CP
from paper_2512_11269_b200.errors import BadStride, NotPeriodic
from paper_2512_11269_b200.params import gen_params

CFG = {"p16": dict(N=16, num_levels=2, d=1, seed=7), "desk": dict(N=4096, num_levels=6, d=3, seed=0)}
CASES = [("p16", s) for s in (1, 2, 4, 8)] + [("desk", 4), ("desk", 64)]


@pytest.mark.parametrize("name,stride", CASES)
def test_unique_rows_match_reference(name, stride):
    z = load_npz("compress.npz")
    p = gen_params(**CFG[name])
    for level in (p.max_level, 1):
        key = f"{name}_s{stride}_l{level}"
        got = CP.unique_rows(z[key + "_v"], p, level, p.scale, stride)
        assert np.array_equal(got, z[key])


def test_descriptor_and_errors():
    p = gen_params(**CFG["p16"])
    d = CP.CompressionDescriptor.for_params(p, 2)
    assert (d.block, d.unique_count) == (4, 4)
    assert np.array_equal(d.index_map(), np.arange(16) // 4)
    with pytest.raises(BadStride):
        CP.CompressionDescriptor.for_params(p, 3)
    rng = np.random.default_rng(0)
    with pytest.raises(NotPeriodic):
        CP.unique_rows(rng.uniform(-1, 1, 8), p, 1, p.scale, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("name,stride", [("p16", 2), ("desk", 4), ("desk", 64)])
def test_gpu_compressed_mul_bit_equals_dense(name, stride):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    z = load_npz("compress.npz")
    p = B.gen_params(**CFG[name], **({"hamming_weight": 8} if name == "p16" else {}))
    sk, pk, rlk = B.keygen(p, seed=11)
    v = z[f"{name}_s{stride}_l{p.max_level}_v"]
    cp = CP.encode_compressed(v, p, stride=stride)
    assert np.array_equal(cp.unique.cpu().numpy().view(np.uint32), z[f"{name}_s{stride}_l{p.max_level}"])
    dense = B.encode(v, p)
    assert np.array_equal(CP.expand(cp, p).poly.numpy(), dense.poly.numpy())
    w = np.random.default_rng(3).uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(w, p), pk, p, np.random.default_rng(4))
    got = CP.mul_plain_compressed(ct, cp, p)
    want = B.mul_plain(ct, dense, p)
    assert got.scale == want.scale
    assert np.array_equal(got.b.numpy(), want.b.numpy()) and np.array_equal(got.a.numpy(), want.a.numpy())
    assert cp.dense_bytes // cp.compressed_bytes == cp.descriptor.block
