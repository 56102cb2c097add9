"""Golden compressed plaintexts (reference compress.py:103-144) for tests/test_compress.py:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_compress.py
"""

import os

import numpy as np

from limbforge.compress import encode_compressed
from limbforge.params import gen_params

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    for name, kw, strides in (("p16", dict(N=16, num_levels=2, d=1, seed=7), (1, 2, 4, 8)),
                              ("desk", dict(N=4096, num_levels=6, d=3, seed=0), (4, 64))):
        p = gen_params(**kw)
        for stride in strides:
            rng = np.random.default_rng(100 + stride)
            v = np.tile(rng.uniform(-1, 1, stride), p.n // stride)
            for level in (p.max_level, 1):
                cp = encode_compressed(v, p, level=level, stride=stride)
                out[f"{name}_s{stride}_l{level}"] = cp.unique_values.astype(np.uint64)
                out[f"{name}_s{stride}_l{level}_v"] = v
    np.savez_compressed(os.path.join(HERE, "compress.npz"), **out)
    print(len(out))


if __name__ == "__main__":
    main()
