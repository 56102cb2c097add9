"""Golden LFHE blobs (reference serial.py) for tests/test_serial.py, produced by the REAL
reference in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_lfhe.py

Config "small" = gen_params(256, 4, d=3, seed=3); keygen(seed=11); rotation key for 1 step
(default_rng(5)); encrypt(encode(v)) with v = default_rng(77).uniform(-1, 1, n) and
encrypt rng default_rng(1); encode(w) plaintext with w from the same rng; a compressed
plaintext of a period-8 vector (compress.encode_compressed, stride 8) at level 3.
"""

import os

import numpy as np

from limbforge import ckks, compress, keys, serial
from limbforge.encoding import encode
from limbforge.params import gen_params

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    p = gen_params(256, 4, d=3, seed=3)
    sk, pk, rlk = keys.keygen(p, seed=11)
    rk = keys.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct = ckks.encrypt(encode(v, p), pk, p, np.random.default_rng(1))
    pt = encode(w, p, level=2)
    blobs = {
        "ciphertext": serial.ciphertext_to_bytes(ct, p),
        "plaintext": serial.plaintext_to_bytes(pt, p),
        "relin": serial.evalkey_to_bytes(rlk, p),
        "rot1": serial.evalkey_to_bytes(rk, p),
        "secret": serial.secret_to_bytes(sk, p),
        "compressed": serial.compressed_to_bytes(
            compress.encode_compressed(np.tile(np.linspace(-0.5, 0.75, 8), p.n // 8), p, stride=8, level=3), p),
    }
    np.savez_compressed(os.path.join(HERE, "lfhe_small.npz"),
                        **{k: np.frombuffer(b, dtype=np.uint8) for k, b in blobs.items()})
    print({k: len(b) for k, b in blobs.items()})


if __name__ == "__main__":
    main()
