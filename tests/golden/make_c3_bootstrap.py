"""One-off: digest of a full C3 bootstrap (N=2^16, L=47, d=4, scale 2^26, h=64, full slots,
BootConfig()) computed by the CPU ORACLE composition (oracle/boot_backend.py over
oracle/lf_oracle.py, the restatement of the reference primitives), on the exact keys and input
the GPU test regenerates (tests/test_gpu_c3_parity.py::test_c3_bootstrap_digest_vs_oracle).

Keys: keygen(seed=11); conjugation key then the rotation keys in sorted order from ONE
default_rng(99) stream (bootstrap.make_bootstrap_keys).  The rotation keys are not all held in
memory: the RNG state before each key is recorded and the key is regenerated when the
composition asks for it (identical draws, identical key).

Writes tests/golden/c3_bootstrap.json.  Runtime: tens of minutes on one core.
    python tests/golden/make_c3_bootstrap.py
"""

import copy
import hashlib
import json
import os
import sys
import time
from collections.abc import Mapping

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lf_oracle as O  # noqa: E402
from oracle.boot_backend import OracleBackend  # noqa: E402
from paper_2512_11269_b200 import bootstrap as BT  # noqa: E402

KW = dict(N=65536, num_levels=47, d=4, seed=0, scale=2 ** 26)


class LazyRotKeys(Mapping):
    def __init__(self, P, keys, rots, rng):
        self.P, self.keys, self.states = P, keys, {}
        for s in sorted(rots):
            self.states[s] = copy.deepcopy(rng.bit_generator.state)
            O.rotation_key(P, keys, s, rng)          # advance the stream exactly as generation does
        self._cache = {}

    def __getitem__(self, s):
        if s not in self._cache:
            g = np.random.default_rng()
            g.bit_generator.state = copy.deepcopy(self.states[s])
            self._cache = {s: O.rotation_key(self.P, self.keys, s, g)}   # keep one key resident
        return self._cache[s]

    def __iter__(self):
        return iter(self.states)

    def __len__(self):
        return len(self.states)


def digest(ct):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ct.b.rows.astype(np.uint32)).tobytes())
    h.update(np.ascontiguousarray(ct.a.rows.astype(np.uint32)).tobytes())
    return h.hexdigest()


def main():
    t0 = time.time()
    P = O.gen_params(**KW)
    keys = O.keygen(P, seed=11)

    class _Plan:
        N = P.N
        main_primes = P.main
    rots = BT.Bootstrapper(_Plan, BT.BootConfig()).required_rotations()
    rng = np.random.default_rng(99)
    ck = O.conj_key(P, keys, rng)
    rk = LazyRotKeys(P, keys, rots, rng)
    print(f"keys ready ({len(rots)} rotations) in {time.time() - t0:.0f} s", flush=True)
    v = np.random.default_rng(77).uniform(-1, 1, P.n)
    ct = O.encrypt(O.encode(v, P, level=0, scale=2 ** 26), keys, P, np.random.default_rng(5))
    in_digest = digest(ct)
    out = BT.Bootstrapper(OracleBackend(P, keys.rlk, ck, rk)).bootstrap(ct)
    dout = O.decrypt(out, keys, P)[: P.n]
    din = O.decrypt(ct, keys, P)[: P.n]
    rec = {"params": KW, "keygen_seed": 11, "rot_seed": 99, "input_seed": [77, 5],
           "rotations": len(rots), "input_sha256": in_digest, "level": out.level,
           "scale": [out.scale.numerator, out.scale.denominator], "sha256": digest(out),
           "max_err_vs_input": float(np.abs(dout - din).max()), "cpu_seconds": round(time.time() - t0)}
    print(rec, flush=True)
    json.dump(rec, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_bootstrap.json"), "w"),
              indent=1)


if __name__ == "__main__":
    main()
