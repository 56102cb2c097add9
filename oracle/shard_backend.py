"""Oracle row primitives and a gloo all-gather for the limb-sharded keyswitch — TEST
INFRASTRUCTURE ONLY.  Implements `paper_2512_11269_b200.shard`'s RowOps interface with the
oracle restatement of the reference row primitives (poly.py:85-178, ntt.py:70-126) on numpy
uint64 rows, so tests can run the sharded algorithm on CPU ranks (gloo) and compare it with
the single-device oracle keyswitch (ckks.py:134-140)."""

import numpy as np

from . import lf_oracle as O

U64 = np.uint64


class OracleRowOps:
    def __init__(self, P: O.Params):
        self.P = P

    def _q(self, ids):
        return np.array([self.P.prime(b) for b in ids], dtype=U64)[:, None]

    def empty(self, n):
        return np.zeros((n, self.P.N), dtype=U64)

    def select(self, rows, idx):
        return rows[list(idx)] if idx else self.empty(0)

    def take_rows(self, pairs):
        return np.stack([blk[i] for blk, i in pairs]) if pairs else self.empty(0)

    def concat(self, blocks):
        return np.concatenate(blocks)

    def scalar_mul(self, rows, ids, scalars):
        if not ids:
            return self.empty(0)
        s = np.array([v % self.P.prime(b) for v, b in zip(scalars, ids)], dtype=U64)[:, None]
        return rows * s % self._q(ids)

    def intt(self, rows, ids):
        return np.stack([O.ntt_inv(r.copy(), self.P.prime(b)) for r, b in zip(rows, ids)]) if ids else self.empty(0)

    def ntt(self, rows, ids):
        return np.stack([O.ntt_fwd(r.copy(), self.P.prime(b)) for r, b in zip(rows, ids)]) if ids else self.empty(0)

    def bconv(self, rows, src_ids, tgt_ids):
        return O.base_convert(self.P, O.Poly(rows, tuple(src_ids), False), tuple(tgt_ids)).rows

    def mulacc(self, acc, a, b, ids):
        if not ids:
            return self.empty(0)
        q = self._q(ids)
        return (a * b % q) if acc is None else (acc + a * b % q) % q

    def modstep(self, a, b, ids, scalars):
        q = self._q(ids)
        s = np.array([v % self.P.prime(x) for v, x in zip(scalars, ids)], dtype=U64)[:, None]
        return (a + q - b) % q * s % q

    def automorph(self, rows, g):
        return rows[:, O.automorphism_perm(self.P.N, g)] if rows.shape[0] else rows


class GlooNumpyComm:
    """torch.distributed all-gather of numpy uint64 row blocks (values < 2^28)."""

    def __init__(self):
        import torch.distributed as dist
        self.k = dist.get_world_size()
        self.group = None

    def all_gather(self, rows):
        import torch
        from paper_2512_11269_b200.shard import TorchComm
        t = torch.from_numpy(np.ascontiguousarray(rows).astype(np.int64))
        return [r.numpy().astype(U64) for r in TorchComm().all_gather(t)]
