"""Compressed plaintexts for stride-periodic slot vectors (reference
compress.py:1-176).

A vector with period p embeds to a polynomial whose nonzeros sit at multiples of r = n/p; its
bit-reversed evaluation rows are constant on contiguous blocks of length r, so each limb keeps
only N/r values (the reference's index map pos // r).  The unique values are computed on the
host exactly as the reference does (one representative root per block, compress.py:103-144)
and live in HBM; `mul_plain_compressed` multiplies a ciphertext by reading them through the
index map inside the kernel (`lf_mul_compressed`), bit-equal to mul_plain with the expanded
plaintext, with r-times less plaintext memory and traffic.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .encoding import embed_inverse
from .errors import BadStride, BaseMismatch, NotPeriodic
from .modmath import bit_reverse_indices, primitive_root_of_unity
from .params import CkksParams
from .poly import main_ids, prime_for_id


@dataclass(frozen=True)
class CompressionDescriptor:
    N: int
    stride: int          # repeat period p
    block: int           # r = n/p: length of each constant run
    unique_count: int    # N/r distinct values per limb

    @classmethod
    def for_params(cls, params: CkksParams, stride: int):
        n = params.n
        if stride < 1 or stride & (stride - 1):
            raise BadStride(f"stride {stride} is not a power of two")
        if n % stride:
            raise BadStride(f"stride {stride} does not divide {n} slots")
        r = n // stride
        return cls(N=params.N, stride=stride, block=r, unique_count=params.N // r)

    def index_map(self) -> np.ndarray:
        return np.arange(self.N) // self.block


@dataclass
class CompressedPlaintext:
    unique: object               # (level+1, unique_count) int32 device tensor (uint32 residues)
    descriptor: CompressionDescriptor
    scale: Fraction
    level: int

    @property
    def compressed_bytes(self):          # in the reference's uint64 accounting (compress.py:60-67)
        return (self.level + 1) * self.descriptor.unique_count * 8

    @property
    def dense_bytes(self):
        return (self.level + 1) * self.descriptor.N * 8


def _smallest_period(values: np.ndarray) -> int:
    n = len(values)
    p = 1
    while p < n:
        if np.array_equal(values, np.tile(values[:p], n // p)):
            return p
        p *= 2
    return n


def unique_rows(values, params: CkksParams, level: int, scale, stride: int) -> np.ndarray:
    """Host computation of the stored values (compress.py:103-144): the sparse coefficients
    (2p of them) evaluated at one representative root per block, for every main prime."""
    desc = CompressionDescriptor.for_params(params, stride)
    coeffs = np.rint(embed_inverse(values, params.N) * float(scale)).astype(np.int64)
    r = desc.block
    support = np.arange(0, params.N, r)
    if np.delete(coeffs, support).any():
        raise NotPeriodic("periodic vector must embed to a sparse polynomial")
    sparse = [int(m) for m in coeffs[support]]
    rev = bit_reverse_indices(params.N)
    two_n = 2 * params.N
    reps = [int(rev[b * r]) for b in range(desc.unique_count)]
    rows = np.empty((level + 1, desc.unique_count), dtype=np.uint64)
    for li, bid in enumerate(main_ids(level)):
        q = prime_for_id(params, bid)
        psi = primitive_root_of_unity(2 * params.N, q)
        for b, k in enumerate(reps):
            acc = 0
            for u, m in enumerate(sparse):
                if m:
                    acc = (acc + (m % q) * pow(psi, (2 * k + 1) * u * r % two_n, q)) % q
            rows[li, b] = acc
    return rows


def encode_compressed(values, params: CkksParams, level=None, scale=None,
                      stride=None) -> CompressedPlaintext:
    """Encode an exactly stride-periodic vector keeping only the unique evaluation values
    (compress.py:103-144); the values are uploaded once and stay resident."""
    from .poly import to_device
    level = params.max_level if level is None else level
    scale = Fraction(params.scale if scale is None else scale)
    values = np.asarray(values, dtype=np.float64)
    n = params.n
    if len(values) != n:
        values = np.resize(values, n) if len(values) and n % len(values) == 0 else values
    if len(values) != n:
        raise NotPeriodic(f"need all {n} slots to check periodicity")
    if stride is None:
        stride = _smallest_period(values)
    desc = CompressionDescriptor.for_params(params, stride)
    if not np.array_equal(values, np.tile(values[:stride], n // stride)):
        raise NotPeriodic(f"vector is not exactly periodic with stride {stride}")
    rows = unique_rows(values, params, level, scale, stride)
    return CompressedPlaintext(to_device(rows), desc, scale, level)


def expand(cp: CompressedPlaintext, params: CkksParams):
    """Dense evaluation-domain plaintext: row[i] = unique[i // r] (compress.py:147-155)."""
    from .encoding import Plaintext
    from .poly import Domain, RnsPolynomial
    rows = cp.unique.repeat_interleave(cp.descriptor.block, dim=1).contiguous()
    return Plaintext(RnsPolynomial(rows, Domain.EVAL, main_ids(cp.level)), cp.scale, cp.level)


def mul_plain_compressed(ct, cp: CompressedPlaintext, params: CkksParams):
    """ct * cp without expanding the plaintext (compress.py:158-176 for every limb of b and a);
    level and base checks as mul_plain (ckks.py:171-179)."""
    import torch
    from . import _native
    from .ckks import Ciphertext, as_device_ct
    from .context import dptr, get_context, stream_handle
    from .errors import LevelMismatch
    from .fused import ct_block
    from .poly import Domain, RnsPolynomial
    if ct.level != cp.level:
        if ct.level > cp.level:
            raise BaseMismatch(f"compressed plaintext has no limb for base {cp.level + 1}")
        raise LevelMismatch(f"mulPlain: ciphertext level {ct.level}, plaintext level {cp.level}")
    ct = as_device_ct(ct)
    c = ct_block(ct)
    out = torch.empty_like(c)
    ctx = get_context(params)
    _native.check(_native.lib().lf_mul_compressed(ctx.handle, dptr(out), dptr(c), dptr(cp.unique),
                                                  ct.level + 1, cp.descriptor.unique_count,
                                                  stream_handle()), "lf_mul_compressed")
    ids = main_ids(ct.level)
    return Ciphertext(RnsPolynomial(out[0], Domain.EVAL, ids), RnsPolynomial(out[1], Domain.EVAL, ids),
                      ct.scale * cp.scale, ct.level)
