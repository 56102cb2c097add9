"""Device-resident RNS polynomials and the row primitives (reference poly.py:1-287).

`RnsPolynomial.limbs` is a CUDA int32 tensor of shape (num_limbs, N) whose words are the
uint32 residues (the reference stores the same values as uint64, poly.py:50).  Every
primitive runs a kernel of libcerium_b200.so on the current torch stream.
"""

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native
from .context import SPECIAL_BASE, dptr, get_context, stream_handle
from .params import CkksParams

LF_OP_ADD, LF_OP_SUB, LF_OP_MUL, LF_OP_NEG = 0, 1, 2, 3
LF_OP_SCALAR_MUL, LF_OP_MULACC, LF_OP_MODSTEP, LF_OP_MUL_SCALAR_ADD = 4, 5, 6, 7
LF_OP_ADD_SCALAR = 8


class Domain(Enum):
    COEFF = "coeff"
    EVAL = "eval"


def prime_for_id(params: CkksParams, bid: int) -> int:
    if bid >= SPECIAL_BASE:
        return params.special_basis[bid - SPECIAL_BASE]
    return params.rns_basis[bid]


def main_ids(level: int) -> tuple:
    return tuple(range(level + 1))


def special_ids(params: CkksParams) -> tuple:
    return tuple(SPECIAL_BASE + j for j in range(params.num_special))


def extended_ids(params: CkksParams, level: int) -> tuple:
    return main_ids(level) + special_ids(params)


def to_device(arr) -> torch.Tensor:
    a = np.ascontiguousarray(np.asarray(arr).astype(np.uint32))
    return torch.from_numpy(a.view(np.int32)).cuda()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32).astype(np.uint64)


@dataclass
class RnsPolynomial:
    limbs: torch.Tensor          # (num_limbs, N) int32 on CUDA (uint32 residues)
    domain: Domain
    basis_ids: tuple

    def __post_init__(self):
        if isinstance(self.limbs, np.ndarray):
            self.limbs = to_device(self.limbs)
        assert self.limbs.dim() == 2 and self.limbs.dtype == torch.int32
        assert len(self.basis_ids) == self.limbs.shape[0]
        assert len(set(self.basis_ids)) == len(self.basis_ids)
        self.basis_ids = tuple(self.basis_ids)

    @property
    def N(self) -> int:
        return self.limbs.shape[1]

    def row(self, bid: int) -> torch.Tensor:
        return self.limbs[self.basis_ids.index(bid)]

    def numpy(self) -> np.ndarray:
        """Reference layout: (num_limbs, N) uint64."""
        return to_host(self.limbs)

    def validate(self, params: CkksParams):
        h = self.numpy()
        for bid, row in zip(self.basis_ids, h):
            assert row.max(initial=0) < prime_for_id(params, bid), f"residue >= prime on base {bid}"

    def clone(self):
        return RnsPolynomial(self.limbs.clone(), self.domain, self.basis_ids)

    @staticmethod
    def from_reference(p) -> "RnsPolynomial":
        """Upload a reference `limbforge.poly.RnsPolynomial` (uint64 numpy rows)."""
        dom = Domain.EVAL if getattr(p.domain, "value", p.domain) == "eval" else Domain.COEFF
        return RnsPolynomial(to_device(p.limbs), dom, tuple(p.basis_ids))


def as_device_poly(p) -> RnsPolynomial:
    if isinstance(p, RnsPolynomial):
        return p
    return RnsPolynomial.from_reference(p)


def empty_like(p: RnsPolynomial, ids=None, domain=None) -> RnsPolynomial:
    ids = p.basis_ids if ids is None else tuple(ids)
    return RnsPolynomial(torch.empty((len(ids), p.N), dtype=torch.int32, device=p.limbs.device),
                         p.domain if domain is None else domain, ids)


def zero_poly(params: CkksParams, basis_ids, domain=Domain.EVAL) -> RnsPolynomial:
    return RnsPolynomial(torch.zeros((len(basis_ids), params.N), dtype=torch.int32, device="cuda"),
                         domain, tuple(basis_ids))


# --- device row primitives ------------------------------------------------------------

def ewise(params, op, out: torch.Tensor, a: torch.Tensor, ids, b=None, c=None, scalars=None):
    ctx = get_context(params)
    lib = _native.lib()
    sc = None
    if scalars is not None:
        sc = _native.u32_array([int(s) % ctx.prime(b) for s, b in zip(scalars, ids)])
    _native.check(lib.lf_ewise(ctx.handle, op, dptr(out), dptr(a),
                               dptr(b) if b is not None else None,
                               dptr(c) if c is not None else None,
                               len(ids), ctx.pidx_array(ids), sc, stream_handle()), "lf_ewise")
    return out


def ntt_rows(params, rows: torch.Tensor, ids, inverse=False):
    ctx = get_context(params)
    lib = _native.lib()
    fn = lib.lf_ntt_inv if inverse else lib.lf_ntt_fwd
    _native.check(fn(ctx.handle, dptr(rows), len(ids), ctx.pidx_array(ids), stream_handle()),
                  "lf_ntt")
    return rows


def automorph_rows(params, out: torch.Tensor, rows: torch.Tensor, g: int):
    ctx = get_context(params)
    _native.check(_native.lib().lf_automorph(ctx.handle, dptr(out), dptr(rows), g & 0xFFFFFFFF,
                                             rows.shape[0], stream_handle()), "lf_automorph")
    return out


def _binary(op):
    def run(a: RnsPolynomial, b: RnsPolynomial, params: CkksParams) -> RnsPolynomial:
        assert a.basis_ids == b.basis_ids and a.domain == b.domain
        out = empty_like(a)
        ewise(params, op, out.limbs, a.limbs, a.basis_ids, b=b.limbs)
        return out
    return run


poly_add = _binary(LF_OP_ADD)
poly_sub = _binary(LF_OP_SUB)
poly_mul = _binary(LF_OP_MUL)


def poly_neg(a: RnsPolynomial, params: CkksParams) -> RnsPolynomial:
    out = empty_like(a)
    ewise(params, LF_OP_NEG, out.limbs, a.limbs, a.basis_ids)
    return out


def poly_scalar_mul(a: RnsPolynomial, scalars, params: CkksParams) -> RnsPolynomial:
    """Per-limb scalar multiply; scalars maps basis id -> int (poly.py:204-209)."""
    out = empty_like(a)
    sc = [scalars[b] % prime_for_id(params, b) for b in a.basis_ids]
    ewise(params, LF_OP_SCALAR_MUL, out.limbs, a.limbs, a.basis_ids, scalars=sc)
    return out


def poly_ntt(a: RnsPolynomial, params: CkksParams) -> RnsPolynomial:
    assert a.domain == Domain.COEFF
    out = RnsPolynomial(a.limbs.clone(), Domain.EVAL, a.basis_ids)
    ntt_rows(params, out.limbs, a.basis_ids)
    return out


def poly_intt(a: RnsPolynomial, params: CkksParams) -> RnsPolynomial:
    assert a.domain == Domain.EVAL
    out = RnsPolynomial(a.limbs.clone(), Domain.COEFF, a.basis_ids)
    ntt_rows(params, out.limbs, a.basis_ids, inverse=True)
    return out


def poly_automorph(a: RnsPolynomial, g: int, params: CkksParams) -> RnsPolynomial:
    assert a.domain == Domain.EVAL
    if g % 2 == 0:
        raise ValueError("automorphism index must be odd")
    out = empty_like(a)
    automorph_rows(params, out.limbs, a.limbs, g)
    return out


def base_convert(a: RnsPolynomial, target_ids, params: CkksParams) -> RnsPolynomial:
    """Exact conversion of coefficient-domain residues onto target primes; targets already in
    the source pass through unchanged (poly.py:234-248)."""
    assert a.domain == Domain.COEFF
    ctx = get_context(params)
    target_ids = tuple(target_ids)
    out = torch.empty((len(target_ids), a.N), dtype=torch.int32, device=a.limbs.device)
    conv = tuple(b for b in target_ids if b not in a.basis_ids)
    if conv:
        blob, k, m, W = ctx.bconv_table(a.basis_ids, conv)
        tmp = torch.empty((m, a.N), dtype=torch.int32, device=a.limbs.device)
        _native.check(_native.lib().lf_bconv(ctx.handle, dptr(tmp), dptr(a.limbs), dptr(blob),
                                             k, m, W, stream_handle()), "lf_bconv")
    for i, bid in enumerate(target_ids):
        out[i] = a.row(bid) if bid in a.basis_ids else tmp[conv.index(bid)]
    return RnsPolynomial(out, Domain.COEFF, target_ids)


def mod_down(a: RnsPolynomial, target_ids, params: CkksParams) -> RnsPolynomial:
    """Floor-divide by the product of the dropped primes (poly.py:251-281): INTT of the dropped
    rows, exact conversion onto the kept primes, NTT, then (a - conv) * P^-1."""
    target_ids = tuple(target_ids)
    drop_ids = tuple(b for b in a.basis_ids if b not in target_ids)
    assert drop_ids, "mod_down needs at least one dropped prime"
    assert all(b in a.basis_ids for b in target_ids)
    p_prod = 1
    for b in drop_ids:
        p_prod *= prime_for_id(params, b)
    drop = RnsPolynomial(torch.stack([a.row(b) for b in drop_ids]), a.domain, drop_ids)
    if a.domain == Domain.EVAL:
        drop = poly_intt(drop, params)
    conv = base_convert(drop, target_ids, params)
    if a.domain == Domain.EVAL:
        conv = poly_ntt(conv, params)
    kept = torch.stack([a.row(b) for b in target_ids])
    out = torch.empty_like(kept)
    sc = [pow(p_prod, -1, prime_for_id(params, b)) for b in target_ids]
    ewise(params, LF_OP_MODSTEP, out, kept, target_ids, b=conv.limbs, scalars=sc)
    return RnsPolynomial(out, a.domain, target_ids)


def rescale_poly(a: RnsPolynomial, params: CkksParams) -> RnsPolynomial:
    assert a.basis_ids == main_ids(len(a.basis_ids) - 1), "rescale wants a full main basis"
    return mod_down(a, a.basis_ids[:-1], params)
