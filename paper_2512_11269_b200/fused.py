"""Host side of the fused keyswitch pipeline (csrc/lf_ks.cu via the C ABI).

Ciphertexts are handed to the kernels as one (2, level+1, N) block (b rows then a rows,
include/lf_b200.h); results come back the same way and are exposed as two views, so chained
operations never copy.
"""

import torch

from . import _native
from .context import dptr, get_context, stream_handle
from .poly import Domain, RnsPolynomial, extended_ids, main_ids


def ct_block(ct) -> torch.Tensor:
    """(2, l+1, N) view of a ciphertext's residues; stacks only if b and a are not adjacent."""
    b, a = ct.b.limbs, ct.a.limbs
    n = b.numel()
    if (b.is_contiguous() and a.is_contiguous() and a.data_ptr() == b.data_ptr() + 4 * n
            and a.untyped_storage().data_ptr() == b.untyped_storage().data_ptr()):
        return b.as_strided((2, *b.shape), (n, b.shape[1], 1), b.storage_offset())
    return torch.stack([b, a])


def _pair(out: torch.Tensor, ids):
    return (RnsPolynomial(out[0], Domain.EVAL, ids), RnsPolynomial(out[1], Domain.EVAL, ids))


def keyswitch(params, x: RnsPolynomial, evk):
    ctx = get_context(params)
    level = len(x.basis_ids) - 1
    ws = ctx.ks_workspace_cached(level)
    out = torch.empty((2, level + 1, params.N), dtype=torch.int32, device=x.limbs.device)
    xl = x.limbs.contiguous()
    _native.check(_native.lib().lf_keyswitch(ctx.handle, level, dptr(xl), 0, dptr(ctx.check_evk(evk)), 0,
                                             dptr(out), 0, 1, dptr(ws), stream_handle()),
                  "lf_keyswitch")
    return _pair(out, main_ids(level))


def hom_mul(params, ct1, ct2, rlk):
    ctx = get_context(params)
    level = ct1.level
    ws = ctx.ks_workspace_cached(level)
    c1, c2 = ct_block(ct1), ct_block(ct2)
    out = torch.empty_like(c1)
    _native.check(_native.lib().lf_hom_mul(ctx.handle, level, dptr(c1), dptr(c2), 0, dptr(ctx.check_evk(rlk)),
                                           dptr(out), 0, 1, dptr(ws), stream_handle()), "lf_hom_mul")
    return _pair(out, main_ids(level))


def hom_mul_rescale(params, ct1, ct2, rlk, ndrop: int = 1):
    """hom_mul then `ndrop` rescales (ckks.py:182-194, 220-225), one pipeline: the rescale is
    folded into the relinearisation's ModDown (lf_hom_mul_rescale).  Returns (b, a) at level
    ct1.level - ndrop."""
    ctx = get_context(params)
    level = ct1.level
    ws = ctx.ks_workspace_cached(level)
    c1, c2 = ct_block(ct1), ct_block(ct2)
    out = torch.empty((2, max(level + 1 - ndrop, 1), params.N), dtype=torch.int32, device=c1.device)
    _native.check(_native.lib().lf_hom_mul_rescale(ctx.handle, level, ndrop, dptr(c1), dptr(c2), 0,
                                                   dptr(ctx.check_evk(rlk)), dptr(out), 0, 1, dptr(ws),
                                                   stream_handle()), "lf_hom_mul_rescale")
    return _pair(out, main_ids(level - ndrop))


def rotate(params, ct, g: int, key):
    ctx = get_context(params)
    level = ct.level
    ws = ctx.ks_workspace_cached(level)
    c = ct_block(ct)
    out = torch.empty_like(c)
    _native.check(_native.lib().lf_rotate(ctx.handle, level, dptr(c), 0, g, dptr(ctx.check_evk(key)), 0,
                                          dptr(out), 0, 1, dptr(ws), stream_handle()), "lf_rotate")
    return _pair(out, main_ids(level))


def rotate_hoisted(params, ct, gs, keys, out=None):
    """One shared ModUp of ct.a, then one (inner product, ModDown, sigma_g(b) + .) per key;
    `out`: an (n, 2, level+1, N) contiguous tensor to write into."""
    import ctypes
    ctx = get_context(params)
    level = ct.level
    n = len(gs)
    lib = _native.lib()
    ws = torch.empty(lib.lf_rotate_hoisted_workspace_bytes(ctx.handle, level, n) // 4,
                     dtype=torch.int32, device="cuda")
    c = ct_block(ct)
    if out is None:
        out = torch.empty((n, 2, level + 1, params.N), dtype=torch.int32, device=c.device)
    karr = (ctypes.c_void_p * n)(*[ctx.check_evk(k).data_ptr() for k in keys])
    _native.check(lib.lf_rotate_hoisted(ctx.handle, level, dptr(c), n, _native.u32_array(gs), karr,
                                        dptr(out), out[0].numel(), dptr(ws), stream_handle()),
                  "lf_rotate_hoisted")
    return [_pair(out[r], main_ids(level)) for r in range(n)]


def permute_rotation_key(params, key, g: int) -> torch.Tensor:
    """The permuted form of a rotation key for Galois element g (every row composed with
    sigma_g^-1, lf_automorph by g^-1 mod 2N), as the *_pk rotation entry points take it."""
    ctx = get_context(params)
    ginv = pow(int(g), -1, 2 * params.N)
    src = key.data
    out = torch.empty_like(src)
    nrows = src.numel() // params.N
    _native.check(_native.lib().lf_automorph(ctx.handle, dptr(out), dptr(src), ginv, nrows, stream_handle()),
                  "lf_automorph")
    return out


def rotate_batch(params, level: int, cts: torch.Tensor, gs, keys, permuted: bool = False):
    """cts: (n, 2, level+1, N) -> n rotations with their own Galois elements and keys
    (permuted=True: keys in permute_rotation_key form, lf_rotate_batch_pk)."""
    import ctypes
    ctx = get_context(params)
    n = cts.shape[0]
    lib = _native.lib()
    ws = ctx.ks_workspace(level, min(n, 64))
    out = torch.empty_like(cts)
    karr = (ctypes.c_void_p * n)(*[ctx.check_evk(k).data_ptr() for k in keys])
    fn = lib.lf_rotate_batch_pk if permuted else lib.lf_rotate_batch
    _native.check(fn(ctx.handle, level, dptr(cts), cts[0].numel(), n, _native.u32_array(gs),
                     karr, dptr(out), out[0].numel(), dptr(ws), stream_handle()),
                  "lf_rotate_batch")
    return out


def rescale(params, ct):
    ctx = get_context(params)
    level = ct.level
    ws = ctx.rescale_workspace(level)
    c = ct_block(ct)
    out = torch.empty((2, level, params.N), dtype=torch.int32, device=c.device)
    _native.check(_native.lib().lf_rescale(ctx.handle, level, dptr(c), 0, dptr(out), 0, 1, dptr(ws),
                                           stream_handle()), "lf_rescale")
    return _pair(out, main_ids(level - 1))


def rescale_multi(params, ct, ndrop: int):
    """Drop the top `ndrop` (1 or 2) primes in one pass; ndrop=2 equals two rescales."""
    ctx = get_context(params)
    level = ct.level
    ws = ctx.rescale_workspace(level)
    c = ct_block(ct)
    out = torch.empty((2, level + 1 - ndrop, params.N), dtype=torch.int32, device=c.device)
    _native.check(_native.lib().lf_rescale_multi(ctx.handle, level, ndrop, dptr(c), 0, dptr(out), 0, 1,
                                                 dptr(ws), stream_handle()), "lf_rescale_multi")
    return _pair(out, main_ids(level - ndrop))


def decompose(params, x: RnsPolynomial):
    ctx = get_context(params)
    level = len(x.basis_ids) - 1
    ext = extended_ids(params, level)
    beta = min(params.ks.d, level + 1)
    ws = ctx.ks_workspace_cached(level)
    pieces = torch.empty((beta, len(ext), params.N), dtype=torch.int32, device=x.limbs.device)
    xl = x.limbs.contiguous()
    _native.check(_native.lib().lf_ks_decompose(ctx.handle, level, dptr(xl), dptr(pieces), dptr(ws),
                                                stream_handle()), "lf_ks_decompose")
    return [(j, RnsPolynomial(pieces[j], Domain.EVAL, ext)) for j in range(beta)]


# --- batched entry points (bench / bootstrap) -------------------------------------------

def keyswitch_batch(params, level: int, xs: torch.Tensor, evk, out: torch.Tensor = None,
                    ws: torch.Tensor = None):
    """xs: (B, level+1, N) -> out (B, 2, level+1, N); one shared key."""
    ctx = get_context(params)
    B = xs.shape[0]
    if ws is None:
        ws = ctx.ks_workspace(level, B)
    if out is None:
        out = torch.empty((B, 2, level + 1, params.N), dtype=torch.int32, device=xs.device)
    _native.check(_native.lib().lf_keyswitch(ctx.handle, level, dptr(xs), xs[0].numel(), dptr(ctx.check_evk(evk)), 0,
                                             dptr(out), out[0].numel(), B, dptr(ws), stream_handle()),
                  "lf_keyswitch")
    return out


def keyswitch_batch_profiled(params, level: int, xs: torch.Tensor, evk, out: torch.Tensor,
                             ws: torch.Tensor):
    """As keyswitch_batch, returning the CUDA-event duration (ms) of each fused kernel:
    [modup_in, modup_bconv, ks_inner, moddown_bconv, moddown_out]."""
    import ctypes
    ctx = get_context(params)
    ms = (ctypes.c_float * 5)()
    _native.check(_native.lib().lf_keyswitch_profiled(
        ctx.handle, level, dptr(xs), xs[0].numel(), dptr(ctx.check_evk(evk)), 0, dptr(out), out[0].numel(),
        xs.shape[0], dptr(ws), stream_handle(), ms), "lf_keyswitch_profiled")
    return list(ms)
