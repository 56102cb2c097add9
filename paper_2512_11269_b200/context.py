"""Device context: one per parameter set.

Holds the native `lf_ctx` (per-prime constants and twiddle tables resident in HBM, built by
lf_ctx_create from the reference's psi = g^((q-1)/2N), ntt.py:22-67) and the host-built
constant blobs (base-conversion tables, keyswitch plans) uploaded once and cached.

Prime indexing inside the context: main prime i -> i, special prime j -> L+1+j.  That is the
basis-id order of the reference's extended basis (poly.py:28-43) with the special offset
SPECIAL_BASE removed.
"""

import ctypes
import math
from functools import lru_cache

import numpy as np
import torch

from . import _native
from .modmath import primitive_root_of_unity
from .params import CkksParams

SPECIAL_BASE = 1 << 16


def require_cuda():
    if not torch.cuda.is_available():
        raise _native.NativeError("a CUDA device is required (no CPU fallback)")


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dptr(t: torch.Tensor, strided: bool = False):
    """Raw device pointer for the C ABI: the kernels index rows densely, so a strided view or
    a tensor on another GPU than the current one is rejected instead of read out of bounds.
    `strided=True` (the pitched entry points, which take the strides explicitly) only requires
    whole contiguous rows."""
    if not t.is_cuda:
        raise _native.NativeError("expected a CUDA tensor")
    if strided:
        if t.stride(-1) != 1 or (t.dim() > 1 and t.stride(-2) != t.shape[-1]):
            raise _native.NativeError(f"expected contiguous rows (strides {t.stride()})")
    elif not t.is_contiguous():
        raise _native.NativeError(f"expected a contiguous tensor (shape {tuple(t.shape)}, strides {t.stride()})")
    if t.device.index != torch.cuda.current_device():
        raise _native.NativeError(f"tensor on cuda:{t.device.index}, current device cuda:{torch.cuda.current_device()}")
    return ctypes.c_void_p(t.data_ptr())


class DeviceContext:
    def __init__(self, params: CkksParams):
        require_cuda()
        self.params = params
        self.N = params.N
        self.logN = params.N.bit_length() - 1
        self.L = params.max_level
        self.alpha = params.num_special
        self.primes = tuple(params.rns_basis) + tuple(params.special_basis)
        psis = [primitive_root_of_unity(2 * params.N, q) for q in self.primes]
        self._lib = _native.lib()
        h = ctypes.c_void_p()
        _native.check(self._lib.lf_ctx_create(self.logN, len(self.primes),
                                              _native.u32_array(self.primes),
                                              _native.u32_array(psis), ctypes.byref(h)),
                      "lf_ctx_create")
        self.handle = h
        self._blobs = {}
        self._pidx = {}
        self._ws = {}
        _native.check(self._lib.lf_ctx_enable_keyswitch(h, self.L + 1, params.ks.d),
                      "lf_ctx_enable_keyswitch")

    def ks_workspace(self, level: int, batch: int = 1) -> torch.Tensor:
        nbytes = self._lib.lf_ks_workspace_bytes(self.handle, level, batch)
        return torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")

    def ks_workspace_cached(self, level: int, batch: int = 1) -> torch.Tensor:
        """A keyswitch workspace reused by every call on the current stream (kernels of one
        stream run in order, so consecutive calls cannot overlap in it); grown on demand."""
        need = self._lib.lf_ks_workspace_bytes(self.handle, level, batch) // 4
        if torch.cuda.is_current_stream_capturing():      # a captured graph keeps its own
            return torch.empty(need, dtype=torch.int32, device="cuda")
        key = torch.cuda.current_stream().cuda_stream
        ws = self._ws.get(key)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.int32, device="cuda")
            self._ws[key] = ws
        return ws[:need]

    def check_evk(self, evk):
        """The fused entry points read an evaluation key as ONE dense (d, 2, L+1+alpha, N)
        tensor (keys.EvalKey) on this context's device."""
        t = getattr(evk, "data", None)
        want = (self.params.ks.d, 2, self.L + 1 + self.alpha, self.N)
        if not isinstance(t, torch.Tensor) or tuple(t.shape) != want or t.dtype != torch.int32:
            raise _native.NativeError(f"evaluation key must be an int32 tensor of shape {want}, got "
                                      f"{getattr(t, 'shape', None)} {getattr(t, 'dtype', None)}")
        return t

    def rescale_workspace(self, level: int, batch: int = 1) -> torch.Tensor:
        nbytes = self._lib.lf_rescale_workspace_bytes(self.handle, level, batch)
        return torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.lf_ctx_destroy(self.handle)
        except Exception:
            pass

    # --- basis ids ---------------------------------------------------------------------
    def pidx(self, bid: int) -> int:
        return bid if bid < SPECIAL_BASE else self.L + 1 + (bid - SPECIAL_BASE)

    def prime(self, bid: int) -> int:
        return self.primes[self.pidx(bid)]

    def pidx_array(self, ids):
        ids = tuple(ids)
        arr = self._pidx.get(ids)
        if arr is None:
            arr = _native.i32_array([self.pidx(b) for b in ids])
            self._pidx[ids] = arr
        return arr

    # --- constant blobs ----------------------------------------------------------------
    def blob(self, key, builder):
        """Device-resident constant blob (int32 tensor) cached under `key`."""
        t = self._blobs.get(key)
        if t is None:
            host = builder()
            t = torch.from_numpy(np.ascontiguousarray(host).view(np.int32)).cuda()
            self._blobs[key] = t
        return t

    def bconv_table(self, src_ids, tgt_ids, extra=None):
        """(device blob, k, m, W) for exact conversion src -> tgt (poly.py:140-178).
        `extra[i]` (optional) is folded into the y-multiplier of source i."""
        src_ids, tgt_ids = tuple(src_ids), tuple(tgt_ids)
        extra = tuple(extra) if extra is not None else None
        key = ("bconv", src_ids, tgt_ids, extra)
        src = [self.prime(b) for b in src_ids]
        k, m = len(src_ids), len(tgt_ids)
        W = bconv_words(src)

        def build():
            return bconv_blob(src, [self.pidx(b) for b in src_ids],
                              [self.prime(b) for b in tgt_ids], [self.pidx(b) for b in tgt_ids],
                              extra)
        return self.blob(key, build), k, m, W


def bconv_words(src_primes) -> int:
    S = 1
    for s in src_primes:
        S *= s
    return (S.bit_length() + 31) // 32 + 1


def bconv_blob(src, src_pidx, tgt, tgt_pidx, extra=None) -> np.ndarray:
    """Host build of the BConv table blob (layout: lf_bconv.cuh / DESIGN.md):
    inv_s f64[k] | src_pi[k] | c[k] | c'[k] | tgt_pi[m] | negS[m] | w[m][k] | shat[k][W] | S[W]."""
    k, m = len(src), len(tgt)
    S = 1
    for s in src:
        S *= s
    W = bconv_words(src)
    inv_s = np.array([1.0 / s for s in src], dtype=np.float64).view(np.uint32)
    c = []
    for i, s in enumerate(src):
        v = pow(S // s, -1, s)
        if extra is not None:
            v = v * (extra[i] % s) % s
        c.append(v)
    cp = [(v << 32) // s for v, s in zip(c, src)]
    negS = [(t - S % t) % t for t in tgt]
    w = [[(S // s) % t for s in src] for t in tgt]      # target-major

    def words(x):
        return [(x >> (32 * i)) & 0xFFFFFFFF for i in range(W)]

    shat = [words(S // s) for s in src]
    parts = [inv_s, np.array(src_pidx, np.uint32), np.array(c, np.uint32), np.array(cp, np.uint32),
             np.array(tgt_pidx, np.uint32), np.array(negS, np.uint32),
             np.array(w, np.uint32).reshape(-1), np.array(shat, np.uint32).reshape(-1),
             np.array(words(S), np.uint32)]
    blob = np.concatenate([p.astype(np.uint32) for p in parts])
    assert blob.size == 5 * k + 2 * m + k * m + k * W + W
    return blob


_CTX = {}


def get_context(params: CkksParams) -> DeviceContext:
    """One context per (parameter set, device): tables and plans live on the device that was
    current when the context was built."""
    require_cuda()
    key = (params, torch.cuda.current_device())
    ctx = _CTX.get(key)
    if ctx is None:
        ctx = DeviceContext(params)
        _CTX[key] = ctx
    return ctx
