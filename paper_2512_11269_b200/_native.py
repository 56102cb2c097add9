"""ctypes binding of libcerium_b200.so (the C ABI declared in include/lf_b200.h).

The product path has no CPU fallback: importing this module on a machine without the built
library, or calling into it without a CUDA device, raises immediately.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LF_LIB_PATH") or os.path.join(_HERE, "libcerium_b200.so")

_u32p = ctypes.c_void_p          # device pointers are passed as raw addresses
_i32_host = ctypes.POINTER(ctypes.c_int32)
_u32_host = ctypes.POINTER(ctypes.c_uint32)


class NativeError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise NativeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "lf_shard_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
        "lf_shard_destroy": (ctypes.c_int, [ctypes.c_void_p]),
        "lf_shard_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 4),
        "lf_shard_ws_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_shard_gather_layout": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
        "lf_shard_ks_phase": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_comm_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
        "lf_comm_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
        "lf_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
        "lf_shard_attach_comm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
        "lf_shard_keyswitch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_abi_version": (ctypes.c_int, []),
        "lf_last_error": (ctypes.c_char_p, []),
        "lf_set_bconv_engine": (ctypes.c_int, [ctypes.c_int]),
        "lf_get_bconv_engine": (ctypes.c_int, []),
        "lf_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _u32_host, _u32_host,
                                         ctypes.POINTER(ctypes.c_void_p)]),
        "lf_ctx_destroy": (ctypes.c_int, [ctypes.c_void_p]),
        "lf_ntt_fwd": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, _i32_host, ctypes.c_void_p]),
        "lf_ntt_inv": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, _i32_host, ctypes.c_void_p]),
        "lf_ewise": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, _u32p, _u32p, _u32p,
                                    ctypes.c_int, _i32_host, _u32_host, ctypes.c_void_p]),
        "lf_automorph": (ctypes.c_int, [ctypes.c_void_p, _u32p, _u32p, ctypes.c_uint32, ctypes.c_int,
                                        ctypes.c_void_p]),
        "lf_bconv": (ctypes.c_int, [ctypes.c_void_p, _u32p, _u32p, _u32p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_void_p]),
        "lf_ctx_enable_keyswitch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_ks_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_keyswitch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, _u32p,
                                        ctypes.c_size_t, _u32p, ctypes.c_size_t, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]),
        "lf_keyswitch_profiled": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, _u32p,
                                                 ctypes.c_size_t, _u32p, ctypes.c_size_t, ctypes.c_int,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]),
        "lf_hom_mul": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, _u32p, ctypes.c_size_t, _u32p,
                                      _u32p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_hom_mul_rescale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, _u32p,
                                              ctypes.c_size_t, _u32p, _u32p, ctypes.c_size_t, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p]),
        "lf_hom_mul_rescale_p": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, ctypes.c_size_t,
                                                ctypes.c_int, _u32p, ctypes.c_size_t, ctypes.c_int, _u32p, _u32p,
                                                ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_hom_mul_rescale_list": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_void_p, _u32p, _u32p,
                                                   ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_moddown_ext_rescale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, ctypes.c_size_t,
                                                  _u32p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rescale_multi_p": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, ctypes.c_size_t,
                                              ctypes.c_int, _u32p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                              ctypes.c_void_p]),
        "lf_rotate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, ctypes.c_uint32,
                                     _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rotate_hoisted_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_rotate_hoisted": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_int, _u32_host,
                                             ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_size_t,
                                             ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rotate_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, ctypes.c_int,
                                           _u32_host, ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_size_t,
                                           ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rotate_batch_pk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, ctypes.c_int,
                                              _u32_host, ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_size_t,
                                              ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rescale_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_rescale": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, _u32p,
                                      ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rescale_multi": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, ctypes.c_size_t,
                                            _u32p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_lincomb": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                      _u32_host, ctypes.c_void_p]),
        "lf_lincomb_c": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                        _u32_host, _u32_host, ctypes.c_void_p]),
        "lf_rows_from_u64": (ctypes.c_int, [_u32p, _u32p, ctypes.c_size_t, ctypes.c_void_p]),
        "lf_rows_to_u64": (ctypes.c_int, [_u32p, _u32p, ctypes.c_size_t, ctypes.c_void_p]),
        "lf_rotate_hoisted_ext": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_int, _u32_host,
                                                 ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_size_t,
                                                 ctypes.c_void_p, ctypes.c_void_p]),
        "lf_rotate_hoisted_ext_pk": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_int, _u32_host,
                                                    ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_size_t,
                                                    ctypes.c_void_p, ctypes.c_void_p]),
        "lf_bsgs_ext": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_int, _u32_host,
                                       ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_void_p), _u32p, ctypes.c_void_p,
                                       ctypes.c_void_p]),
        "lf_plan_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
        "lf_moddown_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
        "lf_moddown_ext": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, ctypes.c_size_t, _u32p,
                                          ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
        "lf_ptmac_rows": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, _i32_host, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]),
        "lf_mul_compressed": (ctypes.c_int, [ctypes.c_void_p, _u32p, _u32p, _u32p, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_void_p]),
        "lf_ks_decompose": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _u32p, _u32p, ctypes.c_void_p,
                                           ctypes.c_void_p]),
        "lf_modraise": (ctypes.c_int, [ctypes.c_void_p, _u32p, _u32p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_void_p]),
        "lf_ptmac": (ctypes.c_int, [ctypes.c_void_p, _u32p, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib, sig


_LIB = None
EXPORTS = ()


def lib():
    global _LIB, EXPORTS
    if _LIB is None:
        _LIB, sig = _load()
        EXPORTS = tuple(sig)
    return _LIB


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = lib().lf_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (rc={rc}): {msg}")


def i32_array(values):
    arr = (ctypes.c_int32 * len(values))(*[int(v) for v in values])
    return arr


def u32_array(values):
    return (ctypes.c_uint32 * len(values))(*[int(v) & 0xFFFFFFFF for v in values])
