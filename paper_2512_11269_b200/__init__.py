"""paper_2512_11269_b200 — B200-native CKKS core behind the reference `limbforge` operator API.

Python host code mirroring `limbforge` (/root/reference/pkg/src/limbforge/__init__.py:10-34)
over hand-written sm_100a CUDA kernels reached through the C ABI of libcerium_b200.so
(include/lf_b200.h).  There is no CPU fallback: every homomorphic operation runs on the GPU.
"""

from .params import CkksParams, KeySwitchConfig, gen_params
from .poly import Domain, RnsPolynomial
from .encoding import Plaintext, decode, encode
from .keys import (EvalKey, PublicKey, SecretKey, keygen, make_conjugation_key, make_galois_key,
                   make_rotation_key)
from .ckks import (Ciphertext, add_plain, apply_galois, decrypt, encrypt, hom_add, hom_conjugate,
                   hom_mul, hom_rotate, hom_rotate_hoisted, hom_sub, keyswitch, keyswitch_decompose,
                   keyswitch_inner_product, mul_plain, rescale)

__all__ = [
    "CkksParams", "KeySwitchConfig", "gen_params",
    "Plaintext", "decode", "encode",
    "EvalKey", "PublicKey", "SecretKey", "keygen", "make_rotation_key", "make_conjugation_key",
    "make_galois_key",
    "Ciphertext", "add_plain", "decrypt", "encrypt", "hom_add", "hom_mul", "hom_rotate",
    "hom_sub", "mul_plain", "rescale", "keyswitch", "keyswitch_decompose",
    "keyswitch_inner_product", "apply_galois", "hom_conjugate", "hom_rotate_hoisted",
    "Domain", "RnsPolynomial",
]

__version__ = "0.1.0"
