"""Host-side NTT helpers that stay on the CPU in the reference as well: the Galois element of a
rotation and the automorphism index table (ntt.py:108-132).  The transforms themselves run on
the GPU (poly.ntt_rows)."""

from functools import lru_cache

import numpy as np

from .modmath import bit_reverse_indices


@lru_cache(maxsize=None)
def automorphism_permutation(N: int, g: int) -> np.ndarray:
    """perm[i] = brv(((2 brv(i) + 1) g mod 2N - 1)/2); eval-domain gather x[..., perm]."""
    if g % 2 == 0:
        raise ValueError("automorphism index must be odd")
    rev = bit_reverse_indices(N)
    e = (2 * rev + 1) * g % (2 * N)
    return rev[(e - 1) // 2]


@lru_cache(maxsize=None)
def galois_element(N: int, steps: int) -> int:
    """Automorphism index of a cyclic left rotation by `steps` slots: 5^steps mod 2N."""
    return pow(5, steps % (N // 2), 2 * N)
