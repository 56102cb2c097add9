"""Frozen numeric tolerances of the reference (tolerance.py:1-13)."""

DEPTH4_TAU = 0.2876
ENCODE_ROUNDTRIP = 2.0 ** -12
OP_TOL = 0.05  # single-op decryption bound used by the reference tests (test_ckks_ops.py:27)
