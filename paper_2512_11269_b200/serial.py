"""LFHE serialisation straight into / out of device memory (reference
serial.py:1-209).

Same wire layout as the reference, byte for byte (little-endian):

    magic "LFHE" | version u16 | kind u8 | N u32 | count u16 | primes u64[count] |
    level u8 | scale f64 | domain u8 | kind-specific payload, limb rows as u64[N]

Two layers:
  * host layer (`pack_*` / `parse_*`): header and payload on numpy uint64 rows, no device;
  * device layer (`*_to_bytes` / `*_from_bytes`): the u64 rows travel as raw bytes through a
    pinned staging buffer and are narrowed to / widened from the device's u32 residues by the
    `lf_rows_from_u64` / `lf_rows_to_u64` kernels, so a 90 MiB key lands in HBM with one copy
    and one kernel instead of a host-side conversion.
"""

from __future__ import annotations

import struct
from fractions import Fraction

import numpy as np

MAGIC = b"LFHE"
VERSION = 1
KIND_POLY, KIND_PLAINTEXT, KIND_CIPHERTEXT, KIND_SECRET, KIND_EVALKEY, KIND_COMPRESSED = range(6)

_HEADER = struct.Struct("<4sHBIH")
_TAIL = "<Bd B"


# ------------------------------------------------------------------------------------------
# host layer (serial.py:42-69)
# ------------------------------------------------------------------------------------------

def pack_header(kind, N, primes, level, scale, domain) -> bytes:
    return (_HEADER.pack(MAGIC, VERSION, kind, N, len(primes)) +
            np.asarray(primes, dtype="<u8").tobytes() +
            struct.pack(_TAIL, level & 0xFF, float(scale), domain))


def parse_header(data, off=0):
    magic, version, kind, N, count = _HEADER.unpack_from(data, off)
    if magic != MAGIC:
        raise ValueError("not a limbforge LFHE blob")
    if version != VERSION:
        raise ValueError(f"unsupported version {version}")
    off += _HEADER.size
    primes = tuple(int(p) for p in np.frombuffer(data, dtype="<u8", count=count, offset=off))
    off += 8 * count
    level, scale, domain = struct.unpack_from(_TAIL, data, off)
    off += struct.calcsize(_TAIL)
    return kind, N, primes, level, scale, domain, off


def detect_kind(data) -> int:
    return parse_header(data)[0]


def ids_for_primes(params, primes) -> tuple:
    """serial.py:82-88: basis ids by prime value (main i, special 65536 + j)."""
    from .context import SPECIAL_BASE
    lookup = {q: i for i, q in enumerate(params.rns_basis)}
    lookup.update({q: SPECIAL_BASE + j for j, q in enumerate(params.special_basis)})
    unknown = [q for q in primes if q not in lookup]
    if unknown:
        raise ValueError(f"LFHE blob primes {unknown[:3]} are not in this parameter set's basis")
    return tuple(lookup[q] for q in primes)


def _check_blob(params, N, primes, expected_ids=None, what="blob"):
    """Reject blobs built for other parameters before anything reaches the device: the fused
    kernels index device rows with the context's N, level and digit counts, so a foreign
    shape would be read out of bounds instead of failing like the reference's numpy code."""
    if N != params.N:
        raise ValueError(f"LFHE {what}: N={N} but the parameters have N={params.N}")
    if len(set(primes)) != len(primes):
        raise ValueError(f"LFHE {what}: repeated primes in the header")
    ids = ids_for_primes(params, primes)
    if expected_ids is not None and tuple(ids) != tuple(expected_ids):
        raise ValueError(f"LFHE {what}: basis {ids[:4]}... is not the expected {tuple(expected_ids)[:4]}...")
    return ids


def _check_residues(rows, primes, what):
    """Every residue below its prime (lf_rows_from_u64 narrows u64 -> u32 without a check)."""
    q = np.asarray(primes, dtype=np.uint64)
    if (rows.reshape(-1, len(primes), rows.shape[-1]) >= q[None, :, None]).any():
        raise ValueError(f"LFHE {what}: residue not below its prime")


def primes_for_ids(params, ids) -> list:
    from .poly import prime_for_id
    return [prime_for_id(params, b) for b in ids]


def rows_view(data, off, count, N):
    """Zero-copy view of `count` u64 rows at `off`; returns (view, end offset)."""
    return np.frombuffer(data, dtype="<u8", count=count * N, offset=off).reshape(count, N), off + 8 * count * N


# ------------------------------------------------------------------------------------------
# device layer
# ------------------------------------------------------------------------------------------

def _upload_rows(raw_u64: np.ndarray):
    """(n, N) little-endian u64 host rows -> (n, N) int32 device residues."""
    import torch
    from . import _native
    from .context import dptr, stream_handle
    n = raw_u64.size
    import warnings
    with warnings.catch_warnings():          # a read-only view of the blob: only read (pinned copy)
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(np.ascontiguousarray(raw_u64).view(np.int64)).reshape(raw_u64.shape)
    stage = host.pin_memory() if torch.cuda.is_available() else host
    wide = stage.to("cuda", non_blocking=True)
    out = torch.empty(raw_u64.shape, dtype=torch.int32, device="cuda")
    _native.check(_native.lib().lf_rows_from_u64(dptr(out), dptr(wide), n, stream_handle()),
                  "lf_rows_from_u64")
    return out


def _download_rows(rows) -> bytes:
    """(n, N) int32 device residues -> little-endian u64 bytes."""
    import torch
    from . import _native
    from .context import dptr, stream_handle
    rows = rows.contiguous()
    wide = torch.empty(rows.shape, dtype=torch.int64, device=rows.device)
    _native.check(_native.lib().lf_rows_to_u64(dptr(wide), dptr(rows), rows.numel(), stream_handle()),
                  "lf_rows_to_u64")
    return wide.cpu().numpy().astype("<u8").tobytes()


def poly_to_bytes(poly, params, scale=0.0, level=None, kind=KIND_POLY) -> bytes:
    from .poly import Domain
    level = len(poly.basis_ids) - 1 if level is None else level
    head = pack_header(kind, poly.N, primes_for_ids(params, poly.basis_ids), level, scale,
                       0 if poly.domain == Domain.COEFF else 1)
    return head + _download_rows(poly.limbs)


def poly_from_bytes(data, params):
    from .poly import Domain, RnsPolynomial
    kind, N, primes, level, scale, domain, off = parse_header(data)
    _check_blob(params, N, primes, what="polynomial")
    rows, off = rows_view(data, off, len(primes), N)
    _check_residues(rows, primes, "polynomial")
    poly = RnsPolynomial(_upload_rows(rows), Domain.COEFF if domain == 0 else Domain.EVAL,
                         ids_for_primes(params, primes))
    return kind, poly, level, scale, off


def plaintext_to_bytes(pt, params) -> bytes:
    return poly_to_bytes(pt.poly, params, scale=pt.scale, level=pt.level, kind=KIND_PLAINTEXT)


def plaintext_from_bytes(data, params):
    from .encoding import Plaintext
    from .poly import main_ids
    if detect_kind(data) != KIND_PLAINTEXT:
        raise ValueError(f"LFHE kind {detect_kind(data)} is not a plaintext")
    kind, poly, level, scale, _ = poly_from_bytes(data, params)
    if tuple(poly.basis_ids) != main_ids(level):
        raise ValueError(f"LFHE plaintext: basis does not match level {level}")
    return Plaintext(poly=poly, scale=Fraction(scale), level=level)


def ciphertext_to_bytes(ct, params) -> bytes:
    """serial.py:110-112: the b polynomial with the ciphertext header, then a's rows."""
    head = poly_to_bytes(ct.b, params, scale=ct.scale, level=ct.level, kind=KIND_CIPHERTEXT)
    return head + _download_rows(ct.a.limbs)


def ciphertext_from_bytes(data, params):
    from .ckks import Ciphertext
    from .poly import RnsPolynomial
    kind, N, primes, level, scale, domain, off = parse_header(data)
    if kind != KIND_CIPHERTEXT:
        raise ValueError(f"LFHE kind {kind} is not a ciphertext")
    from .poly import main_ids
    if level > params.max_level:
        raise ValueError(f"LFHE ciphertext: level {level} above the parameters' {params.max_level}")
    _check_blob(params, N, primes, main_ids(level), "ciphertext")
    rows, _ = rows_view(data, off, 2 * len(primes), N)         # b rows then a rows, one upload
    _check_residues(rows, primes, "ciphertext")
    dev = _upload_rows(rows)
    from .poly import Domain
    dom = Domain.COEFF if domain == 0 else Domain.EVAL
    ids = ids_for_primes(params, primes)
    n = len(primes)
    return Ciphertext(b=RnsPolynomial(dev[:n], dom, ids), a=RnsPolynomial(dev[n:], dom, ids),
                      scale=Fraction(scale), level=level)


def evalkey_to_bytes(evk, params) -> bytes:
    """serial.py:177-192: header, purpose tag, then per digit b rows and a rows."""
    if evk.purpose == "relin":
        tag, rot = 0, 0
    else:
        tag, rot = 1, evk.purpose[1]
    head = pack_header(KIND_EVALKEY, params.N, primes_for_ids(params, evk.ids), params.max_level,
                       0.0, 1)
    return head + struct.pack("<BIH", tag, rot, evk.data.shape[0]) + _download_rows(
        evk.data.reshape(-1, params.N))


def evalkey_from_bytes(data, params):
    """serial.py:195-209, into the (d, 2, rows, N) device layout of keys.EvalKey."""
    from .keys import EvalKey
    kind, N, primes, _, _, _, off = parse_header(data)
    if kind != KIND_EVALKEY:
        raise ValueError(f"LFHE kind {kind} is not an evaluation key")
    from .poly import extended_ids
    _check_blob(params, N, primes, extended_ids(params, params.max_level), "evaluation key")
    tag, rot, ndig = struct.unpack_from("<BIH", data, off)
    off += struct.calcsize("<BIH")
    if ndig != params.ks.d:
        raise ValueError(f"LFHE evaluation key: {ndig} digits but the parameters use d={params.ks.d}")
    if tag not in (0, 1):
        raise ValueError(f"LFHE evaluation key: purpose tag {tag}")
    rows, _ = rows_view(data, off, ndig * 2 * len(primes), N)
    _check_residues(rows, primes, "evaluation key")
    dev = _upload_rows(rows).view(ndig, 2, len(primes), N)
    purpose = "relin" if tag == 0 else ("rot", rot)
    return EvalKey(purpose, dev, ids_for_primes(params, primes))


def secret_to_bytes(sk, params) -> bytes:
    """serial.py:121-125: header over the main basis, then the ternary coefficients (i8)."""
    return pack_header(KIND_SECRET, params.N, params.rns_basis, params.max_level, 0.0, 0) + \
        np.asarray(sk.coeffs, dtype="<i1").tobytes()


def secret_from_bytes(data, params):
    from .encoding import signed_to_eval
    from .keys import SecretKey
    from .poly import extended_ids
    kind, N, primes, _, _, _, off = parse_header(data)
    if kind != KIND_SECRET:
        raise ValueError(f"LFHE kind {kind} is not a secret key")
    _check_blob(params, N, primes, what="secret key")
    coeffs = np.frombuffer(data, dtype="<i1", count=N, offset=off).copy()
    s_eval = signed_to_eval(coeffs.astype(np.int64), params, extended_ids(params, params.max_level))
    return SecretKey(coeffs=coeffs, s_eval=s_eval)


def compressed_to_bytes(cp, params) -> bytes:
    """serial.py:144-151: header over the main basis of cp.level, (stride, unique count), then
    the unique-value rows (u64)."""
    head = pack_header(KIND_COMPRESSED, params.N, params.rns_basis[: cp.level + 1], cp.level, cp.scale, 1)
    return head + struct.pack("<II", cp.descriptor.stride, cp.descriptor.unique_count) + \
        _download_rows(cp.unique)


def compressed_from_bytes(data, params):
    """serial.py:154-166, the unique rows straight into HBM (compress.CompressedPlaintext)."""
    from .compress import CompressedPlaintext, CompressionDescriptor
    from .poly import main_ids
    kind, N, primes, level, scale, _, off = parse_header(data)
    if kind != KIND_COMPRESSED:
        raise ValueError(f"LFHE kind {kind} is not a compressed plaintext")
    _check_blob(params, N, primes, main_ids(level), "compressed plaintext")
    stride, unique = struct.unpack_from("<II", data, off)
    off += struct.calcsize("<II")
    desc = CompressionDescriptor.for_params(params, stride)
    if desc.unique_count != unique:
        raise ValueError(f"LFHE compressed plaintext: {unique} unique values, stride {stride} implies "
                         f"{desc.unique_count}")
    rows = np.frombuffer(data, dtype="<u8", count=len(primes) * unique, offset=off).reshape(len(primes), unique)
    _check_residues(rows, primes, "compressed plaintext")
    return CompressedPlaintext(unique=_upload_rows(rows), descriptor=desc, scale=Fraction(scale), level=level)


def load_plaintext_auto(data, params):
    """serial.py:169-174: dense or compressed plaintext, dispatched on the header's kind."""
    if detect_kind(data) == KIND_COMPRESSED:
        return compressed_from_bytes(data, params)
    return plaintext_from_bytes(data, params)


def evalkey_shard_from_bytes(data, params, k: int, rank: int):
    """This rank's rows of an LFHE evaluation key, uploaded straight from the blob: only the
    rows the limb-sharded pipeline reads on `rank` of `k` (main row i on rank i % k, special j
    on rank j % k, multidev.py:55-56) cross PCIe; returns (purpose, (d, 2, n_key_rows, N))."""
    from .poly import extended_ids
    kind, N, primes, _, _, _, off = parse_header(data)
    if kind != KIND_EVALKEY:
        raise ValueError(f"LFHE kind {kind} is not an evaluation key")
    _check_blob(params, N, primes, extended_ids(params, params.max_level), "evaluation key")
    tag, rot, ndig = struct.unpack_from("<BIH", data, off)
    off += struct.calcsize("<BIH")
    if ndig != params.ks.d:
        raise ValueError(f"LFHE evaluation key: {ndig} digits but the parameters use d={params.ks.d}")
    L, alpha = params.max_level, params.num_special
    local = list(range(rank, L + 1, k)) + [L + 1 + j for j in range(rank, alpha, k)]
    rows, _ = rows_view(data, off, ndig * 2 * len(primes), N)
    rows = rows.reshape(ndig, 2, len(primes), N)[:, :, local]
    _check_residues(np.ascontiguousarray(rows).reshape(-1, N), [primes[i] for i in local], "evaluation key")
    dev = _upload_rows(np.ascontiguousarray(rows).reshape(-1, N)).view(ndig, 2, len(local), N)
    return ("relin" if tag == 0 else ("rot", rot)), dev
