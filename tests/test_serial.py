"""LFHE wire format (reference serial.py:1-209) — golden blobs written by the real reference
(tests/golden/make_lfhe.py).  CPU: header/payload parsing and byte-exact re-packing.  GPU:
blobs load straight into device memory (u64 -> u32 kernel), decrypt / match this package's
own keys and ciphertexts, and serialise back to the identical bytes."""

import numpy as np
import pytest

from conftest import load_npz
from paper_2512_11269_b200 import serial as S


@pytest.fixture(scope="module")
def blobs():
    z = load_npz("lfhe_small.npz")
    return {k: z[k].tobytes() for k in z.files}


def test_headers(blobs, golden_params):
    main = golden_params["small"]["params"]["main"]
    special = golden_params["small"]["params"]["special"]
    kind, N, primes, level, scale, domain, off = S.parse_header(blobs["ciphertext"])
    assert (kind, N, list(primes), level, scale, domain) == (S.KIND_CIPHERTEXT, 256, main, 4, 2.0 ** 20, 1)
    assert len(blobs["ciphertext"]) == off + 2 * 5 * 256 * 8
    kind, N, primes, level, scale, domain, off = S.parse_header(blobs["relin"])
    assert kind == S.KIND_EVALKEY and list(primes) == main + special
    assert S.detect_kind(blobs["secret"]) == S.KIND_SECRET
    assert S.detect_kind(blobs["plaintext"]) == S.KIND_PLAINTEXT
    with pytest.raises(ValueError):
        S.parse_header(b"XXXX" + blobs["secret"][4:])


@pytest.mark.parametrize("name", ["ciphertext", "plaintext", "relin", "rot1", "secret"])
def test_repack_is_byte_exact(blobs, name):
    data = blobs[name]
    kind, N, primes, level, scale, domain, off = S.parse_header(data)
    assert S.pack_header(kind, N, primes, level, scale, domain) == data[:off]
    rest = data[off:]
    if kind == S.KIND_EVALKEY:
        rest = rest[7:]
    if kind != S.KIND_SECRET:
        rows = np.frombuffer(rest, dtype="<u8").reshape(-1, N)
        q = np.array(primes, dtype=np.uint64)
        assert (rows.reshape(-1, len(primes), N) < q[None, :, None]).all()   # canonical residues


@pytest.mark.gpu
def test_device_roundtrip_and_parity(blobs, golden_params):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    p = B.gen_params(**golden_params["small"]["kwargs"])
    sk, pk, rlk = B.keygen(p, seed=11)
    rk = B.make_rotation_key(p, sk, 1, np.random.default_rng(5))
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, p.n)
    w = rng.uniform(-1, 1, p.n)
    ct = B.encrypt(B.encode(v, p), pk, p, np.random.default_rng(1))
    # load: device objects equal this package's own (bit-exact with the reference)
    ct2 = S.ciphertext_from_bytes(blobs["ciphertext"], p)
    assert np.array_equal(ct2.b.numpy(), ct.b.numpy()) and np.array_equal(ct2.a.numpy(), ct.a.numpy())
    assert ct2.scale == ct.scale and ct2.level == ct.level
    k2 = S.evalkey_from_bytes(blobs["relin"], p)
    assert k2.purpose == "relin" and torch.equal(k2.data, rlk.data)
    r2 = S.evalkey_from_bytes(blobs["rot1"], p)
    assert r2.purpose == rk.purpose and torch.equal(r2.data, rk.data)
    sk2 = S.secret_from_bytes(blobs["secret"], p)
    assert torch.equal(sk2.s_eval.limbs, sk.s_eval.limbs)
    pt2 = S.plaintext_from_bytes(blobs["plaintext"], p)
    assert np.array_equal(pt2.poly.numpy(), B.encode(w, p, level=2).poly.numpy())
    # store: identical bytes
    assert S.ciphertext_to_bytes(ct, p) == blobs["ciphertext"]
    assert S.evalkey_to_bytes(rlk, p) == blobs["relin"]
    assert S.evalkey_to_bytes(rk, p) == blobs["rot1"]
    assert S.secret_to_bytes(sk, p) == blobs["secret"]
    assert S.plaintext_to_bytes(pt2, p) == blobs["plaintext"]
    # loaded objects compute: rotate with the loaded key, decrypt with the loaded secret
    dec = B.decrypt(B.hom_rotate(ct2, 1, r2, p), sk2, p)
    assert np.abs(dec - np.roll(v, -1)).max() < 0.05


def test_foreign_blobs_rejected_before_upload(blobs, golden_params):
    """Blobs for other parameters fail on the host with ValueError, never reach the device
    (the fused kernels would index them with this context's shapes)."""
    from paper_2512_11269_b200.params import gen_params
    p = gen_params(**golden_params["small"]["kwargs"])
    other_n = gen_params(512, 4, d=3, seed=3)
    other_d = gen_params(256, 4, d=2, seed=3)
    with pytest.raises(ValueError, match="N="):
        S.ciphertext_from_bytes(blobs["ciphertext"], other_n)
    with pytest.raises(ValueError):
        S.evalkey_from_bytes(blobs["relin"], other_d)
    with pytest.raises(ValueError, match="not in this parameter set"):
        S.plaintext_from_bytes(blobs["plaintext"], gen_params(256, 4, d=3, seed=3, scale=2 ** 24))
    with pytest.raises(ValueError, match="is not a ciphertext"):
        S.ciphertext_from_bytes(blobs["plaintext"], p)
    # a residue >= its prime
    kind, N, primes, level, scale, domain, off = S.parse_header(blobs["ciphertext"])
    bad = bytearray(blobs["ciphertext"])
    bad[off: off + 8] = np.array([primes[0]], dtype="<u8").tobytes()
    with pytest.raises(ValueError, match="residue"):
        S.ciphertext_from_bytes(bytes(bad), p)
    # a ciphertext header whose primes are not main 0..level
    hdr = S.pack_header(S.KIND_CIPHERTEXT, N, primes[:3], 3, scale, domain)
    with pytest.raises(ValueError, match="basis"):
        S.ciphertext_from_bytes(hdr + blobs["ciphertext"][off:], p)


def test_compressed_blob_layout(blobs, golden_params):
    kind, N, primes, level, scale, domain, off = S.parse_header(blobs["compressed"])
    assert kind == S.KIND_COMPRESSED and level == 3 and len(primes) == 4
    assert S.detect_kind(blobs["compressed"]) == S.KIND_COMPRESSED


@pytest.mark.gpu
def test_compressed_roundtrip_byte_exact(blobs, golden_params):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_11269_b200 as B
    from paper_2512_11269_b200 import compress as CP
    p = B.gen_params(**golden_params["small"]["kwargs"])
    cp = S.load_plaintext_auto(blobs["compressed"], p)
    assert isinstance(cp, CP.CompressedPlaintext) and cp.descriptor.stride == 8 and cp.level == 3
    own = CP.encode_compressed(np.tile(np.linspace(-0.5, 0.75, 8), p.n // 8), p, stride=8, level=3)
    assert torch.equal(cp.unique, own.unique) and cp.scale == own.scale
    assert S.compressed_to_bytes(cp, p) == blobs["compressed"]
    assert S.compressed_to_bytes(own, p) == blobs["compressed"]
    assert isinstance(S.load_plaintext_auto(blobs["plaintext"], p), B.Plaintext)
