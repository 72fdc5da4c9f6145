"""Bank checkpoint / resume.

CPU: the SHA-256 used for payload digests against FIPS 180-4 known answers
and hashlib.  GPU: save -> load is bit-exact (parameters and Adam state),
training resumed from a checkpoint matches uninterrupted training bit for
bit, and the distinct load errors (digest, version, truncation).
"""
import hashlib
import os

import numpy as np
import pytest
import torch


def test_sha256_known_answers():
    from paper_2011_09463_b200 import api

    assert api.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert api.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert api.sha256(b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq").hex() == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"
    assert api.sha256(b"a" * 1000000).hex() == \
        "cdc76e5c9914fb9281a1c7e284d73e67f1809a48a497200e046d39ccc7112cd0"
    rng = np.random.default_rng(1)
    for n in list(range(0, 130)) + [1000, 4095, 4096, 65537]:
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert api.sha256(data) == hashlib.sha256(data).digest(), n


def _bank(ctx, dims, G=3, seed=5):
    from paper_2011_09463_b200 import api

    bank = api.Bank(ctx, G, dims)
    r = api.Rng(seed)
    for g in range(G):
        bank.init_params(g, r)
    return bank


def _data(G, B, d0, C, seed=1):
    g = torch.Generator().manual_seed(seed)
    X = torch.randn(G, B, d0, generator=g).cuda()
    y = torch.randint(0, C, (G, B), generator=g, dtype=torch.int32).cuda()
    return X, y


@pytest.mark.gpu
@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
def test_save_load_resume_bit_exact(ctx, tmp_path, optimizer):
    from paper_2011_09463_b200 import api

    dims = [64, 48, 40, 10]
    X, y = _data(3, 50, 64, 10)
    kw = dict(lr=0.05 if optimizer == "sgd" else 0.01, optimizer=optimizer, want_loss=False)
    a = _bank(ctx, dims)
    for _ in range(2):
        a.train_step(X, y, **kw)
    path = os.path.join(tmp_path, "bank.ckpt")
    a.save(path)
    b = api.Bank.load(ctx, path)
    assert (b.G, b.dims, b.n_heads) == (a.G, a.dims, a.n_heads)
    for g in range(3):
        for x, z in zip(a.get_params(g)[0] + a.get_params(g)[1], b.get_params(g)[0] + b.get_params(g)[1]):
            assert np.array_equal(x, z)
    for _ in range(3):  # resume: identical trajectories, incl. Adam moments and step count
        a.train_step(X, y, **kw)
        b.train_step(X, y, **kw)
    for g in range(3):
        for x, z in zip(a.get_params(g)[0] + a.get_params(g)[1], b.get_params(g)[0] + b.get_params(g)[1]):
            assert np.array_equal(x, z)


@pytest.mark.gpu
def test_load_errors(ctx, tmp_path):
    from paper_2011_09463_b200 import api, errors

    a = _bank(ctx, [16, 12, 4], G=2)
    path = os.path.join(tmp_path, "bank.ckpt")
    a.save(path)
    raw = open(path, "rb").read()
    hdr_end = raw.index(b"\n\n") + 2
    # one corrupted payload byte -> digest error
    bad = bytearray(raw)
    bad[hdr_end + 40] ^= 0x01
    p2 = os.path.join(tmp_path, "digest.ckpt")
    open(p2, "wb").write(bytes(bad))
    with pytest.raises(errors.DigestError):
        api.Bank.load(ctx, p2)
    # a future format_version -> version error naming both versions
    p3 = os.path.join(tmp_path, "version.ckpt")
    open(p3, "wb").write(raw.replace(b"MTKBANK 2\n", b"MTKBANK 3\n", 1))
    with pytest.raises(errors.VersionError, match="3.*2"):
        api.Bank.load(ctx, p3)
    # truncated payload -> truncation error (a CheckpointError and a DataError)
    p4 = os.path.join(tmp_path, "trunc.ckpt")
    open(p4, "wb").write(raw[:-10])
    with pytest.raises(errors.TruncatedError):
        api.Bank.load(ctx, p4)
    assert issubclass(errors.TruncatedError, errors.CheckpointError)
    assert issubclass(errors.CheckpointError, errors.DataError)


@pytest.mark.gpu
def test_header_is_digested_and_strictly_parsed(ctx, tmp_path):
    """The SHA-256 covers the config lines too (a corrupted Adam step count
    would change the bias correction on resume); integers parse strictly."""
    from paper_2011_09463_b200 import api, errors

    a = _bank(ctx, [16, 12, 4], G=2)
    X, y = _data(2, 20, 16, 4)
    a.train_step(X, y, lr=0.01, optimizer="adam", want_loss=False)
    path = os.path.join(tmp_path, "bank.ckpt")
    a.save(path)
    raw = open(path, "rb").read()
    assert b"\nadam 1 1\n" in raw
    cases = {"step": (b"\nadam 1 1\n", b"\nadam 1 2\n", errors.DigestError),
             "garbage": (b"\nG 2\n", b"\nG 2x\n", errors.CheckpointError),
             "negative": (b"\nheads 1\n", b"\nheads -1\n", errors.CheckpointError),
             "missing": (b"\nheads 1\n", b"\n", errors.CheckpointError)}
    for name, (old, new, exc) in cases.items():
        p = os.path.join(tmp_path, name + ".ckpt")
        open(p, "wb").write(raw.replace(old, new, 1))
        with pytest.raises(exc):
            api.Bank.load(ctx, p)
    b = api.Bank.load(ctx, path)  # the untouched file still loads
    assert b.dims == [16, 12, 4]
