"""Untrusted-input and object-lifetime checks of the C ABI (include/hd.h, serialisation).

* hd_ciphertext_import / hd_eval_keys_import reject a header whose payload size does not
  match its shape, residues >= q, and (keys) out-of-range or duplicate rotation steps;
* a database's cached rotation-key pointers are invalidated when hd_relin_keygen
  reallocates the key storage (query -> relin_keygen -> query stays bit-identical).
"""
import gc

import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2604_00546_b200 as hd  # noqa: E402

HD_E_FORMAT = -10


@pytest.fixture(scope="module")
def toy():
    cfg = CONFIGS["C1"]
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    steps = ctx.rotation_steps(cfg.dim, cfg.n1)
    sk, evk = ctx.keygen(steps)
    qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
    db = ctx.enroll(db_vecs, cfg.n1)
    return cfg, ctx, sk, evk, qct, db


def _expect_format(fn, *a):
    with pytest.raises(hd.HDError) as ei:
        fn(*a)
    assert ei.value.code == HD_E_FORMAT, str(ei.value)


def test_ciphertext_import_roundtrip_and_rejects(toy):
    cfg, ctx, sk, evk, qct, db = toy
    buf = ctx.ciphertext_export(qct)
    back = ctx.ciphertext_import(buf)
    assert (ctx.ciphertext_residues(back) == ctx.ciphertext_residues(qct)).all()
    hdr = buf[:64].copy()
    payload = int(hdr[32:40].view(np.uint64)[0])
    # a payload field larger than the shape implies (the overrun ADVICE r1 found), with a
    # buffer long enough that the old `bytes` check passed
    big = np.concatenate([buf, np.zeros(4096, np.uint8)])
    big[32:40] = np.array([payload + 4096], np.uint64).view(np.uint8)
    _expect_format(ctx.ciphertext_import, big)
    # smaller payload field
    small = buf.copy()
    small[32:40] = np.array([payload - 8], np.uint64).view(np.uint8)
    _expect_format(ctx.ciphertext_import, small)
    # truncated buffer
    _expect_format(ctx.ciphertext_import, buf[:-8].copy())
    # one residue >= q (last coefficient of c1 at the top limb)
    bad = buf.copy()
    bad[-8:] = np.array([np.uint64(2 ** 64 - 1)], np.uint64).view(np.uint8)
    _expect_format(ctx.ciphertext_import, bad)
    # in-place import: header payload must match the target's shape too (HD_E_LEVEL)
    with pytest.raises(hd.HDError) as ei:
        ctx.ciphertext_import_into(back, small)
    assert ei.value.code == hd.HD_E_LEVEL


def test_eval_keys_import_rejects(toy):
    cfg, ctx, sk, evk, qct, db = toy
    buf = ctx.eval_keys_export(evk)
    k2 = ctx.eval_keys_import(buf)  # round trip accepted
    steps, keys = hd.eval_key_residues(ctx, ctx.eval_keys_export(k2))
    s0, k0 = hd.eval_key_residues(ctx, buf)
    assert list(steps) == list(s0) and (keys == k0).all()
    count = int(buf[20:24].view(np.uint32)[0])
    # count claims one more key than the payload holds (the over-read ADVICE r1 found)
    bad = buf.copy()
    bad[20:24] = np.array([count + 1], np.uint32).view(np.uint8)
    _expect_format(ctx.eval_keys_import, bad)
    # duplicate step
    dup = buf.copy()
    st = dup[64:64 + 4 * count].view(np.int32)
    st[1] = st[0]
    _expect_format(ctx.eval_keys_import, dup)
    # out-of-range step
    oor = buf.copy()
    oor[64:68] = np.array([ctx.n], np.int32).view(np.uint8)
    _expect_format(ctx.eval_keys_import, oor)
    # a key residue >= its modulus
    res = buf.copy()
    res[-8:] = np.array([np.uint64(2 ** 64 - 1)], np.uint64).view(np.uint8)
    _expect_format(ctx.eval_keys_import, res)


def test_query_after_relin_keygen_reallocation(toy):
    """hd_relin_keygen reallocates the key storage; the database's cached key pointers must
    follow it (keyed only on the evk address, the second query read freed memory)."""
    cfg, ctx, sk, evk, qct, db = toy
    evk2 = ctx.keygen(ctx.rotation_steps(cfg.dim, cfg.n1))[1]
    # a fresh key set: same secret (same seed) -> identical keys -> identical outputs
    a = [ctx.ciphertext_residues(o) for o in ctx.query(evk2, db, qct)]
    ctx.relin_keygen(sk, evk2)  # frees and reallocates evk2's key storage
    junk = torch.full((64 << 20,), 0x7F, dtype=torch.uint8, device="cuda")  # likely reuses the freed block
    b = [ctx.ciphertext_residues(o) for o in ctx.query(evk2, db, qct)]
    del junk
    for x, y in zip(a, b):
        assert (x == y).all()


def test_torch_allocator_owns_device_memory():
    """device memory comes from the caller's allocator (the torch caching
    allocator in the binding): enrolling a database grows torch's allocated bytes by the
    footprint hd_enroll_footprint reports, and destroying it returns them."""
    cfg = CONFIGS["C2"]
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    gc.collect()  # earlier tests' handles: free them now, not in the middle of the measurement
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    after_ctx = torch.cuda.memory_allocated(0)
    assert after_ctx > base  # the context's NTT / FFT tables live in torch memory
    need = ctx.enroll_footprint(cfg.num_vectors, cfg.dim, cfg.n1)
    db = ctx.enroll(db_vecs, cfg.n1)
    got = torch.cuda.memory_allocated(0) - after_ctx
    assert 0.95 * need <= got <= need + (64 << 20), (need, got)  # footprint: a conservative pre-check
    db.close()
    assert torch.cuda.memory_allocated(0) - after_ctx < (64 << 20)
    ctx.close()


def test_default_pool_allocator_matches_torch_allocator():
    """The same query with libhd's own stream-ordered pool (allocator=None) and with the
    torch allocator gives identical ciphertexts."""
    cfg = CONFIGS["C1"]
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    res = []
    for alloc in ("torch", None):
        ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1, allocator=alloc)
        sk, evk = ctx.keygen(ctx.rotation_steps(cfg.dim, cfg.n1))
        qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
        db = ctx.enroll(db_vecs, cfg.n1)
        res.append([ctx.ciphertext_residues(o) for o in ctx.query(evk, db, qct)])
    for a, b in zip(*res):
        assert (a == b).all()


def test_enroll_capacity_precheck():
    """a database that cannot fit is refused before any upload (HD_E_CAPACITY)."""
    cfg = CONFIGS["C1"]
    ctx = hd.Context(16, 3, seed=1)
    # 2^24 vectors x 512 at ring 2^16: 512 aggregates x 805 MB = 412 GB > 180 GB
    need = ctx.enroll_footprint(1 << 24, 512, 128)
    assert need > 400e9
    with pytest.raises(hd.HDError) as ei:
        ctx._precheck(1 << 24, 512, 128, 0, 0, "replicated", False)
    assert ei.value.code == hd.HD_E_CAPACITY
