"""Pins for Alg. enroller_bsgs: the paper's worked example,
SPEC.md S:L273, floor-vs-truncation (R3), reconstruction, and the key set."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))


@pytest.fixture(scope="module")
def worked(oracle_mod):
    w = GOLD["paper"]
    o = oracle_mod.Oracle(16, 3)       # numSlots = 32768
    assert o.ns == w["numSlots"]
    rng = np.random.default_rng(11)
    shape = (w["numVectors"], w["VECTOR_DIM"])       # nonzero components: occupancy is checkable
    vecs = (rng.integers(1, 100, size=shape) * rng.choice([-1, 1], size=shape)).astype(np.float32)
    U = o.normalize_rows(vecs)
    return o, w, U


def test_worked_example_slot_map(worked):
    o, w, U = worked
    N, n1 = w["N"], w["n1"]
    for k in (0, 1, 256, 300, 511):
        z = o.enroll_slots(U, 0, w["numVectors"], n1, 0, k)
        for lo, hi in w["zero_slot_ranges"]:
            assert not z[lo:hi + 1].any()
        for lo, hi in w["group_slot_ranges"]:
            assert np.count_nonzero(z[lo:hi + 1]) == N
    # diagonal 0 of group 0 = [v0[0], v1[1], ..., v511[511]], shiftN = 0
    z0 = o.enroll_slots(U, 0, w["numVectors"], n1, 0, 0)
    assert (z0[:N] == np.array([U[j, j] for j in range(N)])).all()
    assert (z0[1024:1024 + N] == np.array([U[512 + j, j] for j in range(N)])).all()
    # aggregate count A = 1: aggregate 1 does not exist
    with pytest.raises(Exception):
        o.enroll_slots(U, 0, w["numVectors"], n1, 1, 0)


def test_worked_example_preshift(worked):
    o, w, U = worked
    N, n1 = w["N"], w["n1"]
    for s in w["shifts"] + [GOLD["floor_vs_trunc"]]:
        k, shift = s["k"], s["shiftN"]
        z = o.enroll_slots(U, 0, w["numVectors"], n1, 0, k)
        diag = np.array([U[t, (t + k) % N] for t in range(N)])
        assert (z[:N] == np.roll(diag, shift)).all()     # right shift by shiftN within the block


def test_spec_S_L273(oracle_mod):
    s = GOLD["spec_S_L273"]
    o = oracle_mod.Oracle(4, 3)                       # numSlots = 8 -> M = 2 blocks of N = 4
    vecs = np.arange(1, 17, dtype=np.float32).reshape(4, 4)
    U = o.normalize_rows(vecs)
    d = [np.array([U[t, (t + s["k"]) % 4] for t in range(4)])]
    z = o.enroll_slots(U, 0, 4, s["n1"], 0, s["k"])
    order = [int(x[1]) for x in s["stored_order"]]
    assert (z[:4] == d[0][order]).all()


@pytest.mark.parametrize("K,log_n,dim,n1", [(256, 12, 64, 8), (320, 8, 8, 2), (264, 9, 16, 4), (1280, 11, 32, 8)])
def test_reconstruct_vectors_from_diagonals(oracle_mod, K, log_n, dim, n1):
    """Undo shift and diagonalisation: every vector comes back exactly, gaps are zero."""
    o = oracle_mod.Oracle(log_n, 3)
    rng = np.random.default_rng(K)
    vecs = rng.integers(-99, 100, size=(K, dim)).astype(np.float32)
    U = o.normalize_rows(vecs)
    N, ns = dim, o.ns
    M = ns // N
    G = -(-K // N)
    A = -(-2 * G // M)
    rec = np.zeros((A * (M // 2) * N, N))
    for a in range(A):
        for k in range(N):
            z = o.enroll_slots(U, 0, K, n1, a, k)
            ks = k if k < N // 2 else k - N
            shift = (n1 * (ks // n1)) % N
            for b in range(M // 2):
                blk = z[b * 2 * N: b * 2 * N + N]
                assert not z[b * 2 * N + N: b * 2 * N + 2 * N].any()   # gap blocks are zero
                diag = np.roll(blk, -shift)
                for t in range(N):
                    rec[(a * (M // 2) + b) * N + t, (t + k) % N] = diag[t]
    assert (rec[:K] == U).all() and not rec[K:].any()


def test_zero_vector_and_layout_errors(oracle_mod):
    o = oracle_mod.Oracle(8, 3)
    v = np.zeros((3, 16), dtype=np.float32)
    v[0, 0] = 1
    with pytest.raises(oracle_mod.OracleError) as e:
        o.normalize_rows(v)
    assert e.value.code == oracle_mod.OR_E_ZERO_VECTOR
    with pytest.raises(oracle_mod.OracleError) as e:     # numSlots mod 2N != 0 -> layout error (R19)
        o.query_slots(np.ones(128, dtype=np.float32))
    assert e.value.code == oracle_mod.OR_E_LAYOUT


def test_rotation_key_set(oracle_mod):
    o = oracle_mod.Oracle(15, 3)
    for n1 in (4, 8, 16, 23, 32, 64):
        steps = o.rotation_steps(512, n1)
        jmin, jmax = o.giant_range(512, n1)
        giant = {o.pre_rot(512, n1, j) for j in range(jmin, jmax + 1)} - {0}
        assert set(range(1, n1)) <= set(steps)                    # S_baby
        assert len(steps) == len(set(range(1, n1)) | giant | {o.ns - 512})
    # n1 = 23, l = 512: |S_baby| = 22 as printed; signed giant range covers
    # k_signed in [-N/2, N/2) exactly once with 24 giant steps (R6)
    jmin, jmax = o.giant_range(512, 23)
    assert (jmin, jmax) == (-12, 11)
    cover = sorted(j * 23 + i for j in range(jmin, jmax + 1) for i in range(23)
                   if -256 <= j * 23 + i < 256)
    assert cover == list(range(-256, 256))
    # C2/C3 (n1 = 16): 15 + 31 + 1 = 47 keys
    assert len(o.rotation_steps(512, 16)) == 47
