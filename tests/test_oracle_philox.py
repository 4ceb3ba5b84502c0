"""Philox4x32-10 known-answer vectors (Random123 kat_vectors) and draw statistics."""
import numpy as np

KAT = [  # (ctr, key, expected) -- Random123 "philox4x32_10" known-answer vectors
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
]


def test_philox_kat(oracle_mod):
    for ctr, key, exp in KAT:
        assert oracle_mod.philox4x32_10(ctr, key) == exp


def test_secret_is_ternary_uniform(oracle_mod):
    o = oracle_mod.Oracle(12, 3)
    s, s_ntt = o.secret_key()
    vals, counts = np.unique(s, return_counts=True)
    assert list(vals) == [-1, 0, 1]
    assert (np.abs(counts / o.n - 1 / 3) < 0.03).all()
    # s_ntt is the NTT of s in every modulus
    for l, m in enumerate(o.p.moduli):
        assert (o.ntt(s_ntt[l], l, inverse=True) == np.array([x % m for x in s.tolist()], dtype=np.uint64)).all()
