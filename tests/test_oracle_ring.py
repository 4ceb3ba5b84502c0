"""Pins for the oracle's ring arithmetic (not gpu): primes, roots, NTT, automorphisms.

Each check is against something other than the oracle itself: primality by a
second independent test (sympy-free trial structure), the O(n^2) NTT
definition, schoolbook negacyclic convolution (the textbook product in
Z_q[X]/(X^n+1)), and the coefficient-domain definition of X -> X^g.
"""
import numpy as np
import pytest


def _py_is_prime(x):
    """Independent deterministic Miller-Rabin in pure Python big ints."""
    if x < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
    for p in small:
        if x % p == 0:
            return x == p
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(s - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


@pytest.mark.parametrize("log_n", [4, 12, 15, 16])
def test_moduli_are_the_pinned_primes(oracle_mod, log_n):
    o = oracle_mod.Oracle(log_n, 3)
    mods = o.p.moduli
    two_n = 2 << (log_n - 1) * 1 if False else 2 * (1 << log_n)
    q0, q1, q2, P = mods
    for m in mods:
        assert _py_is_prime(m) and m % two_n == 1
    assert q0 < 2**60 and P < q0 and q2 < q1 < 2**45
    # "largest": no NTT-friendly prime strictly between each and its upper bound (R5)
    for m, upper in ((q0, 2**60), (P, q0), (q1, 2**45), (q2, q1)):
        c = m + two_n
        while c < upper:
            assert not _py_is_prime(c)
            c += two_n


@pytest.mark.parametrize("log_n", [4, 6, 8])
def test_psi_is_smallest_primitive_root(oracle_mod, log_n):
    o = oracle_mod.Oracle(log_n, 3)
    n = 1 << log_n
    for l, m in enumerate(o.p.moduli):
        psi = int(o.p.psi[l])
        assert pow(psi, n, m) == m - 1          # order exactly 2n
        roots = sorted(pow(psi, 2 * t + 1, m) for t in range(n))
        assert roots[0] == psi


@pytest.mark.parametrize("log_n", [4, 7])
def test_ntt_equals_definition_and_inverts(oracle_mod, log_n):
    o = oracle_mod.Oracle(log_n, 3)
    rng = np.random.default_rng(1)
    n = 1 << log_n
    for l, m in enumerate(o.p.moduli):
        a = rng.integers(0, m, n, dtype=np.uint64)
        fa = o.ntt(a, l)
        # plain definition, written out here in Python big ints
        psi = int(o.p.psi[l])
        br = [int(format(i, f"0{log_n}b")[::-1], 2) for i in range(n)]
        ref = [sum(int(a[j]) * pow(psi, (2 * br[i] + 1) * j, m) for j in range(n)) % m for i in range(n)]
        assert [int(x) for x in fa] == ref
        assert (o.ntt_definition(a, l) == fa).all()
        assert (o.ntt(fa, l, inverse=True) == a).all()


def test_ntt_product_is_negacyclic_convolution(oracle_mod):
    o = oracle_mod.Oracle(5, 3)
    rng = np.random.default_rng(2)
    n = o.n
    for l, m in enumerate(o.p.moduli):
        a = rng.integers(0, m, n, dtype=np.uint64)
        b = rng.integers(0, m, n, dtype=np.uint64)
        prod = np.array([int(x) * int(y) % m for x, y in zip(o.ntt(a, l), o.ntt(b, l))], dtype=np.uint64)
        # schoolbook product in Z_m[X]/(X^n + 1), Python big ints
        ref = [0] * n
        for i in range(n):
            for j in range(n):
                k = i + j
                v = int(a[i]) * int(b[j])
                if k < n:
                    ref[k] = (ref[k] + v) % m
                else:
                    ref[k - n] = (ref[k - n] - v) % m
        assert [int(x) for x in o.ntt(prod, l, inverse=True)] == ref
        assert [int(x) for x in oracle_mod.schoolbook(a, b, m)] == ref


@pytest.mark.parametrize("step", [1, 3, 7, 5, -1])
def test_ntt_automorphism_matches_coefficient_definition(oracle_mod, step):
    o = oracle_mod.Oracle(4, 3)
    n = o.n
    rng = np.random.default_rng(3)
    g = o.galois_elt(step) if step > 0 else 2 * n - 1   # also the conjugation X -> X^{-1}
    a = rng.integers(-50, 50, n).astype(np.int64)
    # definition: a(X) -> a(X^g) in Z[X]/(X^n+1), written out in Python
    ref = [0] * n
    for j in range(n):
        e = j * g % (2 * n)
        if e < n:
            ref[e] += int(a[j])
        else:
            ref[e - n] -= int(a[j])
    assert [int(x) for x in o.automorph_coeff(g, a)] == ref
    for l, m in enumerate(o.p.moduli):
        ahat = o.ntt(np.array([x % m for x in a.tolist()], dtype=np.uint64), l)
        refhat = o.ntt(np.array([x % m for x in ref], dtype=np.uint64), l)
        assert (o.automorph_ntt(g, ahat) == refhat).all()


def test_galois_composition(oracle_mod):
    o = oracle_mod.Oracle(6, 3)
    rng = np.random.default_rng(4)
    m = o.p.moduli[0]
    a = rng.integers(0, m, o.n, dtype=np.uint64)
    g1, g2 = o.galois_elt(3), o.galois_elt(5)
    assert o.galois_elt(8) == g1 * g2 % (2 * o.n)
    assert (o.automorph_ntt(g1, o.automorph_ntt(g2, a)) == o.automorph_ntt(g1 * g2 % (2 * o.n), a)).all()
