"""Pins of the oracle's general hybrid key switching (R31; SURVEY 8(d) "paper-depth" profile:
L = 12 limbs, alpha = 4 limbs per digit, K_sp = 4 special primes, ring 2^15 and scale 2^45 in
the paper).  Not gpu.

(1) the modulus chain: primes, = 1 mod 2n, the special primes the largest NTT primes below q0
    in turn (exhaustive candidate scan), P = prod p_k larger than every digit modulus;
(2) fast basis conversion with centred digits: the converted residues are ONE integer V per
    coefficient (CRT over several target moduli), V = X mod B, |V| <= cnt B / 2, exact on the
    base's own moduli, and the centred lift itself for one modulus;
(3) ModDown(P x) = x exactly, and ModDown of a small polynomial is tiny;
(4) key structure: b_d + a_d s - [l in I_d] P s' is the same CBD(21) polynomial on every
    modulus of a key digit (|e| <= 21), i.e. the gadget sits exactly on the digit's limbs;
(5) decrypt(Rot_r(ct)) is the slot rotation by r (in the clear) at the paper profile;
(6) the whole scan at the paper profile decodes to brute-force cosine <= 1e-6 with the planted
    matches on top.
"""
import numpy as np
import pytest

from synth_inputs import CONFIGS, make_dataset

D45 = 2.0 ** 45


def _is_prime(x):
    if x < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if x % p == 0:
            return x == p
    d, r = x - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(r - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def _crt(residues, moduli):
    M = 1
    for m in moduli:
        M *= m
    x = 0
    for r, m in zip(residues, moduli):
        Mi = M // m
        x += int(r) * Mi * pow(Mi, -1, m)
    x %= M
    return x - M if x > M // 2 else x, M


@pytest.fixture(scope="module")
def paper(oracle_mod):
    return oracle_mod.Oracle(12, 12, seed=1, K_sp=4, alpha=4)


def test_modulus_chain(paper):
    o = paper
    mods = o.p.moduli
    two_n = 2 * o.n
    assert len(mods) == 16 and len(set(mods)) == 16
    assert all(_is_prime(m) and m % two_n == 1 for m in mods)
    assert mods[0] < 2 ** 60 and all(m < 2 ** 45 for m in mods[1:12])
    # special primes: each the largest NTT prime below the previous one (p_0 below q0)
    prev = mods[0]
    for k in range(4):
        pk = mods[12 + k]
        assert pk < prev
        c = pk + two_n
        while c < prev:
            assert not _is_prime(c), (k, c)
            c += two_n
        prev = pk
    P = 1
    for pk in mods[12:]:
        P *= pk
    for d in range(o.num_digits(12)):
        Qd = 1
        for q in mods[4 * d: 4 * d + 4]:
            Qd *= q
        assert P > 4 * Qd  # the special modulus dominates every digit (noise, R31)
    assert o.num_digits(12) == 3 and o.num_digits(11) == 3 and o.num_digits(8) == 2


@pytest.mark.parametrize("base", [[3], [0], [1, 2], [4, 5, 6, 7], [12, 13, 14, 15], [8, 9, 10]])
def test_basis_conversion_is_one_small_integer(paper, base):
    o = paper
    mods = o.p.moduli
    B = 1
    for i in base:
        B *= mods[i]
    rng = np.random.default_rng(len(base) * 100 + base[0])
    X = [int(v) for v in rng.integers(0, 2 ** 62, size=o.n)]
    X = [(a * (2 ** 62) + b) % B for a, b in zip(X, reversed(X))]
    x = np.array([[v % mods[i] for v in X] for i in base], dtype=np.uint64)
    targets = [t for t in range(16) if t not in base][:6] + base
    rows = {t: o.basis_convert(x, base, t) for t in targets}
    tm = [mods[t] for t in targets]
    for j in range(0, o.n, 97):
        V, M = _crt([rows[t][j] for t in targets], tm)
        assert M > 2 * len(base) * B                # enough target moduli to see V itself
        assert (V - X[j]) % B == 0                  # congruent to X modulo the base
        assert abs(V) <= len(base) * B // 2         # the centred digits keep it small
        for i in base:                               # exact on the base's own moduli
            assert int(rows[i][j]) == X[j] % mods[i]
        if len(base) == 1:                           # one modulus: the centred lift (R12)
            assert V == (X[j] - B if X[j] > B // 2 else X[j])


@pytest.mark.parametrize("ell", [12, 11, 5])
def test_moddown_exact_on_multiples_of_P(paper, ell):
    o = paper
    mods = o.p.moduli
    P = 1
    for pk in mods[12:]:
        P *= pk
    rng = np.random.default_rng(ell)
    x = np.array([rng.integers(0, mods[l], o.n, dtype=np.uint64) for l in range(ell)])
    u = np.zeros((ell + 4, o.n), np.uint64)
    for l in range(ell):
        u[l] = np.array([(P % mods[l]) * int(v) % mods[l] for v in x[l]], dtype=np.uint64)
    assert (o.moddown(u, ell) == x).all()
    # a small integer polynomial e (|e| <= 1000) in every modulus: ModDown(e) is the tiny
    # rounding of e / P (|.| <= K / 2 + 1 per coefficient, the same integer on every limb)
    e = rng.integers(-1000, 1001, o.n)
    ue = np.zeros((ell + 4, o.n), np.uint64)
    ext = list(range(ell)) + [12, 13, 14, 15]
    for row, mi in enumerate(ext):
        ue[row] = o.ntt(np.array([int(v) % mods[mi] for v in e], np.uint64), mi)
    md = o.moddown(ue, ell)
    coef = [o.ntt(md[l].copy(), l, inverse=True) for l in range(ell)]
    for j in range(0, o.n, 31):
        V, _ = _crt([coef[l][j] for l in range(ell)], mods[:ell])
        assert abs(V) <= 3


def test_switch_key_gadget_on_digit_limbs(oracle_mod):
    o = oracle_mod.Oracle(6, 6, seed=3, K_sp=2, alpha=4)  # digits {0..3}, {4, 5}
    mods = o.p.moduli
    P = mods[6] * mods[7]
    s, s_ntt = o.secret_key()
    step = 3
    key = o.rotation_key(s_ntt, step)
    sp = o.automorph_coeff(o.galois_elt(step), s)
    for d in range(o.beta):
        e_rows = []
        for l in range(o.M):
            m = mods[l]
            b, a = key[d, 0, l], key[d, 1, l]
            v = [(int(bb) + int(aa) * int(ss)) % m for bb, aa, ss in zip(b, a, s_ntt[l])]
            v = o.ntt(np.array(v, np.uint64), l, inverse=True)
            in_digit = l < 6 and l // 4 == d
            coef = []
            for j in range(o.n):
                c = int(v[j])
                if in_digit:
                    c = (c - (P % m) * (int(sp[j]) % m)) % m
                coef.append(c - m if c > m // 2 else c)
            assert max(abs(c) for c in coef) <= 21, (d, l)
            e_rows.append(coef)
        assert all(r == e_rows[0] for r in e_rows)  # one error polynomial per digit


@pytest.mark.parametrize("L,K,alpha", [(6, 2, 2), (12, 4, 4), (4, 4, 4)])  # (4, 4, 4): one digit, P > Q
def test_rotation_is_slot_shift(oracle_mod, L, K, alpha):
    o = oracle_mod.Oracle(7, L, seed=2, K_sp=K, alpha=alpha)
    s, s_ntt = o.secret_key()
    rng = np.random.default_rng(L)
    z = rng.uniform(-1, 1, o.ns)
    ct = o.encrypt(s_ntt, o.encode(z, D45, L), 77)
    for step in (1, 5, o.ns - 8):
        key = o.rotation_key(s_ntt, step)
        rot = o.rotate(ct, key, step)
        got = o.decode(o.decrypt(s_ntt, rot), D45)
        assert np.abs(got - np.roll(z, -step)).max() < 1e-8
        # at a lower level too (a truncated last digit)
        low = np.ascontiguousarray(ct[:, : L - 1])
        got = o.decode(o.decrypt(s_ntt, o.rotate(low, key, step)), D45)
        assert np.abs(got - np.roll(z, -step)).max() < 1e-8


def test_paper_depth_scan_scores(paper):
    """The encrypted scan (Alg. sender-bsgs) at the paper's depth on the toy workload."""
    o = paper
    cfg = CONFIGS["C1"]
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    s, s_ntt = o.secret_key()
    steps, keys = o.keyset(s_ntt, o.rotation_steps(cfg.dim, cfg.n1))
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, cfg.n1, steps, keys)
    D = o.enroll_aggregate(o.normalize_rows(db), 0, cfg.num_vectors, cfg.n1, 0)
    out = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)
    assert out.shape == (2, 11, o.n)
    sc = o.decrypt_scores(s_ntt, out, cfg.dim, 0, cfg.num_vectors)[: cfg.num_vectors]
    d = db.astype(np.float64)
    cos = d @ q.astype(np.float64) / (np.linalg.norm(d, axis=1) * np.linalg.norm(q.astype(np.float64)))
    assert np.abs(sc - cos).max() < 1e-6
    assert sorted(np.argsort(-sc)[:3]) == sorted(pos.tolist())
