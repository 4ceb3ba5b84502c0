"""CPU oracle for the encrypted BSGS similarity scan (arXiv 2604.00546).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  It wraps ``oracle/hd_oracle.c`` (plain C, built with gcc) through
ctypes and shares no code with the product package ``paper_2604_00546_b200``.

Every wrapper takes/returns numpy arrays in the layouts documented in
``hd_oracle.h``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OR_OK, OR_E_ARG, OR_E_PARAMS, OR_E_LAYOUT, OR_E_ZERO_VECTOR, OR_E_MISSING_KEY, OR_E_RANGE = (
    0, -1, -2, -3, -4, -5, -6)


class OracleError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed with oracle status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction: DESIGN.md R15)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hd_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Params(C.Structure):
    _fields_ = [("log_n", C.c_int32), ("n", C.c_int32), ("num_slots", C.c_int32),
                ("L", C.c_int32), ("q0_bits", C.c_int32), ("scale_bits", C.c_int32),
                ("special_bits", C.c_int32), ("K_sp", C.c_int32), ("alpha", C.c_int32), ("pad_", C.c_int32),
                ("mod", C.c_uint64 * 20), ("psi", C.c_uint64 * 20), ("seed", C.c_uint64)]

    @property
    def moduli(self):
        """q_0..q_{L-1}, then the special primes p_0..p_{K-1}"""
        return [int(self.mod[i]) for i in range(self.L + self.K_sp)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = C.CDLL(build())
            _lib.or_galois_elt.restype = C.c_uint64
            _lib.or_pre_rot.restype = C.c_int32
            _lib.or_is_prime.argtypes = [C.c_uint64]
            _lib.or_galois_elt.argtypes = [C.POINTER(Params), C.c_int64]
        return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(fn, rc):
    if rc != 0:
        raise OracleError(fn, rc)


def u64(shape):
    return np.zeros(shape, dtype=np.uint64)


class Oracle:
    """Thin stateful wrapper: parameters + convenience shapes."""

    def __init__(self, log_n: int, L: int = 3, seed: int = 1, K_sp: int = 1, alpha: int = 1):
        """K_sp special primes and alpha limbs per key-switching digit (R31); the defaults are
        the north-star profile (R11: alpha = 1, one special prime P)."""
        self.p = Params()
        _check("or_params_init_ex", lib().or_params_init_ex(C.byref(self.p), log_n, L, K_sp, alpha,
                                                            C.c_uint64(seed)))
        self.n = self.p.n
        self.ns = self.p.num_slots
        self.L = self.p.L
        self.K = K_sp
        self.alpha = alpha
        self.M = self.L + K_sp          # moduli of a key: Q_L u P
        self.beta = -(-self.L // alpha)  # digits of a top-level key
        self.log_n = log_n

    def num_digits(self, ell):
        return -(-ell // self.alpha)

    # -- ring --------------------------------------------------------------
    def ntt(self, a, l, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        fn = lib().or_ntt_inverse if inverse else lib().or_ntt_forward
        _check("ntt", fn(C.byref(self.p), l, _p(a)))
        return a

    def ntt_definition(self, a, l):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = u64(self.n)
        _check("ntt_definition", lib().or_ntt_definition(C.byref(self.p), l, _p(a), _p(out)))
        return out

    def galois_elt(self, step):
        return int(lib().or_galois_elt(C.byref(self.p), step))

    def automorph_ntt(self, g, a):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = u64(self.n)
        lib().or_automorph_ntt(C.byref(self.p), C.c_uint64(g), _p(a), _p(out))
        return out

    def automorph_coeff(self, g, a):
        a = np.ascontiguousarray(a, dtype=np.int64)
        out = np.zeros(self.n, dtype=np.int64)
        lib().or_automorph_coeff(C.byref(self.p), C.c_uint64(g), _p(a), _p(out))
        return out

    # -- encoding ------------------------------------------------------------
    def encode(self, z, delta, nlimbs):
        z = np.ascontiguousarray(z, dtype=np.float64)
        pt = u64((nlimbs, self.n))
        _check("encode", lib().or_encode(C.byref(self.p), _p(z), C.c_double(delta), nlimbs, _p(pt)))
        return pt

    def encode_coeffs(self, z, delta):
        z = np.ascontiguousarray(z, dtype=np.float64)
        c = np.zeros(self.n, dtype=np.int64)
        _check("encode_coeffs", lib().or_encode_coeffs(C.byref(self.p), _p(z), C.c_double(delta), _p(c)))
        return c

    def decode(self, pt, delta):
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        z = np.zeros(self.ns, dtype=np.float64)
        _check("decode", lib().or_decode(C.byref(self.p), _p(pt), pt.shape[0], C.c_double(delta), _p(z)))
        return z

    # -- keys / encryption --------------------------------------------------------
    def secret_key(self):
        s = np.zeros(self.n, dtype=np.int64)
        s_ntt = u64((self.M, self.n))
        _check("secret_key", lib().or_secret_key(C.byref(self.p), _p(s), _p(s_ntt)))
        return s, s_ntt

    def rotation_key(self, s_ntt, step):
        key = u64((self.beta, 2, self.M, self.n))
        _check("rotation_key", lib().or_rotation_key(C.byref(self.p), _p(s_ntt), step, _p(key)))
        return key

    def encrypt(self, s_ntt, pt, enc_seed):
        nl = pt.shape[0]
        ct = u64((2, nl, self.n))
        _check("encrypt", lib().or_encrypt(C.byref(self.p), _p(s_ntt), _p(np.ascontiguousarray(pt)),
                                           nl, C.c_uint64(enc_seed), _p(ct)))
        return ct

    def decrypt(self, s_ntt, ct):
        nl = ct.shape[1]
        pt = u64((nl, self.n))
        _check("decrypt", lib().or_decrypt(C.byref(self.p), _p(s_ntt), _p(np.ascontiguousarray(ct)), nl, _p(pt)))
        return pt

    # -- key switching -----------------------------------------------------------
    def modup(self, c1):
        ell = c1.shape[0]
        dig = u64((self.num_digits(ell), ell + self.K, self.n))
        _check("modup", lib().or_modup(C.byref(self.p), _p(np.ascontiguousarray(c1)), ell, _p(dig)))
        return dig

    def basis_convert(self, x, bidx, mi):
        """R31 fast basis conversion of coefficient-form rows x[i] (modulo mod[bidx[i]]) into mod[mi]."""
        x = np.ascontiguousarray(x, dtype=np.uint64)
        b = np.ascontiguousarray(bidx, dtype=np.int32)
        out = u64(self.n)
        _check("basis_convert", lib().or_basis_convert(C.byref(self.p), _p(x), _p(b), len(b), mi, _p(out)))
        return out

    def moddown(self, u, ell):
        u = np.ascontiguousarray(u, dtype=np.uint64)
        out = u64((ell, self.n))
        _check("moddown", lib().or_moddown(C.byref(self.p), _p(u), ell, _p(out)))
        return out

    def rotate_hoisted(self, ct, dig, key, step):
        ell = ct.shape[1]
        out = u64((2, ell, self.n))
        _check("rotate_hoisted", lib().or_rotate_hoisted(
            C.byref(self.p), _p(np.ascontiguousarray(ct)), _p(np.ascontiguousarray(dig)), ell,
            _p(np.ascontiguousarray(key)), step, _p(out)))
        return out

    def rotate(self, ct, key, step):
        ell = ct.shape[1]
        out = u64((2, ell, self.n))
        _check("rotate", lib().or_rotate(C.byref(self.p), _p(np.ascontiguousarray(ct)), ell,
                                         _p(np.ascontiguousarray(key)), step, _p(out)))
        return out

    def rescale(self, ct):
        ell = ct.shape[1]
        out = u64((2, ell - 1, self.n))
        _check("rescale", lib().or_rescale(C.byref(self.p), _p(np.ascontiguousarray(ct)), ell, _p(out)))
        return out

    # -- enrollment / query ------------------------------------------------------
    def normalize_rows(self, vecs):
        vecs = np.ascontiguousarray(vecs, dtype=np.float32)
        U = np.zeros(vecs.shape, dtype=np.float64)
        _check("normalize_rows", lib().or_normalize_rows(_p(vecs), vecs.shape[0], vecs.shape[1], _p(U)))
        return U

    def query_slots(self, q):
        q = np.ascontiguousarray(q, dtype=np.float32)
        z = np.zeros(self.ns, dtype=np.float64)
        _check("query_slots", lib().or_query_slots(C.byref(self.p), _p(q), q.shape[0], _p(z)))
        return z

    def enroll_slots(self, U, u_first, num_vectors, n1, agg, k):
        U = np.ascontiguousarray(U, dtype=np.float64)
        z = np.zeros(self.ns, dtype=np.float64)
        _check("enroll_slots", lib().or_enroll_slots(C.byref(self.p), _p(U), C.c_int64(u_first),
                                                     C.c_int64(U.shape[0]), C.c_int64(num_vectors),
                                                     U.shape[1], n1, C.c_int64(agg), k, _p(z)))
        return z

    def enroll_aggregate(self, U, u_first, num_vectors, n1, agg):
        U = np.ascontiguousarray(U, dtype=np.float64)
        dim = U.shape[1]
        N = min(dim, self.ns)
        D = u64((N, self.L, self.n))
        _check("enroll_aggregate", lib().or_enroll_aggregate(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]),
            C.c_int64(num_vectors), dim, n1, C.c_int64(agg), _p(D)))
        return D

    # -- scan -------------------------------------------------------------------
    def giant_range(self, N, n1):
        a, b = C.c_int32(), C.c_int32()
        lib().or_giant_range(N, n1, C.byref(a), C.byref(b))
        return a.value, b.value

    def pre_rot(self, N, n1, j):
        return int(lib().or_pre_rot(N, n1, j))

    def rotation_steps(self, N, n1):
        steps = np.zeros(4096, dtype=np.int32)
        cnt = C.c_int32()
        _check("rotation_steps", lib().or_rotation_steps(C.byref(self.p), N, n1, _p(steps), 4096, C.byref(cnt)))
        return [int(s) for s in steps[:cnt.value]]

    def keyset(self, s_ntt, steps):
        steps = np.asarray(steps, dtype=np.int32)
        keys = u64((len(steps), self.beta, 2, self.M, self.n))
        for i, s in enumerate(steps):
            keys[i] = self.rotation_key(s_ntt, int(s))
        return steps, keys

    def baby_steps(self, q_ct, n1, steps, keys):
        r = u64((n1, 2, self.L, self.n))
        _check("baby_steps", lib().or_baby_steps(C.byref(self.p), _p(np.ascontiguousarray(q_ct)), n1,
                                                 _p(steps), len(steps), _p(keys), _p(r)))
        return r

    def giant_sum(self, r, n1, N, Dagg, j):
        S = u64((2, self.L, self.n))
        rc = lib().or_giant_sum(C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N,
                                _p(np.ascontiguousarray(Dagg)), j, _p(S))
        if rc == OR_E_RANGE:
            return None
        _check("giant_sum", rc)
        return S

    def scan_aggregate(self, r, n1, N, Dagg, steps, keys, want_y=False, hoisted=True):
        """One aggregate's output ciphertext.  hoisted=True (the CUDA path's schedule,
        R23): giant-step rotations accumulated in Q u {P}, one ModDown; False: one
        ModDown per rotation (the textbook rotation of Alg. sender-bsgs)."""
        out = u64((2, self.L - 1, self.n))
        y = u64((2, self.L - 1, self.n))
        fn = lib().or_scan_aggregate_hoisted if hoisted else lib().or_scan_aggregate
        _check("scan_aggregate", fn(
            C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N, _p(np.ascontiguousarray(Dagg)),
            _p(steps), len(steps), _p(keys), _p(out), _p(y)))
        return (out, y) if want_y else out

    # -- flat pre-rotated layout (NEXT-2, R27) ------------------------------------
    def enroll_slots_flat(self, U, u_first, num_vectors, n1, agg, k):
        U = np.ascontiguousarray(U, dtype=np.float64)
        z = np.zeros(self.ns, np.float64)
        _check("enroll_slots_flat", lib().or_enroll_slots_flat(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]), C.c_int64(num_vectors),
            U.shape[1], n1, C.c_int64(agg), k, _p(z)))
        return z

    def enroll_aggregate_flat(self, U, u_first, num_vectors, n1, agg):
        U = np.ascontiguousarray(U, dtype=np.float64)
        D = u64((U.shape[1], self.L, self.n))
        _check("enroll_aggregate_flat", lib().or_enroll_aggregate_flat(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]), C.c_int64(num_vectors),
            U.shape[1], n1, C.c_int64(agg), _p(D)))
        return D

    def rotation_steps_flat(self, N, n1):
        cap = self.ns
        steps = np.zeros(cap, np.int32)
        cnt = C.c_int32()
        _check("rotation_steps_flat", lib().or_rotation_steps_flat(C.byref(self.p), N, n1, _p(steps), cap,
                                                                   C.byref(cnt)))
        return [int(s) for s in steps[:cnt.value]]

    def giant_sum_flat(self, r, n1, N, Dagg, j):
        S = u64((2, self.L, self.n))
        rc = lib().or_giant_sum_flat(C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N,
                                     _p(np.ascontiguousarray(Dagg)), j, _p(S))
        if rc == OR_E_RANGE:
            return None
        _check("giant_sum_flat", rc)
        return S

    def scan_aggregate_flat(self, r, n1, N, Dagg, steps, keys):
        out = u64((2, self.L - 1, self.n))
        _check("scan_aggregate_flat", lib().or_scan_aggregate_flat(
            C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N, _p(np.ascontiguousarray(Dagg)), _p(steps),
            len(steps), _p(keys), _p(out)))
        return out

    def enroll_aggregate_flat_encrypted(self, U, u_first, num_vectors, n1, agg, pk, enc_seed):
        U = np.ascontiguousarray(U, dtype=np.float64)
        D = u64((U.shape[1], 2, self.L, self.n))
        _check("enroll_aggregate_flat_encrypted", lib().or_enroll_aggregate_flat_encrypted(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]), C.c_int64(num_vectors),
            U.shape[1], n1, C.c_int64(agg), _p(pk), C.c_uint64(enc_seed), _p(D)))
        return D

    def enroll_aggregate_flat_tbs(self, U, u_first, num_vectors, n1, agg, pk, enc_seed):
        U = np.ascontiguousarray(U, dtype=np.float64)
        D = u64((U.shape[1], 2, self.L, self.n))
        _check("enroll_aggregate_flat_tbs", lib().or_enroll_aggregate_flat_tbs(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]), C.c_int64(num_vectors),
            U.shape[1], n1, C.c_int64(agg), _p(pk), C.c_uint64(enc_seed), _p(D)))
        return D

    def prerotate_tbs(self, Dct, n1, steps, keys):
        D = np.ascontiguousarray(Dct).copy()
        _check("prerotate_tbs", lib().or_prerotate_tbs(C.byref(self.p), _p(D), D.shape[0], n1, _p(steps), len(steps),
                                                       _p(keys)))
        return D

    def giant_sum_ct_flat(self, r, n1, N, Dct, j):
        S = u64((3, self.L, self.n))
        rc = lib().or_giant_sum_ct_flat(C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N,
                                        _p(np.ascontiguousarray(Dct)), j, _p(S))
        if rc == OR_E_RANGE:
            return None
        _check("giant_sum_ct_flat", rc)
        return S

    def scan_aggregate_flat_ct(self, r, n1, N, Dct, steps, keys, rlk):
        out = u64((2, self.L - 1, self.n))
        _check("scan_aggregate_flat_ct", lib().or_scan_aggregate_flat_ct(
            C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N, _p(np.ascontiguousarray(Dct)), _p(rlk), _p(steps),
            len(steps), _p(keys), _p(out)))
        return out

    def decrypt_scores_flat(self, s_ntt, out_ct, N, agg, num_vectors):
        sc = np.zeros((self.ns // N) * N, dtype=np.float64)
        _check("decrypt_scores_flat", lib().or_decrypt_scores_flat(
            C.byref(self.p), _p(s_ntt), _p(np.ascontiguousarray(out_ct)), N, C.c_int64(agg),
            C.c_int64(num_vectors), _p(sc)))
        return sc

    # -- encrypted-database mode (NEXT-1, R26) ------------------------------------
    def public_key(self, s_ntt):
        pk = u64((2, self.L, self.n))
        _check("public_key", lib().or_public_key(C.byref(self.p), _p(s_ntt), _p(pk)))
        return pk

    def encrypt_pk(self, pk, pt, enc_seed, obj):
        nl = pt.shape[0]
        ct = u64((2, nl, self.n))
        _check("encrypt_pk", lib().or_encrypt_pk(C.byref(self.p), _p(pk), _p(np.ascontiguousarray(pt)), nl,
                                                 C.c_uint64(enc_seed), C.c_uint32(obj), _p(ct)))
        return ct

    def relin_key(self, s_ntt):
        key = u64((self.beta, 2, self.M, self.n))
        _check("relin_key", lib().or_relin_key(C.byref(self.p), _p(s_ntt), _p(key)))
        return key

    def enroll_aggregate_encrypted(self, U, u_first, num_vectors, n1, agg, pk, enc_seed):
        U = np.ascontiguousarray(U, dtype=np.float64)
        dim = U.shape[1]
        N = min(dim, self.ns)
        D = u64((N, 2, self.L, self.n))
        _check("enroll_aggregate_encrypted", lib().or_enroll_aggregate_encrypted(
            C.byref(self.p), _p(U), C.c_int64(u_first), C.c_int64(U.shape[0]),
            C.c_int64(num_vectors), dim, n1, C.c_int64(agg), _p(pk), C.c_uint64(enc_seed), _p(D)))
        return D

    def giant_sum_ct(self, r, n1, N, Dct, j):
        S = u64((3, self.L, self.n))
        rc = lib().or_giant_sum_ct(C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N,
                                   _p(np.ascontiguousarray(Dct)), j, _p(S))
        if rc == OR_E_RANGE:
            return None
        _check("giant_sum_ct", rc)
        return S

    def relinearize(self, S3, rlk):
        ell = S3.shape[1]
        out = u64((2, ell, self.n))
        _check("relinearize", lib().or_relinearize(C.byref(self.p), _p(np.ascontiguousarray(S3)), ell, _p(rlk),
                                                   _p(out)))
        return out

    def scan_aggregate_ct(self, r, n1, N, Dct, steps, keys, rlk, want_y=False):
        out = u64((2, self.L - 1, self.n))
        y = u64((2, self.L - 1, self.n))
        _check("scan_aggregate_ct", lib().or_scan_aggregate_ct(
            C.byref(self.p), _p(np.ascontiguousarray(r)), n1, N, _p(np.ascontiguousarray(Dct)), _p(rlk),
            _p(steps), len(steps), _p(keys), _p(out), _p(y)))
        return (out, y) if want_y else out

    def decrypt_scores(self, s_ntt, out_ct, N, agg, num_vectors):
        M = self.ns // N
        sc = np.zeros((M // 2) * N, dtype=np.float64)
        _check("decrypt_scores", lib().or_decrypt_scores(C.byref(self.p), _p(s_ntt),
                                                         _p(np.ascontiguousarray(out_ct)), N,
                                                         C.c_int64(agg), C.c_int64(num_vectors), _p(sc)))
        return sc

    # -- encrypted comparison and scenario tail (NEXT-3, R29) ---------------------
    def cheb_compare(self, ct, scale, coeffs, rlk, out_limbs=1):
        """ChebyshevCompare (Alg. gpu-chebyshev) to out_limbs limbs: (ct_out, scale_out)."""
        ell = ct.shape[1]
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = u64((2, ell, self.n))
        eo = C.c_int32(0)
        so = C.c_double(0.0)
        _check("cheb_compare", lib().or_cheb_compare_at(
            C.byref(self.p), _p(np.ascontiguousarray(ct)), ell, C.c_double(scale), _p(c), len(c) - 1,
            _p(np.ascontiguousarray(rlk)), out_limbs, _p(out), C.byref(eo), C.byref(so)))
        return np.ascontiguousarray(out.reshape(-1)[: 2 * eo.value * self.n].reshape(2, eo.value, self.n)), so.value

    def relin_rescale(self, S3, rlk):
        """Relinearize + Rescale with one rounding by P q_{ell-1} (R29)."""
        ell = S3.shape[1]
        out = u64((2, ell - 1, self.n))
        _check("relin_rescale", lib().or_relin_rescale(C.byref(self.p), _p(np.ascontiguousarray(S3)), ell,
                                                        _p(np.ascontiguousarray(rlk)), _p(out)))
        return out

    def aggregate_diagonals(self, Ds):
        """Online DB aggregation (Alg. online-aggr Step 2): the per-aggregate diagonals summed."""
        D = np.ascontiguousarray(np.stack(Ds), dtype=np.uint64)
        A, N = D.shape[0], D.shape[1]
        dpoly = 2 if D.ndim == 5 else 1
        out = np.zeros(D.shape[1:], dtype=np.uint64)
        _check("aggregate_diagonals", lib().or_aggregate_diagonals(C.byref(self.p), _p(D), A, N, dpoly, _p(out)))
        return out

    def membership(self, cts, steps, keys):
        """EvalAddMany + RotateAndSum over numSlots (Alg. membership)."""
        cts = np.ascontiguousarray(cts, dtype=np.uint64)
        count, _, ell, _ = cts.shape
        out = u64((2, ell, self.n))
        _check("membership", lib().or_membership(C.byref(self.p), _p(cts), count, ell, _p(steps), len(steps),
                                                 _p(keys), _p(out)))
        return out


def cheb_degree(kappa: int) -> int:
    lib().or_cheb_degree.restype = C.c_int32
    return int(lib().or_cheb_degree(kappa))


def ps_split(n: int):
    d1, d2 = C.c_int32(0), C.c_int32(0)
    _check("ps_split", lib().or_ps_split(n, C.byref(d1), C.byref(d2)))
    return d1.value, d2.value


def cheb_coeffs(delta: float, n: int) -> np.ndarray:
    c = np.zeros(n + 1, dtype=np.float64)
    _check("cheb_coeffs", lib().or_cheb_coeffs(C.c_double(delta), n, _p(c)))
    return c


def philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def is_prime(x: int) -> bool:
    return bool(lib().or_is_prime(C.c_uint64(x)))


def schoolbook(a, b, m):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.zeros_like(a)
    lib().or_negacyclic_schoolbook(_p(a), _p(b), len(a), C.c_uint64(m), _p(out))
    return out
