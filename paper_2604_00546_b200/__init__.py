"""paper_2604_00546_b200 -- B200-native encrypted BSGS similarity scan (arXiv 2604.00546).

Thin ctypes binding of ``libhd.so`` (include/hd.h).  Every function named
``hd_*`` here marshals arguments to the C ABI function of the same name; all
arithmetic runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback:
if ``libhd.so`` cannot be built/loaded, or no CUDA device is present, calls
raise :class:`HDError`.

The small classes (:class:`Context`, :class:`Database`, ...) only own handles
and call the ``hd_*`` functions.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import threading

import numpy as np

from ._build import LIB as _LIB_PATH
from ._build import build as _build_lib

__all__ = ["HDError", "Params", "Layout", "Context", "Database", "load", "lib_path"]

HD_OK, HD_E_INVALID_ARG, HD_E_PARAMS, HD_E_LAYOUT, HD_E_ZERO_VECTOR, HD_E_MISSING_KEY = 0, -1, -2, -3, -4, -5
HD_E_LEVEL, HD_E_CAPACITY, HD_E_CUDA, HD_E_STATE, HD_E_FORMAT = -6, -7, -8, -9, -10

ABI_FUNCTIONS = [
    "hd_status_string", "hd_last_error", "hd_context_create", "hd_context_destroy", "hd_context_set_stream",
    "hd_context_moduli", "hd_rotation_steps", "hd_keygen", "hd_encrypt_query", "hd_decrypt_scores", "hd_decrypt",
    "hd_enroll", "hd_database_layout", "hd_query", "hd_query_stats", "hd_launch_count", "hd_ciphertext_export",
    "hd_ciphertext_import", "hd_ciphertext_import_into", "hd_ciphertext_limbs", "hd_eval_keys_export",
    "hd_eval_keys_import", "hd_secret_key_export", "hd_ciphertext_destroy", "hd_eval_keys_destroy",
    "hd_secret_key_destroy", "hd_database_destroy", "hd_test_ntt", "hd_test_stage", "hd_test_rotate",
    "hd_test_rescale", "hd_ciphertext_export_async", "hd_context_synchronize", "hd_enroll_encrypted",
    "hd_public_keygen", "hd_public_key_export", "hd_public_key_import", "hd_relin_keygen", "hd_public_key_destroy",
    "hd_enroll_ex", "hd_rotation_steps_ex", "hd_prerotation_steps", "hd_database_prerotate",
    "hd_chebyshev_degree", "hd_chebyshev_coefficients", "hd_compare", "hd_membership_steps", "hd_membership",
    "hd_ciphertext_scale", "hd_decrypt_slots", "hd_query_batch", "hd_eval_add_many", "hd_baby_steps",
    "hd_query_baby", "hd_database_aggregate", "hd_compare_ex", "hd_enroll_footprint",
    "hd_ciphertext_export_level", "hd_encrypt_query_ex", "hd_test_inject", "hd_database_diagonal_bytes",
]


class HDError(RuntimeError):
    def __init__(self, fn, code, detail=""):
        self.code = code
        super().__init__(f"{fn}: status {code} ({_status_string(code)}){': ' + detail if detail else ''}")


class Params(C.Structure):
    _fields_ = [("log_n", C.c_uint32), ("num_limbs", C.c_uint32), ("q0_bits", C.c_uint32),
                ("scale_bits", C.c_uint32), ("special_bits", C.c_uint32), ("num_special", C.c_uint32),
                ("digit_limbs", C.c_uint32), ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class Layout(C.Structure):
    _fields_ = [("vector_dim", C.c_uint32), ("n1", C.c_uint32), ("num_slots", C.c_uint32),
                ("block_n", C.c_uint32), ("blocks_m", C.c_uint32), ("groups_per_ct", C.c_uint32),
                ("num_vectors", C.c_uint64), ("num_groups", C.c_uint64), ("num_aggregates", C.c_uint64),
                ("giant_min", C.c_int32), ("giant_max", C.c_int32), ("agg_begin", C.c_uint32),
                ("agg_end", C.c_uint32), ("packing", C.c_uint32), ("reserved", C.c_uint32)]


PACKING = {"replicated": 0, "flat": 1, "flat_tbs": 2}  # HD_PACKING_* (flat: NEXT-2, R27; flat_tbs: TBS)


class EnrollOptions(C.Structure):
    _fields_ = [("packing", C.c_uint32), ("reserved", C.c_uint32), ("pk", C.c_void_p), ("enc_seed", C.c_uint64)]


_lib = None
_lock = threading.Lock()
VP = C.c_void_p


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load libhd.so (building it with nvcc if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is None:
            # HD_LIBHD: an alternative in-tree build of libhd (kernel A/B runs; tools/ntt_variants.sh)
            path = os.environ.get("HD_LIBHD") or _build_lib()
            L = C.CDLL(path)
            L.hd_status_string.restype = C.c_char_p
            L.hd_status_string.argtypes = [C.c_int]
            L.hd_last_error.restype = C.c_char_p
            for name in ABI_FUNCTIONS:
                f = getattr(L, name)
                if name not in ("hd_status_string", "hd_last_error"):
                    f.restype = C.c_int
            for name in ("hd_context_destroy", "hd_ciphertext_destroy", "hd_eval_keys_destroy",
                         "hd_secret_key_destroy", "hd_database_destroy", "hd_public_key_destroy"):
                getattr(L, name).restype = None
                getattr(L, name).argtypes = [VP]
            L.hd_context_create.argtypes = [C.POINTER(Params), C.c_int, VP, C.POINTER(Allocator), C.POINTER(VP)]
            L.hd_enroll_footprint.argtypes = [VP, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, VP,
                                              C.POINTER(C.c_size_t)]
            L.hd_context_set_stream.argtypes = [VP, VP]
            L.hd_context_moduli.argtypes = [VP, VP, VP, C.c_size_t]
            L.hd_rotation_steps.argtypes = [VP, C.c_uint32, C.c_uint32, VP, C.c_size_t, C.POINTER(C.c_size_t)]
            L.hd_keygen.argtypes = [VP, VP, C.c_size_t, C.POINTER(VP), C.POINTER(VP)]
            L.hd_encrypt_query.argtypes = [VP, VP, VP, C.c_uint32, C.c_uint64, C.POINTER(VP)]
            L.hd_encrypt_query_ex.argtypes = [VP, VP, VP, C.c_uint32, C.c_uint64, C.c_double, C.POINTER(VP)]
            L.hd_decrypt_scores.argtypes = [VP, VP, C.POINTER(Layout), VP, C.c_size_t, VP, C.c_size_t,
                                            C.POINTER(C.c_size_t)]
            L.hd_decrypt.argtypes = [VP, VP, VP, VP, C.c_size_t]
            L.hd_enroll.argtypes = [VP, VP, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(VP)]
            L.hd_database_layout.argtypes = [VP, C.POINTER(Layout)]
            L.hd_database_diagonal_bytes.argtypes = [VP, C.POINTER(C.c_size_t), C.POINTER(C.c_int)]
            L.hd_query.argtypes = [VP, VP, VP, VP, VP, C.c_size_t]
            L.hd_query_stats.argtypes = [VP, VP, C.c_size_t]
            L.hd_launch_count.argtypes = [VP, C.POINTER(C.c_uint64)]
            L.hd_ciphertext_export.argtypes = [VP, VP, C.c_size_t, C.c_int, C.POINTER(C.c_size_t)]
            L.hd_ciphertext_import.argtypes = [VP, VP, C.c_size_t, C.c_int, C.POINTER(VP)]
            L.hd_ciphertext_import_into.argtypes = [VP, VP, C.c_size_t, C.c_int]
            L.hd_ciphertext_export_level.argtypes = [VP, C.c_uint32, VP, C.c_size_t, C.c_int, C.POINTER(C.c_size_t)]
            L.hd_ciphertext_export_async.argtypes = [VP, C.c_uint32, VP, C.c_size_t, C.c_int, C.POINTER(C.c_size_t)]
            L.hd_context_synchronize.argtypes = [VP]
            L.hd_enroll_encrypted.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                              C.c_uint64, C.POINTER(VP)]
            L.hd_public_keygen.argtypes = [VP, VP, C.POINTER(VP)]
            L.hd_enroll_ex.argtypes = [VP, VP, VP, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.POINTER(VP)]
            L.hd_rotation_steps_ex.argtypes = [VP, C.c_uint32, C.c_uint32, C.c_uint32, VP, C.c_size_t,
                                               C.POINTER(C.c_size_t)]
            L.hd_prerotation_steps.argtypes = [VP, C.c_uint32, C.c_uint32, VP, C.c_size_t, C.POINTER(C.c_size_t)]
            L.hd_database_prerotate.argtypes = [VP, VP, VP]
            L.hd_public_key_export.argtypes = [VP, VP, C.c_size_t]
            L.hd_public_key_import.argtypes = [VP, VP, C.c_size_t, C.POINTER(VP)]
            L.hd_relin_keygen.argtypes = [VP, VP, VP]
            L.hd_ciphertext_limbs.argtypes = [VP, C.POINTER(C.c_uint32)]
            L.hd_eval_keys_export.argtypes = [VP, VP, C.c_size_t, C.c_int, C.POINTER(C.c_size_t)]
            L.hd_eval_keys_import.argtypes = [VP, VP, C.c_size_t, C.c_int, C.POINTER(VP)]
            L.hd_secret_key_export.argtypes = [VP, VP, C.c_size_t]
            L.hd_test_ntt.argtypes = [VP, VP, C.c_uint32, VP, C.c_int]
            L.hd_test_stage.argtypes = [VP, C.c_int, C.c_uint32, C.c_int32, VP, C.c_size_t]
            L.hd_test_rotate.argtypes = [VP, VP, VP, C.c_int32, C.POINTER(VP)]
            L.hd_test_rescale.argtypes = [VP, VP, C.POINTER(VP)]
            L.hd_test_inject.argtypes = [VP, C.c_uint32, C.c_int32, C.c_uint64, C.c_uint64]
            L.hd_chebyshev_degree.argtypes = [C.c_uint32, C.POINTER(C.c_uint32)]
            L.hd_chebyshev_coefficients.argtypes = [C.c_double, C.c_uint32, VP, C.c_size_t]
            L.hd_compare.argtypes = [VP, VP, VP, C.c_size_t, VP, C.c_uint32, VP]
            L.hd_membership_steps.argtypes = [VP, VP, C.c_size_t, C.POINTER(C.c_size_t)]
            L.hd_membership.argtypes = [VP, VP, VP, C.c_size_t, C.POINTER(VP)]
            L.hd_ciphertext_scale.argtypes = [VP, C.POINTER(C.c_double)]
            L.hd_decrypt_slots.argtypes = [VP, VP, VP, VP, C.c_size_t]
            L.hd_query_batch.argtypes = [VP, VP, VP, VP, C.c_size_t, VP, C.c_size_t]
            L.hd_eval_add_many.argtypes = [VP, VP, C.c_size_t, C.POINTER(VP)]
            L.hd_baby_steps.argtypes = [VP, VP, VP, VP, C.c_uint32, C.c_uint32, VP]
            L.hd_query_baby.argtypes = [VP, VP, VP, VP, VP, C.c_size_t]
            L.hd_database_aggregate.argtypes = [VP, VP, C.POINTER(VP)]
            L.hd_compare_ex.argtypes = [VP, VP, VP, C.c_size_t, VP, C.c_uint32, C.c_uint32, VP]
            _lib = L
        return _lib


def _status_string(code):
    try:
        return load().hd_status_string(code).decode()
    except Exception:  # noqa: BLE001
        return "?"


# ---- device memory: the torch caching allocator behind hd_allocator (include/hd.h) ----------------
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", VP)]


_ALLOCATORS = {}    # device -> Allocator (the ctypes callbacks must outlive every context)
_FINALIZING = False  # at interpreter exit frees become no-ops (the process releases the memory)


def _at_exit():
    global _FINALIZING
    _FINALIZING = True


atexit.register(_at_exit)


def torch_allocator(device: int) -> Allocator:
    """hd_allocator over torch.cuda.caching_allocator_alloc/delete on ``device``: libhd's
    device memory then lives in (and is accounted by) PyTorch's caching allocator."""
    if device in _ALLOCATORS:
        return _ALLOCATORS[device]
    import torch

    def _alloc(nbytes, stream, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=device, stream=int(stream or 0))
        except Exception:  # noqa: BLE001  (out of memory -> NULL -> HD_E_CAPACITY)
            return None

    def _free(ptr, _stream, _user):
        if _FINALIZING or not ptr:
            return
        try:
            torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:  # noqa: BLE001
            pass

    a = Allocator(ALLOC_FN(_alloc), FREE_FN(_free), None)
    _ALLOCATORS[device] = a
    return a


def _check(fn, rc):
    if rc != HD_OK:
        raise HDError(fn, rc, load().hd_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(VP)


class _Handle:
    _destroy = None

    def __init__(self, h, owner=None):
        self.h = h
        self.owner = owner  # keeps the context alive

    def close(self):
        if self.h:
            if not _FINALIZING:  # at interpreter exit the process releases everything: no C calls
                getattr(load(), self._destroy)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class SecretKey(_Handle):
    _destroy = "hd_secret_key_destroy"


class EvalKeys(_Handle):
    _destroy = "hd_eval_keys_destroy"


class PublicKey(_Handle):
    _destroy = "hd_public_key_destroy"


class Ciphertext(_Handle):
    _destroy = "hd_ciphertext_destroy"

    @property
    def limbs(self):
        v = C.c_uint32()
        _check("hd_ciphertext_limbs", load().hd_ciphertext_limbs(self.h, C.byref(v)))
        return v.value


class Database(_Handle):
    _destroy = "hd_database_destroy"

    @property
    def layout(self) -> Layout:
        lay = Layout()
        _check("hd_database_layout", load().hd_database_layout(self.h, C.byref(lay)))
        return lay

    @property
    def diagonal_bytes(self):
        """(bytes of one stored diagonal, packed?) -- hd_database_diagonal_bytes (R34)."""
        b, p = C.c_size_t(0), C.c_int(0)
        _check("hd_database_diagonal_bytes", load().hd_database_diagonal_bytes(self.h, C.byref(b), C.byref(p)))
        return b.value, bool(p.value)

    @property
    def num_local(self):
        lay = self.layout
        return lay.agg_end - lay.agg_begin


class Context(_Handle):
    """One CUDA device + one stream (``stream``: a torch.cuda.Stream, an int handle or None)."""

    _destroy = "hd_context_destroy"

    def __init__(self, log_n, limbs=3, seed=1, device=0, stream=None, scale_bits=45, q0_bits=60,
                 allocator="torch", num_special=1, digit_limbs=1):
        """allocator: "torch" (default: PyTorch's caching allocator owns libhd's device
        memory) or None (libhd's default, the device's stream-ordered pool).
        num_special / digit_limbs: the key-switching profile (R11: 1 / 1; the paper-depth
        profile of SURVEY 8(d), R31: limbs 12, num_special 4, digit_limbs 4)."""
        p = Params(log_n=log_n, num_limbs=limbs, q0_bits=q0_bits, scale_bits=scale_bits,
                   special_bits=q0_bits, num_special=num_special, digit_limbs=digit_limbs, reserved=0, seed=seed)
        h = VP()
        alloc = C.byref(torch_allocator(device)) if allocator == "torch" else None
        _check("hd_context_create", load().hd_context_create(C.byref(p), device, _stream_handle(stream),
                                                             alloc, C.byref(h)))
        super().__init__(h.value)
        self.device = device
        self.allocator = allocator
        self.K, self.alpha = num_special, digit_limbs
        self.M = limbs + num_special              # moduli of a key: Q_L u P
        self.beta = -(-limbs // digit_limbs)      # digits of a top-level key
        self.log_n, self.L, self.n, self.ns = log_n, limbs, 1 << log_n, 1 << (log_n - 1)

    def set_stream(self, stream):
        _check("hd_context_set_stream", load().hd_context_set_stream(self.h, _stream_handle(stream)))

    def moduli(self):
        m = np.zeros(self.M, np.uint64)
        p = np.zeros(self.M, np.uint64)
        _check("hd_context_moduli", load().hd_context_moduli(self.h, _ptr(m), _ptr(p), self.M))
        return [int(x) for x in m], [int(x) for x in p]

    # -- client -------------------------------------------------------------------------------------
    def rotation_steps(self, vector_dim, n1, packing="replicated"):
        pk_ = PACKING[packing]
        cnt = C.c_size_t()
        _check("hd_rotation_steps_ex", load().hd_rotation_steps_ex(self.h, vector_dim, n1, pk_, None, 0,
                                                                   C.byref(cnt)))
        steps = np.zeros(cnt.value, np.int32)
        _check("hd_rotation_steps_ex", load().hd_rotation_steps_ex(self.h, vector_dim, n1, pk_, _ptr(steps),
                                                                   cnt.value, C.byref(cnt)))
        return steps

    def keygen(self, steps):
        steps = np.ascontiguousarray(steps, dtype=np.int32)
        sk, evk = VP(), VP()
        _check("hd_keygen", load().hd_keygen(self.h, _ptr(steps), len(steps), C.byref(sk), C.byref(evk)))
        return SecretKey(sk.value, self), EvalKeys(evk.value, self)

    def encrypt_query(self, sk, q, enc_seed, msg_scale=1.0):
        """hd_encrypt_query (msg_scale 1) / hd_encrypt_query_ex (the normalised query times msg_scale)."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        out = VP()
        if msg_scale == 1.0:
            _check("hd_encrypt_query", load().hd_encrypt_query(self.h, sk.h, _ptr(q), len(q), C.c_uint64(enc_seed),
                                                               C.byref(out)))
        else:
            _check("hd_encrypt_query_ex", load().hd_encrypt_query_ex(
                self.h, sk.h, _ptr(q), len(q), C.c_uint64(enc_seed), C.c_double(msg_scale), C.byref(out)))
        return Ciphertext(out.value, self)

    def decrypt_scores(self, sk, layout, cts):
        arr = (VP * len(cts))(*[c.h for c in cts])
        per = layout.groups_per_ct * layout.block_n
        v0 = layout.agg_begin * per
        v1 = min(layout.num_vectors, (layout.agg_begin + len(cts)) * per)
        scores = np.zeros(v1 - v0, np.float64)
        w = C.c_size_t()
        _check("hd_decrypt_scores", load().hd_decrypt_scores(self.h, sk.h, C.byref(layout), arr, len(cts),
                                                             _ptr(scores), len(scores), C.byref(w)))
        return scores

    def decrypt(self, sk, ct):
        out = np.zeros((ct.limbs, self.n), np.uint64)
        _check("hd_decrypt", load().hd_decrypt(self.h, sk.h, ct.h, _ptr(out), out.size))
        return out

    # -- enroller / server ---------------------------------------------------------------------------
    def enroll_footprint(self, num_vectors, vector_dim, n1, agg_begin=0, agg_end=0, packing="replicated",
                         encrypted=False):
        """hd_enroll_footprint: device bytes of the database handle (P:L662-664 pre-check)."""
        opt = EnrollOptions(PACKING[packing], 0, VP(1) if encrypted else None, 0)  # only pk != NULL matters
        b = C.c_size_t()
        _check("hd_enroll_footprint", load().hd_enroll_footprint(self.h, num_vectors, vector_dim, n1, agg_begin,
                                                                 agg_end, C.byref(opt), C.byref(b)))
        return b.value

    def _precheck(self, num_vectors, vector_dim, n1, agg_begin, agg_end, packing, encrypted):
        """The paper's footprint check before the upload against what the torch
        allocator can hand out: free device memory plus its own cached, unused blocks."""
        if self.allocator != "torch":
            return  # libhd checks against free device memory itself
        import torch
        need = self.enroll_footprint(num_vectors, vector_dim, n1, agg_begin, agg_end, packing, encrypted)
        free = torch.cuda.mem_get_info(self.device)[0]
        cached = torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
        if need + (256 << 20) > free + cached:
            raise HDError("hd_enroll_footprint", HD_E_CAPACITY,
                          f"database of {need >> 20} MiB exceeds available device memory "
                          f"({(free + cached) >> 20} MiB); shard the aggregates over more GPUs")

    def enroll(self, vectors, n1, agg_begin=0, agg_end=0, packing="replicated", pk=None, enc_seed=0):
        """hd_enroll_ex: plaintext (pk None) or encrypted (NEXT-1) diagonals, replicated or flat (NEXT-2)."""
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        self._precheck(vectors.shape[0], vectors.shape[1], n1, agg_begin, agg_end, packing, pk is not None)
        opt = EnrollOptions(PACKING[packing], 0, pk.h if pk is not None else None, enc_seed)
        out = VP()
        _check("hd_enroll_ex", load().hd_enroll_ex(self.h, C.byref(opt), _ptr(vectors), vectors.shape[0],
                                                   vectors.shape[1], n1, agg_begin, agg_end, C.byref(out)))
        db = Database(out.value, self)
        db.encrypted = pk is not None
        return db

    # -- encrypted-database mode (NEXT-1, R26) ------------------------------------------------
    def public_keygen(self, sk):
        out = VP()
        _check("hd_public_keygen", load().hd_public_keygen(self.h, sk.h, C.byref(out)))
        return PublicKey(out.value, self)

    def public_key_export(self, pk):
        buf = np.zeros((2, self.L, self.n), np.uint64)
        _check("hd_public_key_export", load().hd_public_key_export(pk.h, _ptr(buf), buf.size))
        return buf

    def public_key_import(self, arr):
        arr = np.ascontiguousarray(arr, dtype=np.uint64)
        out = VP()
        _check("hd_public_key_import", load().hd_public_key_import(self.h, _ptr(arr), arr.size, C.byref(out)))
        return PublicKey(out.value, self)

    def prerotation_steps(self, vector_dim, n1):
        """Negative giant-step keys of the TBS server-side pre-rotation."""
        cnt = C.c_size_t()
        _check("hd_prerotation_steps", load().hd_prerotation_steps(self.h, vector_dim, n1, None, 0, C.byref(cnt)))
        steps = np.zeros(cnt.value, np.int32)
        _check("hd_prerotation_steps", load().hd_prerotation_steps(self.h, vector_dim, n1, _ptr(steps), cnt.value,
                                                                   C.byref(cnt)))
        return steps

    def database_aggregate(self, db):
        """hd_database_aggregate: one aggregate holding the sums of db's diagonals (NEXT-4)."""
        out = VP()
        _check("hd_database_aggregate", load().hd_database_aggregate(self.h, db.h, C.byref(out)))
        agg = Database(out.value, self)
        agg.encrypted = getattr(db, "encrypted", False)
        return agg

    def database_prerotate(self, evk, db):
        _check("hd_database_prerotate", load().hd_database_prerotate(self.h, evk.h, db.h))

    def relin_keygen(self, sk, evk):
        _check("hd_relin_keygen", load().hd_relin_keygen(self.h, sk.h, evk.h))

    def enroll_encrypted(self, pk, vectors, n1, enc_seed, agg_begin=0, agg_end=0):
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        self._precheck(vectors.shape[0], vectors.shape[1], n1, agg_begin, agg_end, "replicated", True)
        out = VP()
        _check("hd_enroll_encrypted", load().hd_enroll_encrypted(
            self.h, pk.h, _ptr(vectors), vectors.shape[0], vectors.shape[1], n1, agg_begin, agg_end,
            C.c_uint64(enc_seed), C.byref(out)))
        db = Database(out.value, self)
        db.encrypted = True
        return db

    # -- encrypted comparison and scenario tail (NEXT-3, R29) ---------------------------------
    def compare(self, evk, cts, coeffs, outs=None, out_limbs=1):
        """hd_compare_ex: ChebyshevCompare of every ciphertext (identification, Alg. index)."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        if outs is None:
            outs = [None] * len(cts)
        src = (VP * len(cts))(*[c.h for c in cts])
        arr = (VP * len(cts))(*[(o.h if o is not None else None) for o in outs])
        _check("hd_compare_ex", load().hd_compare_ex(self.h, evk.h, src, len(cts), _ptr(coeffs), len(coeffs) - 1,
                                                     out_limbs, arr))
        return [o if o is not None else Ciphertext(arr[i], self) for i, o in enumerate(outs)]

    def membership_steps(self):
        cnt = C.c_size_t()
        _check("hd_membership_steps", load().hd_membership_steps(self.h, None, 0, C.byref(cnt)))
        steps = np.zeros(cnt.value, np.int32)
        _check("hd_membership_steps", load().hd_membership_steps(self.h, _ptr(steps), cnt.value, C.byref(cnt)))
        return steps

    def membership(self, evk, cts, out=None):
        src = (VP * len(cts))(*[c.h for c in cts])
        o = VP(out.h if out is not None else None)
        _check("hd_membership", load().hd_membership(self.h, evk.h, src, len(cts), C.byref(o)))
        return out if out is not None else Ciphertext(o.value, self)

    def eval_add_many(self, cts, out=None):
        src = (VP * len(cts))(*[c.h for c in cts])
        o = VP(out.h if out is not None else None)
        _check("hd_eval_add_many", load().hd_eval_add_many(self.h, src, len(cts), C.byref(o)))
        return out if out is not None else Ciphertext(o.value, self)

    def ciphertext_scale(self, ct):
        v = C.c_double()
        _check("hd_ciphertext_scale", load().hd_ciphertext_scale(ct.h, C.byref(v)))
        return v.value

    def decrypt_slots(self, sk, ct):
        z = np.zeros(self.n // 2, np.float64)
        _check("hd_decrypt_slots", load().hd_decrypt_slots(self.h, sk.h, ct.h, _ptr(z), z.size))
        return z

    def query(self, evk, db, query, outs=None):
        nloc = db.num_local
        if outs is None:
            outs = [None] * nloc
        arr = (VP * nloc)(*[(o.h if o is not None else None) for o in outs])
        _check("hd_query", load().hd_query(self.h, evk.h, db.h, query.h, arr, nloc))
        return [o if o is not None else Ciphertext(arr[i], self) for i, o in enumerate(outs)]

    def query_batch(self, evk, db, queries, outs=None):
        """hd_query_batch: outs[q][i] = score ciphertext of local aggregate i for queries[q] (NEXT-4)."""
        nloc, Q = db.num_local, len(queries)
        flat = [None] * (Q * nloc) if outs is None else [o for row in outs for o in row]
        qs = (VP * Q)(*[x.h for x in queries])
        arr = (VP * (Q * nloc))(*[(o.h if o is not None else None) for o in flat])
        _check("hd_query_batch", load().hd_query_batch(self.h, evk.h, db.h, qs, Q, arr, Q * nloc))
        res = [o if o is not None else Ciphertext(arr[i], self) for i, o in enumerate(flat)]
        return [res[q * nloc:(q + 1) * nloc] for q in range(Q)]

    def baby_steps(self, evk, db, query, i_begin, i_end, r_dev_ptr):
        """hd_baby_steps: r[i] for i in [i_begin, i_end) into the device buffer at r_dev_ptr."""
        _check("hd_baby_steps", load().hd_baby_steps(self.h, evk.h, db.h, query.h, i_begin, i_end,
                                                     C.c_void_p(r_dev_ptr)))

    def query_baby(self, evk, db, r_dev_ptr, outs=None):
        nloc = db.num_local
        if outs is None:
            outs = [None] * nloc
        arr = (VP * nloc)(*[(o.h if o is not None else None) for o in outs])
        _check("hd_query_baby", load().hd_query_baby(self.h, evk.h, db.h, C.c_void_p(r_dev_ptr), arr, nloc))
        return [o if o is not None else Ciphertext(arr[i], self) for i, o in enumerate(outs)]

    def query_stats(self):
        """[baby, mac, rescale, giant, fold, baby_kip] ms averaged over the queries since the last call."""
        ms = np.zeros(6, np.float64)
        _check("hd_query_stats", load().hd_query_stats(self.h, _ptr(ms), 6))
        return ms

    def launch_count(self):
        v = C.c_uint64()
        _check("hd_launch_count", load().hd_launch_count(self.h, C.byref(v)))
        return v.value

    # -- serialisation -----------------------------------------------------------------------------
    def ciphertext_export(self, ct, dst=None, on_device=False):
        """Export to a new numpy uint8 array (host) or into ``dst`` (pointer int + capacity) on device."""
        w = C.c_size_t()
        _check("hd_ciphertext_export", load().hd_ciphertext_export(ct.h, None, 0, 0, C.byref(w)))
        if dst is None:
            buf = np.zeros(w.value, np.uint8)
            _check("hd_ciphertext_export", load().hd_ciphertext_export(ct.h, _ptr(buf), w.value, 0, C.byref(w)))
            return buf
        ptr, cap = dst
        _check("hd_ciphertext_export", load().hd_ciphertext_export(ct.h, VP(ptr), cap, 1 if on_device else 0,
                                                                   C.byref(w)))
        return w.value

    def ciphertext_export_async(self, ct, dst, nlimbs=0, on_device=False):
        """Level-reduced asynchronous export (hd_ciphertext_export_async): ``dst`` is
        (pointer int, capacity) or None to query the size; data valid after synchronize()."""
        w = C.c_size_t()
        if dst is None:
            _check("hd_ciphertext_export_async",
                   load().hd_ciphertext_export_async(ct.h, nlimbs, None, 0, 0, C.byref(w)))
            return w.value
        ptr, cap = dst
        _check("hd_ciphertext_export_async", load().hd_ciphertext_export_async(
            ct.h, nlimbs, VP(ptr), cap, 1 if on_device else 0, C.byref(w)))
        return w.value

    def ciphertext_export_level(self, ct, dst, nlimbs=0, on_device=True):
        """hd_ciphertext_export_level: stream-ordered level-reduced export into ``dst`` = (ptr, cap)
        (None: return the size).  A device destination never synchronises the host."""
        w = C.c_size_t()
        if dst is None:
            _check("hd_ciphertext_export_level",
                   load().hd_ciphertext_export_level(ct.h, nlimbs, None, 0, 0, C.byref(w)))
            return w.value
        ptr, cap = dst
        _check("hd_ciphertext_export_level", load().hd_ciphertext_export_level(
            ct.h, nlimbs, VP(ptr), cap, 1 if on_device else 0, C.byref(w)))
        return w.value

    def synchronize(self):
        _check("hd_context_synchronize", load().hd_context_synchronize(self.h))

    def ciphertext_export_size(self, ct):
        w = C.c_size_t()
        _check("hd_ciphertext_export", load().hd_ciphertext_export(ct.h, None, 0, 0, C.byref(w)))
        return w.value

    def ciphertext_import(self, src, nbytes=None, on_device=False):
        out = VP()
        if isinstance(src, np.ndarray):
            _check("hd_ciphertext_import", load().hd_ciphertext_import(self.h, _ptr(src), src.nbytes, 0,
                                                                       C.byref(out)))
        else:
            _check("hd_ciphertext_import", load().hd_ciphertext_import(self.h, VP(src), nbytes,
                                                                       1 if on_device else 0, C.byref(out)))
        return Ciphertext(out.value, self)

    def ciphertext_import_into(self, ct, src, nbytes=None, on_device=False):
        if isinstance(src, np.ndarray):
            _check("hd_ciphertext_import_into", load().hd_ciphertext_import_into(ct.h, _ptr(src), src.nbytes, 0))
        else:
            _check("hd_ciphertext_import_into", load().hd_ciphertext_import_into(ct.h, VP(src), nbytes,
                                                                                 1 if on_device else 0))

    def ciphertext_residues(self, ct):
        """Residues [2][limbs][n] (host copy, via the canonical export)."""
        buf = self.ciphertext_export(ct)
        return buf[64:].view(np.uint64).reshape(2, -1, self.n).copy()

    def eval_keys_export(self, evk):
        w = C.c_size_t()
        _check("hd_eval_keys_export", load().hd_eval_keys_export(evk.h, None, 0, 0, C.byref(w)))
        buf = np.zeros(w.value, np.uint8)
        _check("hd_eval_keys_export", load().hd_eval_keys_export(evk.h, _ptr(buf), w.value, 0, C.byref(w)))
        return buf

    def eval_keys_import(self, buf):
        out = VP()
        _check("hd_eval_keys_import", load().hd_eval_keys_import(self.h, _ptr(buf), buf.nbytes, 0, C.byref(out)))
        return EvalKeys(out.value, self)

    def secret_key_export(self, sk):
        out = np.zeros((self.M, self.n), np.uint64)
        _check("hd_secret_key_export", load().hd_secret_key_export(sk.h, _ptr(out), out.size))
        return out

    # -- test-only stage entry points ----------------------------------------------------------------
    def test_ntt(self, rows, modulus_idx, inverse=False):
        rows = np.ascontiguousarray(rows, dtype=np.uint64).copy()
        mi = np.ascontiguousarray(modulus_idx, dtype=np.uint32)
        _check("hd_test_ntt", load().hd_test_ntt(self.h, _ptr(rows), rows.shape[0], _ptr(mi), 1 if inverse else 0))
        return rows

    def test_stage(self, db, which, agg, index):
        enc = getattr(db, "encrypted", False)
        ell = self.L if which in (0, 1) else (self.L - 1 if which in (2, 3) else self.L)
        shape = ((2, self.L, self.n) if enc else (self.L, self.n)) if which == 4 else \
            (3 if which == 1 and enc else 2, ell, self.n)
        out = np.zeros(shape, np.uint64)
        _check("hd_test_stage", load().hd_test_stage(db.h, which, agg, index, _ptr(out), out.size))
        return out

    def test_inject(self, db, agg, k, word, mask):
        """hd_test_inject: XOR one word of D[agg][k] on the device (fault injection)."""
        _check("hd_test_inject", load().hd_test_inject(db.h, agg, k, C.c_uint64(word), C.c_uint64(mask)))

    def test_rotate(self, evk, ct, step):
        out = VP()
        _check("hd_test_rotate", load().hd_test_rotate(self.h, evk.h, ct.h, step, C.byref(out)))
        return Ciphertext(out.value, self)

    def test_rescale(self, ct):
        out = VP()
        _check("hd_test_rescale", load().hd_test_rescale(self.h, ct.h, C.byref(out)))
        return Ciphertext(out.value, self)


def chebyshev_degree(kappa):
    d = C.c_uint32()
    _check("hd_chebyshev_degree", load().hd_chebyshev_degree(kappa, C.byref(d)))
    return d.value


def chebyshev_coefficients(delta, degree):
    """Client side (host): coefficients of the Chebyshev sign approximation (R29)."""
    c = np.zeros(degree + 1, np.float64)
    _check("hd_chebyshev_coefficients", load().hd_chebyshev_coefficients(C.c_double(delta), degree, _ptr(c),
                                                                         c.size))
    return c


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return VP(stream)
    return VP(stream.cuda_stream)  # torch.cuda.Stream


def eval_key_residues(ctx: Context, buf: np.ndarray):
    """Split an exported eval-key buffer into (steps, keys[count][L][2][L+1][n])."""
    count = int(buf[20:24].view(np.uint32)[0])
    steps_bytes = ((count * 4 + 63) // 64) * 64
    steps = buf[64:64 + count * 4].view(np.int32).copy()
    keys = buf[64 + steps_bytes:].view(np.uint64).reshape(count, ctx.beta, 2, ctx.M, ctx.n)
    return steps, keys
