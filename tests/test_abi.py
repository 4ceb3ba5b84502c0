"""The C-ABI library loads and exports every symbol include/hd.h declares (not gpu).

No compute call is made here; on a box without a GPU the context constructor
must refuse (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for call in ("hd_keygen", "hd_enroll", "hd_query", "hd_decrypt_scores", "hd_encrypt_query",
                 "hd_rotation_steps", "hd_context_create"):
        assert call in names


def test_library_exports_every_declared_symbol():
    import paper_2604_00546_b200 as hd
    lib = hd.load()
    path = hd.lib_path()
    assert os.path.exists(path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(hd.ABI_FUNCTIONS)
    # every symbol is a plain C symbol (extern "C": unmangled)
    raw = C.CDLL(path)
    for n in _declared():
        getattr(raw, n)


def test_library_is_sm100a():
    import subprocess
    import paper_2604_00546_b200 as hd
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hd.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2604_00546_b200 as hd
    with pytest.raises(hd.HDError) as e:
        hd.Context(12)
    assert e.value.code == hd.HD_E_CUDA


def test_host_chebyshev_coefficients_match_the_oracle(oracle_mod):
    """Client-side host functions (no device): the kappa table of P:L721 and coefficients
    identical to the oracle's, bit for bit (both sides must encode the same constants)."""
    import numpy as np
    import paper_2604_00546_b200 as hd
    assert [hd.chebyshev_degree(k) for k in (7, 8, 9, 10)] == [5, 13, 27, 59]
    with pytest.raises(hd.HDError):
        hd.chebyshev_degree(6)
    for delta, n in ((0.5, 13), (-0.2, 5), (0.0, 27), (0.75, 59)):
        assert (hd.chebyshev_coefficients(delta, n) == oracle_mod.cheb_coeffs(delta, n)).all()


def test_host_chebyshev_error_paths():
    """Client-side host calls reject bad arguments (no device involved)."""
    import ctypes as C

    import numpy as np
    import paper_2604_00546_b200 as hd
    L = hd.load()
    buf = np.zeros(4, np.float64)
    assert L.hd_chebyshev_coefficients(C.c_double(0.5), 13, buf.ctypes.data_as(C.c_void_p), 4) == -1  # cap
    assert L.hd_chebyshev_coefficients(C.c_double(0.5), 0, buf.ctypes.data_as(C.c_void_p), 4) == -1   # degree 0
    d = C.c_uint32()
    assert L.hd_chebyshev_degree(11, C.byref(d)) == -1 and L.hd_chebyshev_degree(8, C.byref(d)) == 0
    assert d.value == 13


def test_baby_slices_cover_every_step_once():
    from paper_2604_00546_b200 import dist as hdd
    for n1 in (1, 7, 8, 23, 128):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                chunk, i0, i1 = hdd.baby_slice(n1, r, world)
                assert 0 <= i1 - i0 <= chunk and chunk * world >= n1
                got += list(range(i0, i1))
            assert got == list(range(n1))
