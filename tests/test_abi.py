"""CPU checks of the C ABI boundary: libholo.so builds, loads without a GPU,
exports exactly the symbols include/holo.h declares, and rejects bad
arguments on the host with the documented status codes (no compute call)."""
import ctypes as C
import os
import re

import pytest

from paper_2004_04049_b200 import build as hb
from paper_2004_04049_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    hb.build()
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "holo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(holo_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    # the Python binding marshals every declared entry point and nothing else
    assert sorted(_lib.SIGNATURES) == syms


def test_version_and_kernel_names(L):
    assert L.holo_version().decode().startswith("holo")
    names = L.holo_kernel_names().decode().split(",")
    assert "ospr_cols" in names and "gs_rows" in names and "lut_generate" in names


def _region(r0, r1, c0, c1):
    return _lib.HoloRegion(r0, r1, c0, c1)


FAKE = C.c_void_p(0x1000)   # never dereferenced: checks fail before any CUDA call


def test_lut_generate_arg_errors(L):
    assert L.holo_lut_generate(1, 0, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_lut_generate(1, 1 << 31, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert b"n_lut" in L.holo_last_error()
    assert L.holo_lut_generate(1, 5, None, None) == _lib.HOLO_ERR_INVALID_ARG
    assert b"NULL" in L.holo_last_error()


def test_ospr_arg_errors(L):
    ok = dict(n=64, F=1, S=8, lut=FAKE, nl=256, b=0, e=8, om=_region(1, 32, 0, 64), ws=FAKE,
              wsb=L.holo_ospr_workspace_size(64, 1, 8))

    def call(**kw):
        a = dict(ok, **kw)
        return L.holo_ospr_generate(FAKE, a["n"], a["F"], a["S"], a["lut"], a["nl"], 0, a["b"], a["e"], None,
                                    FAKE, None, a["om"], a["ws"], a["wsb"], None)

    assert call(n=100) == _lib.HOLO_ERR_INVALID_ARG
    assert call(n=8192) == _lib.HOLO_ERR_INVALID_ARG
    assert call(n=8) == _lib.HOLO_ERR_INVALID_ARG
    assert call(S=0) == _lib.HOLO_ERR_INVALID_ARG
    assert call(b=3, e=3) == _lib.HOLO_ERR_INVALID_ARG
    assert call(e=9) == _lib.HOLO_ERR_INVALID_ARG
    assert call(lut=None) == _lib.HOLO_ERR_INVALID_ARG          # lut NULL but n_lut > 0
    assert call(nl=0) == _lib.HOLO_ERR_INVALID_ARG             # lut given but n_lut == 0
    assert call(om=_region(5, 5, 0, 64)) == _lib.HOLO_ERR_INVALID_ARG
    assert call(om=_region(0, 65, 0, 64)) == _lib.HOLO_ERR_INVALID_ARG
    assert call(wsb=16) == _lib.HOLO_ERR_WORKSPACE
    # mse requested for a partial range
    r = L.holo_ospr_generate(FAKE, 64, 1, 8, FAKE, 256, 0, 0, 4, None, FAKE, FAKE, _region(1, 32, 0, 64), FAKE,
                             ok["wsb"], None)
    assert r == _lib.HOLO_ERR_INVALID_ARG


def test_gs_arg_errors(L):
    ws = L.holo_gs_workspace_size(64, 2, 3)
    assert ws > 0
    om = _region(0, 64, 0, 64)

    def call(levels=0, iters=3, lev_out=None, wsb=ws, n=64):
        return L.holo_gs_generate(FAKE, n, 2, iters, FAKE, 97, 0, levels, FAKE, lev_out, FAKE, FAKE, FAKE, om, FAKE,
                                  wsb, None)

    assert call(levels=1) == _lib.HOLO_ERR_UNSUPPORTED
    assert call(levels=70000) == _lib.HOLO_ERR_UNSUPPORTED
    assert call(levels=0, lev_out=FAKE) == _lib.HOLO_ERR_INVALID_ARG
    assert call(levels=512, lev_out=FAKE) == _lib.HOLO_ERR_INVALID_ARG
    assert call(iters=0) == _lib.HOLO_ERR_INVALID_ARG
    assert call(wsb=ws - 1) == _lib.HOLO_ERR_WORKSPACE
    assert call(n=48) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_gs_step(FAKE, FAKE, 64, 1, 0, FAKE, None, None, None, None, None, om, FAKE, 0, None) == \
        _lib.HOLO_ERR_INVALID_ARG   # r_in aliases r_out


def test_debug_pairs_arg_errors(L):
    def call(n=64, S=4, lut=FAKE, nl=97, prng=0, b=0, e=4, z=FAKE):
        return L.holo_debug_ospr_pairs(FAKE, n, S, lut, nl, prng, 7, 0, b, e, z, None)

    assert call(n=96) == _lib.HOLO_ERR_INVALID_ARG
    assert call(z=None) == _lib.HOLO_ERR_INVALID_ARG
    assert call(e=5) == _lib.HOLO_ERR_INVALID_ARG              # sub-frame range outside [0, n_sub)
    assert call(b=2, e=2) == _lib.HOLO_ERR_INVALID_ARG
    assert call(lut=None) == _lib.HOLO_ERR_INVALID_ARG         # lut NULL but n_lut > 0
    assert call(prng=1) == _lib.HOLO_ERR_INVALID_ARG           # the on-the-fly source excludes a LUT
    assert b"prng" in L.holo_last_error()


def test_workspace_sizes_monotone(L):
    assert L.holo_ospr_workspace_size(1024, 1, 24) >= 8 * 1024 * 1024 + 4 * 1024 * 1024
    assert L.holo_ospr_workspace_size(100, 1, 24) == 0
    assert L.holo_gs_workspace_size(1024, 64, 50) > L.holo_gs_workspace_size(1024, 8, 50)


def test_profile_read_unknown_name(L):
    n = C.c_uint64()
    ms = C.c_double()
    assert L.holo_profile_read(b"nope", C.byref(n), C.byref(ms)) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_profile_read(b"ospr_cols", C.byref(n), C.byref(ms)) == _lib.HOLO_OK
    assert n.value == 0


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: a missing libholo.so raises instead of silently degrading."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libholo.so"))
    with pytest.raises(ImportError):
        _lib.lib()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2004_04049_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "holo_oracle" not in txt and "liboracle" not in txt, f


def test_plan_queries(L):
    assert L.holo_ospr_chunk_pairs(1024, 24) == 12          # C3: one chunk of 12 pairs
    assert L.holo_ospr_chunk_pairs(2048, 32) == 16          # C5: one chunk of 16 pairs (512 MiB)
    assert L.holo_ospr_chunk_pairs(2048, 200) == 32         # capped by the 1 GiB budget
    assert L.holo_ospr_chunk_pairs(64, 7) == 4
    assert L.holo_ospr_chunk_pairs(100, 7) == 0 and L.holo_ospr_chunk_pairs(64, 0) == 0
    assert L.holo_gs_group_frames(1024, 64) == 64
    assert L.holo_gs_group_frames(64, 3) == 3
    assert L.holo_gs_group_frames(64, 0) == 0
    assert L.holo_ospr_finalize_workspace_size() >= 592 * 5 * 8 + 4
    assert L.holo_ospr_workspace_size(1024, 1, 24) >= L.holo_ospr_finalize_workspace_size()


def test_round2_entry_points_arg_errors(L):
    """The row-slice a7, MSE-from-sums and sin/cos-table entry points validate their arguments on
    the host (no device work before the checks)."""
    om = _region(1, 32, 0, 64)
    fin = L.holo_ospr_finalize_workspace_size()
    # row slice empty, reversed or outside the frame
    for r0, r1 in ((5, 5), (9, 3), (-1, 4), (60, 65)):
        assert L.holo_ospr_finalize_rows(FAKE, FAKE, 64, r0, r1, 8, om, FAKE, FAKE, FAKE, fin, None) == \
            _lib.HOLO_ERR_INVALID_ARG
    assert b"row slice" in L.holo_last_error()
    assert L.holo_ospr_finalize_rows(FAKE, FAKE, 64, 0, 8, 0, om, FAKE, FAKE, FAKE, fin, None) == \
        _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_finalize_rows(FAKE, FAKE, 64, 0, 8, 8, om, FAKE, None, FAKE, fin, None) == \
        _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_finalize_rows(FAKE, FAKE, 64, 0, 8, 8, om, FAKE, FAKE, FAKE, fin - 8, None) == \
        _lib.HOLO_ERR_WORKSPACE
    assert L.holo_ospr_finalize_rows(FAKE, FAKE, 100, 0, 8, 8, om, FAKE, FAKE, FAKE, fin, None) == \
        _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_mse_from_sums(None, 1, om, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_mse_from_sums(FAKE, 0, om, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_mse_from_sums(FAKE, 1, _region(3, 3, 0, 8), FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    # phase table: 1 <= phase_bits <= 16
    for q in (0, 17, -3):
        assert L.holo_phase_table(q, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert b"phase_bits" in L.holo_last_error()
    assert L.holo_phase_table(8, None, None) == _lib.HOLO_ERR_INVALID_ARG
    ws = L.holo_ospr_workspace_size(64, 1, 8)
    for q, tbl in ((0, FAKE), (17, FAKE), (8, None)):
        assert L.holo_ospr_generate_prng_table(FAKE, 64, 1, 8, 7, tbl, q, 0, 0, 8, None, FAKE, FAKE, om, FAKE, ws,
                                               None) == _lib.HOLO_ERR_INVALID_ARG


def test_ospr_stream_arg_errors(L):
    """The frame stream's create/submit checks run on the host before any CUDA call."""
    h = C.c_void_p()
    slots = (C.c_void_p * 7)(*([FAKE] * 6 + [None]))
    ws_ok = L.holo_ospr_workspace_size(64, 1, 4)

    def create(**kw):
        a = dict(n=64, S=4, depth=1, lut=FAKE, nl=256, regen=0, slots=slots, ws=FAKE, wsb=ws_ok)
        a.update(kw)
        return L.holo_ospr_stream_create(a["n"], a["S"], a["depth"], a["lut"], a["nl"], a["regen"], 7, 0, 1, 1,
                                         _region(1, 32, 0, 64), a["slots"], a["ws"], a["wsb"], C.byref(h))

    assert create(n=100) == _lib.HOLO_ERR_INVALID_ARG
    assert create(S=0) == _lib.HOLO_ERR_INVALID_ARG
    assert create(depth=0) == _lib.HOLO_ERR_INVALID_ARG and create(depth=17) == _lib.HOLO_ERR_INVALID_ARG
    assert create(lut=None) == _lib.HOLO_ERR_INVALID_ARG                       # n_lut > 0 without a pool
    assert create(lut=None, nl=0, regen=1) == _lib.HOLO_ERR_INVALID_ARG        # a0 needs a pool
    assert create(slots=None) == _lib.HOLO_ERR_INVALID_ARG
    assert create(slots=(C.c_void_p * 7)(*([FAKE] * 3 + [None] + [FAKE] * 3))) == _lib.HOLO_ERR_INVALID_ARG
    assert create(ws=None) == _lib.HOLO_ERR_INVALID_ARG
    assert create(wsb=ws_ok - 1) == _lib.HOLO_ERR_WORKSPACE
    assert not h.value                                                          # nothing was created
    assert L.holo_ospr_stream_submit(None, FAKE, None) == _lib.HOLO_ERR_INVALID_ARG
    assert L.holo_ospr_stream_done(None, 0) == -1
    L.holo_ospr_stream_destroy(None)                                            # no-op
