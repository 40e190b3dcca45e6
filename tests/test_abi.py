"""C-ABI checks that need no GPU: the in-tree library loads, exports every
entry point include/ssb_api.h declares, and rejects bad descriptors with
SSB_EINVAL / SSB_EUNSUPPORTED before touching the device."""
import ctypes as C
import os
import re

import pytest

from paper_2602_08642_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ssb_api.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load(build_if_missing=True)


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.ssb_version() == 1


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def _desc(**kw):
    d = _lib.PyrDesc()
    d.batch, d.channels, d.height, d.width = 1, 3, 16, 16
    d.levels, d.ksize = 3, 5
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def test_plan_queries(lib):
    d = _desc()
    assert [lib.ssb_pyr_logit_channels(C.byref(d), l) for l in range(3)] == [29, 29, 25]
    d2 = _desc(has_prev=1, blend_mode=1)
    assert [lib.ssb_pyr_logit_channels(C.byref(d2), l) for l in range(3)] == [51, 26, 25]
    h, w = C.c_int32(), C.c_int32()
    d3 = _desc(height=7, width=10, levels=5)
    dims = []
    for l in range(5):
        assert lib.ssb_pyr_level_dims(C.byref(d3), l, C.byref(h), C.byref(w)) == 0
        dims.append((h.value, w.value))
    assert dims == [(7, 10), (4, 5), (2, 3), (1, 2), (1, 1)]  # ref test_pyramid.py:54-55
    tb, wb = C.c_size_t(), C.c_size_t()
    assert lib.ssb_pyr_tape_bytes(C.byref(d), C.byref(tb)) == 0 and tb.value > 0
    assert lib.ssb_pyr_workspace_bytes(C.byref(d), C.byref(wb)) == 0 and wb.value > 0


@pytest.mark.parametrize("field,value,code", [
    ("ksize", 4, -3), ("ksize", 9, -3), ("levels", 0, -1), ("levels", 9, -1),
    ("height", 0, -1), ("logit_dtype", 1, -3), ("blend_mode", 5, -1),
])
def test_bad_descriptors_rejected(lib, field, value, code):
    d = _desc(image_dtype=2, logit_dtype=2)
    setattr(d, field, value)
    io = _lib.PyrFwdIO()
    assert lib.ssb_pyr_forward(C.byref(d), C.byref(io), None, None) == code
    assert lib.ssb_last_error()


def test_missing_buffers_rejected(lib):
    d = _desc()
    io = _lib.PyrFwdIO()
    assert lib.ssb_pyr_forward(C.byref(d), C.byref(io), None, None) == -1
    assert b"required" in lib.ssb_last_error()


def test_infer_small_rejects_before_the_device(lib):
    """ssb_infer_small validates its arguments before any CUDA call: missing
    buffers -> SSB_EINVAL; shapes outside the small-frame path (capacity 3,
    W % 4 != 0, > 2^20 pixels, k = 9) -> SSB_EUNSUPPORTED (the caller then
    runs ssb_place_fused + ssb_pyr_forward)."""
    P = C.c_void_p
    fake = C.c_void_p(0x1000)  # never dereferenced: rejected first
    logits = (C.c_void_p * 3)(fake, fake, fake)

    def call(B=1, H=64, W=64, S=2, k=5, levels=3, scores=fake, lg=logits):
        d = _lib.PlaceDesc(B, H, W, S, _lib.VARIANTS["stochastic"], 0, 1, 0, 0.25)
        return lib.ssb_infer_small(C.byref(d), scores, fake, fake, levels, k, lg, fake, fake, fake, None)

    assert call(scores=P(0)) == -1
    assert call(lg=(C.c_void_p * 3)(fake, None, fake)) == -1
    assert call(levels=0) == -1
    assert call(S=3) == -3
    assert call(W=66) == -3
    assert call(H=1100, W=1000) == -3
    assert call(k=9) == -3
    wb = C.c_size_t()
    assert lib.ssb_infer_small_workspace_bytes(1, 256, 256, 3, C.byref(wb)) == 0 and wb.value > 256 * 256 * 12
    assert lib.ssb_infer_small_workspace_bytes(1, 256, 256, 0, C.byref(wb)) == -1
