"""CPU-side checks of the C ABI library: it loads, exports every symbol include/vp.h declares,
struct layouts agree with the binding, and host-detectable errors are reported synchronously
(no GPU needed for any of these calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "vp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = _declared_symbols()
    for s in ("vp_plan_frames", "vp_resize_normalize_patchify", "vp_rope_index"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    # Load _build.py by path: importing the package needs the library it builds.
    import importlib.util
    spec = importlib.util.spec_from_file_location("_vp_build", os.path.join(ROOT, "paper_2604_16893_b200", "_build.py"))
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)
    lib = C.CDLL(_build.build())
    for s in _declared_symbols():
        assert hasattr(lib, s), s


def test_binding_loads_and_struct_sizes_match():
    import paper_2604_16893_b200 as vp
    from paper_2604_16893_b200 import _lib
    assert set(_declared_symbols()) == set(_lib.EXPORTED)
    assert vp.lib.vp_abi_version() == 1
    assert C.sizeof(vp.VpParams) == 120 and vp.DESC_DTYPE.itemsize == 32 and vp.PLAN_DTYPE.itemsize == 104


def test_host_side_errors_are_synchronous():
    import paper_2604_16893_b200 as vp
    L = vp.lib
    bad = vp.make_params(max_frames=1, temporal_patch_size=2)           # S:33 max_frames >= tp
    assert L.vp_plan_frames(C.byref(bad), None, 0, None, None, 0, None, 0, None, None) == vp.VP_EINVAL
    assert b"max_frames" in L.vp_last_error_detail()
    small = vp.make_params(video_max_pixels=100)                         # S:32 budget >= f^2
    assert L.vp_plan_frames(C.byref(small), None, 0, None, None, 0, None, 0, None, None) == vp.VP_EINVAL
    ok = vp.make_params()
    assert L.vp_plan_frames(C.byref(ok), None, 0, None, None, 0, None, 0, None, None) == vp.VP_EINVAL  # null totals
    assert L.vp_rope_index(C.byref(ok), 7, None, None, 0, 0, None, 0, None, 0, None, 0, None, None, None, None, 0,
                           None) == vp.VP_EINVAL
    assert L.vp_rope_index_workspace_bytes(4, 3) >= (8 + 4) * 8
    with pytest.raises(vp.VpError):
        vp._lib.check(vp.VP_EINVAL, "x")
    assert L.vp_status_string(vp.VP_EMISMATCH).startswith(b"VP_EMISMATCH")


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_16893_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f
                assert "vp_oracle" not in txt, f
