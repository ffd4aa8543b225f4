"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

from __future__ import annotations

import ctypes
import re

from conftest import ROOT


def header_functions():
    text = (ROOT / "include" / "voxelray_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+[\s\*]+(vr_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ("vr_render", "vr_render_to_host", "vr_grid_create", "vr_grid_visibility",
                 "vr_volume_create", "vr_threshold_count", "vr_sample_points"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2005_01442_b200 import _build, _lib

    _build.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(header_functions()) == set(_lib.EXPORTS)
    L = _lib.load()
    assert L.vr_abi_version() == 1


def test_struct_layouts_match_header():
    from paper_2005_01442_b200 import _lib

    # 10 int32 then 14 doubles
    assert ctypes.sizeof(_lib.Camera) == 40 + 14 * 8
    assert _lib.Camera.position.offset == 40
    assert _lib.RenderOutputs.ev_stop.offset == 9 * 8
    assert _lib.RenderParams.margin.offset == ctypes.sizeof(_lib.RenderParams) - 8


def test_errors_without_gpu_are_loud():
    """Argument validation runs before any device work and maps to the
    reference's exception classes."""
    import pytest

    from paper_2005_01442_b200 import _lib, errors

    L = _lib.load()
    h = ctypes.c_void_p()
    st = L.vr_grid_create(None, 64, 3, None, ctypes.byref(h))
    with pytest.raises(errors.InvalidSettings):
        _lib.check(st)
