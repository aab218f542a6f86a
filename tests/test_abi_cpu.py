"""CPU-side checks of the boundary: libwect.so loads and exports every symbol that
include/wect.h declares; the Python binding rejects bad arguments before any
device work.  No compute calls (no GPU here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wect.h")).read()
    return sorted(set(re.findall(r"WECT_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("wect_complex", "wect_images", "ecf_complex", "ecf_images", "wect_complex_backward",
              "ecf_complex_backward", "wect_maxheight", "wect_sync_status", "wect_last_error", "wect_repair_count",
              "wect_abi_version"):
        assert n in names


def test_library_builds_and_exports_every_symbol():
    from paper_2511_03909_b200 import build as b

    lib = b.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, re.M))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    from paper_2511_03909_b200 import _lib

    L = _lib.load()
    assert L.wect_abi_version() == 1
    for n in _lib.EXPORTS:
        assert hasattr(L, n)


def test_sm100a_code_present():
    from paper_2511_03909_b200 import build as b

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_are_synchronous():
    """EINVAL / EOVERFLOW / ENOTSUP are returned before anything touches a device."""
    import numpy as np

    import paper_2511_03909_b200 as w
    from paper_2511_03909_b200 import _lib

    img = np.zeros((1, 4, 4), np.uint8)
    dirs = np.zeros((3, 2), np.float32)
    with pytest.raises(w.WectError) as e:
        w.wect_images(img, dirs, 1)  # T < 2
    assert e.value.status == _lib.EINVAL
    with pytest.raises(w.WectError) as e:
        w.wect_images(img, dirs, 8, d_begin=2, d_count=5)
    assert e.value.status == _lib.EINVAL
    big = np.zeros((1, 256, 256, 256), np.uint8)
    with pytest.raises(w.WectError) as e:
        w.wect_images(big, np.zeros((3, 3), np.float32), 8, out_dtype="int32")  # 255 * 511^3 >= 2^31
    assert e.value.status == _lib.EOVERFLOW
    coords = np.zeros((3, 2), np.float32)
    cells = [(np.array([[0, 1]], np.int32), np.array([1], np.int32), 1)]
    with pytest.raises(w.WectError) as e:
        w.wect_complex(coords, [(np.array([[0, 1]], np.int32), None, 0)], np.zeros((2, 2), np.float32), 8)  # dim 0
    assert e.value.status == _lib.EINVAL
    with pytest.raises(w.WectError) as e:
        w.wect_complex(np.zeros((3, 9), np.float32), cells, np.zeros((2, 9), np.float32), 8)  # n = 9 > 8
    assert e.value.status == _lib.EINVAL


def test_new_entry_points_reject_bad_arguments_synchronously():
    """ecf_images and the backward calls validate before touching a device (no GPU here)."""
    import ctypes

    import numpy as np

    from paper_2511_03909_b200 import _lib

    L = _lib.load()
    img = np.zeros((1, 4, 4), np.uint8)
    out = np.zeros((1, 8), np.int32)
    dims = (ctypes.c_int64 * 2)(4, 4)
    g = _lib.wect_grid(1, 0, 0, 0.0, 0.0, 0.0, 0)  # T < 2
    assert L.ecf_images(img.ctypes.data, 1, 2, dims, ctypes.byref(g), out.ctypes.data, _lib.I32, None) == _lib.EINVAL
    g = _lib.wect_grid(8, 0, 0, 0.0, 0.0, 0.0, 0)
    assert L.ecf_images(img.ctypes.data, 1, 5, dims, ctypes.byref(g), out.ctypes.data, _lib.I32, None) == _lib.EINVAL
    assert L.ecf_images(img.ctypes.data, 1, 2, dims, ctypes.byref(g), out.ctypes.data, _lib.F64, None) == _lib.EINVAL
    # wect_complex_backward: NULL complex, T < 2
    G = np.zeros((2, 8))
    gv = np.zeros(4)
    assert L.wect_complex_backward(None, None, 2, ctypes.byref(g), G.ctypes.data, gv.ctypes.data, None,
                                   None) == _lib.EINVAL
    # Freudenthal volumes are not supported (a synchronous ENOTSUP)
    vol = np.zeros((1, 3, 3, 3), np.uint8)
    d3 = (ctypes.c_int64 * 3)(3, 3, 3)
    dirs = np.zeros((2, 3), np.float32)
    o3 = np.zeros((1, 2, 8), np.int32)
    gf = _lib.wect_grid(8, 0, 0, 0.0, 0.0, 0.0, _lib.FREUDENTHAL)
    assert L.wect_images(vol.ctypes.data, 1, 3, d3, dirs.ctypes.data, 2, ctypes.byref(gf), o3.ctypes.data, _lib.I32,
                         None) == _lib.ENOTSUP


def test_out_argument_is_validated_before_the_call():
    """a caller-supplied out= with the wrong size, dtype or layout is rejected in
    the binding (the C ABI only sees a pointer and would write out of bounds)."""
    import numpy as np
    import torch

    import paper_2511_03909_b200 as w

    img = np.zeros((2, 4, 4), np.uint8)
    dirs = np.zeros((3, 2), np.float32)
    with pytest.raises(ValueError, match="elements"):
        w.wect_images(img, dirs, 8, out=torch.empty((2, 3, 7), dtype=torch.int32))
    with pytest.raises(ValueError, match="dtype"):
        w.wect_images(img, dirs, 8, out=torch.empty((2, 3, 8), dtype=torch.int64))
    with pytest.raises(ValueError, match="contiguous"):
        w.wect_images(img, dirs, 8, out=torch.empty((2, 8, 3), dtype=torch.int32).transpose(1, 2))
    with pytest.raises(ValueError, match="elements"):
        w.ecf_images(img, 16, out=torch.empty((2, 15), dtype=torch.int32))
    coords = np.zeros((3, 2), np.float32)
    cells = [(np.array([[0, 1]], np.int32), np.array([1], np.int32), 1)]
    with pytest.raises(ValueError, match="dtype"):
        w.wect_complex(coords, cells, dirs, 8, out=torch.empty((3, 8), dtype=torch.int32))
