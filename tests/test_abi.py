"""The C-ABI library loads and exports every symbol include/drr_b200.h
declares; argument validation maps onto the reference's exception classes.
No compute call is made (CPU container)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "drr_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(drr_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    from paper_2208_12737_b200 import _lib
    lib = _lib.load()
    declared = header_functions()
    assert declared, "header parse failed"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.drr_version() >= 2
    # the ctypes mirrors have the library's struct layouts (checked on load too)
    import ctypes
    got = [ctypes.c_size_t() for _ in range(4)]
    assert lib.drr_struct_sizes(*[ctypes.byref(g) for g in got]) == 0
    assert [g.value for g in got] == [ctypes.sizeof(t) for t in (
        _lib.DrrGrid, _lib.DrrDetector, _lib.DrrRegConfig, _lib.DrrPeerHandle)]


def test_library_is_sm100a():
    """The fatbin holds sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2208_12737_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_map_to_reference_errors():
    from paper_2208_12737_b200 import _lib
    from paper_2208_12737_b200.errors import InvalidArgumentError
    lib = _lib.load()
    bad = _lib.make_grid((0, 4, 4), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    det = _lib.make_detector(8, 8, 1.0, 1.0)
    rc = lib.drr_forward(None, 0, bad, None, 1, det, None, 0, None)
    assert rc == _lib.DRR_ERR_INVALID_ARGUMENT
    with pytest.raises(InvalidArgumentError, match="dims"):
        _lib.check(rc)
    good = _lib.make_grid((4, 4, 4), (1.0, -1.0, 1.0), (0.0, 0.0, 0.0))
    with pytest.raises(InvalidArgumentError, match="spacing"):
        _lib.check(lib.drr_raysum(None, 0, good, None, None, 1, None, None))
    grid = _lib.make_grid((4, 4, 4), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    zero_det = _lib.make_detector(0, 8, 1.0, 1.0)
    with pytest.raises(InvalidArgumentError, match="detector"):
        _lib.check(lib.drr_forward(None, 0, grid, None, 1, zero_det, None, 0, None))
    pitch_det = _lib.make_detector(8, 8, 0.0, 1.0)
    with pytest.raises(InvalidArgumentError, match="pitch"):
        _lib.check(lib.drr_count_steps(None, 0, grid, None, 1, pitch_det, None, None))
    with pytest.raises(InvalidArgumentError, match="vol_dtype"):
        _lib.check(lib.drr_raysum(None, 7, grid, None, None, 1, None, None))
    # empty work is a no-op success
    assert lib.drr_raysum(None, 0, grid, None, None, 0, None, None) == _lib.DRR_OK
    assert lib.drr_forward(None, 0, grid, None, 0, det, None, 0, None) == _lib.DRR_OK


def test_workspace_size_and_error():
    from paper_2208_12737_b200 import _lib
    from paper_2208_12737_b200.errors import InvalidArgumentError
    lib = _lib.load()
    det = _lib.make_detector(200, 200, 3.6, 3.6, ray_split=1)
    # one thread per ray: 13 x 25 CTA tiles of 16 x 8 pixels, 12 doubles each, per pose
    assert lib.drr_backward_workspace_size(3, det) == 3 * 13 * 25 * 12 * 8
    # auto split: one pose's 200^2 rays < 0.6 waves of resident threads (148 x 6 x 128;
    # no device here: 148 SMs assumed) -> 2 threads per ray, 8 x 8 pixel tiles; three
    # poses fill it -> one thread per ray
    auto = _lib.make_detector(200, 200, 3.6, 3.6)
    assert lib.drr_backward_workspace_size(1, auto) == 1 * 25 * 25 * 12 * 8
    assert lib.drr_backward_workspace_size(3, auto) == 3 * 13 * 25 * 12 * 8
    # a large batch needs no split
    assert lib.drr_backward_workspace_size(64, auto) == 64 * 13 * 25 * 12 * 8
    bad = _lib.make_detector(200, 200, 3.6, 3.6, ray_split=3)
    assert lib.drr_backward_workspace_size(3, bad) == 0
    grid = _lib.make_grid((4, 4, 4), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    with pytest.raises(Exception, match="ray_split"):
        _lib.check(lib.drr_forward(None, 0, grid, None, 1, bad, None, 0, None))
    rc = lib.drr_backward(None, 0, grid, None, 3, det, None, 0, None, None, 0, None, 16, None)
    assert rc == _lib.DRR_ERR_WORKSPACE
    with pytest.raises(Exception, match="workspace"):
        _lib.check(rc)
    # the Jacobian contraction validates its workspace the same way
    rc = lib.drr_backward_jac(None, 3, det, None, 0, None, None, 16, None)
    assert rc == _lib.DRR_ERR_WORKSPACE
    assert lib.drr_backward_jac(None, 0, det, None, 0, None, None, 0, None) == _lib.DRR_OK
    with pytest.raises(InvalidArgumentError, match="NULL"):
        _lib.check(lib.drr_forward_jac(None, 0, grid, None, 1, det, None, 0, None, None))
    assert lib.drr_forward_jac(None, 0, grid, None, 0, det, None, 0, None, None) == _lib.DRR_OK


def test_volume_size_limit():
    from paper_2208_12737_b200 import _lib
    from paper_2208_12737_b200.errors import InvalidArgumentError
    lib = _lib.load()
    grid = _lib.make_grid((2048, 2048, 1024), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    with pytest.raises(InvalidArgumentError, match="voxels"):
        _lib.check(lib.drr_raysum(None, 0, grid, None, None, 1, None, None))
