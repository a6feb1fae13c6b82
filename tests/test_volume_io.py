"""Volume ingest (volume_io.py) vs the reference's .dvol / raw formats
(volume.py:149-222): round trips through the device layout pass
(drr_volume_pack, -m gpu) and the same error classes (CPU: they are raised
before anything reaches the device)."""

import json

import numpy as np
import pytest
import torch

from oracle import oracle as O


def _write_dvol(path, data, spacing=(1.0, 2.0, 0.5), origin=(-1.0, 0.0, 3.0)):
    header = {"dims": list(data.shape), "spacing": list(spacing), "origin": list(origin), "dtype": "f64"}
    with open(path, "wb") as fh:
        fh.write(json.dumps(header).encode() + b"\n")
        fh.write(np.asarray(data, dtype="<f8").ravel(order="F").tobytes())


@pytest.mark.gpu
def test_dvol_round_trip(tmp_path, cuda_device):
    from paper_2208_12737_b200.volume_io import load_dvol, save_dvol
    data = np.random.default_rng(0).random((4, 5, 6))
    p = tmp_path / "v.dvol"
    _write_dvol(p, data)
    vol = load_dvol(p, device=cuda_device, dtype=torch.float64)
    assert vol.dims == (4, 5, 6) and vol.spacing == (1.0, 2.0, 0.5) and vol.origin == (-1.0, 0.0, 3.0)
    np.testing.assert_array_equal(vol.flat.cpu().numpy(), data.ravel(order="F"))
    vol32 = load_dvol(p, device=cuda_device)
    np.testing.assert_array_equal(vol32.flat.cpu().numpy(), data.ravel(order="F").astype(np.float32))
    q = tmp_path / "w.dvol"
    save_dvol(vol, q)
    assert q.read_bytes() == p.read_bytes()


@pytest.mark.gpu
def test_dvol_matches_reference_writer(tmp_path, cuda_device):
    dt = O.reference_module()
    if dt is None:
        pytest.skip("reference not built here")
    from paper_2208_12737_b200.volume_io import load_dvol
    ref = dt.make_phantom("sphere", (6, 7, 8), (1.0, 0.5, 2.0))
    p = tmp_path / "r.dvol"
    dt.save_volume(ref, p)
    vol = load_dvol(p, device=cuda_device, dtype=torch.float64)
    np.testing.assert_array_equal(vol.flat.cpu().numpy(), ref.flat_data())
    assert vol.dims == ref.dims and vol.spacing == ref.spacing and vol.origin == ref.plane_origin


def test_dvol_errors(tmp_path):
    from paper_2208_12737_b200.errors import CorruptFileError, HeaderParseError
    from paper_2208_12737_b200.volume_io import load_dvol
    p = tmp_path / "bad.dvol"
    p.write_bytes(b'{"dims": [2,2,2], "spacing": [1,1,1], "origin": [0,0,0], "dtype": "f64"}\n' + b"\0" * 56)
    with pytest.raises(CorruptFileError):
        load_dvol(p, device="cpu")
    p.write_bytes(b'{"dims": [2,2,2], "spac')
    with pytest.raises(HeaderParseError):
        load_dvol(p, device="cpu")
    p.write_bytes(b'{"dims": [2,2,2\n' + b"\0" * 64)
    with pytest.raises(HeaderParseError) as e:
        load_dvol(p, device="cpu")
    assert e.value.offset >= 0
    p.write_bytes(b'{"dims": [2,2,2], "spacing": [1,1,1], "origin": [0,0,0], "dtype": "f32"}\n' + b"\0" * 64)
    with pytest.raises(HeaderParseError):
        load_dvol(p, device="cpu")


@pytest.mark.gpu
def test_import_raw(tmp_path, cuda_device):
    from paper_2208_12737_b200.volume_io import import_raw
    data = np.arange(-12, 12, dtype=np.int16).reshape((2, 3, 4), order="F")
    p = tmp_path / "v.raw"
    p.write_bytes(data.ravel(order="F").astype("<i2").tobytes())
    vol = import_raw(p, (2, 3, 4), 1.5, element_type="i16", device=cuda_device, dtype=torch.float64)
    np.testing.assert_array_equal(vol.flat.cpu().numpy(), data.ravel(order="F").astype(np.float64))
    vol = import_raw(p, (2, 3, 4), 1.5, element_type="i16", clamp_negative=True, device=cuda_device)
    assert float(vol.flat.min()) == 0.0 and float(vol.flat.max()) == 11.0


def test_import_raw_errors(tmp_path):
    from paper_2208_12737_b200.errors import CorruptFileError, InvalidArgumentError
    from paper_2208_12737_b200.volume_io import import_raw
    data = np.arange(-12, 12, dtype=np.int16).reshape((2, 3, 4), order="F")
    p = tmp_path / "v.raw"
    p.write_bytes(data.ravel(order="F").astype("<i2").tobytes())
    with pytest.raises(CorruptFileError):
        import_raw(p, (2, 3, 5), 1.0, element_type="i16", device="cpu")
    with pytest.raises(InvalidArgumentError):
        import_raw(p, (2, 3, 4), 1.0, element_type="f16", device="cpu")
