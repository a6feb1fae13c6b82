"""Volume ingest straight into the device layout.

Restates the reference's ``load_volume`` / ``import_raw``
(``pkg/src/drrtrace/volume.py:149-222``): the ``.dvol`` format is one JSON
header line (dims, spacing, origin, dtype "f64") followed by little-endian
float64 densities in x-fastest order -- which IS the device layout, so the
payload is uploaded as-is and narrowed to fp32 on the GPU by
``drr_volume_pack`` (no host-side transpose or cast).  ``import_raw`` reads
headerless f32 / i16 / u8 voxels, uploads them in their own element type and
lets the same kernel cast (no Hounsfield rescaling) and clamp negatives.  Errors mirror the reference (HeaderParseError with the byte
offset, CorruptFileError on size mismatches, InvalidArgumentError).
"""

from __future__ import annotations

import json

import numpy as np
import torch

from .errors import CorruptFileError, HeaderParseError, InvalidArgumentError
from .renderer import DeviceVolume

_RAW_DTYPES = {"f32": "<f4", "i16": "<i2", "u8": "u1"}


def load_dvol(path, device=None, dtype=torch.float32) -> DeviceVolume:
    """``volume.load_volume`` (volume.py:167-193) into device memory."""
    with open(path, "rb") as fh:
        line = fh.readline()
        payload = fh.read()
    if not line.endswith(b"\n"):
        raise HeaderParseError(f"{path}: header line is not newline-terminated", len(line))
    try:
        header = json.loads(line.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        offset = getattr(exc, "pos", getattr(exc, "start", 0))
        raise HeaderParseError(f"{path}: malformed JSON header", offset) from exc
    if not isinstance(header, dict):
        raise HeaderParseError(f"{path}: header is not a JSON object", 0)
    missing = {"dims", "spacing", "origin", "dtype"} - header.keys()
    if missing:
        raise HeaderParseError(f"{path}: header missing keys {sorted(missing)}", len(line))
    if header["dtype"] != "f64":
        raise HeaderParseError(f"{path}: unsupported dtype {header['dtype']!r}", len(line))
    dims = tuple(int(n) for n in header["dims"])
    if len(dims) != 3 or any(n < 1 for n in dims):
        raise InvalidArgumentError(f"dims must be three integers >= 1, got {dims}")
    expected = int(np.prod(dims)) * 8
    if len(payload) != expected:
        raise CorruptFileError(f"{path}: payload has {len(payload)} bytes, header declares {expected}")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    flat = torch.frombuffer(bytearray(payload), dtype=torch.float64).to(dev)
    return DeviceVolume.from_flat(flat, dims, header["spacing"], header["origin"], device=dev,
                                  dtype=dtype)


def save_dvol(vol: DeviceVolume, path) -> None:
    """``volume.save_volume`` (volume.py:149-164) from a device volume."""
    header = {"dims": list(vol.dims), "spacing": list(vol.spacing),
              "origin": list(vol.origin), "dtype": "f64"}
    with open(path, "wb") as fh:
        fh.write(json.dumps(header).encode("utf-8") + b"\n")
        fh.write(vol.flat.to(torch.float64).cpu().numpy().astype("<f8", copy=False).tobytes())


def import_raw(path, dims, spacing, plane_origin=(0.0, 0.0, 0.0), element_type: str = "f32",
               clamp_negative: bool = False, device=None, dtype=torch.float32) -> DeviceVolume:
    """``volume.import_raw`` (volume.py:196-222): headerless little-endian voxels,
    x-fastest, cast directly (no HU rescale), optional clamp at 0 -- on the device."""
    if element_type not in _RAW_DTYPES:
        raise InvalidArgumentError(
            f"element_type must be one of {sorted(_RAW_DTYPES)}, got {element_type!r}")
    if np.isscalar(dims):
        dims = (dims, dims, dims)
    dims = tuple(int(n) for n in dims)
    np_dtype = np.dtype(_RAW_DTYPES[element_type])
    with open(path, "rb") as fh:
        payload = fh.read()
    expected = int(np.prod(dims)) * np_dtype.itemsize
    if len(payload) != expected:
        raise CorruptFileError(f"{path}: payload has {len(payload)} bytes, expected {expected} "
                               f"for dims {dims} and element type {element_type}")
    host = np.frombuffer(payload, dtype=np_dtype)
    if not host.dtype.isnative:
        host = host.astype(host.dtype.newbyteorder("="))
    dev = torch.device(device) if device is not None else torch.device("cuda")
    raw = torch.from_numpy(host.copy()).to(dev)  # the file's own element type
    return DeviceVolume.from_flat(raw, dims, spacing, plane_origin, device=dev, dtype=dtype,
                                  clamp_negative=clamp_negative)
