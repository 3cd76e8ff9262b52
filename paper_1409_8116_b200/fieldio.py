"""Field files: a JSON header plus a raw little-endian payload (fieldio.py:1-116).

The format is the reference's, byte for byte: ``<name>.json`` (format version,
dims, extents, grid specs, precision, byte order, payload name; ``indent=2``,
sorted keys, trailing newline) and ``<name>.bin`` (the raw scalars in C order,
little-endian, no framing).  Errors raise ``FieldFormatError`` (a
``ValueError``) with the reference's messages.

B200 addition: ``read_field(..., device="cuda")`` streams the
payload from disk straight into HBM through two pinned staging buffers (the
disk read of chunk i+1 overlaps the host-to-device copy of chunk i), and
``write_field`` accepts a CUDA tensor and streams it back the same way, so a
multi-GB field never exists as a pageable host copy.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .grid import BoundaryCondition, GridKind, GridSpec

FORMAT_VERSION = 1

_PRECISION_TO_DTYPE = {"double": "<f8", "single": "<f4"}
_DTYPE_TO_PRECISION = {np.dtype(np.float64): "double", np.dtype(np.float32): "single"}
_CHUNK_BYTES = 64 << 20


class FieldFormatError(ValueError):
    """Raised when a field file is malformed or has an unsupported version."""


def grid_to_dict(spec: GridSpec) -> dict:
    return {"n": spec.n, "length": spec.length, "bc": spec.bc.value, "kind": spec.kind.value}


def grid_from_dict(d: dict) -> GridSpec:
    try:
        return GridSpec(int(d["n"]), float(d["length"]), BoundaryCondition(d["bc"]), GridKind(d["kind"]))
    except (KeyError, ValueError) as exc:
        raise FieldFormatError(f"bad grid entry {d!r}: {exc}") from exc


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _header(base: Path, shape, precision, grids) -> dict:
    return {
        "format_version": FORMAT_VERSION,
        "dims": len(shape),
        "extents": [int(e) for e in shape],
        "grids": None if grids is None else [grid_to_dict(g) for g in grids],
        "precision": precision,
        "byte_order": "little",
        "order": "C",
        "payload": base.with_suffix(".bin").name,
    }


def write_field(basepath, array, grids=None) -> Path:
    """Write ``<basepath>.json`` + ``<basepath>.bin``; returns the header path
    (fieldio.py:49-75).  ``array``: numpy array, or a torch tensor (a CUDA
    tensor is streamed device -> pinned host -> file in chunks)."""
    base = Path(basepath)
    if _is_tensor(array):
        import torch

        precision = {torch.float64: "double", torch.float32: "single"}.get(array.dtype)
        if precision is None:
            raise FieldFormatError(f"unsupported dtype {array.dtype}; use float32/float64")
        shape = tuple(array.shape)
    else:
        array = np.asarray(array)
        precision = _DTYPE_TO_PRECISION.get(array.dtype)
        if precision is None:
            raise FieldFormatError(f"unsupported dtype {array.dtype}; use float32/float64")
        shape = array.shape
    header = _header(base, shape, precision, grids)
    base.parent.mkdir(parents=True, exist_ok=True)
    with open(base.with_suffix(".json"), "w") as fh:
        json.dump(header, fh, indent=2, sort_keys=True)
        fh.write("\n")
    with open(base.with_suffix(".bin"), "wb") as fh:
        if _is_tensor(array) and array.is_cuda:
            _stream_device_to_file(array, fh)
        else:
            host = array.cpu().numpy() if _is_tensor(array) else array
            fh.write(np.ascontiguousarray(host, dtype=_PRECISION_TO_DTYPE[precision]).tobytes())
    return base.with_suffix(".json")


def _validate_header(header_path: Path):
    try:
        with open(header_path) as fh:
            header = json.load(fh)
    except json.JSONDecodeError as exc:
        raise FieldFormatError(f"{header_path}: invalid JSON header: {exc}") from exc
    for key in ("format_version", "dims", "extents", "precision", "byte_order", "payload"):
        if key not in header:
            raise FieldFormatError(f"{header_path}: missing header key {key!r}")
    if header["format_version"] != FORMAT_VERSION:
        raise FieldFormatError(f"{header_path}: unsupported format version {header['format_version']}")
    if header["byte_order"] != "little":
        raise FieldFormatError(f"{header_path}: unsupported byte order {header['byte_order']!r}")
    if header.get("order", "C") != "C":
        raise FieldFormatError(f"{header_path}: unsupported storage order {header['order']!r}")
    dtype = _PRECISION_TO_DTYPE.get(header["precision"])
    if dtype is None:
        raise FieldFormatError(f"{header_path}: unsupported precision {header['precision']!r}")
    extents = tuple(int(e) for e in header["extents"])
    if len(extents) != header["dims"]:
        raise FieldFormatError(f"{header_path}: dims {header['dims']} != extents rank {len(extents)}")
    payload_path = header_path.parent / header["payload"]
    expected = int(np.prod(extents)) * np.dtype(dtype).itemsize
    size = payload_path.stat().st_size
    if size != expected:
        raise FieldFormatError(
            f"{payload_path}: payload is {size} bytes, expected {expected} for extents {extents}")
    grids = header.get("grids")
    if grids is not None:
        grids = tuple(grid_from_dict(g) for g in grids)
        if tuple(g.n for g in grids) != extents:
            raise FieldFormatError(
                f"{header_path}: grid point counts {tuple(g.n for g in grids)} != extents {extents}")
    return extents, np.dtype(dtype), payload_path, grids


def read_field(header_path, device=None):
    """Read a field file; returns ``(array, grids_or_None)`` (fieldio.py:78-116).

    ``device=None``: a numpy array, as the reference.  ``device="cuda"`` (or a
    torch.device): a CUDA tensor filled straight from the file (pinned, chunked,
    disk reads overlapped with the host-to-device copies)."""
    header_path = Path(header_path)
    extents, dtype, payload_path, grids = _validate_header(header_path)
    if device is None:
        raw = payload_path.read_bytes()
        array = np.frombuffer(raw, dtype=dtype).reshape(extents)
        return array.astype(array.dtype.newbyteorder("=")), grids
    return _stream_file_to_device(payload_path, extents, dtype, device), grids


# -- pinned, double-buffered streaming between files and HBM --------------------
def _staging(torch, nbytes):
    n = max(1, min(_CHUNK_BYTES, nbytes))
    return [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]


def _stream_file_to_device(payload_path: Path, extents, dtype, device):
    import torch

    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError(f"read_field: device must be a CUDA device, got {device}")
    tdt = torch.float64 if dtype == np.dtype("<f8") else torch.float32
    out = torch.empty(extents, dtype=tdt, device=device)
    total = out.numel() * out.element_size()
    if total == 0:
        return out
    dst = out.view(-1).view(torch.uint8)
    bufs = _staging(torch, total)
    stream = torch.cuda.Stream(device=device)
    done = [None, None]
    with open(payload_path, "rb", buffering=0) as fh:
        off, k = 0, 0
        while off < total:
            n = min(bufs[k].numel(), total - off)
            if done[k] is not None:
                done[k].synchronize()               # the copy out of this buffer has finished
            view = bufs[k].numpy()[:n]
            got = fh.readinto(memoryview(view))
            if got != n:
                raise FieldFormatError(f"{payload_path}: short read ({got} of {n} bytes)")
            with torch.cuda.stream(stream):
                dst[off:off + n].copy_(bufs[k][:n], non_blocking=True)
                done[k] = torch.cuda.Event()
                done[k].record(stream)
            off += n
            k ^= 1
    torch.cuda.current_stream(device).wait_stream(stream)
    out.record_stream(stream)
    stream.synchronize()
    return out


def _stream_device_to_file(tensor, fh):
    import torch

    src = tensor.contiguous().view(-1).view(torch.uint8)
    total = src.numel()
    if total == 0:
        return
    bufs = _staging(torch, total)
    stream = torch.cuda.Stream(device=tensor.device)
    stream.wait_stream(torch.cuda.current_stream(tensor.device))
    pending = []   # (event, buffer index, nbytes) in file order
    off, k = 0, 0
    while off < total or pending:
        if off < total and len(pending) < 2:
            n = min(bufs[k].numel(), total - off)
            with torch.cuda.stream(stream):
                bufs[k][:n].copy_(src[off:off + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            pending.append((ev, k, n))
            off += n
            k ^= 1
            continue
        ev, kb, n = pending.pop(0)
        ev.synchronize()                            # chunk landed in pinned memory
        fh.write(memoryview(bufs[kb].numpy()[:n]))  # ... while the next chunk copies
