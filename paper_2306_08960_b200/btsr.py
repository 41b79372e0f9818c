"""BTSR containers: the reference's tensor file format (tensor_io.hpp:14-37) read straight into
device memory, and written from host objects.

- `read_header(path)` / `load_dev(path, kind=None)` go through the C ABI
  (`bitmm_btsr_read_header` / `bitmm_btsr_load_dev`): the payload streams through pinned
  chunks into CUDA tensors, with the reference's IoError checks (tensor_io.cpp:139-215) and
  object checks (BitMatrix padding, CsrMatrix::validate, finite dense values).
- `store_tensor(path, obj)` writes the byte layout of the reference's store_tensor
  (tensor_io.cpp:120-137); `store_thm_planes` / `load_thm_planes_dev` handle the plane triple
  plus its JSON sidecar (tensor_io.cpp:200-230).
"""
from __future__ import annotations

import ctypes as C
import json
import struct
from typing import Optional, Union

import numpy as np

from . import _lib
from .api import BitMatrix, CsrMatrix, ThmPlanes, _raise

DENSE, BIT, CSR = 0, 1, 2
_KINDS = {"dense": DENSE, "bit": BIT, "csr": CSR}


def _header(kind: int, rows: int, cols: int) -> bytes:
    return b"BTSR" + struct.pack("<IBQQ", 1, kind, rows, cols)


def store_tensor(path: str, obj: Union[np.ndarray, BitMatrix, CsrMatrix]) -> None:
    """store_tensor (tensor_io.cpp:120-137): dense fp32 ndarray, BitMatrix or CsrMatrix."""
    with open(path, "wb") as f:
        if isinstance(obj, BitMatrix):
            f.write(_header(BIT, obj.rows(), obj.cols()))
            f.write(struct.pack("<Q", obj.words_per_row()))
            f.write(np.ascontiguousarray(obj.words, dtype="<u8").tobytes())
        elif isinstance(obj, CsrMatrix):
            obj.validate()
            f.write(_header(CSR, obj.rows, obj.cols))
            f.write(struct.pack("<Q", obj.nnz()))
            f.write(np.ascontiguousarray(obj.row_ptr, dtype="<u8").tobytes())
            f.write(np.ascontiguousarray(obj.col_idx, dtype="<u8").tobytes())
            f.write(np.ascontiguousarray(obj.vals, dtype="<f4").tobytes())
        else:
            a = np.ascontiguousarray(obj, dtype="<f4")
            if a.ndim != 2:
                raise ValueError("dense tensors are 2-D")
            f.write(_header(DENSE, a.shape[0], a.shape[1]))
            f.write(a.tobytes())


def read_header(path: str) -> dict:
    """Header of a BTSR file (kind, rows, cols, words_per_row, nnz); raises api.IoError."""
    h = _lib.BtsrHeader()
    _raise(_lib.load().bitmm_btsr_read_header(path.encode(), C.byref(h)))
    return {"kind": ("dense", "bit", "csr")[h.kind], "rows": h.rows, "cols": h.cols,
            "words_per_row": h.words_per_row, "nnz": h.nnz}


def load_dev(path: str, kind: Optional[str] = None, device=None, stream=None) -> dict:
    """Load a BTSR file into CUDA tensors. `kind` ('dense' | 'bit' | 'csr') makes a mismatch
    fail like load_dense / load_bit / load_csr. Returns a dict with the header fields and
    `data` (dense float32 [rows, cols] / bit int64 words [rows, wpr]) or `row_ptr`,
    `col_idx` (int64 views of the u64 indices) and `vals` (float32)."""
    import torch

    from .device import _ptr, _stream
    h = read_header(path)
    dev = torch.device("cuda") if device is None else torch.device(device)
    want = -1 if kind is None else _KINDS[kind]
    out = dict(h)
    payload = row_ptr = col_idx = vals = None
    if h["kind"] == "dense":
        payload = torch.empty((h["rows"], h["cols"]), dtype=torch.float32, device=dev)
    elif h["kind"] == "bit":
        payload = torch.empty((h["rows"], h["words_per_row"]), dtype=torch.int64, device=dev)
    else:
        row_ptr = torch.empty(h["rows"] + 1, dtype=torch.int64, device=dev)
        col_idx = torch.empty(h["nnz"], dtype=torch.int64, device=dev)
        vals = torch.empty(h["nnz"], dtype=torch.float32, device=dev)
    p = lambda t: None if t is None or t.numel() == 0 else _ptr(t)  # noqa: E731
    _raise(_lib.load().bitmm_btsr_load_dev(path.encode(), want, p(payload), p(row_ptr), p(col_idx),
                                           p(vals), _stream(stream)))
    if payload is not None:
        out["data"] = payload
    else:
        out.update(row_ptr=row_ptr, col_idx=col_idx, vals=vals)
    return out


def store_thm_planes(prefix: str, planes: ThmPlanes) -> None:
    """store_thm_planes (tensor_io.cpp:200-213): <prefix>.{t,h,m}.btsr + <prefix>.json."""
    planes.validate()
    for name in ("t", "h", "m"):
        store_tensor(f"{prefix}.{name}.btsr", getattr(planes, name))
    with open(prefix + ".json", "w") as f:
        # nlohmann::json objects keep keys sorted; dump(2) indents by two
        json.dump({"s": float(planes.scale),
                   "gamma": None if planes.gamma is None else float(planes.gamma)}, f, indent=2,
                  sort_keys=True)
        f.write("\n")


def store_apb_layer(prefix: str, bin_: BitMatrix, residual: CsrMatrix, alpha: float) -> None:
    """store_apb_layer (apb.cpp:212-221): <prefix>.bin.btsr, <prefix>.res.btsr and
    <prefix>.json holding {"alpha": alpha} (nlohmann dump(2): the float as a double)."""
    store_tensor(prefix + ".bin.btsr", bin_)
    store_tensor(prefix + ".res.btsr", residual)
    with open(prefix + ".json", "w") as f:
        json.dump({"alpha": float(np.float32(alpha))}, f, indent=2)
        f.write("\n")


def load_thm_planes_dev(prefix: str, device=None, stream=None) -> dict:
    """load_thm_planes (tensor_io.cpp:215-235) into device tensors: t, h, m word tensors plus
    scale / gamma from the sidecar."""
    from .api import IoError
    out = {name: load_dev(f"{prefix}.{name}.btsr", "bit", device, stream) for name in ("t", "h", "m")}
    try:
        with open(prefix + ".json") as f:
            j = json.load(f)
        scale = float(j["s"])
        gamma = None if j["gamma"] is None else float(j["gamma"])
    except OSError:
        raise IoError("cannot open for reading: " + prefix + ".json") from None
    except (ValueError, KeyError, TypeError) as e:
        raise IoError(f"bad sidecar: {e}: {prefix}.json") from None
    # ThmPlanes::validate, its InvalidEncoding rethrown as IoError (tensor_io.cpp:230-234)
    from .api import InvalidEncoding
    from .device import _ptr, _stream
    shapes = {(v["rows"], v["cols"], v["words_per_row"]) for v in out.values()}
    try:
        if len(shapes) != 1:
            raise InvalidEncoding("plane shapes differ")
        r, c, w = shapes.pop()
        p = lambda x: None if x.numel() == 0 else _ptr(x)  # noqa: E731
        _raise(_lib.load().bitmm_validate_planes_dev(p(out["t"]["data"]), p(out["h"]["data"]),
                                                      p(out["m"]["data"]), r, c, w, scale,
                                                      _stream(stream)))
    except InvalidEncoding as e:
        raise IoError(f"{e}: {prefix}") from None
    return {"t": out["t"]["data"], "h": out["h"]["data"], "m": out["m"]["data"],
            "rows": out["t"]["rows"], "cols": out["t"]["cols"],
            "words_per_row": out["t"]["words_per_row"], "scale": scale, "gamma": gamma}
