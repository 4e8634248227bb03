"""Index persistence in the reference's file format (grid.py:204-277).

Layout (byte-identical to the reference for the same index): the magic
``GHNIDX\\x01\\n``, a little-endian uint32 header length, the JSON header
(``sort_keys=True``: version, metric, per-array dtype and shape) and the raw
C-order bytes of widths, origin, splits, coords (f8), labels, cell_ids,
offsets, order.  ``save_index`` exports the device CSR (perm, cell table) to
those host arrays; ``load_index`` rebuilds the device index from the file's
points and grid (the fit is deterministic, and the rebuilt cell table is
checked against the file's).
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .grid import GridIndex, GridParams, build_arrays

MAGIC = b"GHNIDX\x01\n"
FIELDS = ("widths", "origin", "splits", "coords", "labels", "cell_ids", "offsets", "order")


def _arrays(index: GridIndex) -> dict:
    labels = np.asarray(index.labels)
    if labels.dtype == object:
        raise ValueError("labels must be numeric or strings to serialize")
    starts = index.bucket_starts
    return {
        "widths": np.asarray(index.params.widths, dtype=np.float64),
        "origin": np.asarray(index.params.origin, dtype=np.float64),
        "splits": np.asarray(index.params.splits, dtype=np.int64),
        "coords": np.ascontiguousarray(index.coords, dtype=np.float64),
        "labels": np.ascontiguousarray(labels),
        "cell_ids": np.ascontiguousarray(index.cell_array, dtype=np.int64),
        "offsets": np.ascontiguousarray(starts - starts[0], dtype=np.int64),
        "order": np.ascontiguousarray(index.order, dtype=np.int64),
    }


def save_index(index: GridIndex, path) -> None:
    """Write the index (grid.py:211-246)."""
    arrays = _arrays(index)
    header = {
        "version": 1,
        "metric": index.metric,
        "arrays": {k: {"dtype": arrays[k].dtype.str, "shape": list(arrays[k].shape)} for k in FIELDS},
    }
    blob = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<I", len(blob)))
        fh.write(blob)
        for k in FIELDS:
            fh.write(np.ascontiguousarray(arrays[k]).tobytes())


def read_index_arrays(path) -> tuple[dict, dict]:
    """(header, arrays) of an index file; ValueError on a bad magic / version."""
    with open(path, "rb") as fh:
        if fh.read(len(MAGIC)) != MAGIC:
            raise ValueError(f"{path}: not a grid index file")
        (n,) = struct.unpack("<I", fh.read(4))
        header = json.loads(fh.read(n))
        if header.get("version") != 1:
            raise ValueError(f"{path}: unsupported index version")
        arrays = {}
        for k in FIELDS:
            meta = header["arrays"][k]
            dt = np.dtype(meta["dtype"])
            shape = tuple(meta["shape"])
            count = int(np.prod(shape)) if shape else 1
            arrays[k] = np.frombuffer(fh.read(dt.itemsize * count), dtype=dt).reshape(shape).copy()
    return header, arrays


def load_index(path) -> GridIndex:
    """Read an index written by save_index or by the reference (grid.py:249-277)."""
    header, arr = read_index_arrays(path)
    params = GridParams(arr["widths"], arr["origin"], arr["splits"])
    labels = arr["labels"]
    index = build_arrays(arr["coords"], labels.tolist() if labels.dtype.kind in "US" else labels,
                         params=params, metric=header["metric"])
    if not (np.array_equal(index.order, arr["order"]) and np.array_equal(index.cell_array, arr["cell_ids"])):
        raise ValueError(f"{path}: cell table does not match the rebuilt index")
    return index
