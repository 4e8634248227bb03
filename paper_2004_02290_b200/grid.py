"""Grid fit and the device CSR cell table (drop-in for gridneighbors/grid.py).

Reference: pkg/src/gridneighbors/grid.py:23-201.  ``build`` keeps the
reference signature (grid.py:165-170) and the same ValueError cases; the
work runs in csrc/ghn_fit.cu through the C ABI (include/ghn.h):

  ghn_fit_bounds   floor(x/w) bounds, origin, finite check      grid.py:109,125
  ghn_fit_build    stable radix sort by cell -> CSR              grid.py:184-195

The resulting ``GridIndex`` lives on the GPU.  The reference's attributes
(``cell_array``, ``buckets``, ``table``, ``coords``) are materialised on the
host lazily, on first access, for drop-in compatibility and tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .core import LabeledPoint, check_metric

CellId = tuple[int, ...]


@dataclass(frozen=True)
class GridParams:
    """Per-dimension cell widths, training origin and split counts (grid.py:23-44)."""

    widths: np.ndarray
    origin: np.ndarray
    splits: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "widths", np.asarray(self.widths, dtype=float))
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=float))
        object.__setattr__(self, "splits", np.asarray(self.splits, dtype=np.int64))
        if np.any(self.widths <= 0):
            raise ValueError("all cell widths must be positive")

    @property
    def dim(self) -> int:
        return self.widths.shape[0]


def hash_cell(p, params: GridParams) -> CellId:
    """Cell id floor(p / w) of one point (grid.py:112-121).  Host utility:
    the batched hash runs on the device inside build / knn_query."""
    p = np.asarray(p, dtype=float)
    if p.shape != (params.dim,):
        raise ValueError(f"dimension mismatch: point {p.shape}, grid {params.dim}")
    return tuple(int(v) for v in np.floor(p / params.widths))


class _Labels:
    """Label storage: int32 codes for the vote, fp64 targets for the mean."""

    def __init__(self, values, device):
        import torch

        self.values = values                  # python list (original objects) or None
        self.decode = None                    # code -> label (None = identity)
        self.codes = None                     # device int32 (n,)
        self._targets = None                  # device float64 (n,), built on first use
        self._targets_from_codes = False
        arr = None
        if isinstance(values, torch.Tensor):
            t = values.to(device)
            if t.dtype.is_floating_point:
                self._targets = t.to(torch.float64).contiguous()
            else:
                wide = t.dtype not in (torch.int32, torch.int16, torch.int8, torch.uint8, torch.bool)
                if wide and t.numel():
                    # only a wider dtype needs the range check before the int32 cast; the
                    # code range itself (n_codes: which vote kernel a predict may use) is
                    # found on first use, not by the fit -- the reference's build never
                    # looks at the labels either (grid.py:165-195)
                    lo, hi = (int(v) for v in torch.aminmax(t))
                    if lo < -2**31 or hi >= 2**31:
                        raise ValueError("integer labels must fit in int32")
                    self._n_codes = hi + 1 if lo >= 0 else 0
                self.codes = t if t.dtype == torch.int32 and t.is_contiguous() else t.to(torch.int32).contiguous()
                self._targets_from_codes = True
            return
        try:
            arr = np.asarray(values)
        except Exception:
            arr = None
        if arr is not None and arr.ndim == 1 and arr.dtype.kind in "biu":
            a64 = arr.astype(np.int64)
            if a64.size and (a64.min() < -2**31 or a64.max() >= 2**31):
                uniq, inv = np.unique(a64, return_inverse=True)
                self.codes = torch.as_tensor(inv.astype(np.int32), device=device)
                self.decode = uniq.tolist()
            else:
                self.codes = torch.as_tensor(a64.astype(np.int32), device=device)
            self._targets = torch.as_tensor(a64.astype(np.float64), device=device)
        elif arr is not None and arr.ndim == 1 and arr.dtype.kind == "f":
            f64 = arr.astype(np.float64)
            self._targets = torch.as_tensor(f64, device=device)
            uniq, inv = np.unique(f64, return_inverse=True)
            self.codes = torch.as_tensor(inv.astype(np.int32), device=device)
            self.decode = uniq.tolist()
        else:
            # arbitrary hashable labels: codes in first-appearance order
            table: dict = {}
            codes = np.empty(len(values), np.int32)
            for i, v in enumerate(values):
                codes[i] = table.setdefault(v, len(table))
            self.codes = torch.as_tensor(codes, device=device)
            self.decode = list(table.keys())
            try:
                self._targets = torch.as_tensor(np.array([float(v) for v in values]), device=device)
            except (TypeError, ValueError):
                self._targets = None

    @property
    def targets(self):
        """fp64 regression targets float(label) (predict.py:43), built lazily."""
        if self._targets is None and self._targets_from_codes:
            import torch

            self._targets = self.codes.to(torch.float64)
        return self._targets

    @property
    def n_codes(self) -> int:
        """Codes lie in [0, n_codes) (0 = unknown / negative codes)."""
        if not hasattr(self, "_n_codes"):
            self._n_codes = 0
            if self.codes is not None and self.codes.numel():
                import torch

                lo, hi = (int(v) for v in torch.aminmax(self.codes))   # one pass, one read-back
                self._n_codes = hi + 1 if lo >= 0 and hi < 2**31 - 1 else 0
        return self._n_codes

    def label_of(self, code: int):
        return self.decode[code] if self.decode is not None else code


class GridIndex:
    """Immutable device cell table over a training set (grid.py:128-162).

    Device tensors: ``X`` (original order, (n, d)), ``perm`` (CSR slot ->
    point), ``coords_soa`` (permuted SoA), ``cell_start``, ``cell_ids``
    (relative to ``lo``), and for the DENSE layout ``pt_off`` / ``ne_off``.
    """

    def __init__(self, params, metric, X, labels, plan, t, n_cells):
        self.params = params
        self.metric = metric
        self.X = X
        self._labels = labels
        self.plan = plan
        self.perm = t["perm"]
        self.coords_soa = t["coords"]
        self.cell_start = t["cell_start"]
        self.cell_ids = t["cell_ids"]
        self.pt_off = t.get("pt_off")
        self.ne_off = t.get("ne_off")
        self.labels_perm = t.get("labels_perm")
        self.n_cells = int(n_cells)
        self._subgrids = None
        self.lo = np.array(plan.lo[: plan.d], dtype=np.int64)
        self.ext = np.array(plan.ext[: plan.d], dtype=np.int64)
        self._cache: dict = {}

    # -- reference attributes -------------------------------------------------
    @property
    def size(self) -> int:
        return int(self.X.shape[0])

    @property
    def dim(self) -> int:
        return int(self.X.shape[1])

    @property
    def layout(self) -> str:
        return "dense" if self.plan.layout == _lib.GHN_LAYOUT_DENSE else "list"

    @property
    def labels(self):
        v = self._labels.values
        if isinstance(v, np.ndarray):
            return v.tolist()
        if v is None or not isinstance(v, (list, tuple)):
            if "labels" not in self._cache:
                src = self._labels.codes if self._labels.codes is not None else self._labels.targets
                self._cache["labels"] = src.cpu().tolist()
            return self._cache["labels"]
        return v

    @property
    def coords(self) -> np.ndarray:
        """(n, d) fp64 coordinates in input order (grid.py:138)."""
        if "coords" not in self._cache:
            self._cache["coords"] = self.X.double().cpu().numpy()
        return self._cache["coords"]

    @property
    def order(self) -> np.ndarray:
        """Concatenated buckets: CSR slot -> original index (int64)."""
        if "order" not in self._cache:
            self._cache["order"] = self.perm.cpu().numpy().astype(np.int64)
        return self._cache["order"]

    @property
    def cell_array(self) -> np.ndarray:
        """(C_ne, d) int64 absolute cell ids, lexicographic (grid.py:193)."""
        if "cell_array" not in self._cache:
            rel = self.cell_ids[: self.n_cells * self.dim].view(self.n_cells, self.dim).cpu().numpy()
            self._cache["cell_array"] = rel.astype(np.int64) + self.lo
        return self._cache["cell_array"]

    @property
    def bucket_starts(self) -> np.ndarray:
        if "starts" not in self._cache:
            self._cache["starts"] = self.cell_start[: self.n_cells + 1].cpu().numpy().astype(np.int64)
        return self._cache["starts"]

    @property
    def buckets(self) -> list:
        """Per-cell int64 point-index arrays in input order (grid.py:194)."""
        if "buckets" not in self._cache:
            self._cache["buckets"] = np.split(self.order, self.bucket_starts[1:-1])
        return self._cache["buckets"]

    @property
    def table(self) -> dict:
        """dict cell id -> bucket (grid.py:151-154)."""
        if "table" not in self._cache:
            self._cache["table"] = {
                tuple(int(v) for v in row): b for row, b in zip(self.cell_array, self.buckets)}
        return self._cache["table"]

    # -- device view ----------------------------------------------------------
    def view(self, density: bool = True, targets: bool = True, label_range: bool = True) -> _lib.IndexView:
        """ctypes ghn_index_view of the device tables (density=False skips
        the tiled predict's density hint, which costs a kernel + sync once;
        targets=False leaves the fp64 regression targets unmaterialised;
        label_range=False leaves the label code range -- one reduction over
        the labels on first use -- to the first predict)."""
        # (built once per flag combination: the tables never move; the nested
        # grids, attached once after the fit, drop the cached views)
        vkey = (density, targets, label_range)
        cached = self._cache.get("views", {}).get(vkey)
        if cached is not None:
            return cached
        v = _lib.IndexView()
        p = self.plan
        v.n, v.d, v.dtype, v.layout, v.n_cells, v.E = p.n, p.d, p.dtype, p.layout, self.n_cells, p.E
        for j in range(p.d):
            v.widths[j] = p.widths[j]
            v.lo[j] = p.lo[j]
            v.ext[j] = p.ext[j]
        v.min_width = float(np.min(self.params.widths))
        v.coords = _lib.ptr(self.coords_soa)
        v.perm = _lib.ptr(self.perm)
        v.cell_start = _lib.ptr(self.cell_start)
        v.cell_ids = _lib.ptr(self.cell_ids)
        v.pt_off = _lib.ptr(self.pt_off)
        v.ne_off = _lib.ptr(self.ne_off)
        v.labels = _lib.ptr(self._labels.codes)
        v.targets = _lib.ptr(self._labels.targets) if targets else 0
        v.labels_perm = _lib.ptr(self.labels_perm)
        v.n_labels = self._labels.n_codes if label_range else 0
        v.metric = _lib.GHN_METRIC[self.metric]
        v.density_hint = self.density_hint(v) if density else 0.0
        sg = self._subgrids
        if sg is not None:
            v.n_sub, v.sub_min = sg["n_sub"], sg["min_points"]
            v.sub_of_cell, v.subs = _lib.ptr(sg["sub_of_cell"]), _lib.ptr(sg["subs"])
            v.sub_off, v.sub_coords, v.sub_idx = _lib.ptr(sg["sub_off"]), _lib.ptr(sg["coords"]), _lib.ptr(sg["idx"])
            v.n_subpts = sg["n_points"]
        self._cache.setdefault("views", {})[vkey] = v
        return v

    @property
    def n_subgrids(self) -> int:
        """Overfull cells carrying a nested grid (0 for most data)."""
        return 0 if self._subgrids is None else self._subgrids["n_sub"]

    def density_hint(self, v=None) -> float:
        """Points per cell the tiled predict sizes its tiles for (2-D DENSE):
        the 90th percentile, over points, of the mean occupancy of the 9x9
        cells around them (ghn_window_density; one small kernel + sync the
        first time).  Equal to the mean for uniform data, the cluster
        density for clustered data.  0 elsewhere."""
        if "density" not in self._cache:
            hint = 0.0
            if self.dim == 2 and self.plan.layout == _lib.GHN_LAYOUT_DENSE and self.n_cells > 0:
                import torch

                if v is None:
                    v = self.view()
                samples = int(min(4096, self.size))
                out = torch.empty(samples, dtype=torch.float32, device=self.X.device)
                _lib.check(_lib.lib().ghn_window_density(ctypes.byref(v), 4, samples, _lib.ptr(out),
                                                         _lib.stream_handle()), "ghn_window_density")
                hint = float(torch.quantile(out.double(), 0.9))
            self._cache["density"] = hint
        return self._cache["density"]


def _coords_matrix(data: Sequence[LabeledPoint]) -> np.ndarray:
    """(n, d) fp64 from points with the reference's checks (grid.py:85-91)."""
    if len(data) == 0:
        raise ValueError("empty dataset")
    dims = {p.dim for p in data}
    if len(dims) != 1:
        raise ValueError(f"points have mixed dimensions: {sorted(dims)}")
    return np.stack([p.coords for p in data])


def dense_limit_for(n: int) -> int:
    """Largest id bounding box kept as a dense table (8 bytes per cell)."""
    return int(min(1 << 30, max(1 << 20, 16 * n)))


def build(
    data: Sequence[LabeledPoint],
    metric: str = "euclidean",
    params: GridParams | None = None,
    max_splits: int | None = None,
) -> GridIndex:
    """Build the grid index on the GPU (grid.py:165-195).

    Same signature, defaults and ValueError cases as the reference.  With
    params=None the widths come from fit_cell_measurements (grid.py:94-109).
    """
    check_metric(metric)
    data = list(data)
    X = _coords_matrix(data)
    labels = [p.label for p in data]
    if params is None:
        from .fitwidths import fit_cell_measurements_arrays

        params = fit_cell_measurements_arrays(X, max_splits)
    elif params.dim != X.shape[1]:
        raise ValueError("params dimension does not match the data")
    return build_arrays(X, labels, params=params, metric=metric)


def build_arrays(X, y=None, params: GridParams | None = None, cells_per_axis=None,
                 metric: str = "euclidean", max_splits: int | None = None,
                 stream=None) -> GridIndex:
    """Array / tensor entry point (new API).

    X: (n, d) numpy array or torch tensor (float32 or float64; float32 is
    kept in float32 on the device, every key is still fp64).  y: labels or
    targets (list / numpy / torch).  Grid: explicit ``params``, or
    ``cells_per_axis`` C (widths 1/C, BASELINE.json's configs), or the
    max-splits fit.
    """
    import torch

    check_metric(metric)
    L = _lib.require_device()
    if stream is not None:
        # every allocation, host read and launch on the caller's stream
        with torch.cuda.stream(stream):
            return build_arrays(X, y, params=params, cells_per_axis=cells_per_axis, metric=metric,
                                max_splits=max_splits)
    dev = torch.device("cuda", torch.cuda.current_device())
    Xt = torch.as_tensor(X)
    if Xt.dtype not in (torch.float32, torch.float64):
        Xt = Xt.to(torch.float64)
    if Xt.ndim != 2:
        raise ValueError("coords must be an (n, d) matrix")
    n, d = int(Xt.shape[0]), int(Xt.shape[1])
    if n == 0:
        raise ValueError("empty dataset")
    if y is not None and len(y) != n:
        raise ValueError("labels length must match the number of rows")
    C = None
    if params is None:
        if cells_per_axis is not None:
            # origin (the per-dimension minimum) comes from the bounds kernel below
            C = np.broadcast_to(np.asarray(cells_per_axis, dtype=np.float64), (d,))
            params = GridParams(1.0 / C, np.zeros(d), C.astype(np.int64))
        else:
            from .fitwidths import fit_cell_measurements_arrays

            params = fit_cell_measurements_arrays(Xt, max_splits)
    if params.dim != d:
        raise ValueError("params dimension does not match the data")
    Xd = Xt.to(dev).contiguous()
    dtype = _lib.GHN_F32 if Xd.dtype == torch.float32 else _lib.GHN_F64
    s = _lib.stream_handle()
    widths = np.ascontiguousarray(params.widths, dtype=np.float64)
    wptr = widths.ctypes.data_as(ctypes.c_void_p)
    # bounds (2d int64), origin (d fp64) and the non-finite flag in one buffer: one read-back
    kbuf = torch.zeros(3 * d + 1, dtype=torch.int64, device=dev)
    bounds, origin, flags = kbuf[:2 * d], kbuf[2 * d:3 * d].view(torch.float64), kbuf[3 * d:].view(torch.int32)
    _lib.check(L.ghn_fit_bounds(_lib.ptr(Xd), dtype, n, d, wptr, _lib.ptr(bounds), _lib.ptr(origin),
                                _lib.ptr(flags), s), "ghn_fit_bounds")
    kh = kbuf.cpu()
    if int(kh[3 * d:].view(torch.int32)[0]) & 1:
        raise ValueError("non-finite coordinate")
    bh = np.ascontiguousarray(kh[:2 * d].numpy())
    if C is not None:
        params = GridParams(params.widths, kh[2 * d:3 * d].view(torch.float64).numpy().copy(), params.splits)
    plan = _lib.FitPlan()
    _lib.check(L.ghn_fit_plan_init(ctypes.byref(plan), n, d, dtype, wptr,
                                   bh.ctypes.data_as(ctypes.c_void_p), dense_limit_for(n)),
               "ghn_fit_plan_init")
    i32 = torch.int32
    t = {
        "perm": torch.empty(n, dtype=i32, device=dev),
        "coords": torch.empty(d * n, dtype=Xd.dtype, device=dev),
        "cell_start": torch.empty(n + 1, dtype=i32, device=dev),
        "cell_ids": torch.empty(n * d, dtype=i32, device=dev),
        "n_cells": torch.zeros(1, dtype=i32, device=dev),
    }
    if plan.layout == _lib.GHN_LAYOUT_DENSE:
        t["pt_off"] = torch.empty(plan.E + 1, dtype=i32, device=dev)
        t["ne_off"] = torch.empty(plan.E + 1, dtype=i32, device=dev)
    labels = _Labels(y if y is not None else [0] * n, dev)
    if labels.codes is not None:
        t["labels_perm"] = torch.empty(n, dtype=i32, device=dev)   # gathered by the fit
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
    out = _lib.FitOut(
        perm=_lib.ptr(t["perm"]), coords=_lib.ptr(t["coords"]), cell_start=_lib.ptr(t["cell_start"]),
        cell_ids=_lib.ptr(t["cell_ids"]), n_cells=_lib.ptr(t["n_cells"]),
        pt_off=_lib.ptr(t.get("pt_off")), ne_off=_lib.ptr(t.get("ne_off")),
        labels_in=_lib.ptr(labels.codes), labels_perm=_lib.ptr(t.get("labels_perm")))
    _lib.check(L.ghn_fit_build(ctypes.byref(plan), _lib.ptr(Xd), ctypes.byref(out), _lib.ptr(ws),
                               plan.workspace_bytes, s), "ghn_fit_build")
    n_cells = int(t["n_cells"].item())
    del ws
    index = GridIndex(params, metric, Xd, labels, plan, t, n_cells)
    _build_subgrids(index)
    return index


# Cells holding more than SUBGRID_MIN_POINTS points get a nested grid of about
# SUBGRID_POINTS_PER_CELL points per sub-cell (csrc/ghn_subgrid.cu; cfg3's
# cell (0,0,0,0) holds 36M points).  Pure acceleration: results are unchanged.
SUBGRID_MIN_POINTS = 1024
SUBGRID_POINTS_PER_CELL = 8


def subgrid_resolution(bmin, bmax, count, points_per_cell=SUBGRID_POINTS_PER_CELL):
    """Sub-cells per dimension for a cell's bounding box: about
    count / points_per_cell cubes of a common side, one split along
    dimensions of zero extent (host logic)."""
    ext = np.asarray(bmax, dtype=np.float64) - np.asarray(bmin, dtype=np.float64)
    d = ext.shape[0]
    pos = ext > 0
    if not pos.any():
        return np.ones(d, dtype=np.int64)
    m = max(1, int(count) // points_per_cell)
    h = float(np.exp(np.log(ext[pos]).sum() / pos.sum() - np.log(m) / pos.sum()))
    for _ in range(200):
        s = np.where(pos, np.clip(np.ceil(ext / h), 1, 1 << 16), 1).astype(np.int64)
        if float(np.prod(s, dtype=np.float64)) <= 2 * m + 16:
            return s
        h *= 1.1
    return s


def _build_subgrids(index: GridIndex, min_points: int = SUBGRID_MIN_POINTS) -> None:
    import torch

    L = _lib.lib()
    n, d = index.size, index.dim
    if index.n_cells == 0 or n <= min_points:
        return
    dev = index.X.device
    s = _lib.stream_handle()
    v = index.view(density=False, targets=False, label_range=False)
    cap = n // (min_points + 1) + 1
    cells = torch.empty(cap, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(L.ghn_subgrid_select(ctypes.byref(v), min_points, _lib.ptr(cells), _lib.ptr(cnt), s),
               "ghn_subgrid_select")
    n_sub = int(cnt.item())
    if n_sub == 0:
        return
    cells = torch.sort(cells[:n_sub])[0].contiguous()
    bmin = torch.empty((n_sub, d), dtype=torch.float64, device=dev)
    bmax = torch.empty((n_sub, d), dtype=torch.float64, device=dev)
    _lib.check(L.ghn_subgrid_bounds(ctypes.byref(v), _lib.ptr(cells), n_sub, _lib.ptr(bmin), _lib.ptr(bmax), s),
               "ghn_subgrid_bounds")
    cells_h = cells.cpu().numpy()
    starts = index.cell_start[cells.long()].cpu().numpy()
    ends = index.cell_start[cells.long() + 1].cpu().numpy()
    bmin_h, bmax_h = bmin.cpu().numpy(), bmax.cpu().numpy()
    recs = (_lib.SubGrid * n_sub)()
    off = 0
    for g in range(n_sub):
        cnt_g = int(ends[g] - starts[g])
        ext = subgrid_resolution(bmin_h[g], bmax_h[g], cnt_g)
        r = recs[g]
        for j in range(d):
            span = float(bmax_h[g, j] - bmin_h[g, j])
            h = span / float(ext[j]) if span > 0 else 1.0
            r.origin[j] = float(bmin_h[g, j])
            r.h[j] = h
            r.inv_h[j] = 1.0 / h
            r.ext[j] = int(ext[j])
        r.off, r.cell, r.start, r.count = off, int(cells_h[g]), int(starts[g]), cnt_g
        off += int(np.prod(ext))
    e_tot = off
    n_points = int((ends - starts).sum())
    subs = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).to(dev)
    sub_off = torch.empty(e_tot + 1, dtype=torch.int32, device=dev)
    coords = torch.empty(d * n_points, dtype=index.coords_soa.dtype, device=dev)
    idx = torch.empty(n_points, dtype=torch.int32, device=dev)
    sub_of_cell = torch.empty(index.n_cells, dtype=torch.int32, device=dev)
    wsz = int(L.ghn_subgrid_workspace_size(e_tot))
    ws = torch.empty(wsz, dtype=torch.uint8, device=dev)
    _lib.check(L.ghn_subgrid_build(ctypes.byref(v), _lib.ptr(subs), n_sub, e_tot, _lib.ptr(sub_off),
                                   _lib.ptr(coords), _lib.ptr(idx), n_points, _lib.ptr(sub_of_cell),
                                   _lib.ptr(ws), wsz, s), "ghn_subgrid_build")
    index._cache.pop("views", None)
    index._subgrids = {"n_sub": n_sub, "min_points": min_points, "sub_of_cell": sub_of_cell, "subs": subs,
                       "sub_off": sub_off, "coords": coords, "idx": idx, "n_points": n_points,
                       "records": recs}


def _max_splits_1d(values, cap):
    """(splits, width) of one dimension (grid.py:52-82), on the device: the
    max-splits width fit of the column as an (n, 1) matrix."""
    from .fitwidths import fit_cell_measurements_arrays

    v = np.asarray(values, dtype=np.float64).reshape(-1, 1)
    params = fit_cell_measurements_arrays(v, cap)
    return int(params.splits[0]), float(params.widths[0])


def cell_points(index: GridIndex, cell) -> list[int]:
    """Point indices of one cell, empty for absent cells (grid.py:198-201)."""
    bucket = index.table.get(tuple(int(v) for v in cell))
    return [] if bucket is None else [int(i) for i in bucket]
