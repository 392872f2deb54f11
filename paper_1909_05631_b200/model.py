"""Boundary types of the drop-in, shaped like the reference's data model
(sdnnbench/model.py:51-219): CSR with int64 indices and float64 values,
canonical (ascending columns, no explicit zeros), immutable arrays.

The engine is duck-typed: it reads ``n_rows / n_cols / row_offsets /
col_indices / values`` from any matrix, ``weights / bias`` from any layer,
``neurons_per_layer / layers`` from any model and ``data`` from any batch,
so the reference's own objects work unchanged and are returned in kind.
These classes exist so the package runs where the reference does not.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from .errors import BoundsError, ShapeError


def _ro(a, dtype) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    a.flags.writeable = False
    return a


class SparseMatrix:
    """Immutable CSR matrix of float64 (model.py:51-125 layout)."""

    __slots__ = ("n_rows", "n_cols", "row_offsets", "col_indices", "values")

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values, check=True):
        object.__setattr__(self, "n_rows", int(n_rows))
        object.__setattr__(self, "n_cols", int(n_cols))
        object.__setattr__(self, "row_offsets", _ro(row_offsets, np.int64))
        object.__setattr__(self, "col_indices", _ro(col_indices, np.int64))
        object.__setattr__(self, "values", _ro(values, np.float64))
        if check:
            if self.row_offsets.shape != (self.n_rows + 1,):
                raise ValueError("row_offsets must have n_rows + 1 entries")
            nnz = int(self.row_offsets[-1])
            if self.col_indices.shape != (nnz,) or self.values.shape != (nnz,):
                raise ValueError("index/value arrays do not match row_offsets")
            if nnz and (self.col_indices.min() < 0 or self.col_indices.max() >= self.n_cols):
                raise ValueError("column index out of range")

    def __setattr__(self, name, value):
        raise AttributeError("SparseMatrix is immutable")

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def row_counts(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.shape, np.float64)
        d[np.repeat(np.arange(self.n_rows), self.row_counts()), self.col_indices] = self.values
        return d

    @classmethod
    def empty(cls, n_rows: int, n_cols: int) -> "SparseMatrix":
        return cls(n_rows, n_cols, np.zeros(n_rows + 1, np.int64), np.empty(0, np.int64),
                   np.empty(0, np.float64), check=False)

    @classmethod
    def from_dense(cls, dense) -> "SparseMatrix":
        d = np.asarray(dense, np.float64)
        mask = d != 0.0
        off = np.zeros(d.shape[0] + 1, np.int64)
        np.cumsum(mask.sum(axis=1), out=off[1:])
        return cls(d.shape[0], d.shape[1], off, np.nonzero(mask)[1], d[mask], check=False)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "row_offsets"):
            return NotImplemented
        return (self.shape == (other.n_rows, other.n_cols)
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and self.values.tobytes() == np.asarray(other.values, np.float64).tobytes())

    def __hash__(self):
        return hash((self.shape, self.nnz))

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


@dataclass(frozen=True, eq=False)
class LayerWeights:
    """One N x N weight matrix plus its scalar bias (model.py:128-139)."""

    weights: SparseMatrix
    bias: float

    def __post_init__(self):
        if self.weights.n_rows != self.weights.n_cols:
            raise ShapeError(f"layer weights must be square, got {self.weights.shape}")


@dataclass(frozen=True, eq=False)
class NetworkModel:
    """Ordered stack of square layers over a fixed neuron count (model.py:142-162)."""

    neurons_per_layer: int
    layers: tuple

    def __post_init__(self):
        object.__setattr__(self, "layers", tuple(self.layers))
        if len(self.layers) < 1:
            raise ShapeError("a model needs at least one layer")
        for i, lw in enumerate(self.layers):
            if lw.weights.shape != (self.neurons_per_layer, self.neurons_per_layer):
                raise ShapeError(f"layer {i + 1} is {lw.weights.shape}")

    @property
    def n_layers(self) -> int:
        return len(self.layers)


@dataclass(frozen=True, eq=False)
class FeatureBatch:
    """Sparse (images x neurons) activations (model.py:165-177)."""

    data: SparseMatrix

    @property
    def n_images(self) -> int:
        return self.data.n_rows

    @property
    def n_neurons(self) -> int:
        return self.data.n_cols


class CategorySet:
    """Sorted set of 1-based image rows (model.py:180-219)."""

    __slots__ = ("image_rows",)

    def __init__(self, image_rows: Iterable[int]):
        arr = np.unique(np.asarray(list(image_rows) if not isinstance(image_rows, np.ndarray)
                                   else image_rows, dtype=np.int64))
        if arr.size and arr[0] < 1:
            raise BoundsError(f"image index {arr[0]} is below 1")
        object.__setattr__(self, "image_rows", _ro(arr, np.int64))

    def __setattr__(self, name, value):
        raise AttributeError("CategorySet is immutable")

    def __len__(self) -> int:
        return int(self.image_rows.size)

    def __iter__(self) -> Iterator[int]:
        return iter(int(i) for i in self.image_rows)

    def __eq__(self, other) -> bool:
        if not hasattr(other, "image_rows"):
            return NotImplemented
        return np.array_equal(self.image_rows, other.image_rows)

    def __hash__(self):
        return hash(self.image_rows.tobytes())

    def __repr__(self):
        return f"CategorySet(n={len(self)})"
