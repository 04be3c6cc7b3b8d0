"""Cost model (cost_model.hpp:16-93): GBT fit on host, scoring on the GPU (K1).

`CostModel.predict(features)` is the reference seam `CostModel::predict
(const MatrixXd&)` (cost_model.cpp:231-236); `predict_idx` scores knob-index
rows directly with the exact integer-threshold transform.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from .context import Context, Space, default_context, ptr_of
from .errors import ConfigError


@dataclass
class GbtParams:  # cost_model.hpp:20-25
    num_trees: int = 50
    max_depth: int = 4
    learning_rate: float = 0.3
    min_samples_leaf: int = 2


@dataclass
class GbtModel:  # cost_model.hpp:47-53, flat pre-order nodes per tree
    base_prediction: float
    learning_rate: float
    num_features: int
    offsets: np.ndarray   # int32 [T+1]
    feature: np.ndarray   # int32, -1 = leaf
    left: np.ndarray
    right: np.ndarray
    threshold: np.ndarray
    value: np.ndarray
    training_sse: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @property
    def num_trees(self) -> int:
        return len(self.offsets) - 1

    def nodes_c(self):
        n = len(self.feature)
        arr = (L.TreeNode * max(1, n))()
        for i in range(n):
            arr[i].feature = int(self.feature[i])
            arr[i].left = int(self.left[i])
            arr[i].right = int(self.right[i])
            arr[i].threshold = float(self.threshold[i])
            arr[i].value = float(self.value[i])
        return arr


def fit_gbt(features, fitness, params: GbtParams = GbtParams(), seed: int = 0) -> GbtModel:
    """fit_gbt (cost_model.cpp:126-177), native host implementation in libktune_cuda."""
    X = np.ascontiguousarray(features, np.float64)
    y = np.ascontiguousarray(fitness, np.float64).reshape(-1)
    if X.ndim != 2 or len(X) != len(y):
        raise ConfigError("cost model: inconsistent feature dimensions in training set")
    m = L.GbtModelC()
    L.check(L.lib().ktune_gbt_fit(X.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), len(y),
                                  X.shape[1] if len(y) else 0, params.num_trees, params.max_depth,
                                  params.learning_rate, params.min_samples_leaf, seed, C.byref(m)))
    try:
        T = m.num_trees
        offs = np.array([m.tree_offsets[i] for i in range(T + 1)], np.int32)
        n = int(offs[-1])
        feat = np.array([m.nodes[i].feature for i in range(n)], np.int32)
        left = np.array([m.nodes[i].left for i in range(n)], np.int32)
        right = np.array([m.nodes[i].right for i in range(n)], np.int32)
        thr = np.array([m.nodes[i].threshold for i in range(n)], np.float64)
        val = np.array([m.nodes[i].value for i in range(n)], np.float64)
        sse = np.array([m.training_sse[i] for i in range(T)], np.float64)
        return GbtModel(m.base_prediction, m.learning_rate, m.num_features, offs, feat, left, right,
                        thr, val, sse)
    finally:
        L.lib().ktune_gbt_model_free(C.byref(m))


class DeviceGbt:
    """A fitted ensemble uploaded to the GPU (ktune_gbt)."""

    def __init__(self, model: GbtModel, space: Optional[Space] = None, ctx: Optional[Context] = None):
        self.ctx = ctx or (space.ctx if space is not None else default_context())
        self.model = model
        self.space = space
        offs = np.ascontiguousarray(model.offsets, np.int32)
        nodes = model.nodes_c()
        h = C.c_void_p()
        self.ctx.check(L.lib().ktune_gbt_create(self.ctx.h, space.h if space else None, model.num_features,
                                                model.base_prediction, model.learning_rate,
                                                model.num_trees, offs.ctypes.data_as(C.c_void_p), nodes,
                                                C.byref(h)))
        self.h = h

    def predict_idx(self, idx, out=None):
        """Scores knob-index rows (B x D uint8/uint16; numpy or CUDA tensor)."""
        if self.space is None:
            raise ConfigError("cost model: uploaded without a design space")
        dt = self.space.idx_dtype
        p, dev, keep = ptr_of(idx, None if hasattr(idx, "is_cuda") else dt)
        B = (idx.numel() if dev else keep.size) // self.space.D
        if dev:
            if out is None:
                import torch
                out = torch.empty(B, dtype=torch.float64, device=idx.device)
            self.ctx.check(L.lib().ktune_gbt_predict_idx(self.ctx.h, self.h, p, self.space.index_bytes, B,
                                                         C.c_void_p(out.data_ptr()), L.F_DEVICE))
            return out
        res = np.zeros(B, np.float64) if out is None else out
        self.ctx.check(L.lib().ktune_gbt_predict_idx(self.ctx.h, self.h, p, self.space.index_bytes, B,
                                                     res.ctypes.data_as(C.c_void_p), 0))
        return res

    def predict_features(self, X):
        X = np.ascontiguousarray(X, np.float64)
        if X.size and X.shape[-1] != self.model.num_features:
            raise ConfigError(f"cost model: feature dimension {X.shape[-1]} does not match training "
                              f"dimension {self.model.num_features}")
        B = X.shape[0] if X.ndim == 2 else 0
        out = np.zeros(B, np.float64)
        if B:
            self.ctx.check(L.lib().ktune_gbt_predict_features(self.ctx.h, self.h, X.ctypes.data_as(C.c_void_p),
                                                              B, out.ctypes.data_as(C.c_void_p), 0))
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().ktune_gbt_destroy(self.h)
        except Exception:
            pass


def predict_batch(model: GbtModel, features, ctx: Optional[Context] = None) -> np.ndarray:
    """predict_batch (cost_model.cpp:189-199) on the GPU."""
    return DeviceGbt(model, None, ctx).predict_features(features)


class CostModel:
    """Mirror of ktune::CostModel (cost_model.hpp:72-93): host refit, GPU predict."""

    def __init__(self, params: GbtParams = GbtParams(), min_training_size: int = 16,
                 space: Optional[Space] = None, ctx: Optional[Context] = None):
        self.params = params
        self.min_training_size = min_training_size
        self.space = space
        self.ctx = ctx or (space.ctx if space is not None else default_context())
        self._model: Optional[GbtModel] = None
        self._dev: Optional[DeviceGbt] = None
        self._fitted = 0

    def fit(self, features, fitness, seed: int) -> None:
        self._model = fit_gbt(features, fitness, self.params, seed)
        self._fitted = len(np.asarray(fitness).reshape(-1))
        self._dev = DeviceGbt(self._model, self.space, self.ctx)

    def set_model(self, model: GbtModel, fitted_examples: int) -> None:
        self._model = model
        self._fitted = fitted_examples
        self._dev = DeviceGbt(model, self.space, self.ctx)

    def predict(self, features) -> np.ndarray:
        if self._dev is None:
            raise ConfigError("cost model: predict called before fit")
        return self._dev.predict_features(features)

    def predict_idx(self, idx):
        if self._dev is None:
            raise ConfigError("cost model: predict called before fit")
        return self._dev.predict_idx(idx)

    def is_trained(self) -> bool:
        return self._model is not None and self._fitted >= self.min_training_size

    @property
    def model(self) -> GbtModel:
        if self._model is None:
            raise ConfigError("cost model: no fitted model")
        return self._model

    @property
    def device(self) -> DeviceGbt:
        if self._dev is None:
            raise ConfigError("cost model: no fitted model")
        return self._dev
