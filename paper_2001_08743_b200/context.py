"""Device context and device-resident design spaces (C-ABI ktune_ctx / ktune_space)."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib as L
from .errors import ConfigError
from .spaces import DesignSpace


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(getattr(a, "is_cuda"))


_NP_TO_TORCH = None


def host_empty(shape, dtype) -> np.ndarray:
    """Output buffer for host-pointer calls: page-locked memory from torch's caching host
    allocator when torch is present (device->host copies at PCIe speed and no page faults;
    blocks return to the cache when the array dies and are reused by the next call), else a
    plain numpy array. Contents are uninitialised: every element is written by the call."""
    global _NP_TO_TORCH
    try:
        import torch
        if not torch.cuda.is_available():
            raise ImportError
    except ImportError:
        return np.empty(shape, dtype)
    if _NP_TO_TORCH is None:
        _NP_TO_TORCH = {np.dtype(np.uint8): torch.uint8, np.dtype(np.int8): torch.int8,
                        np.dtype(np.uint16): torch.int16, np.dtype(np.int16): torch.int16,
                        np.dtype(np.int32): torch.int32, np.dtype(np.uint32): torch.int32,
                        np.dtype(np.float32): torch.float32,
                        np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64}
    dt = np.dtype(dtype)
    t = torch.empty(shape, dtype=_NP_TO_TORCH[dt], pin_memory=True)
    return t.numpy().view(dt)


def ptr_of(a, dtype=None):
    """(pointer, is_device, keepalive) for a numpy array or a CUDA torch tensor."""
    if a is None:
        return None, False, None
    if _is_torch_cuda(a):
        if not a.is_contiguous():
            raise ConfigError("device tensors must be contiguous")
        return C.c_void_p(a.data_ptr()), True, a
    arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    return arr.ctypes.data_as(C.c_void_p), False, arr


class Context:
    """One per (host thread, GPU): stream, workspaces, optional NCCL communicator."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        h = C.c_void_p()
        if world > 1 or nccl_id is not None:  # one-rank communicator: tests of the sharded paths
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            L.check(L.lib().ktune_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            L.check(L.lib().ktune_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.rank = rank
        self.world = world

    @classmethod
    def with_host_transport(cls, device: int, rank: int, world: int, allreduce, allgather) -> "Context":
        """A context whose collectives run through caller-supplied HOST functions
        (ktune_ctx_create_hostcomm): allreduce(np_array) sums in place, allgather(send_u8,
        recv_u8) fills recv with every rank's send in rank order. The product's sharded
        code paths run unchanged; several processes can share one GPU (tests)."""
        import numpy as np
        ar_t = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)
        ag_t = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

        def _ar(buf, count, dtype, user):
            try:
                ct = C.c_double if dtype == 1 else C.c_int64
                allreduce(np.ctypeslib.as_array((ct * count).from_address(buf)))
                return 0
            except Exception:  # reported through the library's error path
                return 1

        def _ag(send, recv, nbytes, user):
            try:
                snd = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send))
                rcv = np.ctypeslib.as_array((C.c_uint8 * (nbytes * world)).from_address(recv))
                allgather(snd, rcv)
                return 0
            except Exception:
                return 1

        self = cls.__new__(cls)
        self._callbacks = (ar_t(_ar), ag_t(_ag))  # kept alive with the context
        h = C.c_void_p()
        L.check(L.lib().ktune_ctx_create_hostcomm(device, rank, world, C.cast(self._callbacks[0], C.c_void_p),
                                                  C.cast(self._callbacks[1], C.c_void_p), None, C.byref(h)))
        self.h, self.device, self.rank, self.world = h, device, rank, world
        return self

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        L.check(L.lib().ktune_nccl_get_unique_id(buf))
        return buf.raw

    def check(self, rc: int) -> None:
        L.check(rc, self.h)

    def set_stream(self, stream) -> None:
        """Bind to an external cudaStream_t (int handle or torch.cuda.Stream); None = own stream.
        Handle 0 (torch's default stream) maps to cudaStreamLegacy."""
        if stream is None:
            self.check(L.lib().ktune_ctx_set_stream(self.h, None))
            return
        handle = int(getattr(stream, "cuda_stream", stream))
        self.check(L.lib().ktune_ctx_set_stream(self.h, C.c_void_p(handle if handle else 0x1)))

    def synchronize(self) -> None:
        self.check(L.lib().ktune_ctx_synchronize(self.h))

    def set_option(self, opt: int, value: int) -> None:
        self.check(L.lib().ktune_ctx_set_option(self.h, opt, value))

    def stat(self, s: int) -> int:
        v = C.c_int64()
        self.check(L.lib().ktune_ctx_stat(self.h, s, C.byref(v)))
        return v.value

    def reset_stats(self) -> None:
        self.check(L.lib().ktune_ctx_reset_stats(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            L.lib().ktune_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def compile_rule(source: Optional[str], names) -> list:
    """validity.cpp:124-212 through the C++ compiler in the library (host-only)."""
    if not source:
        return []
    cap = 256
    ops = (L.RuleOp * cap)()
    n = C.c_int(cap)
    arr = (C.c_char_p * len(names))(*[s.encode() for s in names])
    err = C.create_string_buffer(512)
    rc = L.lib().ktune_rule_compile(source.encode(), len(names), arr, ops, C.byref(n), err, 512)
    if rc != 0:
        raise ConfigError(err.value.decode())
    return [(ops[i].code, ops[i].arg) for i in range(n.value)]


class Space:
    """A DesignSpace uploaded to the device (ktune_space)."""

    def __init__(self, space: DesignSpace, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.space = space
        self.D = space.num_knobs
        self.card = np.array(space.cards, np.int32)
        vals = np.array([v for k in space.knobs for v in k.values], np.int64)
        ops = compile_rule(space.validity_rule, space.names)
        self.ops = ops
        arr = (L.RuleOp * max(1, len(ops)))()
        for i, (c, a) in enumerate(ops):
            arr[i].code = c
            arr[i].arg = a
        h = C.c_void_p()
        self.ctx.check(L.lib().ktune_space_create(self.ctx.h, self.D, self.card.ctypes.data_as(C.c_void_p),
                                                  vals.ctypes.data_as(C.c_void_p), arr, len(ops),
                                                  C.byref(h)))
        self.h = h
        self.index_bytes = space.index_bytes
        self.idx_dtype = np.uint8 if self.index_bytes == 1 else np.uint16

    def id_of(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, np.int32).reshape(-1, self.D)
        out = np.zeros(len(idx), np.uint64)
        self.ctx.check(L.lib().ktune_space_id_of(self.h, idx.ctypes.data_as(C.c_void_p), len(idx),
                                                 out.ctypes.data_as(C.c_void_p)))
        return out

    def config_at(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, np.uint64).reshape(-1)
        out = np.zeros((len(ids), self.D), np.int32)
        self.ctx.check(L.lib().ktune_space_config_at(self.h, ids.ctypes.data_as(C.c_void_p), len(ids),
                                                     out.ctypes.data_as(C.c_void_p)))
        return out

    def validate(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, np.int32).reshape(-1, self.D)
        out = np.zeros(len(idx), np.uint8)
        self.ctx.check(L.lib().ktune_space_validate(self.h, idx.ctypes.data_as(C.c_void_p), len(idx),
                                                    out.ctypes.data_as(C.c_void_p)))
        return out.astype(bool)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().ktune_space_destroy(self.h)
        except Exception:
            pass
