"""Activation layout handling and the device counterparts of the reference's channel
primitives (``channel_sum``, ``channel_affine``; /root/reference/pkg/src/bigbatch/tensor.py).

The reference's ``Tensor`` (tensor.py:39-87) is an immutable f64/f32 numpy array that
rejects NaN/Inf on construction. Here activations are torch CUDA fp32 / bf16 / fp16
tensors, NCHW contiguous (or channels_last = NHWC, or 2-D (N, C)); the finiteness contract is kept by
the statistics kernels, which report non-finite statistics through a device status
word instead of an O(E) host scan (see batchnorm.py).
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass

import torch

from . import _lib


class TensorError(ValueError):
    """Invalid shape, layout, or argument for a tensor operation (tensor.py:19-20)."""


class NonFiniteError(FloatingPointError):
    """A public operation produced or received NaN/Inf values (tensor.py:23-24)."""


@dataclass
class Geometry:
    x: torch.Tensor  # the (possibly made-contiguous) tensor the kernels read
    N: int
    C: int
    HW: int
    layout: int  # the C ABI's format word: memory layout | activation dtype (include/cgbn.h)
    mem: int = 0  # memory layout alone (LAYOUT_NCHW / LAYOUT_NHWC)

    @property
    def count(self) -> int:
        return self.N * self.HW


def geometry(x, what: str = "x", err=TensorError) -> Geometry:
    """Validate an activation and describe it for the C ABI.

    Layouts (tensor.py:121-128 supports (N, C) and (N, C, H, W)): 2-D (N, C) is NCHW
    with HW = 1; 4-D NCHW-contiguous -> CGBN_LAYOUT_NCHW; 4-D channels_last ->
    CGBN_LAYOUT_NHWC; any other strides are made NCHW-contiguous.
    """
    if not isinstance(x, torch.Tensor):
        raise err(f"{what} must be a torch.Tensor, got {type(x).__name__}")
    if x.dim() not in (2, 4):
        raise err(f"expected layout (N,C) or (N,C,H,W), got shape {tuple(x.shape)}")
    if any(e <= 0 for e in x.shape):
        raise err(f"tensor extents must be positive, got shape {tuple(x.shape)}")
    if not x.is_cuda:
        raise err(f"{what} must be a CUDA tensor (the CGBN path has no CPU fallback)")
    act = _ACT.get(x.dtype)
    if act is None:
        raise err(f"{what} must be float32, bfloat16 or float16, got {x.dtype}")

    def geo(t, n, c, hw, mem):
        # the kernels move 16-byte units: a view whose storage offset breaks the 16-byte
        # alignment (e.g. x[1:] of an (N, 3) tensor) is copied to fresh, aligned storage
        if t.data_ptr() % 16:
            t = t.clone(memory_format=torch.channels_last if mem == _lib.LAYOUT_NHWC
                        else torch.contiguous_format)
        return Geometry(t, n, c, hw, mem | act, mem)

    if x.dim() == 2:
        x = x.contiguous()
        return geo(x, int(x.shape[0]), int(x.shape[1]), 1, _lib.LAYOUT_NCHW)
    n, c, h, w = (int(e) for e in x.shape)
    if x.is_contiguous():
        return geo(x, n, c, h * w, _lib.LAYOUT_NCHW)
    if x.is_contiguous(memory_format=torch.channels_last):
        return geo(x, n, c, h * w, _lib.LAYOUT_NHWC)
    x = x.contiguous()
    return geo(x, n, c, h * w, _lib.LAYOUT_NCHW)


# Activation dtypes: storage only -- statistics are fp64 and gamma,
# beta and the running statistics stay fp32 for every activation dtype.
_ACT = {torch.float32: _lib.ACT_F32, torch.bfloat16: _lib.ACT_BF16, torch.float16: _lib.ACT_F16}


def same_layout_like(g: Geometry) -> torch.Tensor:
    """Uninitialised output with the input's shape and memory layout."""
    if g.mem == _lib.LAYOUT_NHWC:
        return torch.empty_like(g.x, memory_format=torch.channels_last)
    return torch.empty_like(g.x, memory_format=torch.contiguous_format)


def stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# Workspaces (zero-initialised; the kernels return their tickets to zero) and device
# status words, one per (device, stream).
_CACHE_MAX = 64  # streams remembered per cache (DeviceGroup.run makes fresh streams)
_cache_lock = threading.Lock()
_ws_cache: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()
_status_cache: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()


def _cached(cache, key, make, ok=lambda b: True):
    """LRU lookup. Evicting a buffer is stream-safe: its block returns to the caching
    allocator's pool of the stream it was allocated on, after the work queued there."""
    with _cache_lock:
        buf = cache.get(key)
        if buf is not None and ok(buf):
            cache.move_to_end(key)
            return buf
    new = make(buf)
    with _cache_lock:
        cache[key] = new
        cache.move_to_end(key)
        while len(cache) > _CACHE_MAX:
            cache.popitem(last=False)
    return new


def workspace(device, nbytes: int) -> torch.Tensor:
    """Zero-initialised workspace of at least ``nbytes`` for the current stream (the
    kernels return their tickets to zero, so it is reused as is)."""
    st = torch.cuda.current_stream(device)

    def make(old):
        size = max(nbytes, 1 << 16)
        if old is not None:
            size = max(size, 2 * old.numel())
        return torch.zeros(size, dtype=torch.uint8, device=device)

    return _cached(_ws_cache, (st.device_index, st.cuda_stream), make,
                   lambda b: b.numel() >= nbytes)


def status_word(device) -> torch.Tensor:
    st = torch.cuda.current_stream(device)
    return _cached(_status_cache, (st.device_index, st.cuda_stream),
                   lambda old: torch.zeros(1, dtype=torch.int32, device=device))


@dataclass
class ChannelStats:
    """Per-channel reduction result (tensor.py:101-118); sums are fp64 device tensors."""

    count: int
    sum: torch.Tensor
    sum_sq: torch.Tensor | None = None

    def __post_init__(self):
        if self.count <= 0:
            raise TensorError(f"ChannelStats.count must be positive, got {self.count}")
        if self.sum_sq is not None and self.sum_sq.shape != self.sum.shape:
            raise TensorError("ChannelStats.sum and sum_sq must have equal length")


def channel_sum(x: torch.Tensor, with_sum_sq: bool = False) -> ChannelStats:
    """Per-channel sums over all non-channel axes (tensor.py:143-153), on the device.

    The reference pins a strict left-to-right fold; the kernel uses a fixed tree (same
    input -> bitwise-identical sums, run to run) accumulated in fp64.
    """
    g = geometry(x)
    lib = _lib.load()
    s = torch.empty(g.C, dtype=torch.float64, device=g.x.device)
    ss = torch.empty(g.C, dtype=torch.float64, device=g.x.device) if with_sum_sq else None
    nb = lib.cgbn_workspace_bytes(g.N, g.C, g.HW, g.layout)
    ws = workspace(g.x.device, nb)
    _lib.check(lib.cgbn_channel_sum(g.x.data_ptr(), g.N, g.C, g.HW, g.layout, s.data_ptr(),
                                    ss.data_ptr() if ss is not None else None, ws.data_ptr(),
                                    ws.numel(), stream_ptr(g.x.device)), "cgbn_channel_sum")
    return ChannelStats(count=g.count, sum=s, sum_sq=ss)


def channel_affine(x: torch.Tensor, scale, shift) -> torch.Tensor:
    """Per-channel affine map out[n,c,...] = scale[c] * x[n,c,...] + shift[c]
    (tensor.py:156-170), fp64 coefficients, one rounding to fp32."""
    g = geometry(x)
    scale = torch.as_tensor(scale, dtype=torch.float64, device=g.x.device).contiguous()
    shift = torch.as_tensor(shift, dtype=torch.float64, device=g.x.device).contiguous()
    if tuple(scale.shape) != (g.C,) or tuple(shift.shape) != (g.C,):
        raise TensorError(f"scale/shift must have length C={g.C}, got {tuple(scale.shape)} "
                          f"and {tuple(shift.shape)}")
    out = same_layout_like(g)
    lib = _lib.load()
    _lib.check(lib.cgbn_channel_affine(g.x.data_ptr(), g.N, g.C, g.HW, g.layout,
                                       scale.data_ptr(), shift.data_ptr(), out.data_ptr(),
                                       stream_ptr(g.x.device)), "cgbn_channel_affine")
    return out
