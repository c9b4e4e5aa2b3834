"""Producer fusion: the convolution that feeds a BN emits the BN's
forward partial statistics from its own epilogue, so the BN forward skips its statistics
read of the activation (fwd 12 -> 8 B/elem for fp32).

In the reference model every BN follows a GEMM-shaped producer — conv3x3 as an im2col
GEMM plus bias, or a dense layer (/root/reference/pkg/src/bigbatch/model.py:229-242) —
and the BN's first step re-reads that output for channel_sum (batchnorm.py:118,
tensor.py:143-153). Here the producer is the pointwise (1x1) convolution, NCHW, on the
tcgen05 tensor cores (include/cgbn.h ``cgbn_conv1x1_stats``): bf16 input and weight,
fp32 accumulation, output z stored as float32 or bfloat16. Its epilogue reduces every
output channel of its tile to (mean, centred M2) of z *as stored*, and a fold kernel
merges the tiles into the rank's forward partial — the vector the statistics kernel would
have produced from z — which then goes through the unchanged exchange and normalise.

    conv1x1(x, weight, bias=None, out_dtype=torch.float32) -> z
    conv1x1_bn_forward_local(x, weight, state, bias=None, out_dtype=..., relu=False)
        -> (y, cache, z)                        bn_forward_local(z, state) with fusion
    sync_conv1x1_bn_forward(handle, x, weight, state, bias=None, out_dtype=...,
                            one_pass=False, relu=False) -> (y, cache, z)
                                                sync_bn_forward(handle, z, state) fused

``cache`` is an ordinary BNForwardCache over z: ``bn_backward_local`` /
``sync_bn_backward`` take it unchanged. With ``set_forward_exchange("reference")`` (the
reference-literal statistics) the fused partial does not apply and the conv is followed
by the ordinary BN forward.
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import torch

from . import _lib
from .batchnorm import BatchNormError, BNLayerState, _Span, _local_exchange, _train_forward
from . import batchnorm as _bn
from .collectives import SCOPE_BN_GROUP
from .tensor import stream_ptr

_OUT = {torch.float32: _lib.ACT_F32, torch.bfloat16: _lib.ACT_BF16}

# Per-stream scratch for the per-tile partials (not the BN workspace: that one holds
# tickets the BN kernels expect at zero).
_scratch_lock = threading.Lock()
_scratch: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()


def _tile_scratch(device, nbytes):
    st = torch.cuda.current_stream(device)
    key = (st.device_index, st.cuda_stream)
    with _scratch_lock:
        buf = _scratch.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
            _scratch[key] = buf
        _scratch.move_to_end(key)
        while len(_scratch) > 64:
            _scratch.popitem(last=False)
        return buf


def _check(x, weight, bias, out_dtype):
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise BatchNormError("x must be a CUDA tensor (there is no CPU fallback)")
    if x.dim() != 4:
        raise BatchNormError(f"conv1x1 expects x of shape (N, Cin, H, W), got {tuple(x.shape)}")
    if x.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise BatchNormError("conv1x1 takes bfloat16 x and weight (tcgen05 kind::f16)")
    n, cin, h, w = x.shape
    wt = weight.reshape(weight.shape[0], -1) if weight.dim() == 4 else weight
    if wt.dim() != 2 or wt.shape[1] != cin:
        raise BatchNormError(
            f"weight must be (Cout, {cin}) or (Cout, {cin}, 1, 1), got {tuple(weight.shape)}")
    if out_dtype not in _OUT:
        raise BatchNormError(f"out_dtype must be float32 or bfloat16, got {out_dtype}")
    if (h * w) % 8 != 0 or cin % 8 != 0:
        raise BatchNormError(
            f"conv1x1 needs H*W and Cin multiples of 8 (TMA row strides), got H*W={h * w}, "
            f"Cin={cin}")
    b = None
    if bias is not None:
        b = bias.to(device=x.device, dtype=torch.float32).contiguous()
        if b.shape != (wt.shape[0],):
            raise BatchNormError(f"bias must have length {wt.shape[0]}")
    return x.contiguous(), wt.to(x.device).contiguous(), b, (n, cin, h, w, wt.shape[0])


def conv1x1(x, weight, bias=None, out_dtype=torch.float32):
    """z = conv1x1(x, weight) + bias on the tensor cores (the unfused producer)."""
    x, wt, b, (n, cin, h, w, cout) = _check(x, weight, bias, out_dtype)
    lib = _lib.load()
    z = torch.empty((n, cout, h, w), dtype=out_dtype, device=x.device)
    with _Span("conv1x1", 0):
        _lib.check(lib.cgbn_conv1x1(x.data_ptr(), wt.data_ptr(),
                                    b.data_ptr() if b is not None else None, n, cin, cout,
                                    h * w, _OUT[out_dtype], z.data_ptr(),
                                    stream_ptr(x.device)), "cgbn_conv1x1")
    return z


def conv1x1_stats(x, weight, bias=None, out_dtype=torch.float32):
    """(z, partial): the convolution plus this rank's forward partial of z (2C+1 fp64,
    [mean | M2 | count], the cgbn_fwd_stats format)."""
    x, wt, b, (n, cin, h, w, cout) = _check(x, weight, bias, out_dtype)
    lib = _lib.load()
    dev = x.device
    z = torch.empty((n, cout, h, w), dtype=out_dtype, device=dev)
    partial = torch.empty(2 * cout + 1, dtype=torch.float64, device=dev)
    nb = lib.cgbn_conv1x1_ws_bytes(n, cout, h * w)
    ws = _tile_scratch(dev, nb)
    with _Span("conv1x1_stats", 0):
        _lib.check(lib.cgbn_conv1x1_stats(
            x.data_ptr(), wt.data_ptr(), b.data_ptr() if b is not None else None, n, cin, cout,
            h * w, _OUT[out_dtype], z.data_ptr(), partial.data_ptr(), ws.data_ptr(), ws.numel(),
            stream_ptr(dev)), "cgbn_conv1x1_stats")
    return z, partial


def conv1x1_bn_forward_local(x, weight, state: BNLayerState, bias=None,
                             out_dtype=torch.float32, relu: bool = False):
    """bn_forward_local(conv1x1(x, weight) + bias, state) with the statistics taken in the
    conv epilogue. Returns (y, cache, z); cache is the BN cache over z."""
    if _bn._exchange_mode != "merged":
        z = conv1x1(x, weight, bias, out_dtype)
        y, cache = _bn.bn_forward_local(z, state, relu=relu)
        return y, cache, z
    z, partial = conv1x1_stats(x, weight, bias, out_dtype)
    y, cache = _train_forward(z, state, _local_exchange, 1, None, one_pass=False, relu=relu,
                              what="conv1x1_bn_forward_local", partial=partial)
    return y, cache, z


def sync_conv1x1_bn_forward(handle, x, weight, state: BNLayerState, bias=None,
                            out_dtype=torch.float32, one_pass: bool = False,
                            relu: bool = False):
    """sync_bn_forward(handle, conv1x1(x, weight) + bias, state) with the statistics taken
    in the conv epilogue; the partial goes through the BN group's exchange unchanged.
    Returns (y, cache, z)."""
    if _bn._exchange_mode != "merged":
        z = conv1x1(x, weight, bias, out_dtype)
        y, cache = _bn.sync_bn_forward(handle, z, state, one_pass=one_pass, relu=relu)
        return y, cache, z
    z, partial = conv1x1_stats(x, weight, bias, out_dtype)
    scope_key = f"bn{handle.bn_group_index}"
    y, cache = _train_forward(
        z, state, lambda v, info: handle.exchange(SCOPE_BN_GROUP, "bn_forward", v, info),
        handle.bn_group_size, scope_key, one_pass=one_pass, relu=relu,
        what="sync_conv1x1_bn_forward", partial=partial)
    return y, cache, z
