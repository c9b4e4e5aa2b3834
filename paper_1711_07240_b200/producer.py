"""Producer fusion: the convolution that feeds a BN emits the BN's
forward partial statistics from its own epilogue, so the BN forward skips its statistics
read of the activation (fwd 12 -> 8 B/elem for fp32).

In the reference model every BN follows a GEMM-shaped producer — conv3x3 as an im2col
GEMM plus bias, or a dense layer (/root/reference/pkg/src/bigbatch/model.py:229-242) —
and the BN's first step re-reads that output for channel_sum (batchnorm.py:118,
tensor.py:143-153). Here the producer is the pointwise (1x1) or 3x3 convolution on the
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
    conv3x3 / conv3x3_stats / conv3x3_bn_forward_local / sync_conv3x3_bn_forward
        the 3x3 convolution (stride 1, zero padding 1) — the reference model's own conv
        layer — as an implicit GEMM over TMA im2col loads (channels_last x and z)

NCHW x runs the pointwise kernel on NCHW z (H*W a multiple of 8); channels_last x runs
the NHWC kernels (any H, W) and returns channels_last z, which the BN's native NHWC
kernels consume.

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
            # zero-filled: the split-K tickets must start at zero (each call leaves them so)
            buf = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
            _scratch[key] = buf
        _scratch.move_to_end(key)
        while len(_scratch) > 64:
            _scratch.popitem(last=False)
        return buf


def _check(x, weight, bias, out_dtype, k, stride=1):
    """Validate a k x k convolution's operands (k = 1 or 3); return the device operands,
    whether x is channels_last, and (n, cin, h, w, cout). A 3x3 weight is permuted to
    the kernel's [9][Cout][Cin] tap-major layout."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise BatchNormError("x must be a CUDA tensor (there is no CPU fallback)")
    if x.dim() != 4:
        raise BatchNormError(f"conv{k}x{k} expects x of shape (N, Cin, H, W), got {tuple(x.shape)}")
    if x.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise BatchNormError(f"conv{k}x{k} takes bfloat16 x and weight (tcgen05 kind::f16)")
    n, cin, h, w = x.shape
    nhwc = x.is_contiguous(memory_format=torch.channels_last) and not x.is_contiguous()
    if k == 1:
        wt = weight.reshape(weight.shape[0], -1) if weight.dim() == 4 else weight
        if wt.dim() != 2 or wt.shape[1] != cin:
            raise BatchNormError(
                f"weight must be (Cout, {cin}) or (Cout, {cin}, 1, 1), got {tuple(weight.shape)}")
        cout = wt.shape[0]
    else:
        if weight.dim() != 4 or tuple(weight.shape[1:]) != (cin, 3, 3):
            raise BatchNormError(f"weight must be (Cout, {cin}, 3, 3), got {tuple(weight.shape)}")
        if not nhwc:
            raise BatchNormError(
                "conv3x3 needs channels_last x: the tap shifts use TMA im2col loads, which "
                "take the channel as the innermost dimension (NCHW rows cannot be shifted "
                "by one element in a TMA box)")
        cout = weight.shape[0]
        # [Cout][tap = 3 ky + kx][Cin] (OHWI): a channels_last weight as it is, no copy
        wt = weight.permute(0, 2, 3, 1).reshape(cout, 9, cin)
    if stride not in (1, 2):
        raise BatchNormError(f"stride must be 1 or 2, got {stride}")
    if stride != 1 and not nhwc:
        raise BatchNormError("strided convolutions need channels_last x (TMA im2col)")
    if cin % 8 != 0:
        raise BatchNormError(f"conv{k}x{k} needs Cin a multiple of 8, got {cin}")
    if nhwc and cout % 8 != 0:
        raise BatchNormError(f"channels_last conv{k}x{k} needs Cout a multiple of 8, got {cout}")
    if not nhwc:
        x = x.contiguous()
        if (h * w) % 8 != 0:
            raise BatchNormError(
                f"conv1x1 needs H*W and Cin multiples of 8 (TMA row strides), got H*W={h * w}, "
                f"Cin={cin}")
    if out_dtype not in _OUT:
        raise BatchNormError(f"out_dtype must be float32 or bfloat16, got {out_dtype}")
    b = None
    if bias is not None:
        b = bias.to(device=x.device, dtype=torch.float32).contiguous()
        if b.shape != (cout,):
            raise BatchNormError(f"bias must have length {cout}")
    return x, wt.to(x.device).contiguous(), b, nhwc, (n, cin, h, w, cout)


def _conv(x, weight, bias, out_dtype, k, stats, stride=1, slots_only=False):
    """The convolution; with ``stats``, also this rank's partial (or, ``slots_only``, the
    statistics slot table left in the returned scratch tensor instead of the partial)."""
    x, wt, b, nhwc, (n, cin, h, w, cout) = _check(x, weight, bias, out_dtype, k, stride)
    lib = _lib.load()
    dev = x.device
    pad = k // 2
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    z = torch.empty((n, cout, ho, wo), dtype=out_dtype, device=dev,
                    memory_format=torch.channels_last if nhwc else torch.contiguous_format)
    bp = b.data_ptr() if b is not None else None
    st = stream_ptr(dev)
    od = _OUT[out_dtype]
    partial = None
    if stats and not slots_only:
        partial = torch.empty(2 * cout + 1, dtype=torch.float64, device=dev)
    # slot table (statistics) and split-K scratch
    nb = (lib.cgbn_conv_nhwc_ws_bytes(n, cin, cout, h, w, k, stride) if nhwc
          else lib.cgbn_conv1x1_ws_bytes(n, cin, cout, h * w))
    ws = _tile_scratch(dev, nb)
    name = f"conv{k}x{k}" + ("_stats" if stats else "")
    with _Span(name, 0):
        if nhwc and stats:
            rc = lib.cgbn_conv_nhwc_stats(x.data_ptr(), wt.data_ptr(), bp, n, cin, cout, h, w, k,
                                          stride, od, z.data_ptr(),
                                          partial.data_ptr() if partial is not None else None,
                                          ws.data_ptr(), ws.numel(), st)
        elif nhwc:
            rc = lib.cgbn_conv_nhwc(x.data_ptr(), wt.data_ptr(), bp, n, cin, cout, h, w, k,
                                    stride, od, z.data_ptr(), ws.data_ptr(), ws.numel(), st)
        elif stats:
            rc = lib.cgbn_conv1x1_stats(x.data_ptr(), wt.data_ptr(), bp, n, cin, cout, h * w, od,
                                        z.data_ptr(),
                                        partial.data_ptr() if partial is not None else None,
                                        ws.data_ptr(), ws.numel(), st)
        else:
            rc = lib.cgbn_conv1x1(x.data_ptr(), wt.data_ptr(), bp, n, cin, cout, h * w, od,
                                  z.data_ptr(), ws.data_ptr(), ws.numel(), st)
        _lib.check(rc, "cgbn_" + ("conv_nhwc" if nhwc else "conv1x1") + ("_stats" if stats else ""))
    if slots_only:
        return z, ws
    return z, partial


def conv1x1(x, weight, bias=None, out_dtype=torch.float32, stride=1):
    """z = conv1x1(x, weight, stride) + bias on the tensor cores (the unfused producer).
    NCHW or channels_last x (stride 2: channels_last); z has x's memory format."""
    return _conv(x, weight, bias, out_dtype, 1, False, stride)[0]


def conv1x1_stats(x, weight, bias=None, out_dtype=torch.float32, stride=1):
    """(z, partial): the convolution plus this rank's forward partial of z (2C+1 fp64,
    [mean | M2 | count], the cgbn_fwd_stats format)."""
    return _conv(x, weight, bias, out_dtype, 1, True, stride)


def conv3x3(x, weight, bias=None, out_dtype=torch.float32, stride=1):
    """z = conv3x3(x, weight, padding=1, stride) + bias on the tensor cores (implicit GEMM
    over TMA im2col loads; channels_last x and z) — the reference model's conv layer
    (model.py:235-242)."""
    return _conv(x, weight, bias, out_dtype, 3, False, stride)[0]


def conv3x3_stats(x, weight, bias=None, out_dtype=torch.float32, stride=1):
    """(z, partial) for the 3x3 convolution, as conv1x1_stats."""
    return _conv(x, weight, bias, out_dtype, 3, True, stride)


def _fused_local(k, x, weight, state, bias, out_dtype, relu, what, stride=1):
    if _bn._exchange_mode != "merged":
        z = _conv(x, weight, bias, out_dtype, k, False, stride)[0]
        y, cache = _bn.bn_forward_local(z, state, relu=relu)
        return y, cache, z
    # single rank: the slot table goes straight to the finalize (no partial, no fold)
    z, slots = _conv(x, weight, bias, out_dtype, k, True, stride, slots_only=True)
    y, cache = _train_forward(z, state, _local_exchange, 1, None, one_pass=False, relu=relu,
                              what=what, slots=slots)
    return y, cache, z


def _fused_sync(k, handle, x, weight, state, bias, out_dtype, one_pass, relu, what,
                stride=1):
    if _bn._exchange_mode != "merged":
        z = _conv(x, weight, bias, out_dtype, k, False, stride)[0]
        y, cache = _bn.sync_bn_forward(handle, z, state, one_pass=one_pass, relu=relu)
        return y, cache, z
    z, partial = _conv(x, weight, bias, out_dtype, k, True, stride)
    scope_key = f"bn{handle.bn_group_index}"
    y, cache = _train_forward(
        z, state, lambda v, info: handle.exchange(SCOPE_BN_GROUP, "bn_forward", v, info),
        handle.bn_group_size, scope_key, one_pass=one_pass, relu=relu, what=what,
        partial=partial)  # (the partial comes from the conv: a fused P2P push does not apply)
    return y, cache, z


def conv3x3_bn_forward_local(x, weight, state: BNLayerState, bias=None,
                             out_dtype=torch.float32, relu: bool = False, stride: int = 1):
    """bn_forward_local(conv3x3(x, weight) + bias, state), statistics from the conv
    epilogue (the reference model's conv -> bn pair, model.py:235-258). Returns
    (y, cache, z)."""
    return _fused_local(3, x, weight, state, bias, out_dtype, relu, "conv3x3_bn_forward_local",
                        stride)


def sync_conv3x3_bn_forward(handle, x, weight, state: BNLayerState, bias=None,
                            out_dtype=torch.float32, one_pass: bool = False,
                            relu: bool = False, stride: int = 1):
    """sync_bn_forward(handle, conv3x3(x, weight) + bias, state), statistics from the
    conv epilogue. Returns (y, cache, z)."""
    return _fused_sync(3, handle, x, weight, state, bias, out_dtype, one_pass, relu,
                       "sync_conv3x3_bn_forward", stride)


def conv1x1_bn_forward_local(x, weight, state: BNLayerState, bias=None,
                             out_dtype=torch.float32, relu: bool = False, stride: int = 1):
    """bn_forward_local(conv1x1(x, weight) + bias, state) with the statistics taken in the
    conv epilogue. Returns (y, cache, z); cache is the BN cache over z."""
    return _fused_local(1, x, weight, state, bias, out_dtype, relu, "conv1x1_bn_forward_local",
                        stride)


def sync_conv1x1_bn_forward(handle, x, weight, state: BNLayerState, bias=None,
                            out_dtype=torch.float32, one_pass: bool = False,
                            relu: bool = False, stride: int = 1):
    """sync_bn_forward(handle, conv1x1(x, weight) + bias, state) with the statistics taken
    in the conv epilogue; the partial goes through the BN group's exchange unchanged.
    Returns (y, cache, z)."""
    return _fused_sync(1, handle, x, weight, state, bias, out_dtype, one_pass, relu,
                       "sync_conv1x1_bn_forward", stride)
