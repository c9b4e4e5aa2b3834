"""Cross-GPU batch normalization (CGBN) — the drop-in surface of the reference's
``bigbatch.batchnorm`` (/root/reference/pkg/src/bigbatch/batchnorm.py), running on
hand-written sm_100a kernels through the C ABI of include/cgbn.h.

Same names, arguments, return tuples and exceptions as the reference:

    BNLayerState, BNForwardCache, BatchNormError,
    bn_forward_local(x, state, mode="train"|"eval")          batchnorm.py:147-166
    sync_bn_forward(handle, x_local, state, one_pass=False)  batchnorm.py:169-185
    bn_backward_local(dy, cache, state)                      batchnorm.py:213-218
    sync_bn_backward(handle, dy_local, cache, state)         batchnorm.py:221-236
    bn_update_running(state, mu, var, count)                 batchnorm.py:239-252

Differences (by design):

* Activations are torch CUDA float32, bfloat16 or float16 (NCHW, channels_last, or
  (N, C)); statistics are computed and exchanged in fp64, gamma / beta / running
  statistics stay float32. ``relu=True`` fuses the ReLU that follows BN in the
  reference model (model.py:243-246) into the forward and its mask into the backward.
* One statistics exchange per pass by default (``set_forward_exchange("merged")``). The
  forward exchanges each rank's (mean, centred M2, count) and folds them with Chan's
  pairwise update in ascending rank order; this has the reference two-pass algorithm's
  numerics (no E[x^2]-E[x]^2 cancellation) at the cost of one collective, so
  ``one_pass`` changes neither cost nor outcome here (the reference's own
  test_trainer.py:377-387 states "one-pass changes cost, not outcome").
  ``set_forward_exchange("reference")`` runs the reference's literal arithmetic (two
  exchanges for ``one_pass=False``).
* ``BNForwardCache`` keeps the input and the per-channel (mean, var, inv_std, m) on the
  device instead of a full x_hat tensor (the backward recomputes x_hat); ``x_hat``,
  ``mu``, ``var`` and ``total_count`` remain available as attributes.
* dgamma/dbeta are BN-group sums, identical on every rank, exactly as the reference
  (batchnorm.py:203); the model divides them by bn_group_size (model.py:344-346).
* Data-dependent errors (NaN/Inf in the statistics, total count < 2 where the host
  cannot see the global count) are detected on the device. With strict checking (the
  default, ``set_strict``) they are raised synchronously by the call, as in the
  reference; with strict checking off they are collected by ``check_status()``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .collectives import SCOPE_BN_GROUP, CollectiveTimeoutError
from .tensor import NonFiniteError, geometry, same_layout_like, status_word, stream_ptr, workspace


class BatchNormError(ValueError):
    """Invalid state, layout, or cache for a batch-norm operation (batchnorm.py:32-33)."""


_strict = True

# Optional kernel timer (bench.py): an object with ``begin(name, nbytes)`` / ``end()``
# called around every native launch on the current stream. None = no instrumentation.
kernel_timer = None


class _Span:
    __slots__ = ("name", "nbytes")

    def __init__(self, name, nbytes):
        self.name = name
        self.nbytes = nbytes

    def __enter__(self):
        if kernel_timer is not None:
            kernel_timer.begin(self.name, self.nbytes)

    def __exit__(self, *exc):
        if kernel_timer is not None:
            kernel_timer.end()
        return False


_fused = False


def set_fused(flag: bool) -> bool:
    """Enable/disable the single-launch fused kernels for single-rank groups (G == 1);
    returns the previous setting. Disabled, G == 1 runs the split two-kernel path."""
    global _fused
    prev = _fused
    _fused = bool(flag)
    return prev


def set_strict(flag: bool) -> bool:
    """Enable/disable synchronous device-status checks; returns the previous setting."""
    global _strict
    prev = _strict
    _strict = bool(flag)
    return prev


def _to_param(v, device, name):
    if isinstance(v, torch.Tensor):
        t = v
        if t.device != device or t.dtype != torch.float32 or not t.is_contiguous():
            t = t.to(device=device, dtype=torch.float32).contiguous()
        return t
    a = np.asarray(v, dtype=np.float64)
    if a.ndim != 1:
        raise BatchNormError(f"{name} must be a 1-D vector")
    return torch.as_tensor(a, dtype=torch.float32).to(device)


def _default_device():
    if not torch.cuda.is_available():
        raise BatchNormError("CGBN needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class BNLayerState:
    """Per-channel affine parameters plus running statistics (batchnorm.py:36-87).

    All four vectors are CUDA float32 tensors (numpy/torch inputs are converted);
    the running statistics are updated in place by training-mode forwards.
    """

    gamma: torch.Tensor
    beta: torch.Tensor
    eps: float = 1e-5
    running_mean: torch.Tensor = None
    running_var: torch.Tensor = None
    running_momentum: float = 0.1

    @classmethod
    def create(cls, channels: int, eps: float = 1e-5, running_momentum: float = 0.1,
               device=None):
        dev = torch.device(device) if device is not None else _default_device()
        return cls(gamma=torch.ones(channels, device=dev), beta=torch.zeros(channels, device=dev),
                   eps=eps, running_mean=torch.zeros(channels, device=dev),
                   running_var=torch.ones(channels, device=dev),
                   running_momentum=running_momentum)

    def __post_init__(self):
        dev = self.gamma.device if isinstance(self.gamma, torch.Tensor) and self.gamma.is_cuda \
            else _default_device()
        self.gamma = _to_param(self.gamma, dev, "gamma")
        if self.gamma.dim() != 1:
            raise BatchNormError("gamma must be a 1-D vector")
        c = self.gamma.shape[0]
        self.beta = _to_param(self.beta, dev, "beta")
        self.running_mean = (torch.zeros(c, device=dev) if self.running_mean is None
                             else _to_param(self.running_mean, dev, "running_mean"))
        self.running_var = (torch.ones(c, device=dev) if self.running_var is None
                            else _to_param(self.running_var, dev, "running_var"))
        self.validate()

    def validate(self):
        c = self.gamma.shape[0]
        for name in ("beta", "running_mean", "running_var"):
            if tuple(getattr(self, name).shape) != (c,):
                raise BatchNormError(f"{name} must have length {c}")
        if not self.eps > 0:
            raise BatchNormError(f"eps must be positive, got {self.eps}")
        if bool((self.running_var < 0).any()):
            raise BatchNormError("running_var must be elementwise nonnegative")
        if not 0.0 <= self.running_momentum <= 1.0:
            raise BatchNormError(
                f"running_momentum must lie in [0, 1], got {self.running_momentum}")

    @property
    def channels(self) -> int:
        return self.gamma.shape[0]

    @property
    def device(self) -> torch.device:
        return self.gamma.device


@dataclass
class BNForwardCache:
    """Values saved by a forward for the backward (batchnorm.py:90-103).

    ``saved`` is the device vector [mean (C) | var (C) | inv_std (C) | m (1)] (fp64);
    x_hat is recomputed from ``x`` on demand instead of being stored.
    """

    x: torch.Tensor
    saved: torch.Tensor
    train: bool
    scope_key: str | None = None  # None for a purely local forward
    relu: bool = False
    one_pass: bool = False
    _total_count: int | None = field(default=None, repr=False)
    _x_version: int | None = field(default=None, repr=False)

    def __post_init__(self):
        # x is saved by reference (the backward recomputes x_hat and the ReLU mask from
        # it), so an in-place change of x before the backward is detected, as autograd
        # does for saved tensors
        if self._x_version is None:
            self._x_version = self.x._version

    @property
    def channels(self) -> int:
        return (self.saved.numel() - 1) // 3

    @property
    def mu(self) -> torch.Tensor:
        return self.saved[: self.channels]

    @property
    def var(self) -> torch.Tensor:
        c = self.channels
        return self.saved[c: 2 * c]

    @property
    def inv_std(self) -> torch.Tensor:
        c = self.channels
        return self.saved[2 * c: 3 * c]

    @property
    def total_count(self) -> int:
        """Global per-channel element count the statistics cover (synchronises the
        device if the host did not see every rank's count)."""
        if self._total_count is None:
            self._total_count = int(round(float(self.saved[3 * self.channels].item())))
        return self._total_count

    @property
    def x_hat(self) -> torch.Tensor:
        """(x - mean) * inv_std, recomputed by the device kernel."""
        g = geometry(self.x, "x", BatchNormError)
        out = same_layout_like(g)
        lib = _lib.load()
        ws = workspace(g.x.device, lib.cgbn_workspace_bytes(g.N, g.C, g.HW, g.layout))
        _lib.check(lib.cgbn_xhat(g.x.data_ptr(), g.N, g.C, g.HW, g.layout,
                                 self.saved.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                 ws.numel(), stream_ptr(g.x.device)), "cgbn_xhat")
        return out


def _check_layout(x, state: BNLayerState):
    g = geometry(x, "x", BatchNormError)
    if g.C != state.channels:
        raise BatchNormError(f"input has {g.C} channels but state has {state.channels}")
    if g.x.device != state.device:
        raise BatchNormError(f"input is on {g.x.device} but the state is on {state.device}")
    return g


def _raise_status(what: str, status: torch.Tensor, count=None):
    """Synchronously check (and clear) the device status word under strict mode."""
    if not _strict or torch.cuda.is_current_stream_capturing():
        return
    v = int(status.item())
    if v == 0:
        return
    status.zero_()
    if v & _lib.STATUS_EXCHANGE_TIMEOUT:
        raise CollectiveTimeoutError(
            f"{what}: a peer did not join the P2P statistics exchange in time")
    if v & _lib.STATUS_NONFINITE:
        raise NonFiniteError(f"{what}: non-finite values in tensor data")
    if v & _lib.STATUS_SMALL_COUNT:
        got = "" if count is None else f", got {count}"
        raise BatchNormError(
            f"training-mode statistics need at least 2 elements per channel{got}")


def check_status(device=None) -> None:
    """Raise for any device-detected error since the last check on the current stream
    (for callers running with ``set_strict(False)``)."""
    dev = torch.device(device) if device is not None else _default_device()
    st = status_word(dev)
    prev = set_strict(True)
    try:
        _raise_status("cgbn", st)
    finally:
        set_strict(prev)


def _local_exchange(vec, info):
    return [vec], [info]


_exchange_mode = "merged"


def set_forward_exchange(mode: str) -> str:
    """How the training forward combines the ranks' statistics; returns the previous mode.

    ``"merged"`` (default): one exchange per forward of each rank's fp64 (mean, M2,
    count), merged with Chan's pairwise update in ascending rank order. It has the
    numerics of the reference's two-pass algorithm (no E[x^2] - mean^2 cancellation)
    for either ``one_pass`` value, at one exchange and two reads of x.

    ``"reference"``: bigbatch's own arithmetic, literally (batchnorm.py:118-132).
    ``one_pass=False`` (the reference default) exchanges [sum | m], reads x again for
    sum (x - mean)^2 and exchanges that (two exchanges, three reads of x);
    ``one_pass=True`` exchanges [sum | sum x^2 | m] and uses max(E[x^2] - mean^2, 0).
    Group sums are folded in ascending rank order, like the reference's allreduce_sum.
    """
    global _exchange_mode
    if mode not in ("merged", "reference"):
        raise ValueError(f"forward exchange must be 'merged' or 'reference', got {mode!r}")
    prev, _exchange_mode = _exchange_mode, mode
    return prev


def _fold_parts(parts, st):
    """Ascending-rank fold of the exchanged fp64 vectors (collectives.py:293-295)."""
    if len(parts) == 1:
        return parts[0]
    lib = _lib.load()
    out = torch.empty_like(parts[0])
    arr, keep = _lib.ptr_array([p.data_ptr() for p in parts])
    _lib.check(lib.cgbn_fold_sum(arr, len(parts), parts[0].numel(), _lib.DTYPE_F64,
                                 out.data_ptr(), st), "cgbn_fold_sum")
    return out


def _train_forward_reference(g, state, exchange, scope_key, one_pass, relu, what):
    """set_forward_exchange("reference"): batchnorm.py:118-132 step by step on the
    device (see include/cgbn.h, cgbn_centered_sumsq / cgbn_fwd_normalize_sums)."""
    c = g.C
    dev = g.x.device
    lib = _lib.load()
    st = stream_ptr(dev)
    e = g.N * c * g.HW
    saved = torch.empty(3 * c + 1, dtype=torch.float64, device=dev)
    y = same_layout_like(g)
    status = status_word(dev)
    ws = workspace(dev, lib.cgbn_workspace_bytes(g.N, c, g.HW, g.layout))
    n = 2 * c + 1 if one_pass else c + 1
    packed = torch.empty(n, dtype=torch.float64, device=dev)
    with _Span("fwd_sums", 4 * e):
        _lib.check(lib.cgbn_channel_sum(
            g.x.data_ptr(), g.N, c, g.HW, g.layout, packed.data_ptr(),
            packed.data_ptr() + 8 * c if one_pass else None, ws.data_ptr(), ws.numel(), st),
            "cgbn_channel_sum")
    packed[n - 1:].fill_(float(g.count))  # local count (batchnorm.py:120, 126)
    parts, infos = exchange(packed, g.count)
    total = None
    if infos is not None and all(i is not None for i in infos):
        total = int(sum(infos))
        if total < 2:
            raise BatchNormError(
                f"training-mode statistics need at least 2 elements per channel, got {total}")
    tot = _fold_parts(parts, st)
    sum_p, cnt_p = tot.data_ptr(), tot.data_ptr() + 8 * (n - 1)
    keep = [tot]
    if one_pass:
        sq_p, centered = tot.data_ptr() + 8 * c, 0
    else:
        sq = torch.empty(c, dtype=torch.float64, device=dev)
        with _Span("fwd_centered_sumsq", 4 * e):
            _lib.check(lib.cgbn_centered_sumsq(
                g.x.data_ptr(), g.N, c, g.HW, g.layout, sum_p, cnt_p, sq.data_ptr(),
                ws.data_ptr(), ws.numel(), st), "cgbn_centered_sumsq")
        parts2, _ = exchange(sq, None)
        sq_t = _fold_parts(parts2, st)
        keep.append(sq_t)
        sq_p, centered = sq_t.data_ptr(), 1
    rm, rv = state.running_mean.data_ptr(), state.running_var.data_ptr()
    with _Span("fwd_normalize", 8 * e):
        _lib.check(lib.cgbn_fwd_normalize_sums(
            g.x.data_ptr(), g.N, c, g.HW, g.layout, sum_p, sq_p, cnt_p, centered,
            state.gamma.data_ptr(), state.beta.data_ptr(), float(state.eps),
            float(state.running_momentum), rm, rv, saved.data_ptr(), int(bool(relu)),
            y.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st),
            "cgbn_fwd_normalize_sums")
    _raise_status(what, status, total)
    return y, BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                             relu=bool(relu), one_pass=bool(one_pass), _total_count=total)


def _train_forward(x, state: BNLayerState, exchange, group_size: int, scope_key,
                   one_pass: bool, relu: bool, what: str, partial=None, slots=None):
    """The CGBN forward (batchnorm.py:115-144) on the device.

    G > 1: stats kernel -> exchange of the per-rank partials -> finalize (fold + running
    update + coefficients) and elementwise normalise. G == 1: the stats kernel finalises
    each channel itself (cgbn_fwd_train_local), or one fused cooperative kernel when
    enabled (set_fused) and the activation fits on chip.

    ``partial``: this rank's forward partial of ``x`` already computed by its producer
    (producer fusion, ``producer.py``); the statistics kernel is skipped and the partial
    goes straight to the exchange and the normalise pass (for any G). ``slots``: for a
    single-rank group, the producer's statistics slot table instead
    (cgbn_fwd_normalize_slots merges it straight into the coefficients).
    """
    g = _check_layout(x, state)
    if partial is not None and _exchange_mode != "merged":
        raise BatchNormError("a producer-computed partial needs set_forward_exchange('merged')")
    if _exchange_mode == "reference":
        if group_size == 1 and g.count < 2:
            raise BatchNormError(
                f"training-mode statistics need at least 2 elements per channel, got {g.count}")
        return _train_forward_reference(g, state, exchange, scope_key, one_pass, relu, what)
    c = g.C
    dev = g.x.device
    lib = _lib.load()
    st = stream_ptr(dev)
    e = g.N * c * g.HW
    saved = torch.empty(3 * c + 1, dtype=torch.float64, device=dev)
    y = same_layout_like(g)
    status = status_word(dev)
    nb = lib.cgbn_workspace_bytes(g.N, c, g.HW, g.layout)
    ws = workspace(dev, nb)
    rm, rv = state.running_mean.data_ptr(), state.running_var.data_ptr()
    if group_size == 1 and slots is not None:
        total = g.count
        if total < 2:
            raise BatchNormError(
                f"training-mode statistics need at least 2 elements per channel, got {total}")
        with _Span("fwd_normalize", 8 * e):
            _lib.check(lib.cgbn_fwd_normalize_slots(
                g.x.data_ptr(), g.N, c, g.HW, g.layout, slots.data_ptr(),
                state.gamma.data_ptr(), state.beta.data_ptr(), float(state.eps),
                float(state.running_momentum), rm, rv, saved.data_ptr(), int(bool(relu)),
                y.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "cgbn_fwd_normalize_slots")
        _raise_status(what, status, total)
        return y, BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                                 relu=bool(relu), one_pass=bool(one_pass), _total_count=total)
    if group_size == 1 and partial is None:
        total = g.count
        if total < 2:
            raise BatchNormError(
                f"training-mode statistics need at least 2 elements per channel, got {total}")
        if _fused and lib.cgbn_fused_supported(g.N, c, g.HW, g.layout, 0):
            with _Span("fwd_fused", 8 * e):
                _lib.check(lib.cgbn_fwd_fused(
                    g.x.data_ptr(), g.N, c, g.HW, g.layout, state.gamma.data_ptr(),
                    state.beta.data_ptr(), float(state.eps), float(state.running_momentum), rm,
                    rv, saved.data_ptr(), int(bool(relu)), y.data_ptr(), status.data_ptr(),
                    ws.data_ptr(), ws.numel(), st), "cgbn_fwd_fused")
            _raise_status(what, status, total)
            return y, BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                                     relu=bool(relu), one_pass=bool(one_pass),
                                     _total_count=total)
        with _Span("fwd_local", 12 * e):
            _lib.check(lib.cgbn_fwd_train_local(
                g.x.data_ptr(), g.N, c, g.HW, g.layout, state.gamma.data_ptr(),
                state.beta.data_ptr(), float(state.eps), float(state.running_momentum), rm, rv,
                saved.data_ptr(), int(bool(relu)), y.data_ptr(), status.data_ptr(),
                ws.data_ptr(), ws.numel(), st), "cgbn_fwd_train_local")
        _raise_status(what, status, total)
        return y, BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                                 relu=bool(relu), one_pass=bool(one_pass), _total_count=total)
    fused = getattr(exchange, "fused", None) if partial is None else None
    if fused is not None:
        # fused P2P exchange (cgbn_fwd_stats_p2p / cgbn_fwd_normalize_p2p): the reduction
        # pushes the partial into every rank's region, the finalize waits for the flags
        with _Span("fwd_stats", 4 * e):
            _lib.check(lib.cgbn_fwd_stats_p2p(
                g.x.data_ptr(), g.N, c, g.HW, g.layout, fused.idx, fused.G, fused.regions,
                fused.max_len, ws.data_ptr(), ws.numel(), st), "cgbn_fwd_stats_p2p")
        with _Span("fwd_normalize", 8 * e):
            _lib.check(lib.cgbn_fwd_normalize_p2p(
                g.x.data_ptr(), g.N, c, g.HW, g.layout, fused.own, fused.G, fused.max_len,
                fused.timeout_s, state.gamma.data_ptr(), state.beta.data_ptr(),
                float(state.eps), float(state.running_momentum), rm, rv, saved.data_ptr(),
                int(bool(relu)), y.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "cgbn_fwd_normalize_p2p")
        _raise_status(what, status, None)
        return y, BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                                 relu=bool(relu), one_pass=bool(one_pass), _total_count=None)
    if partial is None:
        partial = torch.empty(2 * c + 1, dtype=torch.float64, device=dev)
        with _Span("fwd_stats", 4 * e):
            _lib.check(lib.cgbn_fwd_stats(g.x.data_ptr(), g.N, c, g.HW, g.layout,
                                          partial.data_ptr(), ws.data_ptr(), ws.numel(), st),
                       "cgbn_fwd_stats")
    elif partial.numel() != 2 * c + 1 or partial.dtype != torch.float64:
        raise BatchNormError(f"forward partial must be {2 * c + 1} float64 values")
    parts, infos = exchange(partial, g.count)
    total = None
    if infos is not None and all(i is not None for i in infos):
        total = int(sum(infos))
        if total < 2:
            raise BatchNormError(
                f"training-mode statistics need at least 2 elements per channel, got {total}")
    arr, keep = _lib.ptr_array([p.data_ptr() for p in parts])
    with _Span("fwd_normalize", 8 * e):
        _lib.check(lib.cgbn_fwd_normalize(
            g.x.data_ptr(), g.N, c, g.HW, g.layout, arr, len(parts), state.gamma.data_ptr(),
            state.beta.data_ptr(), float(state.eps), float(state.running_momentum), rm, rv,
            saved.data_ptr(), int(bool(relu)), y.data_ptr(), status.data_ptr(), ws.data_ptr(),
            ws.numel(), st), "cgbn_fwd_normalize")
    _raise_status(what, status, total)
    cache = BNForwardCache(x=g.x, saved=saved, train=True, scope_key=scope_key,
                           relu=bool(relu), one_pass=bool(one_pass), _total_count=total)
    return y, cache


def bn_forward_local(x, state: BNLayerState, mode: str = "train",
                     relu: bool = False):
    """Batch normalization over a single device's batch (batchnorm.py:147-166).

    Training mode computes biased per-channel statistics from ``x`` and updates the
    running estimates; eval mode normalizes with the running statistics and leaves the
    state untouched.
    """
    if mode == "train":
        return _train_forward(x, state, _local_exchange, 1, None, one_pass=False, relu=relu,
                              what="bn_forward_local")
    g = _check_layout(x, state)
    if mode != "eval":
        raise BatchNormError(f"mode must be 'train' or 'eval', got {mode!r}")
    lib = _lib.load()
    y = same_layout_like(g)
    ws = workspace(g.x.device, lib.cgbn_workspace_bytes(g.N, g.C, g.HW, g.layout))
    _lib.check(lib.cgbn_fwd_eval(g.x.data_ptr(), g.N, g.C, g.HW, g.layout,
                                 state.gamma.data_ptr(), state.beta.data_ptr(),
                                 state.running_mean.data_ptr(), state.running_var.data_ptr(),
                                 float(state.eps), int(bool(relu)), y.data_ptr(), ws.data_ptr(),
                                 ws.numel(), stream_ptr(g.x.device)), "cgbn_fwd_eval")
    c = g.C
    saved = torch.empty(3 * c + 1, dtype=torch.float64, device=g.x.device)
    saved[:c] = state.running_mean.double()
    saved[c:2 * c] = state.running_var.double()
    saved[2 * c:3 * c] = torch.rsqrt(state.running_var.double() + state.eps)
    saved[3 * c] = float(g.count)
    cache = BNForwardCache(x=g.x, saved=saved, train=False, relu=bool(relu),
                           _total_count=g.count)
    return y, cache


class _GroupExchange:
    """The reduce_vec seam bound to a handle's BN-group exchange (batchnorm.py:183, 236);
    ``fused`` is the handle's fused P2P exchange when it has one (DistHandle
    transport="p2p_fused"), in which case the kernels do the exchange themselves."""

    def __init__(self, handle, kind: str):
        self.handle = handle
        self.kind = kind
        self.fused = getattr(handle, "fused_exchange", None)

    def __call__(self, v, info):
        return self.handle.exchange(SCOPE_BN_GROUP, self.kind, v, info)


def sync_bn_forward(handle, x_local, state: BNLayerState, one_pass: bool = False,
                    relu: bool = False):
    """Training-mode batch normalization synchronized across a BN sub-group
    (batchnorm.py:169-185).

    Every rank of the sub-group must call this with tensors of identical channel and
    spatial extents (per-rank batch sizes may differ; counts travel with the statistics
    so the mean stays exact). All ranks end up with bitwise-identical statistics and the
    output matches ``bn_forward_local`` on the rank-ordered concatenation of the shards.
    """
    _check_layout(x_local, state)
    scope_key = f"bn{handle.bn_group_index}"
    return _train_forward(
        x_local, state, _GroupExchange(handle, "bn_forward"),
        handle.bn_group_size, scope_key, one_pass=one_pass, relu=relu, what="sync_bn_forward")


def _backward_core(dy, cache: BNForwardCache, state: BNLayerState, exchange, group_size: int,
                   what: str):
    """batchnorm.py:188-210 on the device: partial [sum g, sum g*(x-mean)] -> exchange ->
    finalize (fold + dgamma/dbeta + dx coefficients) + elementwise dx. G == 1: the reduce
    kernel finalises each channel itself (cgbn_bwd_local), or one fused cooperative
    kernel when enabled (set_fused) and dy, x fit on chip."""
    if not cache.train:
        raise BatchNormError("backward requires a training-mode forward cache")
    if cache.x._version != cache._x_version:
        raise BatchNormError(
            "the forward input was modified in place after the forward; the backward "
            "recomputes x_hat from it (save a copy, or run the backward first)")
    if not isinstance(dy, torch.Tensor):
        raise BatchNormError(f"dy must be a torch.Tensor, got {type(dy).__name__}")
    if tuple(dy.shape) != tuple(cache.x.shape):
        raise BatchNormError(
            f"cotangent shape {tuple(dy.shape)} does not match cached shape "
            f"{tuple(cache.x.shape)}")
    c = state.channels
    if cache.channels != c:
        raise BatchNormError("cache does not match this layer state")
    gx = geometry(cache.x, "x", BatchNormError)
    if gx.mem == _lib.LAYOUT_NHWC:
        dy = dy.contiguous(memory_format=torch.channels_last)
    else:
        dy = dy.contiguous()
    gd = geometry(dy, "dy", BatchNormError)
    if gd.layout != gx.layout:
        raise BatchNormError(f"dy ({dy.dtype}) and x ({gx.x.dtype}) must share a memory layout "
                             "and dtype")
    dev = gx.x.device
    lib = _lib.load()
    st = stream_ptr(dev)
    e = gx.N * c * gx.HW
    nb = lib.cgbn_workspace_bytes(gx.N, c, gx.HW, gx.layout)
    ws = workspace(dev, nb)
    dx = same_layout_like(gx)
    dgamma = torch.empty(c, dtype=torch.float32, device=dev)
    dbeta = torch.empty(c, dtype=torch.float32, device=dev)
    status = status_word(dev)
    if group_size == 1 and _fused and lib.cgbn_fused_supported(gx.N, c, gx.HW, gx.layout, 1):
        with _Span("bwd_fused", 12 * e):
            _lib.check(lib.cgbn_bwd_fused(
                gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout,
                cache.saved.data_ptr(), state.gamma.data_ptr(), state.beta.data_ptr(),
                float(state.eps), int(cache.relu), dx.data_ptr(), dgamma.data_ptr(),
                dbeta.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "cgbn_bwd_fused")
        _raise_status(what, status)
        return dx, dgamma, dbeta
    if group_size == 1:
        with _Span("bwd_local", 20 * e):
            _lib.check(lib.cgbn_bwd_local(
                gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout,
                cache.saved.data_ptr(), state.gamma.data_ptr(), state.beta.data_ptr(),
                float(state.eps), int(cache.relu), dx.data_ptr(), dgamma.data_ptr(),
                dbeta.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st),
                "cgbn_bwd_local")
        _raise_status(what, status)
        return dx, dgamma, dbeta
    fused = getattr(exchange, "fused", None)
    if fused is not None and group_size > 1:
        with _Span("bwd_reduce", 8 * e):
            _lib.check(lib.cgbn_bwd_reduce_p2p(
                gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout, cache.saved.data_ptr(),
                state.gamma.data_ptr(), state.beta.data_ptr(), int(cache.relu), fused.idx,
                fused.G, fused.regions, fused.max_len, ws.data_ptr(), ws.numel(), st),
                "cgbn_bwd_reduce_p2p")
        with _Span("bwd_dx", 12 * e):
            _lib.check(lib.cgbn_bwd_dx_p2p(
                gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout, fused.own, fused.G,
                fused.max_len, fused.timeout_s, cache.saved.data_ptr(), state.gamma.data_ptr(),
                state.beta.data_ptr(), float(state.eps), int(cache.relu), dx.data_ptr(),
                dgamma.data_ptr(), dbeta.data_ptr(), status.data_ptr(), ws.data_ptr(),
                ws.numel(), st), "cgbn_bwd_dx_p2p")
        _raise_status(what, status)
        return dx, dgamma, dbeta
    partial = torch.empty(2 * c, dtype=torch.float64, device=dev)
    with _Span("bwd_reduce", 8 * e):
        _lib.check(lib.cgbn_bwd_reduce(
            gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout, cache.saved.data_ptr(),
            state.gamma.data_ptr(), state.beta.data_ptr(), int(cache.relu), partial.data_ptr(),
            ws.data_ptr(), ws.numel(), st), "cgbn_bwd_reduce")
    parts = exchange(partial, gx.count)[0]
    arr, keep = _lib.ptr_array([p.data_ptr() for p in parts])
    with _Span("bwd_dx", 12 * e):
        _lib.check(lib.cgbn_bwd_dx(
            gd.x.data_ptr(), gx.x.data_ptr(), gx.N, c, gx.HW, gx.layout, arr, len(parts),
            cache.saved.data_ptr(), state.gamma.data_ptr(), state.beta.data_ptr(),
            float(state.eps), int(cache.relu), dx.data_ptr(), dgamma.data_ptr(),
            dbeta.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), st), "cgbn_bwd_dx")
    _raise_status(what, status)
    return dx, dgamma, dbeta


def bn_backward_local(dy, cache: BNForwardCache, state: BNLayerState):
    """Backward pass matching a local training-mode forward (batchnorm.py:213-218)."""
    if cache.scope_key is not None:
        raise BatchNormError("cache came from a synchronized forward; use sync_bn_backward")
    return _backward_core(dy, cache, state, _local_exchange, 1, "bn_backward_local")


def sync_bn_backward(handle, dy_local, cache: BNForwardCache, state: BNLayerState):
    """Backward pass matching ``sync_bn_forward`` on the same sub-group
    (batchnorm.py:221-236): the per-channel sums of dy and dy*x_hat are aggregated over
    the sub-group, so dgamma/dbeta are identical on every rank."""
    scope_key = f"bn{handle.bn_group_index}"
    if cache.scope_key != scope_key:
        raise BatchNormError(
            f"cache was produced under scope {cache.scope_key!r} but this device "
            f"belongs to {scope_key!r}")
    return _backward_core(dy_local, cache, state, _GroupExchange(handle, "bn_backward"),
                          handle.bn_group_size, "sync_bn_backward")


def bn_update_running(state: BNLayerState, mu, var, count: int) -> BNLayerState:
    """Blend batch statistics into the running estimates, in place (batchnorm.py:239-252).

    The training forward already fuses this update into its normalise kernel; this
    standalone form is kept for API parity (device vector arithmetic).
    """
    if count <= 1:
        raise BatchNormError(f"running-variance update needs count > 1, got {count}")
    rho = float(state.running_momentum)
    dev = state.device
    mu = torch.as_tensor(mu, dtype=torch.float64, device=dev)
    var = torch.as_tensor(var, dtype=torch.float64, device=dev)
    unbiased = var * (count / (count - 1.0))
    state.running_mean.copy_((1.0 - rho) * state.running_mean.double() + rho * mu)
    state.running_var.copy_((1.0 - rho) * state.running_var.double() + rho * unbiased)
    return state
