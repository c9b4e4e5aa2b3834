"""Device groups and the statistics exchange of the CGBN hot path.

Mirrors the reference's ``bigbatch.collectives`` surface (DeviceGroup, DeviceHandle,
allreduce_sum, scopes, CollectiveProtocolError / CollectiveTimeoutError;
/root/reference/pkg/src/bigbatch/collectives.py:24-298), re-designed for GPUs:

* The reference moves numpy vectors between threads through per-(rank, scope) queues
  and folds them at the lowest rank in ascending rank order (collectives.py:260-298).
* Here the per-rank vectors stay in device memory. A collective is split into a
  *transport* that makes every rank's vector visible to every rank of the scope, and a
  *fold* that each consumer kernel performs itself in ascending rank order (so all
  ranks compute bitwise-identical results, like the reference's root fold followed by
  the broadcast of the result).

Two transports:

``DeviceGroup`` (threaded, one process): one host thread per rank, each with its own
  CUDA stream; ranks may share one GPU ("G shards on one GPU", the mode the parity tests
  use) or sit on different GPUs. The transport is a host rendezvous that exchanges
  device pointers plus CUDA events — no device-side waiting, so emulated ranks on one
  GPU can never deadlock. It keeps the reference's diagnostics: per-scope sequence
  numbers, kind/length mismatch -> CollectiveProtocolError naming ranks, timeouts ->
  CollectiveTimeoutError naming the missing ranks, and abort fan-out when a worker dies.

``DistHandle`` (torch.distributed, one process per GPU, NCCL over NVLink/NVSwitch):
  the transport is an all-gather of the fixed-size partial vector on the BN sub-group's
  communicator (contiguous rank blocks of ``bn_group_size``, collectives.py:98-126).
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field
from typing import Any, Callable

import torch

from . import _lib

DEFAULT_TIMEOUT_S = 30.0

SCOPE_WORLD = "world"
SCOPE_BN_GROUP = "bn_group"
_SCOPE_NAMES = (SCOPE_WORLD, SCOPE_BN_GROUP)


class CollectiveError(RuntimeError):
    """Base class for collective failures (collectives.py:31-32)."""


class CollectiveProtocolError(CollectiveError):
    """Mismatched collective calls, payload disagreement, or invalid scope."""

    def __init__(self, msg, from_abort=False):
        super().__init__(msg)
        self.from_abort = from_abort


class CollectiveTimeoutError(CollectiveError):
    """A rank waited longer than the configured timeout for its peers."""


# ------------------------------------------------------------------------------------
# Rendezvous (threaded transport)


@dataclass
class _Post:
    rank: int
    kind: str
    meta: tuple  # (length, dtype string) of the exchanged vector
    tensor: Any
    event: Any
    info: Any = None  # host-side per-rank info (e.g. the local element count)


class _Board:
    """Per-scope exchange board: posts keyed by sequence number."""

    def __init__(self, ranks):
        self.ranks = list(ranks)
        self.cv = threading.Condition()
        self.posts: dict[int, dict[int, _Post]] = {}
        self.taken: dict[int, int] = {}
        self.abort_note: str | None = None

    def exchange(self, scope_key: str, seq: int, post: _Post, timeout_s: float) -> dict:
        g = len(self.ranks)
        with self.cv:
            if self.abort_note is not None:
                raise CollectiveProtocolError(self.abort_note, from_abort=True)
            slot = self.posts.setdefault(seq, {})
            slot[post.rank] = post
            self.cv.notify_all()
            deadline = time.monotonic() + timeout_s
            while len(slot) < g and self.abort_note is None:
                remaining = deadline - time.monotonic()
                if remaining <= 0:
                    missing = sorted(set(self.ranks) - set(slot))
                    note = (f"{post.kind}[{scope_key}#{seq}]: rank {post.rank} timed out "
                            f"after {timeout_s}s waiting for rank(s) {missing}")
                    raise CollectiveTimeoutError(note)
                self.cv.wait(remaining)
            if len(slot) < g:
                raise CollectiveProtocolError(self.abort_note, from_abort=True)
            got = dict(slot)
            self.taken[seq] = self.taken.get(seq, 0) + 1
            if self.taken[seq] == g:
                del self.posts[seq]
                del self.taken[seq]
        kinds = {p.kind for p in got.values()}
        if len(kinds) != 1:
            detail = ", ".join(f"rank {r}: {got[r].kind}" for r in self.ranks)
            raise CollectiveProtocolError(
                f"collective mismatch in {scope_key}#{seq}: ranks issued different "
                f"collectives ({detail})")
        metas = {p.meta for p in got.values()}
        if len(metas) != 1:
            detail = ", ".join(f"rank {r}: len {got[r].meta[0]} ({got[r].meta[1]})"
                               for r in self.ranks)
            raise CollectiveProtocolError(
                f"{post.kind}[{scope_key}#{seq}]: payload mismatch across ranks ({detail})")
        return got

    def abort(self, note: str):
        with self.cv:
            if self.abort_note is None:
                self.abort_note = note
            self.cv.notify_all()


# ------------------------------------------------------------------------------------
# Handles


class _HandleBase:
    """Common scope bookkeeping (collectives.py:56-95)."""

    rank: int
    world_size: int
    bn_group_size: int

    @property
    def bn_group_index(self) -> int:
        return self.rank // self.bn_group_size

    @property
    def bn_group_ranks(self) -> list[int]:
        g = self.bn_group_size
        start = self.bn_group_index * g
        return list(range(start, start + g))

    def _scope_info(self, scope: str) -> tuple[str, list[int]]:
        if scope == SCOPE_WORLD:
            return "world", list(range(self.world_size))
        if scope == SCOPE_BN_GROUP:
            return f"bn{self.bn_group_index}", self.bn_group_ranks
        raise CollectiveProtocolError(
            f"rank {self.rank}: unknown scope {scope!r}; expected one of {_SCOPE_NAMES}")

    def _next_seq(self, scope_key: str) -> int:
        seq = self._seq.get(scope_key, 0)
        self._seq[scope_key] = seq + 1
        return seq

    def exchange(self, scope: str, kind: str, vec: torch.Tensor, info=None):
        """Make every rank's 1-D ``vec`` of ``scope`` visible on this rank's device, in
        ascending rank order, ordered after each producer's writes on this rank's
        current stream. Transport only — the fold is done by the consumer kernel.

        Returns ``(vectors, infos)``: ``infos`` is the per-rank list of the host-side
        ``info`` objects when the transport carries them (threaded group), else None.
        """
        raise NotImplementedError

    @property
    def device(self) -> torch.device:
        raise NotImplementedError


class DeviceHandle(_HandleBase):
    """One rank of a threaded ``DeviceGroup`` (collectives.py:56-95).

    A handle belongs to exactly one group and must only be used from its own worker
    thread; inside ``DeviceGroup.run`` the worker's current CUDA stream is the handle's
    own stream.
    """

    def __init__(self, group: "DeviceGroup", rank: int, device: torch.device):
        self.group = group
        self.rank = rank
        self.world_size = group.world_size
        self.bn_group_size = group.bn_group_size
        self._device = device
        self._seq: dict[str, int] = {}
        self.stream = None  # created in the worker thread

    def __repr__(self):
        return f"DeviceHandle(rank={self.rank}, world={self.world_size}, device={self._device})"

    @property
    def device(self) -> torch.device:
        return self._device

    def exchange(self, scope: str, kind: str, vec: torch.Tensor, info=None):
        scope_key, ranks = self._scope_info(scope)
        seq = self._next_seq(scope_key)
        if vec.dim() != 1:
            raise CollectiveProtocolError(f"rank {self.rank}: collective payload must be a 1-D vector")
        event = None
        if vec.is_cuda:
            event = torch.cuda.Event()
            event.record(torch.cuda.current_stream(vec.device))
        post = _Post(self.rank, kind, (int(vec.numel()), str(vec.dtype)), vec, event, info)
        got = self.group._boards[scope_key].exchange(scope_key, seq, post, self.group.timeout_s)
        out = []
        if vec.is_cuda:
            cur = torch.cuda.current_stream(vec.device)
            cross = False
            for r in ranks:
                p = got[r]
                if r != self.rank:
                    cur.wait_event(p.event)
                t = p.tensor
                if t.device != vec.device:
                    t = t.to(vec.device, non_blocking=True)  # peer copy (NVLink P2P)
                    cross = True
                elif r != self.rank:
                    t.record_stream(cur)
                out.append(t)
            if cross:
                # A peer's tensor lives on its own device, where record_stream cannot
                # reach our stream: finish the copies, then meet every rank once more so
                # no producer releases (and its allocator reuses) a partial that a
                # consumer has not copied yet. Every rank of a group that spans devices
                # has a peer on another device, so all of them take this branch.
                cur.synchronize()
                ack = _Post(self.rank, "ack", (0, "ack"), None, None, None)
                self.group._boards[scope_key].exchange(scope_key, -(seq + 1), ack,
                                                       self.group.timeout_s)
        else:
            out = [got[r].tensor for r in ranks]
        return out, [got[r].info for r in ranks]


class DeviceGroup:
    """A fixed set of ranks 0..n-1 run as threads of this process (collectives.py:98-199).

    Ranks are partitioned into contiguous BN sub-groups of ``bn_group_size``
    ([0..g), [g..2g), ...); ``bn_group_size`` must divide ``world_size``. ``devices``
    maps ranks to CUDA devices (default: every rank on the current device — the
    "G shards on one GPU" mode).
    """

    def __init__(self, world_size: int, bn_group_size: int | None = None, seed: int = 0,
                 timeout_s: float = DEFAULT_TIMEOUT_S, devices=None):
        if world_size < 1:
            raise ValueError(f"world_size must be >= 1, got {world_size}")
        bn_group_size = world_size if bn_group_size is None else bn_group_size
        if bn_group_size < 1 or world_size % bn_group_size != 0:
            raise ValueError(
                f"bn_group_size {bn_group_size} must divide world_size {world_size}")
        self.world_size = world_size
        self.bn_group_size = bn_group_size
        self.seed = seed
        self.timeout_s = timeout_s
        if devices is None:
            if torch.cuda.is_available():
                devices = [torch.device("cuda", torch.cuda.current_device())] * world_size
            else:
                devices = [torch.device("cpu")] * world_size
        devices = [torch.device(d) for d in devices]
        if len(devices) != world_size:
            raise ValueError(f"need {world_size} devices, got {len(devices)}")
        self.devices = devices
        self._boards = {"world": _Board(range(world_size))}
        for i in range(world_size // bn_group_size):
            self._boards[f"bn{i}"] = _Board(range(i * bn_group_size, (i + 1) * bn_group_size))
        self.handles = [DeviceHandle(self, r, devices[r]) for r in range(world_size)]

    def _abort_all(self, note: str):
        for b in self._boards.values():
            b.abort(note)

    def run(self, fn: Callable[[DeviceHandle], Any], timeout_s: float | None = None,
            return_exceptions: bool = False) -> list:
        """Run ``fn(handle)`` concurrently on every rank; return per-rank results.

        Same contract as the reference (collectives.py:146-199): exceptions are
        re-raised preferring the rank with the original diagnostic over ranks that were
        merely aborted; ``return_exceptions`` returns them in the list instead. Each
        rank's device work is complete when ``run`` returns.
        """
        # fresh boards per run so a previous abort does not leak into this one
        self._boards = {k: _Board(b.ranks) for k, b in self._boards.items()}
        for h in self.handles:
            h._seq = {}
        results: list[Any] = [None] * self.world_size
        errors: list[BaseException | None] = [None] * self.world_size

        def runner(handle: DeviceHandle):
            try:
                if handle.device.type == "cuda":
                    torch.cuda.set_device(handle.device)
                    handle.stream = torch.cuda.Stream(device=handle.device)
                    with torch.cuda.stream(handle.stream):
                        results[handle.rank] = fn(handle)
                    handle.stream.synchronize()
                else:
                    results[handle.rank] = fn(handle)
            except BaseException as exc:  # noqa: BLE001 - reported to caller
                errors[handle.rank] = exc
                if not isinstance(exc, CollectiveError):
                    self._abort_all(f"aborted: rank {handle.rank} failed with "
                                    f"{type(exc).__name__}: {exc}")
                elif isinstance(exc, CollectiveTimeoutError):
                    self._abort_all(str(exc))

        threads = [threading.Thread(target=runner, args=(h,), daemon=True,
                                    name=f"cgbn-rank-{h.rank}") for h in self.handles]
        for t in threads:
            t.start()
        join_deadline = self.timeout_s + 10.0 if timeout_s is None else timeout_s
        for r, t in enumerate(threads):
            t.join(timeout=join_deadline)
            if t.is_alive():
                errors[r] = CollectiveTimeoutError(f"rank {r}: worker did not finish")
        if return_exceptions:
            return [errors[r] if errors[r] is not None else results[r]
                    for r in range(self.world_size)]
        primary = None
        for exc in errors:
            if exc is None:
                continue
            if not (isinstance(exc, CollectiveProtocolError) and exc.from_abort):
                raise exc
            primary = primary or exc
        if primary is not None:
            raise primary
        return results


class SoloHandle(_HandleBase):
    """A one-rank group (world 1): the exchange is the identity, as the reference's
    local path binds reduce_vec to ``lambda v: v`` (batchnorm.py:157, 218)."""

    def __init__(self, device=None):
        self.rank = 0
        self.world_size = 1
        self.bn_group_size = 1
        self._seq = {}
        self._device = (torch.device(device) if device is not None
                        else torch.device("cuda", torch.cuda.current_device()))

    @property
    def device(self) -> torch.device:
        return self._device

    def exchange(self, scope: str, kind: str, vec: torch.Tensor, info=None):
        self._scope_info(scope)
        return [vec], [info]


# ------------------------------------------------------------------------------------
# torch.distributed transport (one process per GPU)


class _P2PGroup:
    """One-shot NVLink / NVSwitch exchange for one BN group of a torch.distributed job
    (include/cgbn.h cgbn_p2p_*): each rank's region is shared with the group by CUDA
    IPC, and an exchange is one single-CTA kernel per rank -- push, publish an epoch
    flag, wait for the peers' flags, copy the G rows out in rank order. The consumer
    kernels fold the rows exactly as on the NCCL path, so results are bitwise equal."""

    def __init__(self, ranks, my_rank, pg, device, max_len: int, timeout_s: float):
        import torch.distributed as dist
        lib = _lib.load()
        self.G = len(ranks)
        self.idx = ranks.index(my_rank)
        self.max_len = int(max_len)
        self.timeout_s = float(timeout_s)
        self.device = device
        nbytes = lib.cgbn_p2p_region_bytes(self.G, self.max_len)
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        with torch.cuda.device(device):
            rc = lib.cgbn_p2p_alloc(nbytes, ctypes.byref(own), handle)
        # every rank reaches the gather, so a failure on one rank cannot strand the others
        handles = [None] * self.G
        dist.all_gather_object(handles, bytes(handle) if rc == _lib.OK else None, group=pg)
        if any(h is None for h in handles):
            if rc == _lib.OK:
                lib.cgbn_p2p_free(own.value)
            bad = [ranks[q] for q, h in enumerate(handles) if h is None]
            raise CollectiveError(f"P2P region allocation failed on rank(s) {bad}")
        self._own = own.value
        self._opened = []
        ptrs = []
        with torch.cuda.device(device):
            for q, h in enumerate(handles):
                if q == self.idx:
                    ptrs.append(self._own)
                    continue
                p = ctypes.c_void_p()
                hb = (ctypes.c_char * 64).from_buffer_copy(h)
                _lib.check(lib.cgbn_p2p_open(hb, ctypes.byref(p)), "cgbn_p2p_open")
                self._opened.append(p.value)
                ptrs.append(p.value)
        self._regions, self._keep = _lib.ptr_array(ptrs)

    def exchange(self, vec: torch.Tensor) -> list:
        from .tensor import status_word
        lib = _lib.load()
        n = vec.numel()
        out = torch.empty(self.G * n, dtype=torch.float64, device=vec.device)
        status = status_word(vec.device)
        _lib.check(lib.cgbn_p2p_exchange(
            vec.data_ptr(), n, self.idx, self.G, self._regions, self.max_len, out.data_ptr(),
            status.data_ptr(), self.timeout_s, torch.cuda.current_stream(vec.device).cuda_stream),
            "cgbn_p2p_exchange")
        return [out[q * n:(q + 1) * n] for q in range(self.G)]

    @property
    def regions(self):
        """ctypes array of the group's region pointers (own at [idx])."""
        return self._regions

    @property
    def own(self) -> int:
        return self._own

    def close(self):
        lib = _lib.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize(self.device)
            for p in self._opened:
                lib.cgbn_p2p_close(p)
            if self._own:
                lib.cgbn_p2p_free(self._own)
        self._opened, self._own = [], None


class DistHandle(_HandleBase):
    """This process's rank in a torch.distributed job, with BN sub-groups of
    ``bn_group_size`` contiguous ranks. The exchange is an all-gather of the packed
    partial on the scope's communicator (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, bn_group_size: int | None = None, validate: bool = False,
                 transport: str = "nccl", p2p_max_len: int = 2 * 65535 + 1,
                 p2p_timeout_s: float = 10.0, device=None):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised before DistHandle")
        self.rank = dist.get_rank()
        self.world_size = dist.get_world_size()
        g = self.world_size if bn_group_size is None else bn_group_size
        if g < 1 or self.world_size % g != 0:
            raise ValueError(f"bn_group_size {g} must divide world_size {self.world_size}")
        self.bn_group_size = g
        self.validate = validate
        self._seq = {}
        # every rank must create every sub-group, in the same order
        self._groups = {"world": None}
        if g == self.world_size:
            self._groups[f"bn0"] = None
        else:
            for i in range(self.world_size // g):
                pg = dist.new_group(list(range(i * g, (i + 1) * g)))
                self._groups[f"bn{i}"] = pg
        backend = dist.get_backend()
        if device is not None:
            self._device = torch.device(device)
        else:
            self._device = (torch.device("cuda", torch.cuda.current_device())
                            if backend == "nccl" else torch.device("cpu"))
        # statistics transport of the BN group: "nccl" (all-gather on the group's
        # communicator), "p2p" (one-shot NVLink exchange over CUDA-IPC regions,
        # include/cgbn.h cgbn_p2p_*) or "p2p_fused" (the same regions, with the push fused
        # into the statistics reductions and the wait into the finalize kernels:
        # cgbn_*_p2p, no exchange kernel; BN groups of at most 8); world-scope
        # collectives always use NCCL
        if transport not in ("nccl", "p2p", "p2p_fused"):
            raise ValueError(
                f"transport must be 'nccl', 'p2p' or 'p2p_fused', got {transport!r}")
        if transport == "p2p_fused" and g > 8:
            raise ValueError("the fused P2P exchange supports BN groups of at most 8 ranks")
        self.transport = transport
        self._p2p = None
        if transport in ("p2p", "p2p_fused") and g > 1:
            if self._device.type != "cuda":
                raise ValueError("the p2p transport needs a CUDA device")
            gi = self.rank // g
            self._p2p = _P2PGroup(list(range(gi * g, (gi + 1) * g)), self.rank,
                                  self._groups[f"bn{gi}"], self._device, p2p_max_len,
                                  p2p_timeout_s)

    def __repr__(self):
        return f"DistHandle(rank={self.rank}, world={self.world_size}, g={self.bn_group_size})"

    @property
    def fused_exchange(self):
        """The fused P2P exchange of the BN group (transport "p2p_fused", G > 1), else
        None: the BN forward / backward then call the cgbn_*_p2p kernels instead of
        reduction -> exchange -> finalize. With validate=True the BN layers keep the
        unfused path, whose exchange() runs the protocol check."""
        if self.transport != "p2p_fused" or self._p2p is None or self.validate:
            return None
        return self._p2p

    @property
    def device(self) -> torch.device:
        return self._device

    def exchange(self, scope: str, kind: str, vec: torch.Tensor, info=None):
        import torch.distributed as dist
        scope_key, ranks = self._scope_info(scope)
        seq = self._next_seq(scope_key)
        pg = self._groups[scope_key]
        g = len(ranks)
        if self.validate:
            self._validate(pg, ranks, scope_key, seq, kind, vec)
        if g == 1:
            return [vec], None
        if (self._p2p is not None and scope == SCOPE_BN_GROUP and vec.is_cuda
                and vec.dtype == torch.float64 and vec.numel() <= self._p2p.max_len):
            return self._p2p.exchange(vec.contiguous()), None
        out = _all_gather_rows(vec, g, pg)
        return [out[i] for i in range(g)], None

    def close(self):
        """Release the P2P regions (collective-free; call on every rank)."""
        if self._p2p is not None:
            self._p2p.close()
            self._p2p = None

    def _validate(self, pg, ranks, scope_key, seq, kind, vec):
        """Optional host-side protocol check (one extra tiny all-gather): every rank
        must issue the same collective with the same payload length, as the reference
        diagnoses at its root (collectives.py:243-292)."""
        import torch.distributed as dist
        kind_id = sum(ord(ch) * (i + 1) for i, ch in enumerate(kind)) % (1 << 30)
        dt_id = {torch.float32: 0, torch.float64: 1}.get(vec.dtype, 2)
        meta = torch.tensor([seq, kind_id, vec.numel(), dt_id], dtype=torch.int64,
                            device=vec.device)
        allm = _all_gather_rows(meta, len(ranks), pg).cpu().tolist()
        if any(m[:2] != allm[0][:2] for m in allm):
            raise CollectiveProtocolError(
                f"collective mismatch in {scope_key}#{seq}: per-rank (seq, kind) = "
                + ", ".join(f"rank {r}: {tuple(m[:2])}" for r, m in zip(ranks, allm)))
        if any(m[2:] != allm[0][2:] for m in allm):
            raise CollectiveProtocolError(
                f"{kind}[{scope_key}#{seq}]: payload mismatch across ranks ("
                + ", ".join(f"rank {r}: len {m[2]}" for r, m in zip(ranks, allm)) + ")")


def _all_gather_rows(vec: torch.Tensor, g: int, pg) -> torch.Tensor:
    """(g, n) tensor whose row r is rank r's 1-D ``vec`` (NCHW: one NCCL all-gather into
    a contiguous buffer; gloo on CPU for the transport tests)."""
    import torch.distributed as dist
    vec = vec.contiguous()
    out = torch.empty((g, vec.numel()), dtype=vec.dtype, device=vec.device)
    if vec.is_cuda and dist.get_backend(pg) == "nccl":
        dist.all_gather_into_tensor(out.view(-1), vec, group=pg)
    elif vec.is_cuda:  # host-staged (gloo with CUDA tensors: tests, no NVLink path)
        host = torch.empty((g, vec.numel()), dtype=vec.dtype)
        dist.all_gather(list(host.unbind(0)), vec.cpu(), group=pg)
        out.copy_(host)
    else:
        dist.all_gather(list(out.unbind(0)), vec, group=pg)
    return out


# ------------------------------------------------------------------------------------
# allreduce_sum on device vectors


def _device_fold(rows, out) -> None:
    """out = rows[0] + rows[1] + ... in ascending order (cgbn_fold_sum, device)."""
    lib = _lib.load()
    arr, keep = _lib.ptr_array([p.data_ptr() for p in rows])
    dt = _lib.DTYPE_F64 if out.dtype == torch.float64 else _lib.DTYPE_F32
    _lib.check(lib.cgbn_fold_sum(arr, len(rows), out.numel(), dt, out.data_ptr(),
                                 torch.cuda.current_stream(out.device).cuda_stream),
               "cgbn_fold_sum")


# Vectors at least this long take the sharded path on torch.distributed handles.
SHARDED_MIN_ELEMS = 1 << 16


def _sharded_allreduce(v: torch.Tensor, g: int, pg, fold) -> torch.Tensor:
    """Ascending-rank allreduce of a long vector over torch.distributed, moving 2x the
    vector per rank instead of the all-gather's G x: an all-to-all delivers shard k of
    every rank to rank k (a reduce-scatter), rank k folds its shard's G rows in ascending
    rank order (`fold`, the device kernel in production), and an all-gather returns the
    folded shards. Every element is folded once, by its shard's owner, so the result is
    bitwise identical on every rank and equal to the full-vector fold."""
    import torch.distributed as dist
    n = v.numel()
    shard = -(-n // g)
    pad = shard * g - n
    src = torch.cat([v, v.new_zeros(pad)]) if pad else v
    recv = torch.empty(g * shard, dtype=v.dtype, device=v.device)
    dist.all_to_all_single(recv, src.contiguous(), group=pg)
    rows = list(recv.view(g, shard).unbind(0))  # row r = rank r's copy of my shard
    mine = torch.empty(shard, dtype=v.dtype, device=v.device)
    fold(rows, mine)
    out = torch.empty(g * shard, dtype=v.dtype, device=v.device)
    if v.is_cuda:
        dist.all_gather_into_tensor(out, mine, group=pg)
    else:
        dist.all_gather(list(out.view(g, shard).unbind(0)), mine, group=pg)
    return out[:n]


def allreduce_sum(handle: _HandleBase, scope: str, v) -> torch.Tensor:
    """Elementwise sum of every rank's 1-D device vector; all ranks receive the result.

    Accumulation runs in ascending rank order (collectives.py:260-298), so the result is
    bitwise identical on every rank and across runs. ``v`` must be a CUDA float32 or
    float64 tensor (no CPU fallback). On a torch.distributed handle, vectors of at least
    SHARDED_MIN_ELEMS elements use the sharded reduce-scatter / fold / all-gather path.
    """
    if not isinstance(v, torch.Tensor):
        raise CollectiveProtocolError(f"rank {handle.rank}: payload must be a torch.Tensor")
    if v.dim() != 1:
        raise CollectiveProtocolError(f"rank {handle.rank}: collective payload must be a 1-D vector")
    if not v.is_cuda:
        raise CollectiveProtocolError(
            f"rank {handle.rank}: allreduce_sum needs a CUDA tensor (there is no CPU path)")
    if v.dtype not in (torch.float32, torch.float64):
        raise CollectiveProtocolError(f"rank {handle.rank}: payload dtype {v.dtype} unsupported")
    v = v.contiguous()
    if isinstance(handle, DistHandle) and v.numel() >= SHARDED_MIN_ELEMS:
        scope_key, ranks = handle._scope_info(scope)
        seq = handle._next_seq(scope_key)
        if handle.validate:
            handle._validate(handle._groups[scope_key], ranks, scope_key, seq, "allreduce", v)
        if len(ranks) == 1:
            return v.clone()
        return _sharded_allreduce(v, len(ranks), handle._groups[scope_key], _device_fold)
    parts, _ = handle.exchange(scope, "allreduce", v)
    out = torch.empty_like(v)
    _device_fold(parts, out)
    return out


def world_mean_allreduce(handle: _HandleBase, grads: dict, loss=None):
    """The data-parallel gradient step of the reference trainer (trainer.py:419-428):
    concatenate the gradients in sorted-key order (plus the task loss), allreduce_sum at
    world scope (ascending-rank fold), divide by the world size and split back.

    ``grads`` maps names to CUDA tensors of one float dtype. Returns (mean grads dict,
    mean loss or None). Every rank receives bitwise-identical values."""
    keys = sorted(grads)
    if not keys:
        raise ValueError("world_mean_allreduce needs at least one gradient")
    # fold in fp64 if any gradient is fp64, else fp32 (bf16 / fp16 gradients are widened
    # for the sum and returned in their own dtype)
    dt = torch.float64 if any(grads[k].dtype == torch.float64 for k in keys) else torch.float32
    dev = grads[keys[0]].device
    flat = [grads[k].reshape(-1).to(dt) for k in keys]
    if loss is not None:
        flat.append(torch.as_tensor([float(loss)], dtype=dt, device=dev))
    mean = allreduce_sum(handle, SCOPE_WORLD, torch.cat(flat)) / handle.world_size
    out, off = {}, 0
    for k in keys:
        n = grads[k].numel()
        out[k] = mean[off:off + n].view(grads[k].shape).to(grads[k].dtype)
        off += n
    return out, (float(mean[-1].item()) if loss is not None else None)


class GradBuckets:
    """The world-gradient allreduce of the trainer (trainer.py:419-428), bucketed and
    overlapped with the backward.

    The reference concatenates every gradient after the backward and allreduces once.
    Here gradients are handed over as the backward produces them (``add``); when a bucket
    reaches ``bucket_bytes`` its allreduce is issued on a side CUDA stream, after an
    event on the producing stream, so the exchange and the ascending-rank fold run while
    the backward of the next layers keeps the compute stream busy. ``finish`` adds the
    loss to the last bucket, makes the caller's stream wait for the side stream and
    returns the mean gradients and loss.

    Numerics: every element is the ascending-rank fold of that element over the world
    (allreduce_sum), divided by the world size, so the bucketing changes nothing: the
    result is bitwise identical to world_mean_allreduce on the same gradients when
    ``dtype`` matches its choice (fp64 if any gradient is fp64, else fp32).

    ``reduce_fn(handle, scope, vec) -> vec`` defaults to allreduce_sum (CUDA tensors).
    """

    def __init__(self, handle, bucket_bytes: int = 16 << 20, dtype=torch.float32,
                 reduce_fn=None):
        self.handle = handle
        self.bucket_bytes = int(bucket_bytes)
        self.dtype = dtype
        self.reduce_fn = reduce_fn or allreduce_sum
        self._pending = []   # (name, tensor) of the open bucket
        self._pending_bytes = 0
        self._issued = []    # (names, shapes, dtypes, sizes, result, event)
        self._names = set()
        self._side = None
        self.buckets_issued = 0

    def _stream(self, dev):
        if dev.type != "cuda":
            return None
        if self._side is None:
            self._side = torch.cuda.Stream(device=dev)
        return self._side

    def add(self, name: str, grad: torch.Tensor) -> None:
        """Hand over one gradient (in the order the backward produces them)."""
        if name in self._names:
            raise ValueError(f"gradient {name!r} added twice")
        self._names.add(name)
        self._pending.append((name, grad))
        self._pending_bytes += grad.numel() * torch.finfo(self.dtype).bits // 8
        if self._pending_bytes >= self.bucket_bytes:
            self._issue()

    def _issue(self, loss=None):
        if not self._pending and loss is None:
            return
        items, self._pending, self._pending_bytes = self._pending, [], 0
        dev = items[0][1].device if items else torch.device(self.handle.device)
        side = self._stream(dev)
        flat_in = [g.reshape(-1) for _, g in items]
        if side is not None:
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(dev))
            side.wait_event(ready)
            ctx = torch.cuda.stream(side)
        else:
            ctx = _nullcontext()
        with ctx:
            parts = [t.to(self.dtype) for t in flat_in]
            if loss is not None:
                parts.append(torch.as_tensor([float(loss)], dtype=self.dtype, device=dev))
            summed = self.reduce_fn(self.handle, SCOPE_WORLD, torch.cat(parts))
            mean = summed / self.handle.world_size
            done = None
            if side is not None:
                for t in flat_in:
                    t.record_stream(side)
                done = torch.cuda.Event()
                done.record(side)
        self._issued.append(([n for n, _ in items], [g.shape for _, g in items],
                             [g.dtype for _, g in items], mean, done, loss is not None))
        self.buckets_issued += 1

    def finish(self, loss=None):
        """Issue the last bucket (with the loss), wait on the caller's stream, return
        ({name: mean gradient}, mean loss or None)."""
        self._issue(loss=loss)
        out, mloss = {}, None
        for names, shapes, dtypes, mean, done, has_loss in self._issued:
            if done is not None:
                torch.cuda.current_stream(mean.device).wait_event(done)
                mean.record_stream(torch.cuda.current_stream(mean.device))
            off = 0
            for n, shp, dt in zip(names, shapes, dtypes):
                k = 1
                for e in shp:
                    k *= e
                out[n] = mean[off:off + k].view(shp).to(dt)
                off += k
            if has_loss:
                mloss = float(mean[-1].item())
        self._issued, self._names = [], set()
        return out, mloss


class _nullcontext:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
