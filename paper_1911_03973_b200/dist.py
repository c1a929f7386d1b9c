"""Element-slab multi-GPU path: one process per GPU, NCCL over NVLink.

Partition: rank p owns the elements [lo, hi) of ``np.linspace(0, n_e, P+1)`` -- the
reference's own chunk rule (operators.py:100).  The generators order cells row-major
(2D) / z-outer (3D), so slabs are geometric and meet along one node row / plane.

Per rank: a plan over the slab's local nodes (sorted global ids), the SELL kernel
producing PARTIAL node sums, then a halo step: interface partials go to / come from the
slab neighbours (NCCL send/recv) and every shared node is summed in ascending rank order,
so all ranks hold the same value for it.  Dots and norms sum owned nodes (owner = lowest
rank touching the node) and are all-reduced.  Maps (local node sets, interfaces, owners)
match oracle/ebs_oracle.py halo_maps bit for bit.

The solver loops are written against two small protocols so the same code runs
  * distributed: one ``GpuRankOperator`` per process and ``PeerTransport`` (peer memory:
                 CUDA-IPC windows of the node's ranks, the halo pushed from the SELL sweep
                 epilogue and the PCG dot all-reduce fused into the combine / update kernels,
                 csrc/peer.cu -- the default of bench.py), ``TorchTransport`` (NCCL / gloo
                 through torch.distributed) or ``NativeTransport`` (libebs.so's own NCCL
                 communicator, ebs_dist_*);
  * emulated:    P ``GpuRankOperator``s in one process on one GPU, ``LocalPeerTransport``
                 (the peer kernels and windows, every put before any get) or
                 ``LocalTransport`` (device copies) -- nothing waits on anything;
  * CPU tests:   a torch-CPU rank operator (tests/) over gloo, world size 2.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from ._lib import EBS_APPLY_ADD, call, load


# ------------------------------------------------------------------------ maps --
def element_slabs(n_e: int, P: int) -> np.ndarray:
    """operators.py:100 chunk rule reused for ranks."""
    return np.linspace(0, n_e, P + 1, dtype=int)


def partition_maps(indt: torch.Tensor, n_nodes: int, P: int) -> dict:
    """Local node sets (sorted global ids), pairwise interfaces and owners for P slabs.

    Works on any torch device; identical to oracle.halo_maps (tests)."""
    bounds = element_slabs(indt.shape[1], P)
    local = [torch.unique(indt[:, lo:hi].reshape(-1).to(torch.int64))
             for lo, hi in zip(bounds[:-1], bounds[1:])]
    interface = []
    for p in range(P):
        row = {}
        for q in range(P):
            if q != p:
                common = local[p][torch.isin(local[p], local[q])]
                if common.numel():
                    row[q] = common
        interface.append(row)
    owner = torch.full((n_nodes,), -1, dtype=torch.int64, device=indt.device)
    for p in reversed(range(P)):
        owner[local[p]] = p
    return dict(bounds=bounds, local=local, interface=interface, owner=owner)


# ------------------------------------------------------------------ transports --
class TorchTransport:
    """torch.distributed (NCCL on GPUs, gloo on CPU): one rank per process.

    ``stage_host=True`` moves device buffers through host memory around each collective
    (gloo with GPU ranks -- used to run several GPU rank processes on one device in tests,
    where nothing may wait on another process's kernels)."""

    def __init__(self, group=None, stage_host: bool = False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.stage_host = stage_host

    def exchange_start(self, ops: list, sends: list):
        """Post the halo send/recv pairs (NCCL runs them on its own stream, after the work
        already queued on the current stream); returns a handle for exchange_finish."""
        (op,), (snd,) = ops, sends
        p2p = []
        recvs = {}
        dev = None
        for q in sorted(snd):
            buf = snd[q].contiguous()
            if self.stage_host and buf.is_cuda:
                dev = buf.device
                buf = buf.cpu()
            recvs[q] = torch.empty_like(buf)
            p2p.append(self.dist.P2POp(self.dist.isend, buf, q, self.group))
            p2p.append(self.dist.P2POp(self.dist.irecv, recvs[q], q, self.group))
        works = self.dist.batch_isend_irecv(p2p) if p2p else []
        return works, recvs, dev

    def exchange_finish(self, handle) -> list:
        works, recvs, dev = handle
        for w in works:
            w.wait()  # the current stream waits for the transfers
        if dev is not None:
            recvs = {q: t.to(dev) for q, t in recvs.items()}
        return [recvs]

    def exchange(self, ops: list, sends: list) -> list:
        """sends[i] = {q: tensor} for local rank ops[i] (len 1 here) -> recvs {q: tensor}."""
        return self.exchange_finish(self.exchange_start(ops, sends))

    def agree(self, ok: bool) -> bool:
        """True iff `ok` on every rank (an eager all-reduce MIN, outside any capture)."""
        if self.dist.get_world_size(self.group) == 1:
            return bool(ok)
        dev = "cpu" if (self.stage_host or self.dist.get_backend(self.group) == "gloo") else "cuda"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))

    def allreduce(self, tensors: list):
        (t,) = tensors
        if self.stage_host and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)


class NativeTransport:
    """The halo exchange and reductions through libebs.so's own NCCL communicator
    (ebs_dist_init / ebs_dist_exchange / ebs_dist_allreduce) -- the C-ABI path a caller
    without PyTorch uses.  One GPU rank operator per process; the NCCL unique id travels
    through torch.distributed's store here (any rendezvous works)."""

    def __init__(self, op, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.op = op
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            call("ebs_dist_unique_id", uid)
        if world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        call("ebs_dist_init", op.plan.handle, uid, rank, world)
        self.world = world

    def exchange_start(self, ops: list, sends: list):
        (op,), (snd,) = ops, sends
        peers = sorted(snd)
        bufs = [snd[q].contiguous() for q in peers]
        recvs = {q: torch.empty_like(b) for q, b in zip(peers, bufs)}
        n = len(peers)
        if n:
            P = (ctypes.c_int32 * n)(*peers)
            C = (ctypes.c_int64 * n)(*[b.numel() for b in bufs])
            Sp = (ctypes.c_void_p * n)(*[b.data_ptr() for b in bufs])
            Rp = (ctypes.c_void_p * n)(*[recvs[q].data_ptr() for q in peers])
            call("ebs_dist_exchange", op.plan.handle, n, P, C, Sp, Rp, D.stream())
        return bufs, recvs  # keep the send buffers alive until the stream has used them

    def exchange_finish(self, handle) -> list:
        return [handle[1]]  # stream-ordered: later work on this stream sees the data

    def exchange(self, ops: list, sends: list) -> list:
        return self.exchange_finish(self.exchange_start(ops, sends))

    def allreduce(self, tensors: list):
        (t,) = tensors
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("NativeTransport reduces contiguous float64 device tensors")
        call("ebs_dist_allreduce", self.op.plan.handle, D.ptr(t), t.numel(), D.stream())

    def agree(self, ok: bool) -> bool:
        t = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device="cuda")
        self.allreduce([t])
        self.sync()
        return int(t.item()) == self.world

    def sync(self, timeout: float | None = None):
        """Wait for the current stream while polling NCCL for asynchronous errors; a lost
        peer or a stream still busy after `timeout` s (default EBS_NCCL_TIMEOUT, 600)
        aborts the communicator and raises (ebs_dist_wait) instead of hanging."""
        import os
        if timeout is None:
            timeout = float(os.environ.get("EBS_NCCL_TIMEOUT", "600"))
        call("ebs_dist_wait", self.op.plan.handle, D.stream(), ctypes.c_double(timeout))

    def poll(self):
        call("ebs_dist_poll", self.op.plan.handle)

    def abort(self):
        call("ebs_dist_abort", self.op.plan.handle)


class LocalTransport:
    """All P ranks in this process (one GPU): the exchange is a device copy."""

    def exchange_start(self, ops: list, sends: list):
        return self.exchange(ops, sends)

    def exchange_finish(self, handle) -> list:
        return handle

    def exchange(self, ops: list, sends: list) -> list:
        ranks = {op.rank: i for i, op in enumerate(ops)}
        recvs = [dict() for _ in ops]
        for i, op in enumerate(ops):
            for q, buf in sends[i].items():
                recvs[ranks[q]][op.rank] = buf.clone()
        return recvs

    def agree(self, ok: bool) -> bool:
        return bool(ok)

    def allreduce(self, tensors: list):
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        for t in tensors:
            t.copy_(total)


def _peer_timeout() -> float:
    import os
    return float(os.environ.get("EBS_PEER_TIMEOUT", "600"))


class _PeerBase:
    """Halo exchange and dot all-reduce over peer memory (csrc/peer.cu): no collective
    library on the data path.  The solver loops use the fused form (fused_peer): the slab
    sweep pushes the interface partials into the neighbours' windows from its epilogue and
    the combine kernel waits for them -- 2 launches per Jacobi iteration.  Subclasses hold
    the ops' native peer views (op.peer) and say how the put and get phases are ordered."""

    fused_peer = True
    serialize = False

    def after_put(self):
        """Between the put phase of every local rank and the first get (serialize: host
        barrier, for several rank processes sharing one GPU in tests)."""

    def exchange_start(self, ops: list, sends: list):
        keep = []
        for op, snd in zip(ops, sends):
            nbs = sorted(snd)
            if nbs != sorted(op.if_idx):
                raise ValueError("peer exchange: sends must cover exactly the slab neighbours")
            bufs = [snd[q].contiguous() for q in nbs]
            keep.append(bufs)
            arr = (ctypes.c_void_p * max(len(bufs), 1))(*[b.data_ptr() for b in bufs])
            call("ebs_peer_send", op.peer, arr, D.stream())
        self.after_put()
        return keep

    def exchange_finish(self, handle) -> list:
        out = []
        for op in self._ops:
            nbs = sorted(op.if_idx)
            recvs = {q: D.empty(op.if_idx[q].numel()) for q in nbs}
            arr = (ctypes.c_void_p * max(len(nbs), 1))(*[recvs[q].data_ptr() for q in nbs])
            call("ebs_peer_recv", op.peer, arr, D.ptr(op._ws), D.stream())
            out.append(recvs)
        return out

    def exchange(self, ops: list, sends: list) -> list:
        return self.exchange_finish(self.exchange_start(ops, sends))

    def halo(self, ops: list, vs: list):
        """v[shared] = rank-ordered sum of the partials: push + combine, 2 launches."""
        for op, v in zip(ops, vs):
            op.peer_push(v)
        self.after_put()
        for op, v in zip(ops, vs):
            op.peer_combine(v)

    def allreduce_get(self, tensors: list):
        """The get phase alone (mode 2) of an all-reduce whose put phase already ran (the
        put of peer_combine_q with dots): tensors[i] (<= 256 values) := the rank-ordered sum."""
        for op, t in zip(self._ops, tensors):
            self._check(t)
            call("ebs_peer_allreduce", op.peer, D.ptr(t), t.numel(), 2, D.stream())

    def _check(self, t):
        if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("peer all-reduce takes contiguous float64 device tensors")

    def status(self):
        """Raise (EBS_ENCCL) when a wait of a local rank timed out; synchronises."""
        for op in self._ops:
            call("ebs_peer_status", op.peer, D.stream())

    def sync(self, timeout=None):
        self.status()


class PeerUnavailable(RuntimeError):
    """Raised on EVERY rank (a collective decision) when some rank cannot map the others'
    windows (no CUDA IPC / peer access between the node's GPUs): fall back to NCCL."""


class PeerTransport(_PeerBase):
    """One rank per process, the node's ranks mapping each other's windows through CUDA IPC
    (NVLink P2P stores between GPUs; the handles travel through torch.distributed's object
    collectives -- host plumbing only).  Waits time out after `timeout` s (EBS_PEER_TIMEOUT,
    600) and report EBS_ENCCL instead of hanging.  serialize=True (tests: several rank
    processes on ONE GPU): a host barrier after every put phase, so no kernel ever waits on
    another process's kernels, and no CUDA graphs."""

    def __init__(self, op, group=None, timeout: float | None = None, serialize: bool = False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.serialize = serialize
        self._ops = [op]
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world > 8:
            raise ValueError("PeerTransport spans at most 8 ranks (one NVSwitch node)")
        if rank != op.rank:
            raise ValueError(f"process rank {rank} runs slab {op.rank}")
        cap = max([t.numel() for t in op.if_idx.values()] + [1])
        if world > 1:
            caps = [None] * world
            dist.all_gather_object(caps, cap, group=group)
            cap = max(caps)
        self.world, self.rank, self.cap = world, rank, cap
        own = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        try:
            call("ebs_peer_window_alloc", cap, ctypes.byref(own), handle)
            mine = bytes(handle.raw)
        except Exception as e:  # noqa: BLE001 -- decided collectively below
            own, mine = None, f"{type(e).__name__}: {e}"
        self._own = own
        handles = [mine]
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, mine, group=group)
        bad = next((f"rank {q}: {h}" for q, h in enumerate(handles) if isinstance(h, str)), None)
        if bad is not None:  # some rank has no window: every rank gives up together
            if own is not None:
                call("ebs_peer_window_free", own)
            raise PeerUnavailable(f"peer window allocation failed ({bad})")
        self._opened = []
        wins = []
        err = None
        try:
            for q in range(world):
                if q == rank:
                    wins.append(own.value)
                    continue
                w = ctypes.c_void_p()
                call("ebs_peer_window_open", ctypes.create_string_buffer(handles[q], 64),
                     ctypes.byref(w))
                self._opened.append(w)
                wins.append(w.value)
        except Exception as e:  # noqa: BLE001 -- decided collectively below
            err = f"{type(e).__name__}: {e}"
        if world > 1:  # every rank mapped every window, or all of them give up together
            errs = [None] * world
            dist.all_gather_object(errs, err, group=group)
            err = next((f"rank {q}: {e}" for q, e in enumerate(errs) if e), None)
        if err is not None:
            for w in self._opened:
                call("ebs_peer_window_close", w)
            call("ebs_peer_window_free", own)
            raise PeerUnavailable(f"peer windows cannot be mapped ({err})")
        arr = (ctypes.c_void_p * world)(*wins)
        peer = ctypes.c_void_p()
        t = _peer_timeout() if timeout is None else float(timeout)
        call("ebs_peer_create", rank, world, cap, arr, ctypes.c_double(t), ctypes.byref(peer))
        self.peer = peer
        op.peer_attach(peer)
        if world > 1:  # every window is mapped before anyone writes into it
            torch.cuda.synchronize()
            dist.barrier(group=group)

    def after_put(self):
        if self.serialize and self.world > 1:
            torch.cuda.synchronize()
            self.dist.barrier(group=self.group)

    def sync(self, timeout=None):
        """status() decided collectively: every rank raises when any rank's wait timed out,
        so no rank is left alone in the next collective."""
        err = None
        try:
            self.status()
        except Exception as e:  # noqa: BLE001
            err = str(e)
        if self.world > 1:
            errs = [None] * self.world
            self.dist.all_gather_object(errs, err, group=self.group)
            err = next((f"rank {q}: {e}" for q, e in enumerate(errs) if e), None)
        if err is not None:
            from ._lib import EbsError
            raise EbsError(err)

    def allreduce(self, tensors: list):
        (t,) = tensors
        self._check(t)
        (op,) = self._ops
        if not self.serialize:
            call("ebs_peer_allreduce", op.peer, D.ptr(t), t.numel(), 0, D.stream())
            return
        for a in range(0, t.numel(), 256):
            piece = t[a:a + 256]
            call("ebs_peer_allreduce", op.peer, D.ptr(piece), piece.numel(), 1, D.stream())
            self.after_put()
            call("ebs_peer_allreduce", op.peer, D.ptr(piece), piece.numel(), 2, D.stream())

    def agree(self, ok: bool) -> bool:
        if self.world == 1:
            return bool(ok)
        box = [None] * self.world
        self.dist.all_gather_object(box, bool(ok), group=self.group)
        return all(box)

    def close(self):
        """Release the window mappings (collective: every rank calls it)."""
        if getattr(self, "peer", None) is None:
            return
        torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier(group=self.group)
        call("ebs_peer_destroy", self.peer)
        for w in self._opened:
            call("ebs_peer_window_close", w)
        call("ebs_peer_window_free", self._own)
        self.peer = None
        self._ops[0].peer = None


class LocalPeerTransport(_PeerBase):
    """All P ranks in this process on one GPU (emulation, tests): the same windows, kernels
    and layout as PeerTransport, windows addressed directly; every put phase of all ranks is
    enqueued before any get, so nothing waits."""

    def __init__(self, ops, timeout: float | None = None):
        if len(ops) > 8:
            raise ValueError("peer groups span at most 8 ranks")
        self._ops = list(ops)
        P = len(ops)
        cap = max([t.numel() for op in ops for t in op.if_idx.values()] + [1])
        self.cap = cap
        self._wins = []
        for _ in range(P):
            w = ctypes.c_void_p()
            call("ebs_peer_window_alloc", cap, ctypes.byref(w), None)
            self._wins.append(w)
        arr = (ctypes.c_void_p * P)(*[w.value for w in self._wins])
        t = _peer_timeout() if timeout is None else float(timeout)
        self.peers = []
        for op in ops:
            peer = ctypes.c_void_p()
            call("ebs_peer_create", op.rank, P, cap, arr, ctypes.c_double(t), ctypes.byref(peer))
            self.peers.append(peer)
            op.peer_attach(peer)

    def selftest(self, iters: int = 200) -> int:
        """The peer protocol under real concurrency (ebs_peer_selftest): one cooperative
        kernel whose block groups act as these ranks on their real windows and halo maps,
        skewed; returns the number of wrong values (0)."""
        P = len(self._ops)
        peers = (ctypes.c_void_p * P)(*[op.peer.value for op in self._ops])
        gids = (ctypes.c_void_p * P)(*[op.global_of_int.data_ptr() for op in self._ops])
        n = ctypes.c_int64(-1)
        call("ebs_peer_selftest", peers, gids, P, int(iters), ctypes.byref(n), D.stream())
        return int(n.value)

    def allreduce(self, tensors: list):
        if len(tensors) != len(self._ops):
            raise ValueError(f"emulated all-reduce takes one tensor per rank ({len(self._ops)}), "
                             f"got {len(tensors)}")
        for t in tensors:
            self._check(t)
        n = tensors[0].numel()
        for a in range(0, n, 256):
            pieces = [t[a:a + 256] for t in tensors]
            for op, p in zip(self._ops, pieces):
                call("ebs_peer_allreduce", op.peer, D.ptr(p), p.numel(), 1, D.stream())
            for op, p in zip(self._ops, pieces):
                call("ebs_peer_allreduce", op.peer, D.ptr(p), p.numel(), 2, D.stream())

    def agree(self, ok: bool) -> bool:
        return bool(ok)

    def close(self):
        if not self.peers:
            return
        torch.cuda.synchronize()
        for op, p in zip(self._ops, self.peers):
            call("ebs_peer_destroy", p)
            op.peer = None
        for w in self._wins:
            call("ebs_peer_window_free", w)
        self.peers = []


# ---------------------------------------------------------------- rank operator --
def rank_operator(mesh, nu: float, f, d, P: int, rank: int, maps: dict | None = None):
    """Rank `rank` of P: partition maps of the mesh and a GpuRankOperator whose element
    matrices are assembled for this rank's slab only (memory and setup scale as 1/P)."""
    from .elements import build_element_batch
    from .mesh import Mesh
    if maps is None:
        maps = partition_maps(mesh.conn, mesh.n_nodes, P)
    lo, hi = int(maps["bounds"][rank]), int(maps["bounds"][rank + 1])
    slab = Mesh(mesh.nodes, None, mesh.boundary_nodes, conn=mesh.conn[:, lo:hi].contiguous())
    batch = build_element_batch(slab, nu=nu, f=f)
    object.__setattr__(batch.index, "n_nodes", mesh.n_nodes)
    return GpuRankOperator(batch, mesh.n_nodes, d, maps, rank, slab=True), maps



class GpuRankOperator:
    """Rank p's slab of a global ElementBatch on the current CUDA device.

    Vectors are in this rank's plan-internal numbering ("internal")."""

    def __init__(self, batch, n_nodes: int, d, maps: dict, p: int, slab: bool = False):
        """`batch` is the global ElementBatch, or (slab=True) a batch holding only this
        rank's elements [lo, hi) (see rank_operator), in the global node numbering."""
        from .elements import ElementBatch
        from .mesh import IndexArrays
        from .operators import DirichletData
        self.rank = p
        self.P = len(maps["local"])
        lo, hi = int(maps["bounds"][p]), int(maps["bounds"][p + 1])
        if slab:
            if batch.n_elements != hi - lo:
                raise ValueError("slab batch does not match the partition bounds")
            lo, hi = 0, hi - lo
        gl = maps["local"][p].to(D.device())
        self.global_ids = gl
        n = gl.numel()
        self.n = n
        indt = batch.index.indt
        conn = torch.searchsorted(gl, indt[:, lo:hi].to(torch.int64)).to(torch.int32).contiguous()
        self._conn_local = conn
        A_store = batch._A_store()[lo:hi]
        b_e = batch.b_e[:, lo:hi].contiguous()
        self.batch = ElementBatch(K_e=A_store.permute(1, 2, 0), M_e=A_store.permute(1, 2, 0),
                                  A_e=A_store.permute(1, 2, 0), b_e=b_e, nu=batch.nu,
                                  index=IndexArrays(None, conn, n_nodes=n))
        self.plan = self.batch.operator(n)
        # Dirichlet nodes of this slab (local ids)
        if d is not None and d.nd.numel():
            nd = d.nd.to(gl.device)
            mine = nd[torch.isin(nd, gl)]
            self.d_local = DirichletData(torch.searchsorted(gl, mine),
                                         torch.zeros(mine.numel(), dtype=torch.float64,
                                                     device=gl.device))
        else:
            self.d_local = None
        self.plan.ensure_dirichlet(self.d_local)
        new_of_old, old_of_new = self.plan.node_maps()
        self.new_of_old = new_of_old.to(torch.int64)
        self.old_of_new = old_of_new.to(torch.int64)
        self.global_of_int = gl[self.old_of_new]
        self.if_idx = {q: self.new_of_old[torch.searchsorted(gl, ids.to(gl.device))].contiguous()
                       for q, ids in maps["interface"][p].items()}
        self.all_if = (torch.unique(torch.cat(list(self.if_idx.values())))
                       if self.if_idx else torch.empty(0, dtype=torch.int64, device=gl.device))
        # one gather for all neighbours' send buffers; one kernel for the shared-node sums:
        # sources in ascending rank order (own partials = the nodes themselves)
        peers = sorted(self.if_idx)
        self.send_idx = (torch.cat([self.if_idx[q] for q in peers]).contiguous() if peers
                         else torch.empty(0, dtype=torch.int64, device=gl.device))
        offs = np.cumsum([0] + [self.if_idx[q].numel() for q in peers])
        self.send_slices = {q: (int(offs[k]), int(offs[k + 1])) for k, q in enumerate(peers)}
        self.combine_ranks = sorted(set(peers) | {p})
        cols = []
        for r in self.combine_ranks:
            if r == p:
                cols.append(self.all_if.to(torch.int32))
            else:
                col = torch.full((self.all_if.numel(),), -1, dtype=torch.int32, device=gl.device)
                col[torch.searchsorted(self.all_if, self.if_idx[r])] = torch.arange(
                    self.if_idx[r].numel(), dtype=torch.int32, device=gl.device)
                cols.append(col)
        self.combine_pos = (torch.stack(cols, 1).contiguous() if self.all_if.numel()
                            else torch.empty(0, dtype=torch.int32, device=gl.device))
        owner = maps["owner"].to(gl.device)
        self.owned = (owner[self.global_of_int] == p).to(torch.uint8).contiguous()
        self.free = D.empty(n, torch.uint8)
        call("ebs_plan_free_mask", self.plan.handle, D.ptr(self.free), D.stream())
        # interface flags and the chunk split (interface chunks are swept first so the
        # halo exchange overlaps the interior sweep)
        self.iface = torch.zeros(n, dtype=torch.uint8, device=gl.device)
        if self.all_if.numel():
            self.iface[self.all_if] = 1
        n_chunks = (n + 31) // 32
        has_if = torch.zeros(n_chunks, dtype=torch.bool, device=gl.device)
        if self.all_if.numel():
            has_if[self.all_if // 32] = True
        self.if_chunks = torch.nonzero(has_if).reshape(-1).to(torch.int32).contiguous()
        self.in_chunks = torch.nonzero(~has_if).reshape(-1).to(torch.int32).contiguous()
        m_own = self.owned.bool()
        self.owned_int = torch.nonzero(m_own).reshape(-1)
        self.owned_glob = self.global_of_int[self.owned_int].contiguous()
        self.global_of_int32 = self.global_of_int.to(torch.int32).contiguous()
        # per neighbour: positions in the interface list whose node this rank owns, and
        # their global ids (the fused caller-numbering residual corrects only those)
        self.corr = {}
        self.corr_local = {}
        for q, idx in self.if_idx.items():
            pos = torch.nonzero(m_own[idx]).reshape(-1).contiguous()
            self.corr[q] = (pos, self.global_of_int[idx[pos]].contiguous())
            self.corr_local[q] = (pos, self.old_of_new[idx[pos]].contiguous())
        # the slab's own caller order = its local nodes in ascending global id (the plan's
        # caller numbering): old_of_new as the int32 output map of the SELL pass
        self.old_of_new32 = self.old_of_new.to(torch.int32).contiguous()
        self.owned_local = self.old_of_new[self.owned_int].contiguous()
        self._ws = D.zeros(int(load().ebs_vec_workspace_bytes()), torch.uint8)
        self._acc = D.zeros(n)
        self._flag = D.zeros(1, torch.int32)
        self._stop = None   # device stop flag of a single-reduction PCG (set_stop)
        self.peer = None    # native peer group view (peer_attach)

    # ---- primitives used by the generic loops ----
    def to_internal(self, x_global: torch.Tensor) -> torch.Tensor:
        return x_global.to(D.device())[self.global_of_int].contiguous()

    def scatter_owned(self, v_int: torch.Tensor, out_global: torch.Tensor):
        call("ebs_index_move", self.owned_int.numel(), D.ptr(self.owned_int), D.ptr(v_int),
             D.ptr(self.owned_glob), D.ptr(out_global), D.stream())

    def residual_caller_partial(self, x_int, r_global, s_raw):
        """r_global[g] = b_p - s_p, the slab's partial residual of every node (caller
        numbering), and the same partials in internal order (s_raw) in one SELL pass."""
        call("ebs_plan_apply_map", self.plan.handle, 1, D.ptr(x_int), D.ptr(r_global),
             D.ptr(self.global_of_int32), D.ptr(s_raw), 0, D.stream())

    def residual_caller_sweep(self, chunks, x_int, r_global, s_raw):
        """residual_caller_partial over the SELL chunks in `chunks` only."""
        call("ebs_plan_apply_map_chunks", self.plan.handle, 1, D.ptr(chunks), chunks.numel(),
             D.ptr(x_int), D.ptr(r_global), D.ptr(self.global_of_int32), D.ptr(s_raw), 0,
             D.stream())

    def residual_local_sweep(self, chunks, x_int, r_local, s_raw):
        """Partial residual b_p - s_p of the chunks in `chunks`, ADDED into r_local (the
        slab's nodes in ascending global id, pre-filled with -0.0: bit-identical to a
        store, cheaper for the scattered map) and stored in internal order in s_raw."""
        call("ebs_plan_apply_map_chunks", self.plan.handle, 1, D.ptr(chunks), chunks.numel(),
             D.ptr(x_int), D.ptr(r_local), D.ptr(self.old_of_new32), D.ptr(s_raw),
             EBS_APPLY_ADD, D.stream())

    def correct_owned_local(self, r_local, recvs: dict):
        """Owned interface entries of r_local: add the neighbours' partial residuals."""
        for q in sorted(recvs):
            pos, loc = self.corr_local[q]
            call("ebs_index_add", pos.numel(), D.ptr(pos), D.ptr(recvs[q]), D.ptr(loc),
                 D.ptr(r_local), D.stream())

    def correct_owned(self, r_global, recvs: dict):
        """Owned interface entries: add the neighbours' partial residuals."""
        for q in sorted(recvs):
            pos, glob = self.corr[q]
            call("ebs_index_add", pos.numel(), D.ptr(pos), D.ptr(recvs[q]), D.ptr(glob),
                 D.ptr(r_global), D.stream())

    def gather_global(self, x_global: torch.Tensor, out_int: torch.Tensor):
        """out_int[m] = x_global[global id of internal node m] (caller -> rank numbering)."""
        call("ebs_gather", self.n, D.ptr(self.global_of_int), D.ptr(x_global), D.ptr(out_int),
             D.stream())

    def matvec_partial(self, x: torch.Tensor, out: torch.Tensor):
        call("ebs_plan_apply", self.plan.handle, 0, D.ptr(x), D.ptr(out), 0, 0, D.stream())

    def rhs_partial(self) -> torch.Tensor:
        b = D.empty(self.n)
        call("ebs_plan_internal_rhs", self.plan.handle, D.ptr(b), D.stream())
        return b

    def diag_partial(self) -> torch.Tensor:
        dg = D.empty(self.n)
        call("ebs_plan_internal_diag", self.plan.handle, D.ptr(dg), D.stream())
        return dg

    def gather(self, idx, v):
        buf = D.empty(idx.numel())
        call("ebs_gather", idx.numel(), D.ptr(idx), D.ptr(v), D.ptr(buf), D.stream())
        return buf

    def gather_sends(self, v: torch.Tensor) -> dict:
        """{neighbour: v at the interface nodes shared with it}: one gather, views of it."""
        if not self.if_idx:
            return {}
        buf = self.gather(self.send_idx, v)
        return {q: buf[a:b] for q, (a, b) in self.send_slices.items()}

    def combine(self, v: torch.Tensor, recvs: dict):
        """v[shared] = sum over touching ranks in ascending rank order (own partial at p),
        one kernel (ebs_dist_combine)."""
        if not self.if_idx:
            return
        if len(self.combine_ranks) > 8:  # more sources than the fused kernel takes
            s = D.stream()
            acc = self._acc
            call("ebs_index_fill", self.all_if.numel(), D.ptr(self.all_if), 0.0, D.ptr(acc), s)
            own = self.gather(self.all_if, v)
            for r in self.combine_ranks:
                idx, src = (self.all_if, own) if r == self.rank else (self.if_idx[r], recvs[r])
                call("ebs_scatter_add", idx.numel(), D.ptr(idx), D.ptr(src), D.ptr(acc), s)
            call("ebs_index_copy", self.all_if.numel(), D.ptr(self.all_if), D.ptr(acc), D.ptr(v),
                 s)
            return
        srcs = [v if r == self.rank else recvs[r] for r in self.combine_ranks]
        ptrs = (ctypes.c_void_p * len(srcs))(*[t.data_ptr() for t in srcs])
        call("ebs_dist_combine", self.all_if.numel(), D.ptr(self.all_if), len(srcs), ptrs,
             D.ptr(self.combine_pos), D.ptr(v), D.stream())

    def _combine_srcs(self, v, recvs):
        srcs = [v if r == self.rank else recvs[r] for r in self.combine_ranks]
        return len(srcs), (ctypes.c_void_p * len(srcs))(*[t.data_ptr() for t in srcs])

    def combine_jacobi(self, recvs, omega, b, s_part, dinv, x, x_out, red, prior=None):
        """combine + jacobi_iface in one launch (ebs_dist_combine_jacobi)."""
        if self.if_idx and len(self.combine_ranks) > 8:
            self.combine(s_part, recvs)
            return self.jacobi_iface(omega, b, s_part, dinv, x, x_out, red, prior=prior)
        n_src, ptrs = self._combine_srcs(s_part, recvs)
        call("ebs_dist_combine_jacobi", self.all_if.numel(), D.ptr(self.all_if), n_src, ptrs,
             D.ptr(self.combine_pos), D.ptr(s_part), float(omega), D.ptr(b), D.ptr(dinv),
             D.ptr(self.free), D.ptr(self.owned), D.ptr(x), D.ptr(x_out), D.ptr(prior),
             D.ptr(red), D.ptr(self._ws), D.stream())

    def combine_q(self, recvs, p, q, red, prior=None):
        """combine + q_iface in one launch (ebs_dist_combine_q)."""
        if self.if_idx and len(self.combine_ranks) > 8:
            self.combine(q, recvs)
            return self.q_iface(p, q, red, prior=prior)
        n_src, ptrs = self._combine_srcs(q, recvs)
        call("ebs_dist_combine_q", self.all_if.numel(), D.ptr(self.all_if), n_src, ptrs,
             D.ptr(self.combine_pos), D.ptr(q), D.ptr(self.free), D.ptr(self.owned), D.ptr(p),
             D.ptr(prior), D.ptr(red), D.ptr(self._ws), D.stream())

    def jacobi_sweep(self, chunks, omega, x, x_out, b, dinv, s_part, red):
        call("ebs_dist_jacobi_sweep", self.plan.handle, D.ptr(chunks), chunks.numel(),
             float(omega), D.ptr(x), D.ptr(x_out), D.ptr(b), D.ptr(dinv), D.ptr(self.iface),
             D.ptr(s_part), D.ptr(red), D.ptr(self._ws), D.stream())

    def jacobi_iface(self, omega, b, s_part, dinv, x, x_out, red, prior=None):
        call("ebs_dist_jacobi_iface", self.all_if.numel(), D.ptr(self.all_if), float(omega),
             D.ptr(b), D.ptr(s_part), D.ptr(dinv), D.ptr(self.free), D.ptr(self.owned), D.ptr(x),
             D.ptr(x_out), D.ptr(prior), D.ptr(red), D.ptr(self._ws), D.stream())

    def matvec_sweep(self, chunks, p, q, red):
        call("ebs_dist_matvec_sweep", self.plan.handle, D.ptr(chunks), chunks.numel(), D.ptr(p),
             D.ptr(q), D.ptr(self.iface), D.ptr(red), D.ptr(self._ws), D.stream())

    def q_iface(self, p, q, red, prior=None):
        call("ebs_dist_q_iface", self.all_if.numel(), D.ptr(self.all_if), D.ptr(self.free),
             D.ptr(self.owned), D.ptr(p), D.ptr(q), D.ptr(prior), D.ptr(red), D.ptr(self._ws),
             D.stream())

    def vec_dinv(self, diag):
        dinv = D.empty(self.n)
        call("ebs_vec_dinv", self.n, D.ptr(diag), D.ptr(self.free), D.ptr(dinv), D.stream())
        return dinv

    def vec_jacobi(self, omega, b, s_, dinv, x, x_out, r_out, red):
        call("ebs_vec_jacobi", self.n, float(omega), D.ptr(b), D.ptr(s_), D.ptr(dinv),
             D.ptr(self.free), D.ptr(self.owned), D.ptr(x), D.ptr(x_out), D.ptr(r_out),
             D.ptr(red), D.ptr(self._flag), D.ptr(self._ws), D.stream())

    def vec_pcg_q(self, p, q, red):
        call("ebs_vec_pcg_q", self.n, D.ptr(self.free), D.ptr(self.owned), D.ptr(p), D.ptr(q),
             D.ptr(red), D.ptr(self._ws), D.stream())

    def vec_pcg_update(self, rz, pq, dinv, x, r, p, q, red):
        call("ebs_vec_pcg_update", self.n, D.ptr(rz), D.ptr(pq), D.ptr(self.owned), D.ptr(dinv),
             D.ptr(x), D.ptr(r), D.ptr(p), D.ptr(q), D.ptr(red), D.ptr(self._flag),
             D.ptr(self._ws), D.stream())

    def vec_pcg_direction(self, rz_old, rz_new, dinv, r, p):
        call("ebs_vec_pcg_direction", self.n, D.ptr(rz_old), D.ptr(rz_new), D.ptr(dinv), D.ptr(r),
             D.ptr(p), D.stream())

    def vec_cg1_update(self, cur, prev, rr0, tol, ctl, dinv, x, r, u, w, p, s_, nxt):
        call("ebs_vec_cg1_update", self.n, D.ptr(cur), D.ptr(prev), D.ptr(rr0), float(tol),
             D.ptr(ctl), D.ptr(self.owned), D.ptr(dinv), D.ptr(x), D.ptr(r), D.ptr(u), D.ptr(w),
             D.ptr(p), D.ptr(s_), D.ptr(nxt), D.ptr(self._flag), D.ptr(self._ws), D.stream())

    def set_stop(self, ctl):
        """Fused matvec sweeps of this rank's plan no-op while ctl[0] != 0 (None clears)."""
        call("ebs_dist_set_stop", self.plan.handle, D.ptr(ctl))
        self._stop = ctl

    # ---- peer-memory halo (PeerTransport / LocalPeerTransport; csrc/peer.cu) ----
    def peer_attach(self, peer):
        """Bind this rank's halo to a native peer group view (ebs_peer_set_halo): the
        neighbours' slots hold the interface nodes in ascending global id (if_idx order)."""
        self.peer = peer
        nbs = sorted(self.if_idx)
        n = len(nbs)
        ranks = (ctypes.c_int32 * max(n, 1))(*nbs)
        lens = (ctypes.c_int64 * max(n, 1))(*[self.if_idx[q].numel() for q in nbs])
        idx = (ctypes.c_void_p * max(n, 1))(*[self.if_idx[q].data_ptr() for q in nbs])
        call("ebs_peer_set_halo", peer, self.n, n, ranks, lens, idx, D.stream())
        # the chunk list of the fused peer sweeps: interface chunks first, then the interior,
        # then the chunks with a node sharing an element with a shared node ("near": they
        # read shared-node values, so ebs_peer_jacobi_step sweeps them last)
        near = torch.zeros((self.n + 31) // 32, dtype=torch.bool, device=self.iface.device)
        if self.all_if.numel():
            ci = self.new_of_old[self._conn_local.to(torch.int64)]      # (nb, n_e) internal
            touch = self.iface[ci].bool().any(dim=0)
            near[torch.unique(ci[:, touch]) // 32] = True
        near[self.if_chunks.to(torch.int64)] = False
        deep = self.in_chunks[~near[self.in_chunks.to(torch.int64)]]
        nearc = self.in_chunks[near[self.in_chunks.to(torch.int64)]]
        self.peer_chunks = torch.cat([self.if_chunks, deep, nearc]).contiguous()
        self.n_near = int(nearc.numel())
        self._stop = getattr(self, "_stop", None)

    def peer_jacobi_sweep(self, omega, x, x_out, b, dinv, s_part, red):
        c = self.peer_chunks
        call("ebs_peer_jacobi_sweep", self.plan.handle, self.peer, D.ptr(c), c.numel(),
             self.if_chunks.numel(), float(omega), D.ptr(x), D.ptr(x_out), D.ptr(b), D.ptr(dinv),
             D.ptr(self.iface), D.ptr(s_part), D.ptr(red), D.ptr(self._ws), D.stream())

    def peer_matvec_sweep(self, p, q, red):
        c = self.peer_chunks
        call("ebs_peer_matvec_sweep", self.plan.handle, self.peer, D.ptr(c), c.numel(),
             self.if_chunks.numel(), D.ptr(p), D.ptr(q), D.ptr(self.iface), D.ptr(red),
             D.ptr(self._ws), D.stream())

    def peer_jacobi_step(self, omega, x_prev, x_cur, x_out, b, dinv, s_part, prior, red_prev,
                         part_out):
        """Iteration k >= 1 in one launch: iteration k-1's shared nodes completed (x_cur there,
        red_prev) by the first warps while the interior chunks of iteration k are swept
        (ebs_peer_jacobi_step)."""
        c = self.peer_chunks
        call("ebs_peer_jacobi_step", self.plan.handle, self.peer, D.ptr(c), c.numel(),
             self.if_chunks.numel(), self.n_near, float(omega), D.ptr(x_prev), D.ptr(x_cur),
             D.ptr(x_out), D.ptr(b), D.ptr(dinv), D.ptr(self.iface), D.ptr(self.owned),
             D.ptr(s_part), D.ptr(prior), D.ptr(red_prev), D.ptr(part_out), D.ptr(self._ws),
             D.stream())

    def peer_combine_jacobi(self, omega, b, s_part, dinv, x, x_out, red, prior=None):
        call("ebs_peer_combine_jacobi", self.peer, D.ptr(s_part), float(omega), D.ptr(b),
             D.ptr(dinv), D.ptr(self.free), D.ptr(self.owned), D.ptr(x), D.ptr(x_out),
             D.ptr(prior), D.ptr(red), D.ptr(self._ws), D.stream())

    def peer_combine_q(self, p, q, red, prior=None, dots=None):
        """dots: also put dots[0..3) (after red[0] is written) as this rank's contribution to
        the fused all-reduce that peer_cg1_update consumes."""
        call("ebs_peer_combine_q", self.peer, D.ptr(q), D.ptr(self.free), D.ptr(self.owned),
             D.ptr(p), D.ptr(prior), D.ptr(red), D.ptr(self._stop), D.ptr(dots), D.ptr(self._ws),
             D.stream())

    def peer_matvec_sweep_put(self, p, q, dots):
        """q = A p with the interface partials pushed, dots[1] = the slab's element energies
        (p.mask(A p) summed over the ranks) and [dots[0..3)] put for the all-reduce -- the
        shared nodes of q are completed by peer_cg1_update_halo."""
        c = self.peer_chunks
        call("ebs_peer_matvec_sweep_put", self.plan.handle, self.peer, D.ptr(c), c.numel(),
             self.if_chunks.numel(), D.ptr(p), D.ptr(q), D.ptr(self.iface), D.ptr(dots),
             D.ptr(self._ws), D.stream())

    def peer_cg1_update_halo(self, cur, prev, rr0, tol, ctl, dinv, x, r, u, w, p, s_, nxt):
        """peer_cg1_update that first completes w's shared nodes (the previous sweep's
        pushed partials, rank-ordered, masked)."""
        call("ebs_peer_cg1_update_halo", self.peer, self.n, D.ptr(cur), D.ptr(prev), D.ptr(rr0),
             float(tol), D.ptr(ctl), D.ptr(self.owned), D.ptr(self.free), D.ptr(dinv), D.ptr(x),
             D.ptr(r), D.ptr(u), D.ptr(w), D.ptr(p), D.ptr(s_), D.ptr(nxt), D.ptr(self._flag),
             D.ptr(self._ws), D.stream())

    def peer_cg1_update(self, cur, prev, rr0, tol, ctl, dinv, x, r, u, w, p, s_, nxt):
        """vec_cg1_update with cur[0..2] all-reduced on the device (waits for every rank's
        peer_combine_q put, adds the contributions in rank order)."""
        call("ebs_peer_cg1_update", self.peer, self.n, D.ptr(cur), D.ptr(prev), D.ptr(rr0),
             float(tol), D.ptr(ctl), D.ptr(self.owned), D.ptr(dinv), D.ptr(x), D.ptr(r), D.ptr(u),
             D.ptr(w), D.ptr(p), D.ptr(s_), D.ptr(nxt), D.ptr(self._flag), D.ptr(self._ws),
             D.stream())

    # slabs of at least this many nodes add into a -0.0-filled r (red.add, as the 1-GPU
    # pass); smaller ones store (the fill launch costs more than the stores' L1tex cost)
    PEER_RED_MIN_NODES = 3 << 20

    def peer_residual_sweep(self, x_int, r_local):
        """residual_local_sweep over all chunks (interface chunks first) whose interface
        partials go straight to the neighbours' windows (ebs_peer_residual_sweep): r_local
        filled with -0.0 and added into on large slabs, stored directly on small ones."""
        c = self.peer_chunks
        add = self.n >= self.PEER_RED_MIN_NODES
        if add:
            call("ebs_fill", r_local.numel(), -0.0, D.ptr(r_local), D.stream())
        call("ebs_peer_residual_sweep", self.plan.handle, self.peer, D.ptr(c), c.numel(),
             self.if_chunks.numel(), D.ptr(x_int), D.ptr(r_local), D.ptr(self.old_of_new32),
             D.ptr(self.iface), EBS_APPLY_ADD if add else 0, D.stream())

    def peer_residual_combine(self, r_local):
        """correct_owned_local with the neighbours' partials from the window."""
        call("ebs_peer_residual_combine", self.peer, D.ptr(self.owned), D.ptr(self.old_of_new32),
             D.ptr(r_local), D.ptr(self._ws), D.stream())

    def peer_push(self, v):
        call("ebs_peer_push", self.peer, D.ptr(v), D.stream())

    def peer_combine(self, v):
        call("ebs_peer_combine", self.peer, D.ptr(v), D.ptr(self._ws), D.stream())

    def dot_owned(self, x, y, red):
        call("ebs_vec_dot_owned", self.n, D.ptr(x), D.ptr(y), D.ptr(self.owned), D.ptr(red),
             D.ptr(self._ws), D.stream())

    def zeros(self, n=None):
        return D.zeros(self.n if n is None else n)


# ------------------------------------------------ exact residual on P slabs --
class ExactSlab:
    """Rank p's slab with a ghost layer, for the EXACT (reference-order) residual on P slabs,
    bit for bit the single-GPU / reference `residual(..., deterministic=True)` at every node
    of the slab ("for bitwise identity across P ...").

    The slab's elements are augmented with every element of another slab that touches one of
    its shared nodes (a one-element ghost layer), kept in ascending GLOBAL element order --
    so the plan's per-node slot order (j, then element) is the global (j, e) bincount order
    of operators.py:98 restricted to ALL the elements at that node: the node sums are the
    reference's, not rank-partial sums.  The price is the ghost elements' bytes (one cell row
    per neighbour) and an exchange of x at the ghost-only nodes before the pass (instead of
    the partial sums after it).  Construction is from the global mesh (+ its f) or, in
    emulation, the global ElementBatch."""

    def __init__(self, maps: dict, p: int, indt: torch.Tensor, n_nodes: int, batch=None,
                 mesh=None, nu=None, f=None):
        from .elements import ElementBatch, build_element_batch
        from .mesh import IndexArrays, Mesh
        self.rank, self.P = p, len(maps["local"])
        dev = D.device()
        indt = indt.to(dev)
        lo, hi = int(maps["bounds"][p]), int(maps["bounds"][p + 1])
        own = maps["local"][p].to(dev)
        shared = (torch.unique(torch.cat(list(maps["interface"][p].values()))).to(dev)
                  if maps["interface"][p] else torch.empty(0, dtype=torch.int64, device=dev))
        is_sh = torch.zeros(n_nodes, dtype=torch.bool, device=dev)
        is_sh[shared] = True
        touch = is_sh[indt.to(torch.int64)].any(dim=0)
        touch[lo:hi] = True                                   # own elements
        self.elements = torch.nonzero(touch).reshape(-1)     # ascending global element id
        nodes = torch.unique(indt[:, self.elements].reshape(-1).to(torch.int64))
        self.global_ids = nodes                               # the plan's caller numbering
        self.n = nodes.numel()
        conn = torch.searchsorted(nodes, indt[:, self.elements].to(torch.int64)).to(torch.int32)
        if batch is not None:
            A = batch._A_store()[self.elements]
            b_e = batch.b_e[:, self.elements].contiguous()
            self.batch = ElementBatch(K_e=A.permute(1, 2, 0), M_e=A.permute(1, 2, 0),
                                      A_e=A.permute(1, 2, 0), b_e=b_e, nu=batch.nu,
                                      index=IndexArrays(None, conn.contiguous(), n_nodes=self.n))
        else:
            sub = Mesh(mesh.nodes, None, mesh.boundary_nodes,
                       conn=mesh.conn[:, self.elements].contiguous())
            full = build_element_batch(sub, nu=nu, f=f)
            self.batch = ElementBatch(K_e=full.K_e, M_e=full.M_e, A_e=full.A_e, b_e=full.b_e,
                                      nu=full.nu,
                                      index=IndexArrays(None, conn.contiguous(), n_nodes=self.n))
        self.plan = self.batch.operator(self.n)
        # where the slab's own local nodes (its caller order) sit in the augmented numbering,
        # and the ghost-only nodes with the rank that supplies each (their owner)
        self.own_pos = torch.searchsorted(nodes, own)
        ghost = torch.ones(self.n, dtype=torch.bool, device=dev)
        ghost[self.own_pos] = False
        self.ghost_pos = torch.nonzero(ghost).reshape(-1)
        gids = nodes[self.ghost_pos]
        src = maps["owner"].to(dev)[gids]
        self.recv = {}   # q -> positions (in the augmented numbering) filled from rank q
        self.recv_g = {}  # q -> their global ids (ascending)
        for q in torch.unique(src).tolist():
            sel = src == q
            self.recv[int(q)] = self.ghost_pos[sel]
            self.recv_g[int(q)] = gids[sel]
        self._own_global = own
        self._owner = maps["owner"].to(dev)
        self.send = {}   # q -> positions in this rank's own local order sent to rank q

    def link(self, slabs_or_recv_g: dict):
        """Send lists: for each rank q, the nodes q needs from this rank (q's recv_g[p]),
        as positions in this rank's own local order.  slabs_or_recv_g: {q: global ids}."""
        for q, g in slabs_or_recv_g.items():
            self.send[q] = torch.searchsorted(self._own_global, g.to(self._own_global.device))


def exact_slabs(maps: dict, indt, n_nodes: int, batch=None, mesh=None, nu=None, f=None,
                ranks=None):
    """ExactSlab of each rank in `ranks` (default all), send lists linked (every rank can
    compute every rank's ghost set from the global connectivity)."""
    P = len(maps["local"])
    allr = list(range(P))
    views = [ExactSlab(maps, p, indt, n_nodes, batch=batch, mesh=mesh, nu=nu, f=f)
             if (ranks is None or p in ranks) else None for p in allr]
    need = {}  # need[q][p] = global ids rank p needs from rank q
    for p in allr:  # remote ranks: only their ghost bookkeeping
        v = views[p] if views[p] is not None else _ghost_only(maps, p, indt, n_nodes)
        for q, g in v.recv_g.items():
            need.setdefault(q, {})[p] = g
    for p in allr:
        if views[p] is not None:
            views[p].link(need.get(p, {}))
    return [v for v in views if v is not None]


def _ghost_only(maps, p, indt, n_nodes):
    """The ghost-node bookkeeping of rank p without building its plan."""
    class _G:
        pass
    dev = D.device()
    indt = indt.to(dev)
    lo, hi = int(maps["bounds"][p]), int(maps["bounds"][p + 1])
    own = maps["local"][p].to(dev)
    shared = (torch.unique(torch.cat(list(maps["interface"][p].values()))).to(dev)
              if maps["interface"][p] else torch.empty(0, dtype=torch.int64, device=dev))
    is_sh = torch.zeros(n_nodes, dtype=torch.bool, device=dev)
    is_sh[shared] = True
    touch = is_sh[indt.to(torch.int64)].any(dim=0)
    touch[lo:hi] = True
    nodes = torch.unique(indt[:, torch.nonzero(touch).reshape(-1)].reshape(-1).to(torch.int64))
    isown = torch.zeros(n_nodes, dtype=torch.bool, device=dev)
    isown[own] = True
    gids = nodes[~isown[nodes]]
    src = maps["owner"].to(dev)[gids]
    g = _G()
    g.recv_g = {int(q): gids[src == q] for q in torch.unique(src).tolist()}
    return g


def residual_exact(slabs: list, comm, x_locals: list) -> list:
    """r = b - A x in the reference's exact order on P slabs: each rank's x_locals[i] holds
    its slab's local nodes (ascending global id, as residual_local); returns each rank's r at
    the same nodes, bit for bit the single-GPU / reference residual there.  The ghost x
    values travel through comm's generic exchange (padded to equal sizes both ways)."""
    sends, xa = [], []
    for sl, xl in zip(slabs, x_locals):
        buf = {}
        for q, pos in sl.send.items():
            m = max(pos.numel(), _peer_count(slabs, sl, q))
            t = torch.zeros(m, dtype=torch.float64, device=xl.device)
            t[:pos.numel()] = xl[pos]
            buf[q] = t
        for q in sl.recv:
            if q not in buf:  # receive-only direction: an empty send of the right size
                buf[q] = torch.zeros(sl.recv[q].numel(), dtype=torch.float64, device=xl.device)
        sends.append(buf)
        x_aug = torch.empty(sl.n, dtype=torch.float64, device=xl.device)
        x_aug[sl.own_pos] = xl
        xa.append(x_aug)
    if getattr(comm, "fused_peer", False):
        raise ValueError("residual_exact needs a transport with a generic exchange "
                         "(LocalTransport / TorchTransport / NativeTransport)")
    recvs = comm.exchange(slabs, sends)
    out = []
    for sl, x_aug, rc in zip(slabs, xa, recvs):
        for q, pos in sl.recv.items():
            x_aug[pos] = rc[q][:pos.numel()]
        r_aug = D.empty(sl.n)
        with sl.batch.using(sl.n) as pl:
            call("ebs_residual", pl.handle, D.ptr(x_aug), D.ptr(r_aug), 0, 0, None, D.stream())
        out.append(r_aug[sl.own_pos])
    return out


def _ghost_exchange(slabs, comm, x_augs):
    """Fill every slab's ghost-only entries of x_aug (the augmented numbering) from the ranks
    that own those nodes (the transport's generic exchange, padded to equal sizes)."""
    if getattr(comm, "fused_peer", False):
        raise ValueError("the ghost-layer slabs need a transport with a generic exchange "
                         "(LocalTransport / TorchTransport / NativeTransport)")
    sends = []
    for sl, xa in zip(slabs, x_augs):
        buf = {}
        own = xa[sl.own_pos]
        for q, pos in sl.send.items():
            m = max(pos.numel(), _peer_count(slabs, sl, q))
            t = torch.zeros(m, dtype=torch.float64, device=xa.device)
            t[:pos.numel()] = own[pos]
            buf[q] = t
        for q in sl.recv:
            if q not in buf:
                buf[q] = torch.zeros(sl.recv[q].numel(), dtype=torch.float64, device=xa.device)
        sends.append(buf)
    recvs = comm.exchange(slabs, sends)
    for sl, xa, rc in zip(slabs, x_augs, recvs):
        for q, pos in sl.recv.items():
            xa[pos] = rc[q][:pos.numel()]


def jacobi_exact(slabs: list, comm, d, x_locals0: list, iters: int, omega: float = 0.8):
    """Damped Jacobi on P ghost-layer slabs (ExactSlab) whose iterates are BIT FOR BIT the
    single-GPU solver's (eb.jacobi, fast residual) at every slab node, for any P: each
    iteration exchanges x at the ghost-only nodes, then every slab evaluates the masked
    residual over all the elements at its nodes in the global (j, e) order (the same SELL
    arithmetic as the solver's step) and the update x + omega (dinv r) with dinv from the
    slot-order diagonal.  Returns (x_locals, norms): x on each slab's own local nodes; the
    norms sum the owned nodes in rank order (within rounding of the 1-GPU history)."""
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    dev = x_locals0[0].device
    xa, rs, dinvs, owned = [], [], [], []
    for sl, x0 in zip(slabs, x_locals0):
        nd = d.nd.to(dev) if d is not None else torch.empty(0, dtype=torch.int64, device=dev)
        is_d = torch.zeros(int(max(int(sl.global_ids.max()) + 1, 1)), dtype=torch.bool,
                           device=dev)
        if nd.numel():
            is_d[nd[nd < is_d.numel()]] = True
        local_d = torch.nonzero(is_d[sl.global_ids]).reshape(-1)
        from .operators import DirichletData
        sl.plan.ensure_dirichlet(DirichletData(local_d, torch.zeros(local_d.numel(),
                                                                   dtype=torch.float64,
                                                                   device=dev)))
        diag = D.empty(sl.n)
        call("ebs_diagonal", sl.plan.handle, D.ptr(diag), D.stream())
        free = torch.ones(sl.n, dtype=torch.bool, device=dev)
        free[local_d] = False
        ok = free & (diag != 0.0)
        dinvs.append(torch.where(ok, 1.0 / torch.where(ok, diag, torch.ones_like(diag)),
                                 torch.zeros_like(diag)))
        x = torch.zeros(sl.n, dtype=torch.float64, device=dev)
        x[sl.own_pos] = x0.to(dev, torch.float64)
        xa.append(x)
        rs.append(D.empty(sl.n))
        own_g = sl.global_ids[sl.own_pos]
        owned.append(sl.own_pos[sl._owner[own_g] == sl.rank])
    norm2 = [torch.zeros(iters + 1, dtype=torch.float64, device=dev) for _ in slabs]
    for k in range(iters + 1):
        _ghost_exchange(slabs, comm, xa)
        for i, sl in enumerate(slabs):
            with sl.batch.using(sl.n) as pl:
                call("ebs_residual", pl.handle, D.ptr(xa[i]), D.ptr(rs[i]), 1, 1, None,
                     D.stream())
            r_o = rs[i][owned[i]]
            norm2[i][k] = torch.dot(r_o, r_o)
            if k < iters:  # x + omega (dinv r): the solver's rounding, op by op
                t = dinvs[i] * rs[i]
                t = t * float(omega)
                xa[i] = xa[i] + t
    comm.allreduce(norm2)
    norms = torch.sqrt(norm2[0]).cpu().numpy()
    return [x[sl.own_pos] for sl, x in zip(slabs, xa)], norms


def _peer_count(slabs, sl, q):
    """Size of what rank q sends to this rank (for the symmetric padding)."""
    n = sl.recv.get(q)
    return 0 if n is None else n.numel()


# ------------------------------------------------------------------- loops --
def _peer(comm) -> bool:
    return bool(getattr(comm, "fused_peer", False))


def halo(ops, comm, vs):
    """Exchange interface partials of vs[i] (rank ops[i]) and combine in rank order."""
    if _peer(comm):
        comm.halo(ops, vs)
        return
    sends = [{q: op.gather(idx, v) for q, idx in op.if_idx.items()} for op, v in zip(ops, vs)]
    recvs = comm.exchange(ops, sends)
    for op, v, rc in zip(ops, vs, recvs):
        op.combine(v, rc)


@dataclass
class DistProblem:
    ops: list
    comm: object
    b: list       # full (combined) b per rank, internal numbering
    dinv: list    # Jacobi 1/diag (0 at constrained nodes)
    diverged: bool = False  # last jacobi/pcg: a non-finite iterate or norm on any rank
                            # (solvers.py:138-152 -- flagged, never raised)
    # per-solver device workspaces and their captured CUDA graphs, kept across solves: the
    # graph of a loop is captured once per problem (and solver settings) and replayed by
    # every later solve -- a capture per solve costs host time, graph-pool allocations and
    # their release, which measured as erratic 1.5-4x slower solves
    cache: dict = field(default_factory=dict)


class _Workspace:
    """Named device buffers of one solver loop + its captured graph (None: not captured,
    or capture not possible -- `tried` records the collective decision)."""

    def __init__(self, **bufs):
        self.__dict__.update(bufs)
        self.graph = None
        self.tried = False


def _workspace(prob, key, make):
    ws = prob.cache.get(key)
    if ws is None:
        ws = prob.cache[key] = make()
    return ws


def _graph_for(prob, ws, body):
    """The workspace's captured graph, capturing it on first use (collective decision)."""
    if not ws.tried:
        ws.graph = _capture(prob.comm, body)
        ws.tried = True
    return ws.graph


def _reset_flags(ops):
    for op in ops:
        flag = getattr(op, "_flag", None)
        if flag is not None:
            flag.zero_()


def _diverged(prob, norms) -> bool:
    """Divergence as the reference's _iterate reports it: any rank's vector kernels saw a
    non-finite iterate, or a residual norm is not finite; identical on every rank."""
    bad = not bool(np.isfinite(norms).all())
    for op in prob.ops:
        flag = getattr(op, "_flag", None)
        if flag is not None:
            bad |= bool(int(flag.item()))
    agree = getattr(prob.comm, "agree", None)
    return (not agree(not bad)) if agree is not None else bad


def setup(ops, comm, precondition=True) -> DistProblem:
    bs = [op.rhs_partial() for op in ops]
    halo(ops, comm, bs)
    dgs = [op.diag_partial() for op in ops]
    halo(ops, comm, dgs)
    dinv = [op.vec_dinv(dg if precondition else None) for op, dg in zip(ops, dgs)]
    return DistProblem(ops, comm, bs, dinv)


def residual_caller(prob: DistProblem, x_global: torch.Tensor, r_globals: list, x_ints: list,
                    s_raws: list, overlap: bool = True):
    """r = b - A x with x and r in the caller's (global) numbering on P ranks, fused: one
    SELL pass per rank writes its slab's partial residual b_p - s_p straight into r
    (caller numbering) and keeps a copy in internal order; after the halo exchange each
    rank adds its neighbours' partial residuals on the interface nodes it owns (in
    ascending rank order).  Owned entries of r_globals[i] are the residual (within
    rounding of the reassociated sum).  overlap: sweep the interface chunks first and
    the interior chunks while the halo exchange is in flight (same values)."""
    ops, comm = prob.ops, prob.comm
    if overlap:  # interface chunks, exchange in flight || interior chunks
        for op, xi, rg, sr in zip(ops, x_ints, r_globals, s_raws):
            op.gather_global(x_global, xi)
            op.residual_caller_sweep(op.if_chunks, xi, rg, sr)
        h = comm.exchange_start(ops, [op.gather_sends(sr)
                                      for op, sr in zip(ops, s_raws)])
        for op, xi, rg, sr in zip(ops, x_ints, r_globals, s_raws):
            op.residual_caller_sweep(op.in_chunks, xi, rg, sr)
        recvs = comm.exchange_finish(h)
    else:
        for op, xi, rg, sr in zip(ops, x_ints, r_globals, s_raws):
            op.gather_global(x_global, xi)
            op.residual_caller_partial(xi, rg, sr)
        sends = [op.gather_sends(sr)
                 for op, sr in zip(ops, s_raws)]
        recvs = comm.exchange(ops, sends)
    for op, rg, rc in zip(ops, r_globals, recvs):
        op.correct_owned(rg, rc)


def residual_local(prob: DistProblem, x_locals: list, r_locals: list, x_ints: list,
                   s_raws: list):
    """r = b - A x on P ranks with each rank's x and r in ITS caller order: the slab's
    local nodes in ascending global id (x_locals[i] = x[op.global_ids]).  Per rank: x to
    internal order, r := -0.0, partial residual of the interface chunks added into r,
    NCCL halo of the interface partials in flight while the interior chunks are swept,
    owned interface entries completed in ascending rank order.  The owned entries
    (op.owned_local) are the residual within rounding of the reassociated sum."""
    ops, comm = prob.ops, prob.comm
    if _peer(comm):  # one sweep pushing the interface partials, one combine (s_raws unused)
        for op, xl, rl, xi in zip(ops, x_locals, r_locals, x_ints):
            call("ebs_to_internal", op.plan.handle, D.ptr(xl), D.ptr(xi), None, D.stream())
            op.peer_residual_sweep(xi, rl)
        comm.after_put()
        for op, rl in zip(ops, r_locals):
            op.peer_residual_combine(rl)
        return
    for op, xl, rl, xi, sr in zip(ops, x_locals, r_locals, x_ints, s_raws):
        call("ebs_to_internal", op.plan.handle, D.ptr(xl), D.ptr(xi), None, D.stream())
        call("ebs_fill", rl.numel(), -0.0, D.ptr(rl), D.stream())
        op.residual_local_sweep(op.if_chunks, xi, rl, sr)
    h = comm.exchange_start(ops, [op.gather_sends(sr)
                                  for op, sr in zip(ops, s_raws)])
    for op, xi, rl, sr in zip(ops, x_ints, r_locals, s_raws):
        op.residual_local_sweep(op.in_chunks, xi, rl, sr)
    recvs = comm.exchange_finish(h)
    for op, rl, rc in zip(ops, r_locals, recvs):
        op.correct_owned_local(rl, rc)


def residual(prob: DistProblem, xs, out=None):
    """r = b - A x (unmasked, operators.py:72) on every rank's local nodes (internal
    numbering); shared nodes hold identical values on every rank."""
    ops, comm = prob.ops, prob.comm
    ss = [op.zeros() for op in ops]
    for op, x, s in zip(ops, xs, ss):
        op.matvec_partial(x, s)
    halo(ops, comm, ss)
    return [b - s for b, s in zip(prob.b, ss)]


GRAPH_BATCH = 8  # iterations per captured CUDA graph (even: Jacobi ping-pong buffers)
GRAPH_STATS = {"captured": 0, "fallback": 0, "last_error": None}


def _capture(comm, body):
    """Capture body() into a CUDA graph on every rank.  The decision is collective: the
    graph is used only if every rank captured it (comm.agree), else all ranks drop it and
    run eagerly -- ranks never mix graph replay with eager steps, whose NCCL calls would
    not pair up.  EBS_DIST_GRAPH=0 disables capture."""
    import os
    if os.environ.get("EBS_DIST_GRAPH", "1") == "0" or getattr(comm, "serialize", False):
        return None
    g, err = None, None
    try:
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
    except Exception as e:  # noqa: BLE001 -- capture unsupported here: run eagerly
        g, err = None, e
        if torch.cuda.is_available():
            torch.cuda.synchronize()
    agree = getattr(comm, "agree", None)
    ok = agree(g is not None) if agree is not None else g is not None
    if not ok:
        GRAPH_STATS["fallback"] += 1
        GRAPH_STATS["last_error"] = (f"{type(err).__name__}: {err}" if err is not None
                                     else "another rank could not capture")
        return None
    GRAPH_STATS["captured"] += 1
    return g


def _graph_ok(ops) -> bool:
    return all(getattr(op, "n", 0) and torch.cuda.is_available() and
               isinstance(getattr(op, "free", None), torch.Tensor) and op.free.is_cuda for op in ops)


def _fused_ok(ops) -> bool:
    return all(hasattr(op, "jacobi_sweep") for op in ops)


def jacobi(prob: DistProblem, xs0, iters: int, omega: float = 0.8, richardson: bool = False,
           graph: bool = False, fused=None):
    """Damped Jacobi on P ranks (oracle/ebs_oracle.py jacobi semantics, fixed count).

    Returns (xs, norms) with norms[k] = ||mask(b - A x_k)||, k = 0..iters.  With
    graph=True the iterations are replayed from a captured CUDA graph of GRAPH_BATCH
    iterations (same kernels, same results).  fused (default: GPU ranks) runs the
    overlapped interface/interior sweeps with the update fused into the SELL pass."""
    ops, comm = prob.ops, prob.comm
    _reset_flags(ops)
    fused = _fused_ok(ops) if fused is None else fused
    B = GRAPH_BATCH
    dev = xs0[0].device
    peer = fused and _peer(comm)
    ws = _workspace(prob, ("jacobi", float(omega), bool(richardson), bool(fused), peer),
                    lambda: _Workspace(
                        xa=[op.zeros() for op in ops], xb=[op.zeros() for op in ops],
                        ss=[op.zeros() for op in ops],
                        r3=[torch.zeros(2, dtype=torch.float64, device=dev) for _ in ops],
                        bred=[torch.zeros(B, dtype=torch.float64, device=dev) for _ in ops]))
    for a, x in zip(ws.xa, xs0):
        a.copy_(x)
    xa, xb, ss, r3 = list(ws.xa), list(ws.xb), ws.ss, ws.r3  # sweep partials in r3
    red = [torch.zeros(iters + 1, dtype=torch.float64, device=dev) for _ in ops]

    def step(src, dst, final, rslot):
        if peer:  # one sweep pushing the interface partials to the neighbours, combine
            for i, op in enumerate(ops):
                op.peer_jacobi_sweep(omega, src[i], None if final else dst[i], prob.b[i],
                                     None if richardson else prob.dinv[i], ss[i], r3[i][0:1])
            comm.after_put()
            for i, op in enumerate(ops):
                op.peer_combine_jacobi(omega, prob.b[i], ss[i],
                                       None if richardson else prob.dinv[i], src[i],
                                       None if final else dst[i], rslot[i], prior=r3[i])
            return
        if fused:  # interface chunks, exchange || interior chunks, interface completion
            for i, op in enumerate(ops):
                op.jacobi_sweep(op.if_chunks, omega, src[i], None if final else dst[i], prob.b[i],
                                None if richardson else prob.dinv[i], ss[i], r3[i][0:1])
            h = comm.exchange_start(ops, [op.gather_sends(s_)
                                          for op, s_ in zip(ops, ss)])
            for i, op in enumerate(ops):
                op.jacobi_sweep(op.in_chunks, omega, src[i], None if final else dst[i], prob.b[i],
                                None if richardson else prob.dinv[i], ss[i], r3[i][1:2])
            recvs = comm.exchange_finish(h)
            for i, op in enumerate(ops):
                op.combine_jacobi(recvs[i], omega, prob.b[i], ss[i],
                                  None if richardson else prob.dinv[i], src[i],
                                  None if final else dst[i], rslot[i], prior=r3[i])
            return
        for op, x, s_ in zip(ops, src, ss):
            op.matvec_partial(x, s_)
        halo(ops, comm, ss)
        for i, op in enumerate(ops):
            op.vec_jacobi(omega, prob.b[i], ss[i], None if richardson else prob.dinv[i], src[i],
                          None if final else dst[i], None, rslot[i])

    if peer:
        return _jacobi_peer(prob, ws, xa, xb, ss, r3, red, iters, omega, richardson, graph)

    k = 0
    if graph and iters >= B and _graph_ok(ops):
        bred = ws.bred

        def body():
            for u in range(B):  # B even: xa/xb roles return to the start
                src, dst = (xa, xb) if u % 2 == 0 else (xb, xa)
                step(src, dst, False, [r_[u:u + 1] for r_ in bred])
        g = _graph_for(prob, ws, body)
        if g is not None:
            while k + B <= iters:
                g.replay()
                for i in range(len(ops)):
                    red[i][k:k + B].copy_(bred[i])
                k += B
    for kk in range(k, iters + 1):
        final = kk == iters
        step(xa, xb, final, [r_[kk:kk + 1] for r_ in red])
        if not final:
            xa, xb = xb, xa
    comm.allreduce(red)
    sync = getattr(comm, "sync", None)
    if sync is not None:
        sync()
    norms = torch.sqrt(red[0]).cpu().numpy()
    prob.diverged = _diverged(prob, norms)
    return [x.clone() for x in xa], norms  # fresh arrays: the workspace is reused


def _jacobi_peer(prob, ws, xa, xb, ss, r3, red, iters, omega, richardson, graph):
    """The peer-transport Jacobi loop: ONE launch per iteration (ebs_peer_jacobi_step: the
    first warps complete iteration k-1's shared nodes while the interior chunks of iteration
    k are swept; the interface chunks push their partials), the first sweep alone and the
    last completion alone.  Iterates are bitwise those of the other transports (same
    per-node sums, same rank order)."""
    ops, comm = prob.ops, prob.comm
    B = GRAPH_BATCH
    dinv = [None if richardson else d for d in prob.dinv]

    def step(src, dst, final, red_prev):  # iteration k >= 1: x_{k-1} in dst, x_k in src
        for i, op in enumerate(ops):
            op.peer_jacobi_step(omega, dst[i], src[i], None if final else dst[i], prob.b[i],
                                dinv[i], ss[i], r3[i], red_prev[i], r3[i][0:1])
        comm.after_put()

    for i, op in enumerate(ops):  # iteration 0: the sweep alone
        op.peer_jacobi_sweep(omega, xa[i], None if iters == 0 else xb[i], prob.b[i], dinv[i],
                             ss[i], r3[i][0:1])
    comm.after_put()
    if iters > 0:
        xa, xb = xb, xa
    k = 1
    if graph and iters >= B + 1 and _graph_ok(ops):
        bred = ws.bred

        def body():  # iterations k..k+B-1 (none final); B even: xa/xb roles return
            for u in range(B):
                src, dst = (xa, xb) if u % 2 == 0 else (xb, xa)
                step(src, dst, False, [r_[u:u + 1] for r_ in bred])
        g = _graph_for(prob, ws, body)
        if g is not None:
            while k + B <= iters:  # the final iteration stays eager
                g.replay()
                for i in range(len(ops)):
                    red[i][k - 1:k - 1 + B].copy_(bred[i])
                k += B
    for kk in range(k, iters + 1):
        final = kk == iters
        step(xa, xb, final, [r_[kk - 1:kk] for r_ in red])
        if not final:
            xa, xb = xb, xa
    for i, op in enumerate(ops):  # the last iteration's shared nodes (x_iters, ||r_iters||)
        op.peer_combine_jacobi(omega, prob.b[i], ss[i], dinv[i], xa[i], None,
                               red[i][iters:iters + 1], prior=r3[i])
    comm.allreduce(red)
    sync = getattr(comm, "sync", None)
    if sync is not None:
        sync()
    norms = torch.sqrt(red[0]).cpu().numpy()
    prob.diverged = _diverged(prob, norms)
    return [x.clone() for x in xa], norms  # fresh arrays: the workspace is reused


def pcg(prob: DistProblem, xs0, iters: int, tol=None, graph: bool = False, fused=None,
        reductions: int = 1):
    """Jacobi-PCG on P ranks (oracle/ebs_oracle.py pcg; with prob from setup(..,
    precondition=False) plain CG), same stopping rule and history as _iterate
    (solvers.py:117-160).  Returns (xs, norms); prob.diverged is set.

    reductions=1 (default): the single-reduction (Chronopoulos-Gear) recurrence -- ONE
    all-reduce of [r.u, w.u, r.r] per iteration, the loop rules (tol, divergence) decided on
    the device, CUDA-graph batches also with a tolerance and no host synchronisation inside
    the solve.  reductions=2: the textbook recurrence of the oracle, two all-reduces per
    iteration (p.q, then [r.r, r.z]); a tolerance costs a host read per iteration there."""
    if reductions == 1:
        return _pcg_single_reduction(prob, xs0, iters, tol=tol, graph=graph, fused=fused)
    if reductions != 2:
        raise ValueError(f"reductions must be 1 or 2, got {reductions}")
    return _pcg_two_reductions(prob, xs0, iters, tol=tol, graph=graph, fused=fused)


def _pcg_single_reduction(prob: DistProblem, xs0, iters: int, tol=None, graph: bool = False,
                          fused=None):
    """Chronopoulos-Gear PCG (oracle pcg in exact arithmetic; rounding differs):
        r = mask(b - A x0), u = dinv r, w = mask(A u);  [gamma, delta, rr] all-reduced
        loop k: beta = gamma_k/gamma_{k-1}, alpha = gamma_k/(delta_k - beta gamma_k/alpha_{k-1})
                p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; u = dinv r
                                                      (ebs_vec_cg1_update: r.u, r.r partials)
                w = mask(A u) and w.u                  (fused sweeps / halo / interface)
                all-reduce [r.u, w.u, r.r]             (ONE collective)
    Scalars live in a ring of GRAPH_BATCH slots [gamma, delta, rr, alpha]; iteration k reads
    slot k % B (and k-1 for beta), writes slot k+1.  ctl = [stop, k_stop, k, diverged]
    per rank: the update kernel stops the loop on the device (tol / non-finite norm), after
    which every kernel is a no-op -- so the host enqueues graph batches and reads ctl one
    batch behind (never idling the device), and the returned x is x_{k_stop} exactly."""
    if iters < 0:
        raise ValueError(f"iteration count must be nonnegative, got {iters}")
    ops, comm = prob.ops, prob.comm
    dev = xs0[0].device
    f64 = dict(dtype=torch.float64, device=dev)
    _reset_flags(ops)
    B = GRAPH_BATCH
    fused = _fused_ok(ops) if fused is None else fused
    tol_ = -1.0 if tol is None else float(tol)
    on_dev = dev.type == "cuda"
    peer = fused and _peer(comm)
    wsp = _workspace(prob, ("pcg1", tol_, bool(fused), peer), lambda: _Workspace(
        xs=[op.zeros() for op in ops], rs=[op.zeros() for op in ops],
        us=[op.zeros() for op in ops], ws=[op.zeros() for op in ops],
        ps=[op.zeros() for op in ops], ss=[op.zeros() for op in ops],
        # [gamma, delta, rr, alpha] (+ peer: the reduced rr again -- [0..2] of a slot are
        # overwritten with the next-but-B iteration's partials before a graph batch ends)
        ring=[torch.zeros((B, 5 if peer else 4), **f64) for _ in ops],
        part=[torch.zeros(2, **f64) for _ in ops],        # interface / interior sweep w.u
        ctl=[torch.zeros(4, dtype=torch.int32, device=dev) for _ in ops],
        rr0=[torch.zeros(1, **f64) for _ in ops],
        host_ctl=[torch.zeros((2, 4), dtype=torch.int32, pin_memory=on_dev) for _ in ops]))
    xs, rs, us, ws, ps, ss = wsp.xs, wsp.rs, wsp.us, wsp.ws, wsp.ps, wsp.ss
    ring, part, ctl, rr0, host_ctl = wsp.ring, wsp.part, wsp.ctl, wsp.rr0, wsp.host_ctl
    for i in range(len(ops)):
        xs[i].copy_(xs0[i])
        for t in (us[i], ps[i], ss[i], ring[i], part[i], ctl[i]):
            t.zero_()
    zero = torch.zeros(1, **f64)
    for op, c in zip(ops, ctl):
        if hasattr(op, "set_stop"):
            op.set_stop(c if fused else None)

    def matvec_w(slot):  # w = mask(A u), slot[1] = the rank's owned w.u
        if peer:  # ... w.u from the element energies and [r.u, w.u, r.r] put for the
            # all-reduce the next update takes, which also completes w's shared nodes
            for i, op in enumerate(ops):
                op.peer_matvec_sweep_put(us[i], ws[i], slot[i][0:3])
            comm.after_put()
        elif fused:
            for i, op in enumerate(ops):
                op.matvec_sweep(op.if_chunks, us[i], ws[i], part[i][0:1])
            h = comm.exchange_start(ops, [op.gather_sends(w_) for op, w_ in zip(ops, ws)])
            for i, op in enumerate(ops):
                op.matvec_sweep(op.in_chunks, us[i], ws[i], part[i][1:2])
            recvs = comm.exchange_finish(h)
            for i, op in enumerate(ops):
                op.combine_q(recvs[i], us[i], ws[i], slot[i][1:2], prior=part[i])
        else:
            for op, u_, w_ in zip(ops, us, ws):
                op.matvec_partial(u_, w_)
            halo(ops, comm, ws)
            for i, op in enumerate(ops):
                op.vec_pcg_q(us[i], ws[i], slot[i][1:2])

    # r_0, u_0, w_0 and the first scalars (slot 0); slot B-1 = "iteration -1" (gamma 0)
    for op, x, s_ in zip(ops, xs, ss):
        op.matvec_partial(x, s_)
    halo(ops, comm, ss)
    slot0 = [rg[0] for rg in ring]
    for i, op in enumerate(ops):
        op.vec_jacobi(0.0, prob.b[i], ss[i], None, xs[i], None, rs[i], slot0[i][2:3])
        op.vec_pcg_direction(zero, zero, prob.dinv[i], rs[i], us[i])  # u = dinv r
        op.dot_owned(rs[i], us[i], slot0[i][0:1])
        ss[i].zero_()
    matvec_w(slot0)
    norm2 = [torch.zeros(iters + 1, **f64) for _ in ops]
    if not peer:
        comm.allreduce([sl[0:3] for sl in slot0])
        for i in range(len(ops)):
            rr0[i].copy_(slot0[i][2:3])
            norm2[i][0:1].copy_(slot0[i][2:3])
    # peer: every put of matvec_w is consumed by the next update (ebs_peer_cg1_update: the
    # slot it reads is reduced there, rr0 set at k = 0), so history entry k is recorded after
    # step k, and the put of the last step by one get after the loop

    def step(k):
        cur = [rg[k % B] for rg in ring]
        prev = [rg[(k - 1) % B] for rg in ring]
        nxt = [rg[(k + 1) % B] for rg in ring]
        if peer:  # the all-reduce of cur and w's halo completion happen inside the update
            for i, op in enumerate(ops):
                op.peer_cg1_update_halo(cur[i], prev[i], rr0[i], tol_, ctl[i], prob.dinv[i],
                                        xs[i], rs[i], us[i], ws[i], ps[i], ss[i], nxt[i])
            matvec_w(nxt)
            return
        for i, op in enumerate(ops):
            op.vec_cg1_update(cur[i], prev[i], rr0[i], tol_, ctl[i], prob.dinv[i], xs[i], rs[i],
                              us[i], ws[i], ps[i], ss[i], nxt[i])
        matvec_w(nxt)
        comm.allreduce([sl[0:3] for sl in nxt])

    g = None
    if graph and iters >= B and _graph_ok(ops):
        def body():
            for u in range(B):
                step(u)
        g = _graph_for(prob, wsp, body)  # recorded only: nothing ran, the ring is untouched
    # batches of B iterations (graph replay or eager); the stop flags of batch j are read
    # while batch j+1 is queued, so the device never waits for the host
    pending = None
    k, j = 0, 0
    while k < iters:
        nb = min(B, iters - k)
        if g is not None and nb == B:
            g.replay()
            for i in range(len(ops)):
                if peer:  # iterations k..k+B-1 reduced slots 0..B-1
                    norm2[i][k:k + B].copy_(ring[i][0:B, 4])
                else:  # iterations k..k+B-1 wrote slots 1..B-1, 0
                    norm2[i][k + 1:k + B].copy_(ring[i][1:B, 2])
                    norm2[i][k + B:k + B + 1].copy_(ring[i][0:1, 2])
        else:
            for kk in range(k, k + nb):
                step(kk)
                for i in range(len(ops)):
                    if peer:
                        norm2[i][kk:kk + 1].copy_(ring[i][kk % B, 4:5])
                    else:
                        norm2[i][kk + 1:kk + 2].copy_(ring[i][(kk + 1) % B, 2:3])
        k += nb
        if k >= iters:
            break
        for i in range(len(ops)):
            host_ctl[i][j & 1].copy_(ctl[i], non_blocking=on_dev)
        ev = torch.cuda.Event() if on_dev else None
        if ev is not None:
            ev.record()
        if pending is not None:  # batch j-1's flags, while batch j runs
            pev, pj = pending
            if pev is not None:
                pev.synchronize()
            if any(int(h[pj & 1][0]) for h in host_ctl):
                break
        pending = (ev, j)
        j += 1
    sync = getattr(comm, "sync", None)
    if sync is not None:
        sync()
    c = ctl[0].cpu()
    if peer and not int(c[0]):  # the last sweep's put and halo (same decision on every rank)
        last = [rg[iters % B] for rg in ring]
        comm.allreduce_get([sl[0:3] for sl in last])
        for op, w_ in zip(ops, ws):
            op.peer_combine(w_)
        for i in range(len(ops)):
            norm2[i][iters:iters + 1].copy_(last[i][2:3])
    for op in ops:
        if hasattr(op, "set_stop"):
            op.set_stop(None)
    n = int(c[1]) + 1 if int(c[0]) else iters + 1
    norms = torch.sqrt(norm2[0][:n]).cpu().numpy()
    diverged = _diverged(prob, norms)  # collective: every rank calls it
    prob.diverged = diverged or bool(int(c[3]))
    return [x.clone() for x in xs], norms  # fresh arrays: the workspace is reused


def _pcg_two_reductions(prob: DistProblem, xs0, iters: int, tol=None, graph: bool = False,
                        fused=None):
    """The oracle's recurrence: two scalar all-reduces per iteration, both in place and
    with no copies between the kernels: the rank's p.q (the interface kernel adds the two
    sweep partials to its own) and the iteration's [r.r, r.z] pair, kept in a ring of
    GRAPH_BATCH slots that the next iteration reads as its rz.  graph=True (fixed iteration
    count only) replays captured CUDA graphs of GRAPH_BATCH iterations."""
    ops, comm = prob.ops, prob.comm
    dev = xs0[0].device
    f64 = dict(dtype=torch.float64, device=dev)
    _reset_flags(ops)
    for op in ops:
        if hasattr(op, "set_stop"):
            op.set_stop(None)
    fused = _fused_ok(ops) if fused is None else fused
    B = GRAPH_BATCH
    peer = fused and _peer(comm)
    wsp = _workspace(prob, ("pcg2", bool(fused), peer), lambda: _Workspace(
        xs=[op.zeros() for op in ops], rs=[op.zeros() for op in ops],
        ps=[op.zeros() for op in ops], qs=[op.zeros() for op in ops],
        ss=[op.zeros() for op in ops],
        ring=[torch.zeros((B, 2), **f64) for _ in ops],   # iteration k: slot k % B
        pq=[torch.zeros(1, **f64) for _ in ops],
        part=[torch.zeros(2, **f64) for _ in ops]))       # interface / interior sweep p.q
    xs, rs, ps, qs, ss = wsp.xs, wsp.rs, wsp.ps, wsp.qs, wsp.ss
    ring, pq, part = wsp.ring, wsp.pq, wsp.part
    for i in range(len(ops)):
        xs[i].copy_(xs0[i])
        for t in (ps[i], ring[i]):
            t.zero_()
    zero = torch.zeros(1, **f64)
    for op, x, s in zip(ops, xs, ss):
        op.matvec_partial(x, s)
    halo(ops, comm, ss)
    init = [rg[B - 1] for rg in ring]                  # iteration 0 reads its rz here
    for i, op in enumerate(ops):
        op.vec_jacobi(0.0, prob.b[i], ss[i], None, xs[i], None, rs[i], init[i][0:1])
        op.vec_pcg_direction(zero, zero, prob.dinv[i], rs[i], ps[i])  # p = dinv r
        op.dot_owned(rs[i], ps[i], init[i][1:2])
    comm.allreduce(init)
    norm2 = [torch.zeros(iters + 1, **f64) for _ in ops]  # ||r_k||^2
    for i in range(len(ops)):
        norm2[i][0:1].copy_(init[i][0:1])

    def step(u):
        slot = [rg[u] for rg in ring]
        prev = [rg[(u - 1) % B] for rg in ring]
        if peer:
            for i, op in enumerate(ops):
                op.peer_matvec_sweep(ps[i], qs[i], part[i][0:1])
            comm.after_put()
            for i, op in enumerate(ops):
                op.peer_combine_q(ps[i], qs[i], pq[i], prior=part[i])
        elif fused:  # interface chunks, exchange || interior chunks, interface completion
            for i, op in enumerate(ops):
                op.matvec_sweep(op.if_chunks, ps[i], qs[i], part[i][0:1])
            h = comm.exchange_start(ops, [op.gather_sends(q_)
                                          for op, q_ in zip(ops, qs)])
            for i, op in enumerate(ops):
                op.matvec_sweep(op.in_chunks, ps[i], qs[i], part[i][1:2])
            recvs = comm.exchange_finish(h)
            for i, op in enumerate(ops):
                op.combine_q(recvs[i], ps[i], qs[i], pq[i], prior=part[i])
        else:
            for op, p_, q_ in zip(ops, ps, qs):
                op.matvec_partial(p_, q_)
            halo(ops, comm, qs)
            for i, op in enumerate(ops):
                op.vec_pcg_q(ps[i], qs[i], pq[i])
        comm.allreduce(pq)
        for i, op in enumerate(ops):
            op.vec_pcg_update(prev[i][1:2], pq[i], prob.dinv[i], xs[i], rs[i], ps[i], qs[i],
                              slot[i])
        comm.allreduce(slot)
        for i, op in enumerate(ops):
            op.vec_pcg_direction(prev[i][1:2], slot[i][1:2], prob.dinv[i], rs[i], ps[i])

    k = 0
    if graph and tol is None and iters >= B and _graph_ok(ops):
        def body():
            for u in range(B):
                step(u)
        g = _graph_for(prob, wsp, body)
        if g is not None:
            while k + B <= iters:
                g.replay()
                for i in range(len(ops)):
                    norm2[i][k + 1:k + 1 + B].copy_(ring[i][:, 0])
                k += B
    n0 = None
    k_done = iters
    for kk in range(k, iters):
        if tol is not None:
            nk = float(torch.sqrt(norm2[0][kk]))
            n0 = nk if n0 is None else n0
            if nk <= tol * n0 or not np.isfinite(nk):
                k_done = kk
                break
        step(kk % B)
        for i in range(len(ops)):
            norm2[i][kk + 1:kk + 2].copy_(ring[i][kk % B, 0:1])
    n = k_done + 1
    sync = getattr(comm, "sync", None)
    if sync is not None:
        sync()
    norms = torch.sqrt(norm2[0][:n]).cpu().numpy()
    prob.diverged = _diverged(prob, norms)
    return [x.clone() for x in xs], norms  # fresh arrays: the workspace is reused


def gather_global(ops, vs, n_nodes, comm=None):
    """Assemble a global vector (caller numbering) from owned entries (emulated ranks or
    rank-local with an all-reduce of the disjoint owned parts)."""
    out = torch.zeros(n_nodes, dtype=torch.float64, device=vs[0].device)
    for op, v in zip(ops, vs):
        op.scatter_owned(v, out)
    if comm is not None and not isinstance(comm, (LocalTransport, LocalPeerTransport)):
        comm.allreduce([out])  # owned parts are disjoint: the sum is the global vector
    return out


def emulate(batch, n_nodes, d, P, precondition=True, peer: bool = False):
    """P ranks in this process on the current GPU (tests; nothing waits on anything).
    peer=True: the peer-memory transport (LocalPeerTransport: the windows, fused sweeps and
    combine kernels of PeerTransport), else device copies (LocalTransport)."""
    maps = partition_maps(batch.index.indt, n_nodes, P)
    ops = [GpuRankOperator(batch, n_nodes, d, maps, p) for p in range(P)]
    comm = LocalPeerTransport(ops) if peer else LocalTransport()
    return setup(ops, comm, precondition=precondition), maps
