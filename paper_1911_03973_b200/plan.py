"""Execution plan handle (ebs_plan_t): incidence, internal numbering, slot stream.

A plan is built once per (connectivity, node count) and owns its device
workspace.  An operator (A_e, b_e) is packed into its slot stream on demand;
the plan remembers which element batch and which Dirichlet set are loaded.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import torch

from . import _device as D
from ._lib import call, load


class Plan:
    def __init__(self, indt: torch.Tensor, n_nodes: int):
        indt = D.i32(indt)
        if indt.ndim != 2 or indt.shape[0] not in (3, 4):
            raise ValueError(f"indt must have shape (3|4, n_e), got {tuple(indt.shape)}")
        n_e = indt.shape[1]
        if n_e and int(indt.max()) >= n_nodes:
            raise ValueError("element connectivity references nonexistent nodes")
        h = ctypes.c_void_p()
        call("ebs_plan_create", indt.shape[0], int(n_nodes), n_e, D.ptr(indt), D.stream(),
             ctypes.byref(h))
        self.handle = h
        self.n_b = indt.shape[0]
        self.n_nodes = int(n_nodes)
        self.n_elements = n_e
        self._loaded = None       # weakref to the loaded ElementBatch
        self._loaded_be = False
        self._dirichlet = None    # weakref/key of the loaded Dirichlet set
        # held from ensure_loaded / ensure_dirichlet through the enqueue of the operation
        # that uses them (batches sharing one plan, e.g. A_e and the mass slices, may be
        # used from several threads); re-entrant for solver callbacks
        self.lock = threading.RLock()
        self._finalizer = weakref.finalize(self, _destroy, h.value)

    # ------------------------------------------------------------- info --
    def info(self) -> dict:
        buf = (ctypes.c_int64 * 8)()
        call("ebs_plan_info", self.handle, buf)
        keys = ("n_nodes", "n_elems", "n_b", "n_chunks", "n_rows", "slot_bytes",
                "max_valence", "loaded")
        return dict(zip(keys, (int(v) for v in buf)))

    def node_maps(self):
        """(new_of_old, old_of_new) int32 device tensors."""
        a = D.empty(self.n_nodes, torch.int32)
        b = D.empty(self.n_nodes, torch.int32)
        call("ebs_plan_node_maps", self.handle, D.ptr(a), D.ptr(b), D.stream())
        return a, b

    # ----------------------------------------------------------- operator --
    def ensure_loaded(self, batch, need_be=True):
        cur = self._loaded() if self._loaded is not None else None
        if cur is batch and (self._loaded_be or not need_be):
            return
        A = batch._A_store()
        b_e = batch.b_e if need_be or batch.b_e is not None else None
        call("ebs_plan_load", self.handle, D.ptr(A), D.ptr(b_e), D.stream())
        self._loaded = weakref.ref(batch)
        self._loaded_be = b_e is not None

    def ensure_dirichlet(self, d):
        key = None if d is None else id(d)
        cur = self._dirichlet
        if cur is not None and cur[0] == key and (key is None or cur[1]() is d):
            return
        if d is None:
            call("ebs_plan_set_dirichlet", self.handle, ctypes.c_void_p(0), 0, D.stream())
            self._dirichlet = (None, None)
        else:
            nd = d.nd
            call("ebs_plan_set_dirichlet", self.handle, D.ptr(nd), nd.numel(), D.stream())
            self._dirichlet = (key, weakref.ref(d))


def _destroy(handle):
    try:
        torch.cuda.synchronize()
    except Exception:
        pass
    load().ebs_plan_destroy(ctypes.c_void_p(handle))
