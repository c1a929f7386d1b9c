"""ctypes binding of libebs.so (include/ebs.h).

The library is built in-tree (``paper_1911_03973_b200/libebs.so``, see
``csrc/Makefile`` / ``__graft_entry__.build``).  Loading it needs no GPU; every
compute entry point does.  There is no CPU fallback: when the library or the
device is missing, the first call raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_size_t, c_void_p, c_char_p

LIB_PATH = os.environ.get("EBS_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libebs.so")

EBS_OK = 0
EBS_EINVAL = -1
EBS_ENOMEM = -2
EBS_ECUDA = -3
EBS_ENCCL = -4
EBS_ENONFINITE = -5
EBS_EDEGENERATE = -6
EBS_ECALLBACK = -7

EBS_RES_EXACT = 0
EBS_RES_FAST = 1
EBS_APPLY_MASKED = 1
EBS_APPLY_ADD = 2

EBS_RICHARDSON = 0
EBS_JACOBI = 1
EBS_CG = 2
EBS_PCG = 3
EBS_CHEB2 = 4
EBS_CHEB3 = 5

CALLBACK = ctypes.CFUNCTYPE(c_int, c_void_p, c_int)


class SolveParams(ctypes.Structure):
    """Mirror of ebs_solve_params (include/ebs.h)."""
    _fields_ = [
        ("method", c_int), ("iters", c_int), ("exact", c_int), ("has_tol", c_int),
        ("tol", c_double), ("omega", c_double),
        ("x0", c_void_p), ("x", c_void_p), ("reference", c_void_p),
        ("norms", POINTER(c_double)), ("errors", POINTER(c_double)),
        ("n_norms", POINTER(c_int)), ("diverged", POINTER(c_int)),
        ("callback", CALLBACK), ("user", c_void_p), ("cb_x", c_void_p), ("cb_r", c_void_p),
        ("r_out", c_void_p),
        ("coef_a", POINTER(c_double)), ("coef_b", POINTER(c_double)),
        ("fused", c_int),
    ]


# name -> (restype, argtypes); every symbol declared in include/ebs.h
SIGNATURES = {
    "ebs_version": (c_int, []),
    "ebs_last_error": (c_int, [c_char_p, c_size_t]),
    "ebs_launch_count": (c_int64, []),
    "ebs_mesh_grid2d": (c_int, [c_int64, c_void_p, c_void_p, c_void_p]),
    "ebs_mesh_kuhn3d": (c_int, [c_int64, c_void_p, c_void_p, c_void_p]),
    "ebs_mesh_flags": (c_int, [c_int, c_int64, c_void_p, c_int, c_void_p, c_void_p]),
    "ebs_mesh_check": (c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_mesh_measure": (c_int, [c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_mesh_permute": (c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p]),
    "ebs_centroids": (c_int, [c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_assemble_p1": (c_int, [c_int, c_int64, c_void_p, c_void_p, c_double, c_void_p,
                                c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p]),
    "ebs_combine": (c_int, [c_int64, c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    "ebs_plan_create": (c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, POINTER(c_void_p)]),
    "ebs_plan_destroy": (c_int, [c_void_p]),
    "ebs_plan_info": (c_int, [c_void_p, POINTER(c_int64)]),
    "ebs_plan_node_maps": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_plan_load": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_plan_set_dirichlet": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "ebs_residual": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "ebs_residual_many": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int,
                                  c_int, c_void_p, c_void_p]),
    "ebs_residual_many_host": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                       c_int, c_int, c_void_p, c_void_p]),
    "ebs_matvec": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "ebs_diagonal": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_diagonal_grouped": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_assemble_rhs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_mask": (c_int, [c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ebs_check_finite": (c_int, [c_int64, c_void_p, c_void_p, c_void_p]),
    "ebs_to_internal": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_to_user": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_plan_apply": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "ebs_csr_nnz": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_csr_fill": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_dot": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_nrm2": (c_int, [c_int64, c_void_p, c_void_p, c_void_p]),
    "ebs_axpby": (c_int, [c_int64, c_double, c_void_p, c_double, c_void_p, c_void_p]),
    "ebs_solve": (c_int, [c_void_p, POINTER(SolveParams), c_void_p]),
    "ebs_power_iteration": (c_int, [c_void_p, c_void_p, c_int, c_double, POINTER(c_double),
                                    POINTER(c_int), c_void_p]),
    "ebs_gather": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_refine_tri": (c_int, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                               POINTER(c_int64), c_void_p]),
    "ebs_scatter_add": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_index_fill": (c_int, [c_int64, c_void_p, c_double, c_void_p, c_void_p]),
    "ebs_index_copy": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_index_move": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_index_add": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_plan_apply_map": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                   c_void_p]),
    "ebs_plan_apply_map_chunks": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p,
                                          c_void_p, c_void_p, c_int, c_void_p]),
    "ebs_vec_workspace_bytes": (c_size_t, []),
    "ebs_dist_combine": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "ebs_fill": (c_int, [c_int64, c_double, c_void_p, c_void_p]),
    "ebs_dist_unique_id": (c_int, [c_void_p]),
    "ebs_dist_init": (c_int, [c_void_p, c_void_p, c_int, c_int]),
    "ebs_dist_exchange": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "ebs_dist_allreduce": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "ebs_dist_poll": (c_int, [c_void_p]),
    "ebs_dist_wait": (c_int, [c_void_p, c_void_p, c_double]),
    "ebs_dist_abort": (c_int, [c_void_p]),
    "ebs_dist_set_stop": (c_int, [c_void_p, c_void_p]),
    "ebs_dist_combine_jacobi": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                        c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p]),
    "ebs_dist_combine_q": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p]),
    "ebs_vec_cg1_update": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_double, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_vec_jacobi": (c_int, [c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "ebs_vec_pcg_q": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "ebs_vec_pcg_update": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p]),
    "ebs_vec_pcg_direction": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p]),
    "ebs_vec_dot_owned": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "ebs_vec_dinv": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_dist_jacobi_sweep": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p]),
    "ebs_dist_matvec_sweep": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p]),
    "ebs_dist_jacobi_iface": (c_int, [c_int64, c_void_p, c_double, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p]),
    "ebs_dist_q_iface": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_plan_free_mask": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_plan_internal_rhs": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_plan_internal_diag": (c_int, [c_void_p, c_void_p, c_void_p]),
    # peer-memory halo (peer.cu)
    "ebs_peer_window_bytes": (c_size_t, [c_int64]),
    "ebs_peer_window_alloc": (c_int, [c_int64, POINTER(c_void_p), c_void_p]),
    "ebs_peer_window_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "ebs_peer_window_close": (c_int, [c_void_p]),
    "ebs_peer_window_free": (c_int, [c_void_p]),
    "ebs_peer_create": (c_int, [c_int, c_int, c_int64, c_void_p, c_double, POINTER(c_void_p)]),
    "ebs_peer_destroy": (c_int, [c_void_p]),
    "ebs_peer_set_halo": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p,
                                  c_void_p]),
    "ebs_peer_status": (c_int, [c_void_p, c_void_p]),
    "ebs_peer_allreduce": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "ebs_peer_send": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_peer_recv": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_push": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ebs_peer_combine": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_jacobi_sweep": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_double,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_matvec_sweep": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_residual_sweep": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                        c_void_p]),
    "ebs_peer_residual_combine": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p]),
    "ebs_peer_selftest": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_int64), c_void_p]),
    "ebs_peer_jacobi_step": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                     c_double, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_void_p]),
    "ebs_peer_combine_jacobi": (c_int, [c_void_p, c_void_p, c_double, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p]),
    "ebs_peer_combine_q": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_matvec_sweep_put": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                          c_void_p]),
    "ebs_peer_cg1_update_halo": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                         c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ebs_peer_cg1_update": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_double,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p]),
}

_lib = None


class EbsError(RuntimeError):
    pass


def load():
    """Load libebs.so (no GPU needed); raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make -C paper_1911_03973_b200/csrc`). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    load().ebs_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(code: int, what: str = ""):
    if code == EBS_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if code in (EBS_EINVAL, EBS_ENONFINITE, EBS_EDEGENERATE):
        raise ValueError(msg)
    if code == EBS_ENOMEM:
        raise MemoryError(msg)
    raise EbsError(f"[{code}] {msg}")


def call(name: str, *args):
    """Call an ebs_* entry point and map its status to a Python exception."""
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().ebs_launch_count())
