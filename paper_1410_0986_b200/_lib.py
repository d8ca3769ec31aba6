"""Loader for the in-tree C-ABI library libhydot_b200.so (include/hydot_b200.h).

There is no fallback: if the library is missing the import fails loudly with
the build command.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhydot_b200.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p

HYDOT_OK, HYDOT_EINVAL, HYDOT_ERUNTIME, HYDOT_ENOMEM, HYDOT_ECUDA, HYDOT_ENCCL = range(6)


class Grid7(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("h", C.c_double)]


class Ledger(C.Structure):
    _fields_ = [("leaf", C.c_double), ("agglomeration", C.c_double),
                ("recompress", C.c_double), ("other", C.c_double),
                ("kernel_tally", C.c_double)]

    def category_total(self):
        return self.leaf + self.agglomeration + self.recompress + self.other


BLOCK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, _dp, C.c_int64)


class Provider(C.Structure):
    _fields_ = [("rows_per_source", C.c_int), ("cols", C.c_int64), ("block", BLOCK_FN),
                ("user", C.c_void_p)]


MV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
MM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                    C.c_void_p)


class LinOp(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("mv", MV_FN), ("rmv", MV_FN),
                ("mm", MM_FN), ("rmm", MM_FN), ("user", C.c_void_p)]


class BornFields(C.Structure):
    _fields_ = [("N", C.c_int64), ("n_lambda", C.c_int), ("n_sources", C.c_int),
                ("n_det", C.c_int), ("incident_dev_h", C.POINTER(_dp)),
                ("adjoint_dev_h", C.POINTER(_dp)), ("w_dev", _dp), ("nu", C.c_double),
                ("ready_events_h", C.POINTER(C.c_void_p))]


class RecOpts(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("p", C.c_int), ("kprobe", C.c_int),
                ("hint_mode", C.c_int), ("source_ids", C.POINTER(C.c_int)),
                ("node_offset", C.c_int)]


class GridGeom(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("Lx", C.c_double),
                ("Ly", C.c_double), ("Lz", C.c_double)]


class KrylovConfig(C.Structure):
    _fields_ = [("arnoldi_steps", C.c_int), ("deflation_dim", C.c_int), ("restart", C.c_int),
                ("tol", C.c_double), ("max_restarts", C.c_int), ("center_shifts", C.c_int),
                ("jacobi", C.c_int), ("explicit_qr_update", C.c_int)]


class KrylovStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("matvecs", C.c_int), ("relres", C.c_double),
                ("converged", C.c_int), ("phase1_relres", C.c_double)]


class KrylovFamily(C.Structure):
    _fields_ = [("phase1_steps", C.c_int), ("deflation_k", C.c_int), ("rank_reduced", C.c_int),
                ("pencil_shifted", C.c_int), ("breakdown", C.c_int), ("cholesky_failed", C.c_int),
                ("all_converged", C.c_int), ("first_failure", C.c_int)]


class PalsParams(C.Structure):
    _fields_ = [("np", C.c_int), ("alpha", _dp), ("beta", _dp), ("centers", _dp),
                ("tau_level", C.c_double), ("eps_H", C.c_double), ("nu_norm", C.c_double)]


class Hop(C.Structure):
    _fields_ = [("H", _vp), ("row_perm_dev", _ip)]


class ReconConfig(C.Structure):
    _fields_ = [("max_outer", C.c_int), ("max_inner", C.c_int), ("max_retries", C.c_int),
                ("gamma", C.c_double), ("nu0", C.c_double), ("stagnation_tol", C.c_double),
                ("fixed_c_h", _dp), ("normal_blocks", C.c_int)]


class TraceRowC(C.Structure):
    _fields_ = [("outer", C.c_int), ("inner", C.c_int), ("resnorm", C.c_double),
                ("nu", C.c_double), ("accepted", C.c_int), ("dice", C.c_double)]


class ReconResultC(C.Structure):
    _fields_ = [("p", PalsParams), ("c_h", _dp), ("trace_h", C.POINTER(TraceRowC)),
                ("trace_cap", C.c_int), ("trace_len", C.c_int), ("resnorm", C.c_double),
                ("converged", C.c_int), ("flagged", C.c_int), ("hmv_calls", C.c_int64),
                ("hmv_columns", C.c_int64), ("normal_columns", C.c_int64)]


# name -> (restype, argtypes); exactly the declarations of include/hydot_b200.h
SIGNATURES = {
    "hydot_version": (C.c_int, []),
    "hydot_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "hydot_ctx_destroy": (C.c_int, [_vp]),
    "hydot_last_error": (C.c_char_p, [_vp]),
    "hydot_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "hydot_ctx_synchronize": (C.c_int, [_vp]),
    "hydot_ctx_launch_count": (C.c_int64, [_vp]),
    "hydot_profile_dump": (C.c_int, [C.c_char_p, C.c_int]),
    "hydot_ctx_set_timing": (C.c_int, [_vp, C.c_int]),
    "hydot_ctx_timing_report": (C.c_int, [_vp, C.c_char_p, C.c_int]),
    "hydot_ctx_set_timing_filter": (C.c_int, [_vp, C.c_char_p]),
    "hydot_fields_solve": (C.c_int, [_vp, C.POINTER(Grid7), C.c_int, _dp, _dp, _dp, _i64p, C.c_int,
                                     C.c_double, C.c_int, C.c_int, _dp, _ip, _dp]),
    "hydot_apply7": (C.c_int, [_vp, C.POINTER(Grid7), C.c_double, C.c_double, _dp, _dp]),
    "hydot_born_block": (C.c_int, [_vp, C.c_int64, C.c_int, _dp, C.POINTER(_dp), C.c_int, _dp,
                                   C.c_double, _dp, C.c_int64]),
    "hydot_gaussian": (C.c_int, [_vp, C.c_uint64, C.c_int64, C.c_int64, _dp]),
    "hydot_mt19937_64": (C.c_int, [_vp, C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]),
    "hydot_rng_selftest": (C.c_int, []),
    "hydot_factor_create": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _dp, C.c_int64, _dp,
                                      C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(_vp)]),
    "hydot_factor_info": (C.c_int, [_vp, _i64p, _i64p, _i64p, _dp, _ip, _ip]),
    "hydot_factor_download": (C.c_int, [_vp, _vp, _dp, _dp, C.c_int]),
    "hydot_factor_device_ptrs": (C.c_int, [_vp, C.POINTER(_dp), C.POINTER(_dp)]),
    "hydot_factor_free": (None, [_vp]),
    "hydot_randsvd": (C.c_int, [_vp, C.c_int64, C.c_int64, _dp, C.c_int64, C.c_double, C.c_int,
                                C.c_int, C.c_uint64, C.c_int, C.c_int, C.POINTER(_vp),
                                C.POINTER(Ledger)]),
    "hydot_randsvd_linop": (C.c_int, [_vp, C.POINTER(LinOp), C.c_double, C.c_int, C.c_int,
                                      C.c_uint64, C.c_int, C.c_int, C.POINTER(_vp),
                                      C.POINTER(Ledger)]),
    "hydot_agglomerate": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                    C.c_int, C.POINTER(_vp), C.POINTER(Ledger)]),
    "hydot_tolerance_schedule": (C.c_int, [C.c_double, C.c_int, C.c_int, _dp]),
    "hydot_tree_build": (C.c_int, [_dp, C.c_int, C.c_int, _dp, _dp, C.POINTER(_vp)]),
    "hydot_tree_num_nodes": (C.c_int, [_vp]),
    "hydot_tree_root": (C.c_int, [_vp]),
    "hydot_tree_depth": (C.c_int, [_vp]),
    "hydot_tree_node": (C.c_int, [_vp, C.c_int, _ip, _ip, _ip, _ip]),
    "hydot_tree_leaf_order": (C.c_int, [_vp, _ip]),
    "hydot_tree_node_box": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "hydot_tree_free": (None, [_vp]),
    "hydot_recursive_lowrank": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(Provider),
                                          C.POINTER(BornFields), C.POINTER(RecOpts),
                                          C.POINTER(_vp), _ip, _ip, _ip, C.POINTER(Ledger)]),
    "hydot_recompress": (C.c_int, [_vp, _vp, C.c_double, C.c_int, C.POINTER(_vp),
                                   C.POINTER(Ledger)]),
    "hydot_lr_matmat": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _dp, C.c_int64, _dp, C.c_int64]),
    "hydot_full_forward": (C.c_int, [_vp, C.POINTER(Grid7), C.c_int, _dp, _dp, _dp, _dp, _dp, _i64p, C.c_int,
                                     _i64p, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp, _ip]),
    "hydot_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "hydot_comm_create": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_ubyte), C.POINTER(_vp)]),
    "hydot_comm_destroy": (C.c_int, [_vp]),
    "hydot_comm_info": (C.c_int, [_vp, _ip, _ip]),
    "hydot_comm_allreduce": (C.c_int, [_vp, _vp, _dp, C.c_int64]),
    "hydot_j_matmat_voxel": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _dp, C.c_int64, _dp, C.c_int64, C.c_int64,
                                       _ip, _dp, C.c_int, C.c_int, _dp, C.c_int64, _dp, C.c_int64]),
    "hydot_j_matmat": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _ip, _dp, C.c_int, C.c_int, _dp,
                                 C.c_int64, _dp, C.c_int64]),
    "hydot_thin_svd": (C.c_int, [_vp, C.c_int64, C.c_int64, _dp, C.c_int64, _dp, _dp, _dp]),
    "hydot_householder_qr": (C.c_int, [_vp, C.c_int64, C.c_int64, _dp, C.c_int64, _dp, _dp]),
    "hydot_dgemm": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                              _dp, C.c_int64, _dp, C.c_int64, C.c_double, _dp, C.c_int64]),
    "hydot_pals_eval": (C.c_int, [_vp, C.c_int, C.POINTER(GridGeom), C.POINTER(PalsParams), _dp,
                                  C.c_int64]),
    "hydot_pals_hmv": (C.c_int, [_vp, C.POINTER(Hop), C.c_int, _dp, C.c_int64, _dp, C.c_int64]),
    "hydot_pals_solve_concentrations": (C.c_int, [_vp, C.POINTER(Hop), _dp, _dp, _dp, _dp, C.c_int,
                                                  C.c_int, _dp, _ip]),
    "hydot_pals_lm_step": (C.c_int, [_vp, C.c_int64, C.c_int, _dp, C.c_int64, _dp, C.c_double,
                                     _dp]),
    "hydot_pals_metrics": (C.c_int, [_vp, C.c_int64, _dp, _dp, C.c_double, _dp, _dp, _ip]),
    "hydot_pals_reconstruct": (C.c_int, [_vp, C.POINTER(Hop), C.POINTER(GridGeom), _dp, C.c_int,
                                         C.c_int, _dp, _dp, C.POINTER(PalsParams), C.c_double,
                                         C.POINTER(ReconConfig), _dp, C.POINTER(ReconResultC)]),
    "hydot_factor_save": (C.c_int, [_vp, _vp, _ip, C.c_int64, C.c_char_p]),
    "hydot_factor_file_info": (C.c_int, [C.c_char_p, _i64p, _i64p, _i64p, _i64p]),
    "hydot_factor_load": (C.c_int, [_vp, C.c_char_p, C.POINTER(_vp), _ip, C.c_int64]),
    "hydot_block_save": (C.c_int, [_vp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_char_p]),
    "hydot_block_file_info": (C.c_int, [C.c_char_p, _i64p, _i64p]),
    "hydot_block_load": (C.c_int, [_vp, C.c_char_p, _dp, C.c_int64, C.c_int64, _i64p, _i64p]),
    "hydot_apply_fem": (C.c_int, [_vp, C.POINTER(GridGeom), C.c_double, C.c_double, _dp, _dp]),
    "hydot_fields_solve_fem": (C.c_int, [_vp, C.POINTER(GridGeom), C.c_int, _dp, _dp, _dp, _dp, C.c_int,
                                         C.c_double, C.c_int, C.c_int, _dp, _ip, _dp]),
    "hydot_krylov_config_default": (None, [C.POINTER(KrylovConfig)]),
    "hydot_solve_family_fem": (C.c_int, [_vp, C.POINTER(GridGeom), C.c_int, _dp, _dp, _dp, C.c_int,
                                         C.POINTER(KrylovConfig), _dp, C.POINTER(KrylovStats),
                                         C.POINTER(KrylovFamily)]),
    "hydot_fields_solve_fem_gmres": (C.c_int, [_vp, C.POINTER(GridGeom), C.c_int, _dp, _dp, _dp, _dp,
                                               C.c_int, C.POINTER(KrylovConfig), _dp,
                                               C.POINTER(KrylovStats), C.POINTER(KrylovFamily)]),
}

_LIB = None


def build():
    import subprocess
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(_HERE, "csrc")], check=True)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
                "paper_1410_0986_b200/csrc).  There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


class HydotError(RuntimeError):
    pass


def check(rc, ctx=None):
    if rc == HYDOT_OK:
        return
    msg = lib().hydot_last_error(ctx).decode(errors="replace")
    if rc == HYDOT_EINVAL:
        raise ValueError(msg)
    if rc == HYDOT_ENOMEM:
        raise MemoryError(msg)
    raise HydotError(f"[status {rc}] {msg}")
