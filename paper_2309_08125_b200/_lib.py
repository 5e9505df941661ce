"""Thin ctypes binding of include/oobleck_plan.h (argument marshalling only).

Every step of the planning path runs inside liboobleck_plan.so (CUDA kernels for the DP,
C++ for the host steps).  There is no Python or CPU fallback: if the library is missing,
importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liboobleck_plan.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback for the planner)")

_lib = ctypes.CDLL(LIB_PATH)

c_int32, c_int64, c_double, c_size_t, c_void_p = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                                  ctypes.c_size_t, ctypes.c_void_p)

OOB_OK, OOB_E_PARSE, OOB_E_INVALID, OOB_E_INFEASIBLE, OOB_E_BATCH, OOB_E_TOO_MANY, OOB_E_CUDA, \
    OOB_E_NCCL, OOB_E_NOMEM = range(9)


class OobStage(ctypes.Structure):
    _fields_ = [("layer_begin", c_int32), ("layer_end", c_int32), ("gpus", c_int32),
                ("node", c_int32), ("gpu_offset", c_int32)]


class OobTemplate(ctypes.Structure):
    _fields_ = [("nodes", c_int32), ("num_stages", c_int32), ("kstar", c_int32), ("reserved", c_int32),
                ("t1_ms", c_double), ("t2_ms", c_double), ("t3_ms", c_double), ("tstar_ms", c_double),
                ("iter_ms", c_double), ("stages", ctypes.POINTER(OobStage))]


class OobPlanOpts(ctypes.Structure):
    _fields_ = [("nodes", c_int32), ("gpus_per_node", c_int32), ("f", c_int32), ("n0", c_int32),
                ("gpu_mem_bytes", c_int64), ("util", c_double), ("samples_per_gpu", c_int32),
                ("device", c_int32), ("stream", c_void_p), ("workspace", c_void_p),
                ("workspace_bytes", c_size_t), ("comm", c_void_p), ("world", c_int32), ("rank", c_int32),
                ("tp_pow2", c_int32), ("stage_mem_bytes", c_double), ("exact", c_int32)]


class OobDpInfo(ctypes.Structure):
    _fields_ = [("L", c_int32), ("M", c_int32), ("n_lo", c_int32), ("n_hi", c_int32),
                ("num_profiles", c_int32), ("wavefronts", c_int32),
                ("cells_per_profile", c_int64), ("splits_per_profile", c_int64),
                ("kernel_launches", c_int64), ("workspace_bytes", c_size_t),
                ("packed_template_bytes", c_size_t), ("packed_profile_bytes", c_size_t),
                ("packed_bytes", c_size_t), ("kernel", c_int32), ("pipelined", c_int32),
                ("fused", c_int32), ("seeded", c_int32), ("chunk_max", c_int32), ("refresh", c_int32),
                ("small_pairs", c_int32), ("num_sms", c_int32), ("world", c_int32), ("warp_waves", c_int32),
                ("small_range", c_int32), ("exchange", c_int32)]


class OobAction(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("a", c_int32), ("b", c_int32), ("nodes", c_int32)]


class OobTransfer(ctypes.Structure):
    _fields_ = [("layer", c_int32), ("donor", c_int32), ("receiver", c_int32), ("reserved", c_int32),
                ("bytes", c_int64)]


OOB_ACT_REINSTANTIATE, OOB_ACT_BORROW, OOB_ACT_MERGE, OOB_ACT_REMOVE, OOB_ACT_REPLAN = 1, 2, 3, 4, 5


def _proto(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


P = ctypes.POINTER
_proto("oob_last_error", ctypes.c_char_p, [])
_proto("oob_status_string", ctypes.c_char_p, [ctypes.c_int])
_proto("oob_load_profile", ctypes.c_int, [ctypes.c_char_p, P(c_void_p)])
_proto("oob_profile_from_arrays", ctypes.c_int, [c_int32, c_int32, c_void_p, c_void_p, c_void_p, P(c_void_p)])
_proto("oob_profile_free", None, [c_void_p])
_proto("oob_profile_layers", c_int32, [c_void_p])
_proto("oob_profile_gpus_per_node", c_int32, [c_void_p])
_proto("oob_profile_costs", ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p])
_proto("oob_min_nodes", ctypes.c_int, [c_void_p, c_int32, c_int64, c_double, c_int32, P(c_int32)])
_proto("oob_node_sizes", ctypes.c_int, [c_int32, c_int32, c_int32, c_int32, P(c_int32), P(c_int32)])
_proto("oob_generate_templates", ctypes.c_int, [P(c_void_p), c_int32, P(OobPlanOpts), P(c_void_p)])
_proto("oob_template_set_profiles", c_int32, [c_void_p])
_proto("oob_template_count", c_int32, [c_void_p, c_int32])
_proto("oob_template_get", ctypes.c_int, [c_void_p, c_int32, c_int32, P(OobTemplate)])
_proto("oob_template_set_free", None, [c_void_p])
_proto("oob_dp_plan_create", ctypes.c_int, [c_int32, c_int32, c_int32, c_int32, c_int32, P(c_void_p)])
_proto("oob_dp_plan_free", None, [c_void_p])
_proto("oob_dp_plan_info", ctypes.c_int, [c_void_p, P(OobDpInfo)])
_proto("oob_dp_run", ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p])
_proto("oob_dp_set_timing", ctypes.c_int, [c_void_p, c_int32])
_proto("oob_dp_set_stage_masks", ctypes.c_int, [c_void_p, c_int32, c_void_p, c_double])
_proto("oob_dp_kernel_time", ctypes.c_int, [c_void_p, P(c_double), P(c_int64), c_int32])
_proto("oob_template_set_from_packed", ctypes.c_int, [c_void_p, P(OobDpInfo), P(c_void_p)])
_proto("oob_nccl_unique_id", ctypes.c_int, [c_void_p])
_proto("oob_nccl_comm_create", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, P(c_void_p)])
_proto("oob_nccl_comm_destroy", None, [c_void_p])
_proto("oob_dp_set_comm", ctypes.c_int, [c_void_p, c_void_p, c_int32, c_int32])
_proto("oob_nccl_allgather", ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p])
_proto("oob_dp_set_virtual_shards", ctypes.c_int, [c_void_p, c_int32])
_proto("oob_dp_run_virtual", ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p])
_proto("oob_instantiate", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_int64, c_int32, c_int64,
                                         c_void_p, c_void_p, c_int32, P(c_int32), P(c_double), P(c_double),
                                         P(c_int64), P(c_int64)])
_proto("oob_count_sets", ctypes.c_int, [c_int32, c_int32, c_int32, c_int32, P(c_int64)])
_proto("oob_instantiate_all", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int64, c_int32, c_int64,
                                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p])
_proto("oob_distribute_batch", ctypes.c_int, [c_void_p, c_int32, c_int64, c_int32, c_void_p, P(c_double),
                                              P(c_int64)])
_proto("oob_recommend_batch", c_int64, [c_int32, c_int32, c_int64])
_proto("oob_exec_create", ctypes.c_int, [c_void_p, c_int32, c_int32, c_int64, c_int32, c_void_p, c_void_p, c_int32,
                                         c_void_p, P(c_void_p)])
_proto("oob_exec_free", None, [c_void_p])
_proto("oob_exec_num_pipelines", c_int32, [c_void_p])
_proto("oob_exec_pipeline", ctypes.c_int, [c_void_p, c_int32, c_void_p, c_int32, P(c_int32), P(c_int64)])
_proto("oob_exec_fail", ctypes.c_int, [c_void_p, c_void_p, c_int32, P(c_int64)])
_proto("oob_exec_num_actions", c_int32, [c_void_p])
_proto("oob_exec_action", ctypes.c_int, [c_void_p, c_int32, P(OobAction)])
_proto("oob_exec_num_transfers", c_int32, [c_void_p])
_proto("oob_exec_transfer", ctypes.c_int, [c_void_p, c_int32, P(OobTransfer)])
_proto("oob_exec_sync_group", ctypes.c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, P(c_int32)])
_proto("oob_exact_workspace_bytes", ctypes.c_int, [c_int32, c_int32, c_int32, c_int32, c_int32, P(c_size_t)])
_proto("oob_exact_run", ctypes.c_int, [c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_size_t, c_void_p, c_void_p])

EXPORTED = [
    "oob_last_error", "oob_status_string", "oob_load_profile", "oob_profile_from_arrays",
    "oob_profile_free", "oob_profile_layers", "oob_profile_gpus_per_node", "oob_profile_costs", "oob_min_nodes",
    "oob_node_sizes", "oob_generate_templates", "oob_template_set_profiles", "oob_template_count",
    "oob_template_get", "oob_template_set_free", "oob_dp_plan_create", "oob_dp_plan_free",
    "oob_dp_plan_info", "oob_dp_run", "oob_dp_set_timing", "oob_dp_kernel_time",
    "oob_template_set_from_packed", "oob_instantiate", "oob_count_sets", "oob_distribute_batch",
    "oob_recommend_batch", "oob_nccl_unique_id", "oob_nccl_comm_create", "oob_nccl_comm_destroy",
    "oob_dp_set_comm", "oob_nccl_allgather", "oob_dp_set_virtual_shards", "oob_dp_run_virtual",
    "oob_instantiate_all", "oob_dp_set_stage_masks", "oob_exec_create", "oob_exec_free", "oob_exec_num_pipelines", "oob_exec_pipeline", "oob_exec_fail",
    "oob_exec_num_actions", "oob_exec_action", "oob_exec_num_transfers", "oob_exec_transfer", "oob_exec_sync_group",
    "oob_exact_workspace_bytes", "oob_exact_run",
]
NCCL_ID_BYTES = 128


class OobError(RuntimeError):
    def __init__(self, status: int, msg: str, payload=None):
        super().__init__(f"{_lib.oob_status_string(status).decode()}: {msg}")
        self.status = status
        self.payload = payload


def check(status: int, payload=None):
    if status != OOB_OK:
        raise OobError(status, _lib.oob_last_error().decode(errors="replace"), payload)


lib = _lib
