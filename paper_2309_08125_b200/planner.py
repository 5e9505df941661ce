"""Python API over the C ABI (same names as include/oobleck_plan.h, marshalling only).

    from paper_2309_08125_b200 import planner
    prof = planner.Profile.from_arrays(fwd_ms, bwd_ms)          # host arrays [L][M]
    sets = planner.generate_templates([prof], nodes=N, gpus_per_node=M, f=f, n0=n0)
    plan = planner.instantiate(sets, 0, nodes=N', f=f, global_batch=B, microbatch=b)
    nb, obj = planner.distribute_batch(T, B, b)

The device-resident path used by bench.py is `DPPlan` (inputs already in HBM).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import (OOB_E_BATCH, OOB_E_TOO_MANY, OOB_OK, OobDpInfo, OobError, OobPlanOpts,
                   OobTemplate, check, lib)


class Profile:
    """Owning wrapper of an oob_profile handle."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_arrays(cls, fwd_ms, bwd_ms, state_bytes=None) -> "Profile":
        fwd = np.ascontiguousarray(fwd_ms, dtype=np.float64)
        bwd = np.ascontiguousarray(bwd_ms, dtype=np.float64)
        if fwd.ndim != 2 or fwd.shape != bwd.shape:
            raise ValueError("fwd_ms/bwd_ms must be [L][M] arrays of the same shape")
        L, M = fwd.shape
        st = None
        if state_bytes is not None:
            st = np.ascontiguousarray(state_bytes, dtype=np.int64)
        h = ctypes.c_void_p()
        check(lib.oob_profile_from_arrays(L, M, fwd.ctypes.data, bwd.ctypes.data,
                                          None if st is None else st.ctypes.data, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "Profile":
        h = ctypes.c_void_p()
        check(lib.oob_load_profile(path.encode(), ctypes.byref(h)))
        return cls(h)

    @property
    def L(self) -> int:
        return lib.oob_profile_layers(self._h)

    @property
    def M(self) -> int:
        return lib.oob_profile_gpus_per_node(self._h)

    def costs(self):
        """(fwd_ms, bwd_ms [L][M], state_bytes [L]) as held by the library (oob_profile_costs)."""
        f = np.zeros((self.L, self.M))
        b = np.zeros((self.L, self.M))
        st = np.zeros(self.L, np.int64)
        check(lib.oob_profile_costs(self._h, f.ctypes.data, b.ctypes.data, st.ctypes.data))
        return f, b, st

    def min_nodes(self, nodes: int, gpu_mem_bytes: int, util: float = 0.8, samples_per_gpu: int = 1) -> int:
        out = ctypes.c_int32()
        check(lib.oob_min_nodes(self._h, nodes, gpu_mem_bytes, util, samples_per_gpu, ctypes.byref(out)))
        return out.value

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.oob_profile_free(self._h)
            self._h = None


def load_profile(path: str) -> Profile:
    return Profile.load(path)


def node_sizes(nodes: int, f: int, n0: int, layers: int) -> list[int]:
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    check(lib.oob_node_sizes(nodes, f, n0, layers, ctypes.byref(lo), ctypes.byref(hi)))
    return list(range(lo.value, hi.value + 1))


def _template_dict(t: OobTemplate) -> dict:
    st = [(t.stages[j].layer_begin, t.stages[j].layer_end, t.stages[j].gpus, t.stages[j].node,
           t.stages[j].gpu_offset) for j in range(t.num_stages)]
    return {"nodes": t.nodes, "S": t.num_stages, "stages": st, "T1": t.t1_ms, "T2": t.t2_ms,
            "T3": t.t3_ms, "kstar": t.kstar, "tstar": t.tstar_ms, "total": t.iter_ms}


class TemplateSet:
    """Owning wrapper of an oob_template_set handle."""

    def __init__(self, handle):
        self._h = handle

    @property
    def num_profiles(self) -> int:
        return lib.oob_template_set_profiles(self._h)

    def count(self, profile: int = 0) -> int:
        return lib.oob_template_count(self._h, profile)

    def get(self, profile: int, i: int):
        """Template i (size n_lo + i) as a dict; None when the size has no allowed mapping
        (stage masks)."""
        t = OobTemplate()
        check(lib.oob_template_get(self._h, profile, i, ctypes.byref(t)))
        return _template_dict(t) if t.num_stages > 0 else None

    def templates(self, profile: int = 0) -> list[dict]:
        return [self.get(profile, i) for i in range(self.count(profile))]

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.oob_template_set_free(self._h)
            self._h = None


def generate_templates(profiles, nodes: int, gpus_per_node: int, f: int, n0: int = 0,
                       gpu_mem_bytes: int = 0, util: float = 0.8, samples_per_gpu: int = 1,
                       device: int = -1, stream: int = 0, workspace: int = 0,
                       workspace_bytes: int = 0, comm: "NcclComm | None" = None, tp_pow2: bool = False,
                       stage_mem_bytes: float = 0.0, exact: bool = False) -> TemplateSet:
    """oob_generate_templates: host profiles in, template set out (H2D + GPU DP + D2H).
    exact=True: the exact optimum of the 1F1B objective per size (oob_exact_run) instead of
    the paper's recursion.
    With `comm` (an NcclComm of world > 1, every rank passing the same profiles): one
    profile is sharded per wavefront across the ranks, a batch of profiles in contiguous
    blocks with one all-gather; every rank gets the whole set.  tp_pow2 / stage_mem_bytes:
    the stage masks of reading R31 (infeasible sizes come back as None)."""
    profs = [p if isinstance(p, Profile) else Profile.from_arrays(*p) for p in profiles]
    arr = (ctypes.c_void_p * len(profs))(*[p._h for p in profs])
    opts = OobPlanOpts(nodes=nodes, gpus_per_node=gpus_per_node, f=f, n0=n0,
                       gpu_mem_bytes=gpu_mem_bytes, util=util, samples_per_gpu=samples_per_gpu,
                       device=device, stream=stream or None, workspace=workspace or None,
                       workspace_bytes=workspace_bytes, comm=comm.handle if comm is not None else None,
                       world=comm.world if comm is not None else 1, rank=comm.rank if comm is not None else 0,
                       tp_pow2=1 if tp_pow2 else 0, stage_mem_bytes=stage_mem_bytes, exact=1 if exact else 0)
    h = ctypes.c_void_p()
    check(lib.oob_generate_templates(arr, len(profs), ctypes.byref(opts), ctypes.byref(h)))
    ts = TemplateSet(h)
    ts._keep = profs
    return ts


def exact_workspace_bytes(L: int, M: int, n_lo: int, n_hi: int, num_profiles: int = 1) -> int:
    """oob_exact_workspace_bytes for the current device."""
    b = ctypes.c_size_t(0)
    check(lib.oob_exact_workspace_bytes(L, M, n_lo, n_hi, num_profiles, ctypes.byref(b)))
    return b.value


def exact_run(L: int, M: int, n_lo: int, n_hi: int, num_profiles: int, d_fwd: int, d_bwd: int, d_packed_ub: int,
              d_workspace: int, workspace_bytes: int, d_packed_out: int, stream: int = 0) -> None:
    """oob_exact_run: exact-optimum templates into d_packed_out (oob_dp_run's layout);
    d_packed_ub = the recursion's packed output (bounds the search) or 0."""
    check(lib.oob_exact_run(L, M, n_lo, n_hi, num_profiles, d_fwd, d_bwd, d_packed_ub or None, d_workspace,
                            workspace_bytes, d_packed_out, stream or None))


class DPPlan:
    """oob_dp_plan: the device-resident DP (inputs already in HBM)."""

    def __init__(self, L: int, M: int, n_lo: int, n_hi: int, num_profiles: int = 1):
        h = ctypes.c_void_p()
        check(lib.oob_dp_plan_create(L, M, n_lo, n_hi, num_profiles, ctypes.byref(h)))
        self._h = h
        self.info = OobDpInfo()
        check(lib.oob_dp_plan_info(self._h, ctypes.byref(self.info)))

    def run(self, d_fwd: int, d_bwd: int, d_workspace: int, workspace_bytes: int, d_packed: int,
            stream: int = 0) -> None:
        check(lib.oob_dp_run(self._h, d_fwd, d_bwd, d_workspace, workspace_bytes, d_packed, stream or None))

    def set_comm(self, comm: "NcclComm | None") -> None:
        """oob_dp_set_comm: shard this plan's wavefronts across the communicator's ranks
        (every rank runs the same profile); refreshes `info` (the workspace grows)."""
        if comm is None:
            check(lib.oob_dp_set_comm(self._h, None, 1, 0))
        else:
            check(lib.oob_dp_set_comm(self._h, comm.handle, comm.world, comm.rank))
            self._comm = comm
        check(lib.oob_dp_plan_info(self._h, ctypes.byref(self.info)))

    def set_virtual_shards(self, world: int) -> None:
        """oob_dp_set_virtual_shards: the sharded algorithm with `world` virtual ranks on
        this GPU (test mode); refreshes `info` (per-rank workspace grows)."""
        check(lib.oob_dp_set_virtual_shards(self._h, world))
        check(lib.oob_dp_plan_info(self._h, ctypes.byref(self.info)))

    def run_virtual(self, d_fwd: int, d_bwd: int, d_workspaces, workspace_bytes: int, d_packed,
                    stream: int = 0) -> None:
        """oob_dp_run_virtual: every virtual rank r on this device (workspace / output r)."""
        ws = (ctypes.c_void_p * len(d_workspaces))(*d_workspaces)
        pk = (ctypes.c_void_p * len(d_packed))(*d_packed)
        check(lib.oob_dp_run_virtual(self._h, d_fwd, d_bwd, ws, workspace_bytes, pk, stream or None))

    def set_timing(self, enable: bool) -> None:
        check(lib.oob_dp_set_timing(self._h, 1 if enable else 0))

    def kernel_time(self, reset: bool = True):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        check(lib.oob_dp_kernel_time(self._h, ctypes.byref(ms), ctypes.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def template_set(self, host_packed: np.ndarray) -> TemplateSet:
        buf = np.ascontiguousarray(host_packed)
        if buf.nbytes < self.info.packed_bytes:
            raise ValueError("packed buffer too small")
        h = ctypes.c_void_p()
        check(lib.oob_template_set_from_packed(buf.ctypes.data, ctypes.byref(self.info), ctypes.byref(h)))
        return TemplateSet(h)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.oob_dp_plan_free(self._h)
            self._h = None


class NcclComm:
    """An NCCL communicator owned by the library (oob_nccl_comm_create); the unique id is
    created by rank 0 and broadcast over an existing torch.distributed process group."""

    def __init__(self, world: int, rank: int, device: int, group=None):
        import torch
        import torch.distributed as dist
        buf = torch.zeros(_lib.NCCL_ID_BYTES, dtype=torch.uint8)
        if rank == 0:
            idb = (ctypes.c_uint8 * _lib.NCCL_ID_BYTES)()
            check(lib.oob_nccl_unique_id(idb))
            buf = torch.tensor(list(idb), dtype=torch.uint8)
        if world > 1:
            if dist.get_backend(group) == "nccl":
                dev_buf = buf.cuda(device)
                dist.broadcast(dev_buf, 0, group=group)
                buf = dev_buf.cpu()
            else:
                dist.broadcast(buf, 0, group=group)
        idb = (ctypes.c_uint8 * _lib.NCCL_ID_BYTES)(*buf.tolist())
        h = ctypes.c_void_p()
        check(lib.oob_nccl_comm_create(idb, world, rank, device, ctypes.byref(h)))
        self.handle, self.world, self.rank = h, world, rank

    def allgather(self, d_send: int, d_recv: int, bytes_per_rank: int, stream: int = 0) -> None:
        """oob_nccl_allgather: d_recv[r * bytes_per_rank:] <- rank r's d_send (device)."""
        check(lib.oob_nccl_allgather(self.handle, d_send, d_recv, bytes_per_rank, stream or None))

    def __del__(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.oob_nccl_comm_destroy(self.handle)
            self.handle = None


def dp_info(L: int, M: int, n_lo: int, n_hi: int, num_profiles: int = 1) -> OobDpInfo:
    return DPPlan(L, M, n_lo, n_hi, num_profiles).info


def count_sets(n_lo: int, n_hi: int, nodes: int, f: int) -> int:
    out = ctypes.c_int64()
    check(lib.oob_count_sets(n_lo, n_hi, nodes, f, ctypes.byref(out)))
    return out.value


def instantiate(tset: TemplateSet, profile: int, nodes: int, f: int, global_batch: int,
                microbatch: int, max_enumerated: int = 0) -> dict:
    """oob_instantiate: best plan for `nodes` nodes (Eq.5 + Eq.6 + throughput)."""
    p = tset.count(profile)
    counts = np.zeros(p, np.int32)
    maxp = max(1, nodes)
    nb = np.zeros(maxp, np.int64)
    npipes, thr, it = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
    nfeas, rec = ctypes.c_int64(), ctypes.c_int64()
    st = lib.oob_instantiate(tset._h, profile, nodes, f, global_batch, microbatch, max_enumerated,
                             counts.ctypes.data, nb.ctypes.data, maxp, ctypes.byref(npipes),
                             ctypes.byref(thr), ctypes.byref(it), ctypes.byref(nfeas), ctypes.byref(rec))
    if st not in (OOB_OK, OOB_E_TOO_MANY):
        check(st, {"recommended_global_batch": rec.value})
    return {"counts": tuple(int(c) for c in counts), "nb": tuple(int(x) for x in nb[:npipes.value]),
            "throughput": thr.value, "iteration_ms": it.value, "num_feasible": nfeas.value,
            "capped": st == OOB_E_TOO_MANY}


def instantiate_all(tset: TemplateSet, profile: int, n_min: int, n_max: int, f: int, global_batch: int,
                    microbatch: int, max_enumerated: int = 0) -> list[dict]:
    """oob_instantiate_all: the plan for every node count n_min..n_max (certified bounds)."""
    p = tset.count(profile)
    n = n_max - n_min + 1
    counts = np.zeros((n, p), np.int32)
    thr, ub = np.zeros(n), np.zeros(n)
    exact, status = np.zeros(n, np.int32), np.zeros(n, np.int32)
    check(lib.oob_instantiate_all(tset._h, profile, n_min, n_max, f, global_batch, microbatch, max_enumerated,
                                  counts.ctypes.data, thr.ctypes.data, ub.ctypes.data, exact.ctypes.data,
                                  status.ctypes.data))
    return [{"nodes": n_min + k, "counts": tuple(int(c) for c in counts[k]), "throughput": float(thr[k]),
             "upper_bound": float(ub[k]), "exact": bool(exact[k]), "status": int(status[k])} for k in range(n)]


def distribute_batch(per_microbatch_ms, global_batch: int, microbatch: int):
    """oob_distribute_batch: exact Eq.6; returns (nb tuple, objective)."""
    T = np.ascontiguousarray(per_microbatch_ms, dtype=np.float64)
    nb = np.zeros(T.shape[0], np.int64)
    obj, rec = ctypes.c_double(), ctypes.c_int64()
    st = lib.oob_distribute_batch(T.ctypes.data, T.shape[0], global_batch, microbatch, nb.ctypes.data,
                                  ctypes.byref(obj), ctypes.byref(rec))
    check(st, {"recommended_global_batch": rec.value})
    return tuple(int(x) for x in nb), obj.value


def recommend_batch(x: int, microbatch: int, global_batch: int) -> int:
    return int(lib.oob_recommend_batch(x, microbatch, global_batch))


ACTION_NAMES = {_lib.OOB_ACT_REINSTANTIATE: "reinstantiate", _lib.OOB_ACT_BORROW: "borrow",
                _lib.OOB_ACT_MERGE: "merge", _lib.OOB_ACT_REMOVE: "remove", _lib.OOB_ACT_REPLAN: "replan"}


class ExecState:
    """oob_exec: pipelines instantiated from a template set, reconfigured on failures
    (PAPER §5: reinstantiate / borrow / merge, batch redistribution, copy plan, sync groups)."""

    def __init__(self, tset: TemplateSet, profile: int, f: int, global_batch: int, microbatch: int,
                 counts, node_ids, layer_bytes=None):
        c = np.ascontiguousarray(counts, dtype=np.int32)
        ids = np.ascontiguousarray(node_ids, dtype=np.int32)
        lb = None if layer_bytes is None else np.ascontiguousarray(layer_bytes, dtype=np.int64)
        h = ctypes.c_void_p()
        check(lib.oob_exec_create(tset._h, profile, f, global_batch, microbatch, c.ctypes.data, ids.ctypes.data,
                                  ids.shape[0], None if lb is None else lb.ctypes.data, ctypes.byref(h)))
        self._h = h
        self._keep = tset

    def pipelines(self):
        """[(node ids, microbatches)] per pipeline."""
        out = []
        buf = np.zeros(4096, np.int32)
        for i in range(lib.oob_exec_num_pipelines(self._h)):
            n, nb = ctypes.c_int32(), ctypes.c_int64()
            check(lib.oob_exec_pipeline(self._h, i, buf.ctypes.data, buf.shape[0], ctypes.byref(n), ctypes.byref(nb)))
            out.append((list(int(x) for x in buf[:n.value]), nb.value))
        return out

    def fail(self, failed):
        """oob_exec_fail: returns (actions, transfers) of the reconfiguration."""
        f = np.ascontiguousarray(sorted(failed), dtype=np.int32)
        rec = ctypes.c_int64()
        check(lib.oob_exec_fail(self._h, f.ctypes.data, f.shape[0], ctypes.byref(rec)),
              {"recommended_global_batch": rec.value})
        return self.actions(), self.transfers()

    def actions(self):
        out = []
        a = _lib.OobAction()
        for i in range(lib.oob_exec_num_actions(self._h)):
            check(lib.oob_exec_action(self._h, i, ctypes.byref(a)))
            name = ACTION_NAMES[a.kind]
            out.append((name, a.a) if name in ("remove", "replan") else
                       (name, a.a, a.nodes) if name == "reinstantiate" else (name, a.a, a.b))
        return out

    def transfers(self):
        out = []
        t = _lib.OobTransfer()
        for i in range(lib.oob_exec_num_transfers(self._h)):
            check(lib.oob_exec_transfer(self._h, i, ctypes.byref(t)))
            out.append((t.layer, t.donor, t.receiver, t.bytes))
        return out

    def sync_group(self, layer: int):
        p = np.zeros(1024, np.int32)
        s = np.zeros(1024, np.int32)
        n = ctypes.c_int32()
        check(lib.oob_exec_sync_group(self._h, layer, p.ctypes.data, s.ctypes.data, 1024, ctypes.byref(n)))
        return [(int(a), int(b)) for a, b in zip(p[:n.value], s[:n.value])]

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.oob_exec_free(self._h)
            self._h = None
