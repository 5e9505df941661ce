"""Host logic of the N>1 path on CPU: world-size-2 gloo process group.

Each rank owns a contiguous shard of a batched sweep (paper_2309_08125_b200.dist.shard),
produces the packed template sets of its shard (here with the C oracle standing in for the
GPU, test infrastructure only), all-gathers them (dist.allgather_packed) and rebuilds the
whole set through the C ABI (oob_template_set_from_packed); every profile must equal the
oracle's set.  The GPU itself is exercised by tests/test_gpu_parity.py and bench.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import coracle
from tests.helpers import pack_templates
from workloads import random_profile

L, M, N, F, N0 = 9, 2, 7, 1, 1
N_HI = min(N - F * N0, L)
NUM_PROFILES = 5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _profiles():
    kinds = ["uniform", "lognormal", "integer", "spiky", "constant"]
    return [random_profile(400 + i, L, M, kinds[i % len(kinds)]) for i in range(NUM_PROFILES)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_08125_b200 import dist as odist
        from paper_2309_08125_b200 import planner
        profs = _profiles()
        first, cnt = odist.shard(NUM_PROFILES, world, rank)
        mine = [coracle.template_set(p.fwd_ms, p.bwd_ms, M, N0, N_HI)[0] for p in profs[first:first + cnt]]
        packed = pack_templates(mine, L, M, N0, N_HI)[0] if mine else np.zeros(0, np.uint8)
        per_rank = (NUM_PROFILES + world - 1) // world
        tpl_bytes = (64 + L * 20 + 63) // 64 * 64
        profile_bytes = tpl_bytes * (N_HI - N0 + 1)
        assert packed.nbytes == cnt * profile_bytes
        gathered = odist.allgather_packed(torch.from_numpy(packed.copy()), per_rank * profile_bytes)
        whole = odist.unshard(gathered, NUM_PROFILES, world, profile_bytes).numpy()
        dinfo = planner.OobDpInfo(L=L, M=M, n_lo=N0, n_hi=N_HI, num_profiles=NUM_PROFILES, wavefronts=0,
                                  cells_per_profile=0, splits_per_profile=0, kernel_launches=0,
                                  workspace_bytes=0, packed_template_bytes=tpl_bytes,
                                  packed_profile_bytes=profile_bytes,
                                  packed_bytes=profile_bytes * NUM_PROFILES)
        import ctypes
        h = ctypes.c_void_p()
        planner.check(planner.lib.oob_template_set_from_packed(whole.ctypes.data, ctypes.byref(dinfo),
                                                                ctypes.byref(h)))
        ts = planner.TemplateSet(h)
        ok = True
        for i, p in enumerate(profs):
            want = coracle.template_set(p.fwd_ms, p.bwd_ms, M, N0, N_HI)[0]
            ok = ok and ts.templates(i) == want
        q.put((rank, ok, first, cnt))
    finally:
        dist.destroy_process_group()


def test_shard_covers_every_profile_once():
    from paper_2309_08125_b200 import dist as odist
    for n in (0, 1, 5, 8, 1024, 1023):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, cnt = odist.shard(n, world, r)
                seen.extend(range(first, first + cnt))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        odist.shard(4, 2, 2)


def test_gloo_world2_gather_rebuilds_template_set():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(q.get() for _ in range(world))
    assert [r[0] for r in results] == [0, 1]
    assert all(ok for _, ok, _, _ in results), results
    assert sum(c for *_, c in results) == NUM_PROFILES
    for p in procs:
        assert p.exitcode == 0
