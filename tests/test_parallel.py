"""Multi-rank host logic of the slab decomposition, world size 2
on CPU with the gloo backend; the device path at world size 1 (NCCL) on GPU.

The CPU tests use the oracle's element integration as the per-rank local
compute, so what they check is the decomposition itself: slab partition,
padding of uneven slabs, the all-gather and the reassembly into the full
array must reproduce the single-process result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_03606_b200 import parallel


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slab_rows_partition(world):
    for N in (1, 3, 9, 27, 81, 243, 729, 2187):
        slabs = parallel.all_slabs(N, world)
        covered = [r for a, b in slabs for r in range(a, b)]
        assert covered == list(range(N))  # contiguous, covering, disjoint, ordered
        for a, b in slabs:
            assert (a % 3 == 0 or a == N) and (b % 3 == 0 or b == N)  # level-(D-1) patches never split
        sizes = [b - a for a, b in slabs]
        assert max(sizes) - min(sizes) <= 3


def _worker(rank, world, port, depth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import port as orc
        f = orc.field_from_keys({"setup": "checkerboard", "field-seed": "5", "blocks": "8"})
        N = 3 ** depth
        h = np.power(1.0 / 3, depth)
        full = torch.zeros(N * N * 16, dtype=torch.float64)
        r0, r1 = parallel.slab_rows(N, world, rank)
        for cy in range(r0, r1):
            for cx in range(N):
                c = cy * N + cx
                full[16 * c:16 * c + 16] = torch.from_numpy(orc.integrate_element(f, cx * h, cy * h, h, 3))
        parallel.gather_rows(None, full, 16 * N, N)
        # single-process reference
        want = np.zeros(N * N * 16)
        for c in range(N * N):
            want[16 * c:16 * c + 16] = orc.integrate_element(f, (c % N) * h, (c // N) * h, h, 3)
        same = bool(np.array_equal(full.numpy(), want))
        mx = parallel.max_over_ranks(rank + 1.5)
        sm = parallel.sum_over_ranks([rank, 1.0])
        q.put((rank, same, mx, list(sm), (r0, r1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("depth", [2, 3])
def test_gloo_slab_gather_reproduces_single_process(depth):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N = 3 ** depth
    slabs = sorted(o[4] for o in out)
    assert slabs == parallel.all_slabs(N, world)
    for rank, same, mx, sm, _ in out:
        assert same, f"rank {rank}: gathered operator differs from the single-process one"
        assert mx == world - 1 + 1.5
        assert sm == [sum(range(world)), float(world)]


@pytest.mark.gpu
def test_distributed_assemble_world1_matches_single_gpu():
    """The device path of the decomposition (NCCL, world size 1 on the one GPU
    of this pool): slab assembly + all-gather + replicated cycles reproduce the
    single-grid run bit for bit."""
    import paper_2005_03606_b200 as lzb
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1)
    f = lzb.checkerboard(2, 8)
    d = lzb.make_desc(depth=4, field=f, solver="additive", omega=0.6, rhs=1.0, max_cycles=20)
    a, b = lzb.Grid(d, 3), lzb.Grid(d, 3)
    parallel.distributed_assemble(a, 4)
    b.assemble_fixed(4)
    assert np.array_equal(a.cells(4)["ops"], b.cells(4)["ops"])
    ra, rb = [a.step() for _ in range(5)], [b.step() for _ in range(5)]
    assert [r["residual"] for r in ra] == [r["residual"] for r in rb]
    assert np.array_equal(a.vertices(4, 0), b.vertices(4, 0))
    dist.destroy_process_group()
