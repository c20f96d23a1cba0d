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


# ------------------------------------------------ slab-distributed cycle (§8e)
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slab_vertex_rows_partition(world):
    for depth in range(2, 8):
        N = 3 ** depth
        if N // 3 < world:
            with pytest.raises(ValueError):
                parallel.slab_vertex_rows(N, world, 0)
            continue
        rows = [parallel.slab_vertex_rows(N, world, r) for r in range(world)]
        assert [v for a, b in rows for v in range(a, b)] == list(range(N + 1))  # every vertex row once
        for a, b in rows:
            assert a % 3 == 0 and (b % 3 == 0 or b == N + 1) and b - a >= 3
        # level-(D-1) rows: vertex row 3*IY of the slab, together every coarse row once
        coarse = [(a // 3, (b + 2) // 3) for a, b in rows]
        assert [v for a, b in coarse for v in range(a, b)] == list(range(N // 3 + 1))


def _comm_worker(rank, world, port, depth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = parallel.TorchComm()
        N = 3 ** depth
        n = N + 1
        v0, v1 = parallel.slab_vertex_rows(N, world, rank)
        owner = [parallel.slab_vertex_rows(N, world, r) for r in range(world)]

        def own(row):
            return next(r for r, (a, b) in enumerate(owner) if a <= row < b)

        t = torch.full((n * n,), -1.0, dtype=torch.float64)
        for row in range(v0, v1):
            t[row * n:(row + 1) * n] = 1000.0 * rank + row
        comm.halo_tensor(t, n, v0, v1, 3)
        ok_halo = True
        for row in list(range(max(v0 - 3, 0), v0)) + list(range(v1, min(v1 + 3, n))):
            ok_halo &= bool(torch.all(t[row * n:(row + 1) * n] == 1000.0 * own(row) + row))
        for row in range(v0, v1):  # own rows untouched
            ok_halo &= bool(torch.all(t[row * n:(row + 1) * n] == 1000.0 * rank + row))
        # all-gather of level-(D-1) rows
        nc = N // 3 + 1
        ranges = [(a // 3, (b + 2) // 3) for a, b in owner]
        c = torch.full((nc * nc,), -1.0, dtype=torch.float64)
        a, b = ranges[rank]
        for row in range(a, b):
            c[row * nc:(row + 1) * nc] = 7.0 * row + 0.5
        comm.allgather_tensor(c, nc, ranges)
        ok_gather = bool(torch.all(c.view(nc, nc) == (7.0 * torch.arange(nc, dtype=torch.float64) + 0.5)[:, None]))
        slots = [rank + k for k in range(20)]
        norm2, red = comm.reduce([(0.25 * (rank + 1), slots)])
        q.put((rank, ok_halo, ok_gather, norm2, red))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,depth", [(2, 2), (3, 3), (2, 3)])
def test_gloo_dist_comm_halo_gather_reduce(world, depth):
    """The exchanges of the distributed cycle on CPU tensors (gloo): halo rows
    arrive from their owners, own rows stay, level-(D-1) rows are gathered
    everywhere, and the result slots reduce by sum / max as the C side expects."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_halo, ok_gather, norm2, red in out:
        assert ok_halo, f"rank {rank}: halo rows"
        assert ok_gather, f"rank {rank}: gathered rows"
        assert norm2 == pytest.approx(sum(0.25 * (r + 1) for r in range(world)))
        for k in range(20):
            want = max(r + k for r in range(world)) if k in parallel.MAX_SLOTS else sum(r + k for r in range(world))
            assert red[k] == want


def _dist_vs_single(depth, world, solver, cycles, field=None):
    import paper_2005_03606_b200 as lzb
    f = field or lzb.field_theta(16.0)
    d = lzb.make_desc(depth=depth, field=f, solver=solver, omega=0.6, rhs_kind="sinprod", max_cycles=200,
                      delta_max=1e-8)
    ref = lzb.Grid(d, 42)
    ref.assemble_fixed(3)
    want = [ref.step() for _ in range(cycles)]
    grids = [lzb.Grid(d, 42) for _ in range(world)]
    for g in grids:
        g.assemble_fixed(3)
    slabs = [parallel.Slab(g, r, world) for r, g in enumerate(grids)]
    comm = parallel.LoopbackComm(torch.cuda.ExternalStream(lzb.default_context().solve_stream))
    got = [parallel.dist_cycle(slabs, comm, solver == "adafac-pi") for _ in range(cycles)]
    return ref, grids, want, got


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("solver", ["additive", "adafac-pi"])
def test_dist_cycle_loopback_bit_identical(world, solver):
    """The slab-distributed cycle (phases + exchanges, several slabs on the one
    GPU through device copies) against the one-GPU cycle: u, r and fl on every
    level bit for bit, residual norms to rounding of the regrouped sum."""
    import paper_2005_03606_b200 as lzb
    depth = 4
    ref, grids, want, got = _dist_vs_single(depth, world, solver, 6)
    for w, g in zip(want, got):
        assert g["status"] == w["status"] and g["cycle"] == w["cycle"]
        assert g["residual"] == pytest.approx(w["residual"], rel=1e-12)
        assert g["dof_updates"] == w["dof_updates"] and g["max_n"] == w["max_n"]
        assert g["factor_totals"] == w["factor_totals"]
    N = 3 ** depth
    for r, g in enumerate(grids):
        # leaf level: the slab's rows (a rank never updates the others' rows)
        v0, v1 = parallel.slab_vertex_rows(N, world, r)
        for fld in (lzb.T.V_U, lzb.T.V_R, lzb.T.V_RHAT, lzb.T.V_DIAG):
            a = g.vertices(depth, fld).reshape(N + 1, N + 1)[v0:v1]
            assert np.array_equal(a, ref.vertices(depth, fld).reshape(N + 1, N + 1)[v0:v1]), (r, fld)
        # coarse levels: replicated, everything
        for lvl in range(depth):
            for fld in (lzb.T.V_U, lzb.T.V_FL, lzb.T.V_R):
                assert np.array_equal(g.vertices(lvl, fld), ref.vertices(lvl, fld)), (r, lvl, fld)


@pytest.mark.gpu
def test_dist_cycle_loopback_runs_to_convergence():
    import paper_2005_03606_b200 as lzb
    f = lzb.field_sinusoid(0.9, 6.0)
    d = lzb.make_desc(depth=5, field=f, solver="adafac-pi", omega=0.6, rhs_kind="sinprod", max_cycles=300,
                      target=1e-10)
    ref = lzb.Grid(d, 42)
    ref.assemble_fixed(4)
    want = ref.run()
    grids = [lzb.Grid(d, 42) for _ in range(4)]
    for g in grids:
        g.assemble_fixed(4)
    slabs = [parallel.Slab(g, r, 4) for r, g in enumerate(grids)]
    comm = parallel.LoopbackComm(torch.cuda.ExternalStream(lzb.default_context().solve_stream))
    got = []
    while True:
        got.append(parallel.dist_cycle(slabs, comm, True))
        if got[-1]["status"] != lzb.T.CONTINUE:
            break
    assert len(got) == len(want) and got[-1]["status"] == want[-1]["status"] == lzb.T.CONVERGED
    N = 3 ** 5
    v0, v1 = parallel.slab_vertex_rows(N, 4, 2)
    assert np.array_equal(grids[2].vertices(5, lzb.T.V_U).reshape(N + 1, N + 1)[v0:v1],
                          ref.vertices(5, lzb.T.V_U).reshape(N + 1, N + 1)[v0:v1])


@pytest.mark.gpu
def test_dist_cycle_nccl_world1():
    """The NCCL exchange layer (TorchComm) on the device at world size 1."""
    import paper_2005_03606_b200 as lzb
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1)
    try:
        f = lzb.field_theta(16.0)
        d = lzb.make_desc(depth=4, field=f, solver="adafac-pi", omega=0.6, rhs_kind="sinprod", max_cycles=50)
        ref, g = lzb.Grid(d, 7), lzb.Grid(d, 7)
        ref.assemble_fixed(2)
        g.assemble_fixed(2)
        slab = parallel.Slab(g, 0, 1)
        comm = parallel.TorchComm(stream=torch.cuda.ExternalStream(lzb.default_context().solve_stream))
        for _ in range(4):
            w, r = ref.step(), parallel.dist_cycle([slab], comm, True)
            assert r["residual"] == pytest.approx(w["residual"], rel=1e-12)
        assert np.array_equal(g.vertices(4, lzb.T.V_U), ref.vertices(4, lzb.T.V_U))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_set_slab_rejects_bad_rows():
    import paper_2005_03606_b200 as lzb
    d = lzb.make_desc(depth=3, field=lzb.field_theta(1.0), solver="additive")
    g = lzb.Grid(d, 1)
    for v0, v1 in ((1, 9), (0, 10), (3, 3), (0, 29), (-3, 9)):
        with pytest.raises(lzb.LzbError):
            g.set_slab(v0, v1)
    dj = lzb.make_desc(depth=3, field=lzb.field_theta(1.0), solver="adafac-jac")
    with pytest.raises(lzb.LzbError):
        lzb.Grid(dj, 1).set_slab(0, 9)
