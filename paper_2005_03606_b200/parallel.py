"""Multi-GPU decomposition of the delayed-assembly path.

One process per GPU (torchrun), `torch.distributed` for the plumbing: NCCL on
the GPU box, gloo in the CPU tests. The grid is cut into slabs of whole
leaf-cell rows along y; slab boundaries are multiples of 3 rows so every
level-(D-1) patch (3x3 leaves) lives on one rank.

* Assembly (integration + compression + publish) is embarrassingly parallel
  over cells: each rank integrates its slab, no data-path collective.
* To solve, the assembled slabs are exchanged once with an all-gather of the
  leaf state (operators, markers, change epochs) into every rank's grid, after
  which the cycle runs replicated. The NCCL halo exchange of a slab-distributed
  smoother is the next step.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def slab_rows(n_rows: int, world: int, rank: int, align: int = 3) -> tuple[int, int]:
    """Row range [r0, r1) of `rank`: contiguous, covering, disjoint, boundaries
    at multiples of `align`, sizes balanced to one `align` unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    units = (n_rows + align - 1) // align
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return min(n_rows, u0 * align), min(n_rows, u1 * align)


def all_slabs(n_rows: int, world: int, align: int = 3):
    return [slab_rows(n_rows, world, r, align) for r in range(world)]


def gather_rows(local, full, row_elems: int, n_rows: int, group=None):
    """All-gather slab rows into `full` (a 1-D torch tensor of n_rows*row_elems
    elements on any device the backend supports); `local` holds this rank's
    slab, already written in place inside `full` (it is re-read from there).
    Uneven slabs are padded to the largest slab for the collective."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    slabs = all_slabs(n_rows, world)
    maxr = max(r1 - r0 for r0, r1 in slabs)
    r0, r1 = slabs[rank]
    send = torch.zeros(maxr * row_elems, dtype=full.dtype, device=full.device)
    send[: (r1 - r0) * row_elems] = full[r0 * row_elems:r1 * row_elems]
    recv = torch.empty(world * maxr * row_elems, dtype=full.dtype, device=full.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for q, (a, b) in enumerate(slabs):
        if q == rank or b <= a:
            continue
        full[a * row_elems:b * row_elems] = recv[q * maxr * row_elems:q * maxr * row_elems + (b - a) * row_elems]
    del local
    return full


class _CudaArray:
    """__cuda_array_interface__ view of device memory owned by liblzb."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def device_tensor(ptr: int, count: int, typestr: str):
    """A torch tensor aliasing `count` elements at device pointer `ptr` (no copy)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, (count,), typestr), device="cuda")


def leaf_tensors(grid):
    """Torch views of the leaf level's cell arrays of a paper_2005_03606_b200.Grid."""
    import paper_2005_03606_b200 as lzb

    ptrs = [C.c_void_p() for _ in range(6)]
    lzb._check(lzb.lib().lzb_grid_cell_arrays(grid.h, grid.depth, *[C.byref(p) for p in ptrs]))
    N = 3 ** grid.depth
    nc = N * N
    op, p1, n, p3, ep, chg = (p.value for p in ptrs)
    out = {"op": device_tensor(op, 16 * nc, "<f8"), "p1": device_tensor(p1, nc, "<i4"),
           "n": device_tensor(n, nc, "<i4"), "p3": device_tensor(p3, nc, "|i1"),
           # u32 arrays travel as i32 (same bits; torch's NCCL group has no uint32)
           "epoch": device_tensor(ep, nc, "<i4"), "chg": device_tensor(chg, nc, "<i4")}
    planes, cp3, width = C.c_void_p(), C.c_void_p(), C.c_int()
    lzb._check(lzb.lib().lzb_grid_plane_arrays(grid.h, C.byref(planes), C.byref(cp3), C.byref(width)))
    if width.value:  # the compressed records the residual reads
        out["planes"] = device_tensor(planes.value, 16 * width.value * nc, "|u1")
        out["cp3"] = device_tensor(cp3.value, nc, "|i1")
    return out


def distributed_assemble(grid, n: int, group=None):
    """Fixed-p assembly of this rank's slab, then one all-gather of the leaf
    state so every rank holds the whole assembled operator (replicated solve).
    Returns (r0, r1) of the local slab."""
    import torch
    import torch.distributed as dist

    import paper_2005_03606_b200 as lzb

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    N = 3 ** grid.depth
    r0, r1 = slab_rows(N, world, rank)
    if r1 > r0:
        lzb._check(lzb.lib().lzb_grid_assemble_rows(grid.h, n, r0, r1))
    t = leaf_tensors(grid)
    torch.cuda.synchronize()
    for key, per_cell in (("op", 16), ("p1", 1), ("n", 1), ("epoch", 1), ("chg", 1)):
        gather_rows(None, t[key], per_cell * N, N, group)
    # i8 markers travel as i32 (NCCL has int8, but keep one code path for gloo)
    for key in ("p3", "cp3"):
        if key in t:
            v = t[key].to(torch.int32)
            gather_rows(None, v, N, N, group)
            t[key].copy_(v.to(torch.int8))
    if "planes" in t:
        w = t["planes"].numel() // (N * N)
        gather_rows(None, t["planes"], w * N, N, group)
    torch.cuda.synchronize()
    lzb._check(lzb.lib().lzb_grid_invalidate(grid.h))
    return r0, r1


def max_over_ranks(x: float, group=None, device=None) -> float:
    """Max of a scalar over ranks (device timing: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x, group=None, device=None):
    import torch
    import torch.distributed as dist

    arr = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return arr
    t = torch.tensor(arr, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


# ------------------------------------------------------ slab-distributed cycle
# the leaf level's vertex rows are cut into slabs (multiples of
# 3), one per rank; the coarse levels run replicated. Grid.dist_phase 0..5 do
# the compute (csrc/grid.cu, Grid::dist_phase); this layer does the exchanges
# in between: NCCL point-to-point halos and all-gathers of level-(D-1) rows
# over torch.distributed (TorchComm), or device copies between several slabs
# of one process (LoopbackComm, the one-GPU test of the same plan).

# Result slots reduced by max (S_MAXN, S_MAXDELTA as non-negative double bits,
# S_MAXSAMPLES); every other slot is a count, reduced by sum.
MAX_SLOTS = (11, 14, 15)


def slab_vertex_rows(n_cells: int, world: int, rank: int) -> tuple[int, int]:
    """Leaf vertex rows [v0, v1) of `rank`: the cell-row slab of slab_rows
    (boundaries at multiples of 3); the last rank also owns vertex row N."""
    if n_cells // 3 < world:
        raise ValueError(f"{world} slabs need at least {3 * world} cell rows")
    r0, r1 = slab_rows(n_cells, world, rank)
    return r0, (n_cells + 1 if r1 >= n_cells else r1)


class Slab:
    """One rank's view: its Grid (whole-grid storage) and its leaf rows."""

    def __init__(self, grid, rank: int, world: int):
        self.grid, self.rank, self.world = grid, rank, world
        self.D = grid.depth
        self.N = 3 ** self.D
        self.v0, self.v1 = slab_vertex_rows(self.N, world, rank)
        self.c0, self.c1 = self.v0 // 3, (self.v1 + 2) // 3  # owned rows of level D-1
        grid.set_slab(self.v0, self.v1)

    dims = 2

    def row_elems(self, level: int) -> int:
        """Elements of one slab unit (a vertex row in 2D, a vertex plane in 3D)."""
        return (3 ** level + 1) ** (self.dims - 1)

    def field(self, level: int, fld: int):
        n = 3 ** level + 1
        return device_tensor(self.grid.device_view(level, fld), n ** self.dims, "<f8")


class Slab3(Slab):
    """One rank's view of a Grid3: z-slabs of leaf vertex planes."""

    dims = 3


def _row_ranges(slabs_or_plan, level_is_coarse: bool):
    return [(s.c0, s.c1) if level_is_coarse else (s.v0, s.v1) for s in slabs_or_plan]


class LoopbackComm:
    """All ranks in this process (one GPU): exchanges are device copies on the
    solve stream the slabs' kernels run on."""

    def __init__(self, stream=None):
        self.stream = stream

    def _ctx(self):
        import contextlib

        import torch
        return torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def halo(self, slabs, level, fld, depth):
        n = slabs[0].row_elems(level)
        nrows = 3 ** level + 1
        with self._ctx():
            for i, s in enumerate(slabs):
                t = s.field(level, fld)
                if i > 0:  # rows below the slab from the previous rank
                    a = max(s.v0 - depth, 0)
                    t[a * n:s.v0 * n].copy_(slabs[i - 1].field(level, fld)[a * n:s.v0 * n])
                if i + 1 < len(slabs):
                    b = min(s.v1 + depth, nrows)
                    t[s.v1 * n:b * n].copy_(slabs[i + 1].field(level, fld)[s.v1 * n:b * n])

    def allgather_rows(self, slabs, level, fld):
        n = slabs[0].row_elems(level)
        with self._ctx():
            for s in slabs:
                src = s.field(level, fld)[s.c0 * n:s.c1 * n]
                for o in slabs:
                    if o is not s:
                        o.field(level, fld)[s.c0 * n:s.c1 * n].copy_(src)

    def allgather_planes(self, slabs, level):
        Nc = 3 ** level
        views = [device_tensor(s.grid.level_ops_ptr(level), 27 * Nc ** 3, "<f8").view(27, Nc, Nc * Nc)
                 for s in slabs]
        with self._ctx():
            for s, v in zip(slabs, views):
                p0, p1 = coarse_cell_planes(s)
                for o in views:
                    if o is not v:
                        o[:, p0:p1].copy_(v[:, p0:p1])

    def reduce(self, results):
        norm2 = sum(r[0] for r in results)
        slots = [max(r[1][k] for r in results) if k in MAX_SLOTS else sum(r[1][k] for r in results)
                 for k in range(20)]
        return norm2, slots


class TorchComm:
    """One slab per process over torch.distributed: point-to-point halos
    (batch_isend_irecv) and padded all-gathers of level-(D-1) rows; NCCL on
    the GPU box (tensors alias liblzb device memory), gloo for CPU tensors."""

    def __init__(self, group=None, stream=None):
        self.group, self.stream = group, stream

    def _ctx(self):
        import contextlib

        import torch
        return torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def halo_tensor(self, t, n, v0, v1, depth):
        """Exchange `depth` rows (of n elements) of the flat row-major tensor t
        with the neighbouring ranks: send own boundary rows, receive theirs."""
        import torch.distributed as dist
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        nrows = t.numel() // n
        ops = []
        if rank > 0:
            a = max(v0 - depth, 0)
            ops.append(dist.P2POp(dist.isend, t[v0 * n:min(v0 + depth, v1) * n], rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, t[a * n:v0 * n], rank - 1, self.group))
        if rank + 1 < world:
            b = min(v1 + depth, nrows)
            ops.append(dist.P2POp(dist.isend, t[max(v1 - depth, v0) * n:v1 * n], rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, t[v1 * n:b * n], rank + 1, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def halo(self, slabs, level, fld, depth):
        (s,) = slabs
        with self._ctx():
            self.halo_tensor(s.field(level, fld), s.row_elems(level), s.v0, s.v1, depth)

    def allgather_tensor(self, t, n, ranges):
        """Every rank's rows [r0, r1) of t (n elements per row) into all ranks."""
        import torch
        import torch.distributed as dist
        rank = dist.get_rank(self.group)
        maxr = max(b - a for a, b in ranges)
        send = torch.zeros(maxr * n, dtype=t.dtype, device=t.device)
        a, b = ranges[rank]
        send[:(b - a) * n] = t[a * n:b * n]
        recv = torch.empty(len(ranges) * maxr * n, dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        for q, (a, b) in enumerate(ranges):
            if q != rank and b > a:
                t[a * n:b * n] = recv[q * maxr * n:q * maxr * n + (b - a) * n]

    def allgather_rows(self, slabs, level, fld):
        import torch.distributed as dist
        (s,) = slabs
        world = dist.get_world_size(self.group)
        ranges = []
        for r in range(world):
            v0, v1 = slab_vertex_rows(s.N, world, r)
            ranges.append((v0 // 3, (v1 + 2) // 3))
        with self._ctx():
            self.allgather_tensor(s.field(level, fld), s.row_elems(level), ranges)

    def allgather_planes(self, slabs, level):
        import torch.distributed as dist
        (s,) = slabs
        world = dist.get_world_size(self.group)
        Nc = 3 ** level
        ranges = []
        for r in range(world):
            v0, v1 = slab_vertex_rows(s.N, world, r)
            ranges.append((v0 // 3, min(v1, s.N) // 3))
        ops = device_tensor(s.grid.level_ops_ptr(level), 27 * Nc ** 3, "<f8")
        with self._ctx():
            for q in range(27):  # class plane q: rows of Nc^2 cells, one per coarse z plane
                self.allgather_tensor(ops[q * Nc ** 3:(q + 1) * Nc ** 3], Nc * Nc, ranges)

    def reduce(self, results, device=None):
        import torch
        import torch.distributed as dist
        ((norm2, slots),) = results
        dev = device or ("cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        sums = torch.tensor([0 if k in MAX_SLOTS else int(slots[k]) for k in range(20)], dtype=torch.int64,
                            device=dev)
        maxs = torch.tensor([int(slots[k]) if k in MAX_SLOTS else 0 for k in range(20)], dtype=torch.int64,
                            device=dev)
        n2 = torch.tensor([float(norm2)], dtype=torch.float64, device=dev)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(n2, op=dist.ReduceOp.SUM, group=self.group)
        s, m = sums.cpu().tolist(), maxs.cpu().tolist()
        return float(n2.item()), [m[k] if k in MAX_SLOTS else s[k] for k in range(20)]


def dist_cycle(slabs, comm, adafac_pi: bool) -> dict:
    """One slab-distributed cycle (Grid::dist_phase 0..5 with the exchanges in
    between); returns the cycle report (identical on every rank)."""
    import paper_2005_03606_b200 as lzb

    V = lzb.T
    D = slabs[0].D
    for s in slabs:
        s.grid.dist_phase(0, 1 if s.rank == 0 else 0)
    comm.halo(slabs, D, V.V_RHAT, 3)               # restriction reads r̂ 3 rows beyond the slab
    for s in slabs:
        s.grid.dist_phase(1)
    comm.allgather_rows(slabs, D - 1, V.V_FL)      # restricted load of level D-1
    for s in slabs:
        s.grid.dist_phase(2)
    norm2, slots = comm.reduce([s.grid.dist_result() for s in slabs])
    reps = [s.grid.dist_report(norm2, slots) for s in slabs]
    rep = reps[0]
    if rep["status"] in (V.CONTINUE, V.TIMEOUT):
        for s in slabs:
            s.grid.dist_phase(3)
        if adafac_pi:
            comm.allgather_rows(slabs, D - 1, V.V_AUX)  # injected residual of level D-1
        for s in slabs:
            s.grid.dist_phase(4)
        comm.allgather_rows(slabs, D - 1, V.V_U)        # injected solution of level D-1
        for s in slabs:
            s.grid.dist_phase(5)
        comm.halo(slabs, D, V.V_U, 1)                   # leaf u one row beyond the slab
    return rep


def coarse_cell_planes(s) -> tuple[int, int]:
    """Level-(D-1) cell planes [p0, p1) whose 27 children lie in slab s's leaf cells."""
    return s.v0 // 3, min(s.v1, s.N) // 3


def distributed_assemble3(slabs, comm, n: int):
    """z-slab sharded 3D assembly (assembly needs no exchange):
    each slab assembles the leaf cell planes its cycle reads (its vertex
    planes' cells and one layer below), the Galerkin operators of its
    level-(D-1) cell planes; one all-gather of the level-(D-1) class planes,
    then every rank recomputes the (small) levels below. After init_cycle;
    the result is bit-identical to a one-GPU assembly on the planes read."""
    for s in slabs:
        s.grid.assemble_planes(n, max(s.v0 - 1, 0), min(s.v1, s.N))
        s.grid.galerkin_planes(s.D - 1, *coarse_cell_planes(s))
    comm.allgather_planes(slabs, slabs[0].D - 1)
    for s in slabs:
        s.grid.coarse_below(s.D - 1)


def dist_cycle3(slabs, comm, adafac_pi: bool) -> dict:
    """One slab-distributed 3D cycle (Grid3.dist_phase 0..5 with the exchanges
    in between, z-slabs of vertex planes); returns the cycle report."""
    import paper_2005_03606_b200 as lzb

    V = lzb.T
    D = slabs[0].D
    for s in slabs:
        s.grid.dist_phase(0)
    comm.halo(slabs, D, V.V_RHAT, 3)
    for s in slabs:
        s.grid.dist_phase(1)
    comm.allgather_rows(slabs, D - 1, V.V_FL)
    for s in slabs:
        s.grid.dist_phase(2)
    norm2, _ = comm.reduce([s.grid.dist_result() for s in slabs])
    reps = [s.grid.dist_report(norm2) for s in slabs]
    rep = reps[0]
    if rep["status"] in (V.CONTINUE, V.TIMEOUT):
        for s in slabs:
            s.grid.dist_phase(3)
        if adafac_pi:
            comm.allgather_rows(slabs, D - 1, V.V_AUX)
        for s in slabs:
            s.grid.dist_phase(4)
        comm.allgather_rows(slabs, D - 1, V.V_U)
        for s in slabs:
            s.grid.dist_phase(5)
        comm.halo(slabs, D, V.V_U, 1)
    return rep
