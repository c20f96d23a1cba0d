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
    return {"op": device_tensor(op, 16 * nc, "<f8"), "p1": device_tensor(p1, nc, "<i4"),
            "n": device_tensor(n, nc, "<i4"), "p3": device_tensor(p3, nc, "|i1"),
            # u32 arrays travel as i32 (same bits; torch's NCCL group has no uint32)
            "epoch": device_tensor(ep, nc, "<i4"), "chg": device_tensor(chg, nc, "<i4")}


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
    p3 = t["p3"].to(torch.int32)
    gather_rows(None, p3, N, N, group)
    t["p3"].copy_(p3.to(torch.int8))
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
