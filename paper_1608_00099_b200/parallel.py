"""Slab sharding of the TRIOT hot path over ranks (one process per GPU, torch.distributed).

P:607: "Parallelism could be automatically exploited by specializing the classes in the template
recursion that correspond to the outermost for loops ... This would allow multiple processors,
cores, or GPUs to simultaneously process partitions of tensors", and, for inner products, "each
thread computes its own pre-result and these pre-results are amalgamated together".

Here the partition is a slab of axis 0 (the outermost loop):

* embed and apply_binary need NO collective: rank r owns rows [lo, hi) of the output and reads
  only the matching rows of the inputs (`slab_rows`, `embed_slab`, `apply_binary_slab`);
* the expected value is the one exchange: each rank runs `triot_expected_value_offset` on its
  slab with the slab's origin (lo, 0, ..., 0) -- the kernel weights axis 0 by the global
  coordinate lo + t_0 -- the d-vectors are all-gathered (NCCL over NVLink for CUDA tensors, gloo
  in the CPU tests) and summed in rank order by `triot_sum_rows`, so the result is identical on
  every rank and deterministic run to run (an all-reduce would leave the summation order to the
  collective's algorithm).  No arithmetic happens outside the library's kernels.

`local_ev` / `sum_rows` let the host logic run with stand-ins for the GPU kernels (the CPU tests
pass the oracle); the defaults are the library's kernels.
"""
from __future__ import annotations


def slab_rows(n0: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous slab [lo, hi) of n0 rows for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (rank * n0) // world, ((rank + 1) * n0) // world


def leading_box(shape, world: int, rank: int) -> list[tuple[int, int]]:
    """This rank's box [lo_k, hi_k) per axis of a partition of the outermost loops:
    axis 0 in balanced slabs when it has at least as many indices as ranks; otherwise each
    axis-0 index goes to a contiguous group of ranks (rank r takes index r * n0 // world), which
    split the next axis the same way.  Boxes are disjoint and cover the shape."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    box = [(0, int(n)) for n in shape]
    r, nr = rank, world
    for k, n in enumerate(shape):
        n = int(n)
        if nr <= 1:
            break
        if n >= nr or k == len(shape) - 1:
            box[k] = slab_rows(n, nr, r)
            break
        i = (r * n) // nr
        box[k] = (i, i + 1)
        first, last = -(-i * nr // n), -(-(i + 1) * nr // n)   # ranks sharing index i
        r, nr = r - first, last - first
    return box


def embed_slab(dst_slab, src, lo: int, region_only: bool = False):
    """Rows [lo, lo + dst_slab.shape[0]) of embed(dst, src): dst_slab is this rank's slab of the
    global dst; src is the global src (or at least its rows from lo on) on this device."""
    from . import api
    hi = lo + dst_slab.shape[0]
    s_hi = min(hi, src.shape[0])
    src_part = src[lo:s_hi] if lo < s_hi else src[0:0]
    return api.embed(dst_slab, src_part.contiguous(), region_only=region_only)


def apply_binary_slab(a, b, lo: int, hi: int, op: str = "mul", out_slab=None, iter_shape=None):
    """Rows [lo, hi) of apply_binary(a, b): a, b are the global operands on this device."""
    from . import api
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    hi = min(hi, iter_shape[0])
    ish = (max(0, hi - lo),) + tuple(iter_shape[1:])
    return api.apply_binary(a[lo:hi].contiguous() if lo < hi else a[0:0],
                            b[lo:hi].contiguous() if lo < hi else b[0:0],
                            op, out=out_slab, iter_shape=ish)


def _default_local_ev(p_slab, offset):
    from . import api
    return api.expected_value(p_slab, offset=offset)


def _default_sum_rows(rows):
    from . import api
    return api.sum_rows(rows)


def expected_value_sharded(p_slab, lo: int, group=None, local_ev=None, sum_rows=None):
    """Global expected value of a p whose axis-0 rows [lo, lo + p_slab.shape[0]) this rank holds.

    Returns the same (d,) float64 tensor on every rank of `group`."""
    import torch
    import torch.distributed as dist

    local_ev = local_ev or _default_local_ev
    sum_rows = sum_rows or _default_sum_rows
    d = p_slab.dim()
    part = local_ev(p_slab, (lo,) + (0,) * (d - 1))
    world = dist.get_world_size(group)
    flat = torch.empty(world * d, dtype=torch.float64, device=part.device)
    dist.all_gather_into_tensor(flat, part.reshape(-1)[:d].contiguous(), group=group)
    return sum_rows(flat.view(world, d))
