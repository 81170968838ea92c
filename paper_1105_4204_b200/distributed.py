"""Multi-GPU partitioning of the filter (one process per GPU, torch.distributed).

Two ways the path shards:

* frames -- a batch of independent frames (config 4) is split into
  contiguous per-rank ranges; no collective on the data path.
* terms  -- one huge image (config 5): the filter is a sum over independent
  frequency terms (engines.py:264-300 accumulates num/den term by term), so
  each rank accumulates partial num/den planes for its share of the terms,
  the two planes are summed onto the root with an NCCL reduce over
  NVLink/NVSwitch, and the root applies the guarded ratio.  Term costs are
  not uniform (the zero frequency needs one plane, the others four), so the
  split balances plane counts, not term counts.

The reference has no distributed mode; its only parallelism is a thread pool
over the 4 planes of one term (engines.py:262-303).
"""

from __future__ import annotations

from dataclasses import dataclass


def frame_range(n_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal frame range of `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def term_costs(n_terms: int, has_zero: bool) -> list[int]:
    """Relative cost of each pair: planes to filter (4, or 1 for nu = 0)."""
    return [1 if (has_zero and j == 0) else 4 for j in range(n_terms)]


def term_range(n_terms: int, has_zero: bool, world: int, rank: int, align: int = 2) -> tuple[int, int]:
    """Contiguous term range of `rank` with balanced plane cost.

    Boundaries are multiples of `align` (the device's phasor anchor block) so
    every rank generates bit-identical phasors; a rank may get an empty range
    when there are fewer aligned blocks than ranks.
    """
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    costs = term_costs(n_terms, has_zero)
    nblocks = (n_terms + align - 1) // align
    cum = [0]
    for b in range(nblocks):
        cum.append(cum[-1] + sum(costs[b * align:(b + 1) * align]))
    total = cum[-1]
    idx = [0]
    for r in range(1, world):
        target = total * r / world
        lo = idx[-1]
        idx.append(min(range(lo, nblocks + 1), key=lambda i: (abs(cum[i] - target), i)))
    idx.append(nblocks)
    return min(n_terms, idx[rank] * align), min(n_terms, idx[rank + 1] * align)


@dataclass
class ShardInfo:
    world: int
    rank: int
    mode: str  # "replica" | "frames" | "terms"
    start: int
    stop: int


def reduce_numden(numden, dst: int = 0, group=None) -> None:
    """Sum the stacked partial [num, den] planes onto `dst` in one collective
    (NCCL reduce over NVLink/NVSwitch when the process group is NCCL; gloo on
    CPU tensors in the tests).  One call moves both planes: half the launches
    and protocol rounds of two separate reduces."""
    import torch.distributed as dist

    dist.reduce(numden, dst=dst, op=dist.ReduceOp.SUM, group=group)


def bilateral_trig_term_sharded(f, spatial, kernel, *, partial_fn=None, finalize_fn=None,
                                group=None):
    """Term-sharded filter of one image on every rank of the default group.

    Every rank holds the full input `f` ([B, H, W] float32).  Returns the
    filtered image on rank 0 and None elsewhere.  `partial_fn(f, num, den,
    t0, t1)` / `finalize_fn(num, den, f, out)` default to the device path
    (TrigFilter); tests inject CPU implementations to exercise the
    partitioning and the reduce with the gloo backend.
    """
    import torch
    import torch.distributed as dist

    from .kernels import term_pairs

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pairs = term_pairs(kernel)
    t0, t1 = term_range(pairs.count, pairs.has_zero, world, rank)
    numden = torch.zeros((2, *f.shape), dtype=f.dtype, device=f.device)
    num, den = numden[0], numden[1]
    plan_for_checks = None
    if partial_fn is None or finalize_fn is None:
        from .engines import TrigFilter

        plan = TrigFilter(tuple(f.shape), spatial, kernel, term_range=(t0, t1)) if t1 > t0 else None
        if plan is not None:
            plan_for_checks = plan
        elif rank == 0:  # the root finalises even without terms of its own
            plan_for_checks = TrigFilter(tuple(f.shape), spatial, kernel)

        def partial_fn(f_, n_, d_, a, b):
            if plan is not None:
                plan.partial(f_, n_, d_, accumulate=False)

        def finalize_fn(n_, d_, f_, o_):
            return plan_for_checks.finalize(n_, d_, f_, o_)

    if t1 > t0:
        partial_fn(f, num, den, t0, t1)
    reduce_numden(numden, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.empty_like(f)
    finalize_fn(num, den, f, out)
    if plan_for_checks is not None:
        # engines.py:218-225 on the root's copy of the input (every rank holds
        # the same f); read once, after the filter (one sync)
        plan_for_checks.range_check(f)
        bad, _ = plan_for_checks.read_counters()
        if bad:
            from .errors import ParameterError

            raise ParameterError(f"samples exceed the declared range [0, {kernel.T:g}]; "
                                 "rescale the input or raise T")
    return out


def bilateral_trig_frame_sharded(frames, spatial, kernel, *, gather: bool = False, group=None,
                                 filter_fn=None):
    """Frame batches split across ranks with no collective (SURVEY 8(e),
    config 4): rank r filters frames frame_range(B, world, r) of ``frames``
    ([B, H, W], host or device; every rank passes the same batch).  Returns
    this rank's filtered frames, or with ``gather=True`` the whole batch on
    every rank (all_gather of equal-size shards, padded).  ``filter_fn(frames)``
    defaults to the device ``bilateral_trig``; the gloo tests inject a CPU
    implementation (the gather then runs on CPU tensors)."""
    import torch
    import torch.distributed as dist

    from .engines import bilateral_trig

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    B = int(frames.shape[0])
    f0, f1 = frame_range(B, world, rank)
    if filter_fn is None:
        def filter_fn(x):
            return bilateral_trig(x, spatial, kernel)
    mine = filter_fn(frames[f0:f1].contiguous()) if f1 > f0 else frames[0:0]
    if not gather:
        return mine
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
           else torch.device("cpu"))
    per = max(frame_range(B, world, r)[1] - frame_range(B, world, r)[0] for r in range(world))
    buf = torch.zeros((per, *frames.shape[1:]), dtype=torch.float32, device=dev)
    if f1 > f0:
        buf[: f1 - f0].copy_(torch.as_tensor(mine).to(dev))
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: frame_range(B, world, r)[1] - frame_range(B, world, r)[0]]
                      for r in range(world)])
