"""Multi-GPU partitioning of the filter (one process per GPU, torch.distributed).

Two ways the path shards:

* frames -- a batch of independent frames (config 4) is split into
  contiguous per-rank ranges; no collective on the data path.
* terms  -- one huge image (config 5): the filter is a sum over independent
  frequency terms (engines.py:264-300 accumulates num/den term by term), so
  each rank accumulates partial num/den planes for its share of the terms,
  the two planes are summed onto the root with one NCCL reduce over
  NVLink/NVSwitch, and the root applies the guarded ratio.  The terms left
  over after an even split go whole to the last ranks (the root finalizes);
  splitting them by rows across all ranks balances the term count exactly but
  costs a second call per rank (a full transpose and an under-filled band
  launch), measured slower on one rank's share of 8 (term_shard).

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


ROW_BLOCK = 128  # band granularity of tbf_trig_partial_rows (pass-2 row blocks)
PASS1_SHARE = 0.6  # share of a term's device time in pass 1 (the part with y warm-ups), measured on config 5
# Fixed cost of a rank's leftover-band call in whole-term units (its own full
# transpose and reduce, and a band launch far from filling the GPU): config 5,
# the root's share of 8: 7 whole terms + the band of 4 leftover terms took
# 24.2 ms against 20.0 ms for the 7 terms alone, i.e. 1.77 terms at 2.36 ms per
# term, of which the model's band rows account for 0.61
# (profiles/ab_term_balance_r02.log)
BAND_FIXED_TERMS = 1.2
ROOT_FIXED_TERMS = 0.4  # the root's finalize + range check (0.94 ms on config 5)
TERM_BALANCE = "terms"  # "terms": leftover terms whole to the last ranks; "rows": split by row bands


@dataclass
class TermShard:
    """One rank's share of a term-sharded filter: whole terms [t0, t1) over the
    full image plus the leftover terms [l0, l1) over output rows [r0, r1)."""

    t0: int
    t1: int
    l0: int
    l1: int
    r0: int
    r1: int


def term_shard(n_terms: int, world: int, rank: int, height: int, warm_rows: int = 0,
               balance: str | None = None) -> TermShard:
    """Split of n_terms pairs across `world` ranks.

    balance="terms" (TERM_BALANCE, the default): contiguous whole terms,
    floor(n/world) per rank and the n % world leftover ones one each to the
    last ranks, never to the root while a rank is left (it also finalizes).
    Up to one term of imbalance (config 5 on 8 ranks: 8 vs 7.5 terms).

    balance="rows": every rank takes floor(n/world) consecutive terms over the
    whole image, and the leftover terms are split by rows instead: every rank
    filters them over its own band of whole 128-row blocks
    (tbf_trig_partial_rows; a band costs its rows plus the y warm-ups on both
    sides in pass 1).  Exact in term-rows, but each rank makes a second call
    whose fixed cost (BAND_FIXED_TERMS) outweighs the term it saves.
    """
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of {world}")
    balance = balance or TERM_BALANCE
    if balance not in ("terms", "rows"):
        raise ValueError(f"unknown balance {balance!r}")
    q, r = divmod(n_terms, world)
    if balance == "terms":
        first_extra = world - r  # ranks [world - r, world) take q + 1 terms
        t0 = rank * q + max(0, rank - first_extra)
        t1 = t0 + q + (1 if rank >= first_extra else 0)
        return TermShard(t0, t1, n_terms, n_terms, 0, 0)
    t0, t1 = rank * q, (rank + 1) * q
    l0, l1 = world * q, n_terms
    nrb = -(-height // ROW_BLOCK)
    b0, b1 = frame_range(nrb, world, rank)
    r0, r1 = min(height, b0 * ROW_BLOCK), min(height, b1 * ROW_BLOCK)
    if r == 0 or r1 <= r0:
        l0 = l1 = n_terms
        r0 = r1 = 0
    return TermShard(t0, t1, l0, l1, r0, r1)


def shard_cost(sh: TermShard, height: int, warm_rows: int, root: bool = False) -> float:
    """Model of a rank's device time in whole-image term units: pass 1 (the
    PASS1_SHARE of a term) sweeps a band's rows plus its warm-ups, pass 2
    the band's rows; a band call adds BAND_FIXED_TERMS, the root
    ROOT_FIXED_TERMS."""
    full = float(sh.t1 - sh.t0) + (ROOT_FIXED_TERMS if root else 0.0)
    if sh.l1 <= sh.l0:
        return full
    ext = min(height, sh.r1 + warm_rows) - max(0, sh.r0 - warm_rows)
    frac = PASS1_SHARE * ext / height + (1.0 - PASS1_SHARE) * (sh.r1 - sh.r0) / height
    return full + (sh.l1 - sh.l0) * frac + BAND_FIXED_TERMS


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
                                group=None, balance: str | None = None):
    """Term-sharded filter of one image on every rank of the default group.

    Every rank holds the full input `f` ([B, H, W] float32).  Returns the
    filtered image on rank 0 and None elsewhere.  The split is term_shard's
    (`balance`: whole terms, or whole terms plus a row band of the leftover
    terms per rank).
    `partial_fn(f, num, den, t0, t1, rows=None, accumulate=False)` /
    `finalize_fn(num, den, f, out)` default to the device path (TrigFilter);
    tests inject CPU implementations to exercise the partitioning and the
    reduce with the gloo backend.
    """
    import torch
    import torch.distributed as dist

    from .kernels import term_pairs

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    pairs = term_pairs(kernel)
    H = int(f.shape[-2])
    sh = term_shard(pairs.count, world, rank, H, balance=balance)
    numden = torch.zeros((2, *f.shape), dtype=f.dtype, device=f.device)
    num, den = numden[0], numden[1]
    plan_for_checks = None
    if partial_fn is None or finalize_fn is None:
        from .engines import TrigFilter

        plan = TrigFilter(tuple(f.shape), spatial, kernel, term_range=(sh.t0, sh.t1)) if sh.t1 > sh.t0 else None
        left = (TrigFilter(tuple(f.shape), spatial, kernel, term_range=(sh.l0, sh.l1))
                if sh.l1 > sh.l0 else None)
        if plan is not None:
            plan_for_checks = plan
        elif rank == 0:  # the root finalises even without terms of its own
            plan_for_checks = TrigFilter(tuple(f.shape), spatial, kernel)

        def partial_fn(f_, n_, d_, a, b, rows=None, accumulate=False):
            p = plan if rows is None else left
            if p is not None:
                p.partial(f_, n_, d_, accumulate=accumulate, rows=rows)

        def finalize_fn(n_, d_, f_, o_):
            return plan_for_checks.finalize(n_, d_, f_, o_)

    if sh.t1 > sh.t0:
        partial_fn(f, num, den, sh.t0, sh.t1)
    if sh.l1 > sh.l0:
        partial_fn(f, num, den, sh.l0, sh.l1, rows=(sh.r0, sh.r1), accumulate=sh.t1 > sh.t0)
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
