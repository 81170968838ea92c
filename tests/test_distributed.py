"""Multi-rank host logic on CPU with gloo (world_size 2): term sharding with
an NCCL-style reduce of num/den, and frame sharding.  The per-rank compute
is injected (the float64 oracle restricted to the rank's terms), so this
exercises the partitioning and the collective, not the device kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1105_4204_b200.distributed import frame_range, shard_cost, term_shard


def test_frame_range_partition():
    for n in (1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            rs = [frame_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("balance", ["terms", "rows"])
def test_term_shard_partition(balance):
    """Every (term, row) is covered exactly once: whole terms are contiguous
    and disjoint across ranks; with balance="rows" the leftover terms' row
    bands tile [0, H) in whole 128-row blocks; with balance="terms" the
    leftover terms go one each to the last ranks (the root keeps the fewest)."""
    for n_terms in (60, 22, 133, 16, 3, 34):
        for world in (1, 2, 3, 4, 8):
            for H in (16384, 2048, 300):
                sh = [term_shard(n_terms, world, r, H, balance=balance) for r in range(world)]
                if balance == "terms":
                    counts = [s.t1 - s.t0 for s in sh]
                    assert max(counts) - min(counts) <= 1 and counts[0] == min(counts)
                    assert counts == sorted(counts)
                cover = np.zeros((n_terms, H), dtype=int)
                for s in sh:
                    cover[s.t0:s.t1, :] += 1
                    cover[s.l0:s.l1, s.r0:s.r1] += 1
                    assert s.r0 % 128 == 0 and (s.r1 % 128 == 0 or s.r1 == H or s.r1 == s.r0)
                assert np.all(cover == 1), (n_terms, world, H)


def test_term_shard_balance_config5():
    """Config 5 (60 terms, 16384 rows, y warm-up 384 rows): the row-band split
    evens out the term-rows exactly (within 3% of the mean before its fixed
    cost), but with the measured fixed cost of the band call (a full
    transpose and an under-filled launch: one rank's share of 8 took 24.2 ms
    vs 21.1 ms for the busiest whole-term rank, profiles/ab_term_balance_r02.log)
    the whole-term split (the default) models and measures cheaper; 2 and 4
    ranks divide 60 evenly."""
    from paper_1105_4204_b200 import distributed as d

    H, warm = 16384, 384
    for world in (2, 4, 8):
        rows = [term_shard(60, world, r, H, balance="rows") for r in range(world)]
        terms = [term_shard(60, world, r, H) for r in range(world)]
        band_only = [shard_cost(s, H, warm) - (d.BAND_FIXED_TERMS if s.l1 > s.l0 else 0.0) for s in rows]
        assert max(band_only) <= 1.03 * 60.0 / world, (world, band_only)
        c_rows = max(shard_cost(s, H, warm, root=(r == 0)) for r, s in enumerate(rows))
        c_terms = max(shard_cost(s, H, warm, root=(r == 0)) for r, s in enumerate(terms))
        assert c_terms <= c_rows, (world, c_terms, c_rows)
    counts = [s.t1 - s.t0 for s in (term_shard(60, 8, r, H) for r in range(8))]
    assert counts == [7, 7, 7, 7, 8, 8, 8, 8]  # the root (finalize) among the 7s


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_oracle(plane, sigma_s, kernel, t0, t1):
    from oracle import trigbf_oracle as orc

    pairs = orc.term_pairs(kernel)[t0:t1]
    num = np.zeros_like(plane)
    den = np.zeros_like(plane)
    for nu, w in pairs:
        c, s = np.cos(nu * plane), np.sin(nu * plane)
        sm = [orc.smooth_plane(p, "gauss-recursive", sigma_s) for p in (c, s, plane * c, plane * s)]
        num += w * (c * sm[2] + s * sm[3])
        den += w * (c * sm[0] + s * sm[1])
    return num, den


def _worker(rank, world, port, q, balance="rows"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import trigbf_oracle as orc
        from paper_1105_4204_b200 import SpatialSpec, make_trig_kernel
        from paper_1105_4204_b200.distributed import bilateral_trig_term_sharded

        # 300 rows (three 128-row blocks, the last partial) and N = 5 (3 pairs):
        # on 2 ranks one term each plus the leftover one split by rows
        plane = np.random.default_rng(3).uniform(0, 255, (300, 24))
        k = make_trig_kernel(300.0)
        okern = orc.make_trig_kernel(300.0)
        f = torch.from_numpy(plane)

        def partial_fn(f_, num, den, t0, t1, rows=None, accumulate=False):
            n, d = _partial_oracle(f_.numpy(), 3.0, okern, t0, t1)
            r0, r1 = rows if rows is not None else (0, n.shape[0])
            if not accumulate:
                num[r0:r1].zero_()
                den[r0:r1].zero_()
            num[r0:r1] += torch.from_numpy(n[r0:r1])
            den[r0:r1] += torch.from_numpy(d[r0:r1])

        def finalize_fn(num, den, f_, out):
            o, _ = orc.guarded_ratio(num.numpy(), den.numpy(), f_.numpy())
            out.copy_(torch.from_numpy(o))

        out = bilateral_trig_term_sharded(f, SpatialSpec.gaussian_recursive(3.0), k,
                                          partial_fn=partial_fn, finalize_fn=finalize_fn, balance=balance)
        if rank == 0:
            ref, _ = orc.bilateral_trig(plane, "gauss-recursive", 3.0, okern)
            q.put(float(np.max(np.abs(out.numpy() - ref))))
        else:
            q.put(None if out is None else "non-root got output")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("balance", ["rows", "terms"])
def test_term_sharded_reduce_gloo_world2(balance):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, balance)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if isinstance(r, float)]
    assert len(errs) == 1 and errs[0] < 1e-9, res
    assert all(r is None or isinstance(r, float) for r in res), res


def _frame_worker(rank, world, port, q, gather):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import trigbf_oracle as orc
        from paper_1105_4204_b200 import SpatialSpec, make_trig_kernel
        from paper_1105_4204_b200.distributed import bilateral_trig_frame_sharded, frame_range

        B = 5  # odd: ranks get 3 and 2 frames, the gather pads the short shard
        frames = torch.from_numpy(np.random.default_rng(11).uniform(0, 255, (B, 12, 10)).astype(np.float32))
        k = make_trig_kernel(40.0)
        okern = orc.make_trig_kernel(40.0)
        calls = []

        def filter_fn(x):
            calls.append(int(x.shape[0]))
            out = [orc.bilateral_trig(x[i].double().numpy(), "gauss-recursive", 2.0, okern)[0] for i in range(x.shape[0])]
            return torch.from_numpy(np.stack(out).astype(np.float32))

        got = bilateral_trig_frame_sharded(frames, SpatialSpec.gaussian_recursive(2.0), k, gather=gather,
                                           filter_fn=filter_fn)
        ref = np.stack([orc.bilateral_trig(frames[i].double().numpy(), "gauss-recursive", 2.0, okern)[0]
                        for i in range(B)])
        f0, f1 = frame_range(B, world, rank)
        want = ref if gather else ref[f0:f1]
        q.put((rank, calls, tuple(got.shape), float(np.max(np.abs(got.double().numpy() - want)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("gather", [False, True])
def test_frame_sharded_gloo_world2(gather):
    """Config 4's frame split on two ranks (gloo, CPU compute injected): each
    rank filters only its own contiguous frames (no collective on the data
    path); with gather=True every rank ends with the whole batch in order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frame_worker, args=(r, 2, port, q, gather)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    (r0, c0, s0, e0), (r1, c1, s1, e1) = res
    assert c0 == [3] and c1 == [2]  # frame_range(5, 2, r): 3 + 2 frames, one call each
    if gather:
        assert s0 == s1 == (5, 12, 10)
    else:
        assert s0 == (3, 12, 10) and s1 == (2, 12, 10)
    assert e0 < 1e-4 and e1 < 1e-4
