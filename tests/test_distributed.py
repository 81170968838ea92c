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

from paper_1105_4204_b200.distributed import frame_range, term_range


def test_frame_range_partition():
    for n in (1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            rs = [frame_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_term_range_partition_balanced():
    for n_terms, has_zero in ((60, True), (22, False), (133, True), (16, True), (3, False)):
        for world in (1, 2, 4, 8):
            rs = [term_range(n_terms, has_zero, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n_terms
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(a % 2 == 0 or a == b == n_terms for a, b in rs)


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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import trigbf_oracle as orc
        from paper_1105_4204_b200 import SpatialSpec, make_trig_kernel
        from paper_1105_4204_b200.distributed import bilateral_trig_term_sharded

        plane = np.random.default_rng(3).uniform(0, 255, (20, 24))
        k = make_trig_kernel(30.0)
        okern = orc.make_trig_kernel(30.0)
        f = torch.from_numpy(plane)

        def partial_fn(f_, num, den, t0, t1):
            n, d = _partial_oracle(f_.numpy(), 3.0, okern, t0, t1)
            num.copy_(torch.from_numpy(n))
            den.copy_(torch.from_numpy(d))

        def finalize_fn(num, den, f_, out):
            o, _ = orc.guarded_ratio(num.numpy(), den.numpy(), f_.numpy())
            out.copy_(torch.from_numpy(o))

        out = bilateral_trig_term_sharded(f, SpatialSpec.gaussian_recursive(3.0), k,
                                          partial_fn=partial_fn, finalize_fn=finalize_fn)
        if rank == 0:
            ref, _ = orc.bilateral_trig(plane, "gauss-recursive", 3.0, okern)
            q.put(float(np.max(np.abs(out.numpy() - ref))))
        else:
            q.put(None if out is None else "non-root got output")
    finally:
        dist.destroy_process_group()


def test_term_sharded_reduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
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
