"""Multi-process data parallelism on CPU (gloo, world size 2): sharding, the flat
gradient buffer and the all-reduce reproduce the single-process gradients.

Each rank renders its ray shard with the oracle (the CPU tests have no GPU);
the data-parallel logic under test (paper_2404_19760_b200.dist) is the same
code the CUDA path runs with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import workload as wl
    from tests.helpers import tiny_field_arrays, tiny_rays
    grid, params = tiny_field_arrays(wl.TRIPLANE, (4, 5, 6), 3, (3, 5, 4), sigma_bias=0.4)
    o, d, near, far = tiny_rays(6)
    p = wl.counter_uniform(61, np.arange(18, dtype=np.uint64), -1, 1).reshape(6, 3)
    gt = wl.counter_uniform(62, np.arange(6, dtype=np.uint64), -1, 1)
    return grid, params, (o, d, near, far), p, gt


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2404_19760_b200.dist import FlatGrads, dp_backward
    grid, params, (o, d, near, far), p, gt = _problem()
    F = oracle.Field(0, grid, (3, 5, 4), params)
    S = 9
    grads = FlatGrads([g.shape for g in F.grid] + [F.params.shape], dtype=torch.float64)

    def backward_shard(lo, hi, views):
        R = oracle.Rays(o[lo:hi], d[lo:hi], near[lo:hi], far[lo:hi], S)
        gg, gp = oracle.render_backward(F, R, p[lo:hi], gt[lo:hi])
        for v, a in zip(views, list(gg) + [gp]):
            v += torch.from_numpy(a)

    dp_backward(len(o), backward_shard, grads)
    out_q.put((rank, [v.numpy().copy() for v in grads.views]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_gradients_equal_single_process(world):
    import oracle
    grid, params, (o, d, near, far), p, gt = _problem()
    F = oracle.Field(0, grid, (3, 5, 4), params)
    ref_g, ref_p = oracle.render_backward(F, oracle.Rays(o, d, near, far, 9), p, gt)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in range(world):
        got = res[r]
        for a, b in zip(got, list(ref_g) + [ref_p]):
            assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b)))


def test_shard_range_partitions():
    from paper_2404_19760_b200.dist import shard_range
    for n in (0, 1, 7, 8388608):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_flat_grads_alignment():
    from paper_2404_19760_b200.dist import FlatGrads
    fg = FlatGrads([(3, 5), (7,), (2, 2, 3)])
    for v in fg.views:
        assert (v.data_ptr() - fg.flat.data_ptr()) % 16 == 0
    fg.views[1] += 1
    assert float(fg.flat.sum()) == 7.0
