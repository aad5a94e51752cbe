"""Multi-rank host logic of the sharded configs, on CPU with gloo (world 2),
plus the strip decomposition checked end to end with the CPU oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import shiftbf_oracle as O
from paper_1203_5128_b200.dist import allreduce_max_, gather_strips, shard_images, strip_plan


def test_strip_plan_covers_rows_with_clamped_halos():
    for H, world, halo in [(100, 1, 9), (100, 3, 9), (16384, 8, 36), (7, 4, 3)]:
        strips = strip_plan(H, world, halo)
        assert strips[0].out_lo == 0 and strips[-1].out_hi == H
        for a, b in zip(strips, strips[1:]):
            assert a.out_hi == b.out_lo
        for s in strips:
            assert s.buf_lo == max(0, s.out_lo - halo) and s.buf_hi == min(H, s.out_hi + halo)


def test_shard_images_balances_cost():
    costs = [12.0] * 61 + [11.0, 11.0, 10.0]          # config 4 terms per image
    parts = shard_images(costs, 8)
    assert sorted(i for p in parts for i in p) == list(range(64))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= 12.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, img, params, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    halo = 9
    s = strip_plan(img.shape[0], world, halo)[rank]
    buf = img[s.buf_lo:s.buf_hi]
    # strip-local T over the owned rows only (windows stay inside the buffer)
    M = O.max_filter_2d(buf, halo)
    lo, hi = s.out_lo - s.buf_lo, s.out_hi - s.buf_lo
    T_local = torch.tensor([float(np.max(M[lo:hi] - buf[lo:hi]))], dtype=torch.float64)
    allreduce_max_(T_local)
    res = O.shiftable_bf(buf, params[0], params[1], params[2], fixed_T=float(T_local.item()))
    q.put((rank, float(T_local.item()), res["image"][lo:hi]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_rank_strips_match_full_image():
    rng = np.random.default_rng(3)
    img = rng.uniform(0, 255, (70, 40))
    params = (3.0, 30.0, 0.01)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, img, params, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = O.shiftable_bf(img, *params)
    Ts = {r: t for r, t, _ in got}
    assert Ts[0] == Ts[1] == full["T"]          # max of strip maxima is exact
    outs = {r: o for r, _, o in got}
    strips = strip_plan(img.shape[0], 2, 9)
    stacked = gather_strips([outs[0], outs[1]], strips)
    np.testing.assert_allclose(stacked, full["image"], rtol=1e-10, atol=1e-9)
