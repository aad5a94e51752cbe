"""StripFilter.run() through a real 2-rank process group on the GPU box.

Two processes share cuda:0 (the GPU box has one GPU for tests) and talk over
gloo — NCCL refuses two ranks on one device — so the MAX all-reduce of the
strip-local T values is a real collective between processes; no kernel of
one rank waits on the other.  The gathered strips must equal the
single-process filter of the whole image (T, N, M bit-exact).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, imgs, q):
    import torch
    import torch.distributed as dist

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.dist import StripFilter, strip_halo, strip_plan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    params = P.FilterParams(sigma_s=12.0, sigma_r=15.0, epsilon=0.01)
    H = imgs[0].shape[0]
    s = strip_plan(H, world, strip_halo(params))[rank]
    bufs = [torch.from_numpy(np.ascontiguousarray(a[s.buf_lo:s.buf_hi])).cuda() for a in imgs]
    sf = StripFilter(bufs, s, H, params, overlap=True)
    outs = sf.run()                 # K1, one gloo all-reduce of 2 fp64 values, plan + filter
    plans = sf.check()              # one read-back: plans, fallbacks, non-finite check
    q.put((rank, s.out_lo, s.out_hi, [o.cpu().numpy() for o in outs],
           [(pl.T, pl.N, pl.M, fb) for pl, fb in plans]))
    dist.barrier()
    dist.destroy_process_group()


def test_strip_filter_two_processes_gloo_match_full_image():
    import torch.multiprocessing as mp

    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.workloads import config_image

    imgs = [config_image(5, c, size=384) for c in (0, 2)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, imgs, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(2)], key=lambda g: g[1])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    params = P.FilterParams(sigma_s=12.0, sigma_r=15.0, epsilon=0.01)
    for c, img in enumerate(imgs):
        full = P.shiftable_bf(img, params)
        for _, _, _, _, plans in got:
            T, N, M, fb = plans[c]
            assert (T, N, M) == (full.plan.T, full.plan.N, full.plan.M)
        stacked = np.concatenate([g[3][c] for g in got], axis=0)
        assert stacked.shape == img.shape
        d = stacked.astype(np.float64) - full.image
        assert float(np.abs(d).max()) <= 2e-3 and float(np.sqrt(np.mean(d * d))) <= 2e-4
