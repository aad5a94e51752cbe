import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_dist_gpu as T

def main():
    import torch.multiprocessing as mp
    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.workloads import config_image
    imgs = [config_image(5, c, size=384) for c in (0, 2)]
    ctx = mp.get_context("spawn"); q = ctx.Queue(); port = T._free_port()
    procs = [ctx.Process(target=T._rank, args=(r, 2, port, imgs, q)) for r in range(2)]
    [p.start() for p in procs]
    got = sorted([q.get(timeout=300) for _ in range(2)], key=lambda g: g[1])
    [p.join(timeout=120) for p in procs]
    params = P.FilterParams(sigma_s=12.0, sigma_r=15.0, epsilon=0.01)
    for c, img in enumerate(imgs):
        full = P.shiftable_bf(img, params)
        for rank, lo, hi, outs, plans in got:
            d = np.abs(outs[c].astype(np.float64) - full.image[lo:hi])
            print(c, rank, lo, hi, plans[c], d.max(), d.mean(), outs[c][:2, :4], full.image[lo:lo+2, :4])

if __name__ == "__main__":
    main()
