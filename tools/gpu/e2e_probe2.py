"""e2e variance probe 2: the batch call's timeline (host wall, device events)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())


def main():
    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.workloads import CONFIGS, config_image
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n = 16
    base = config_image(4, 0)
    host = [np.ascontiguousarray(base) for _ in range(n)]
    pin_in = [torch.from_numpy(a).pin_memory() for a in host]
    pin_out = [torch.empty_like(t).pin_memory() for t in pin_in]
    p = CONFIGS[4]
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    for stage in ("ce",):
        for lanes in (2, 3, 4):
            ts = []
            for rep in range(6):
                torch.cuda.synchronize(); t = time.perf_counter()
                P.shiftable_bf_batch(pin_in, params, lanes=lanes, out=pin_out, stage=stage)
                torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
            print(stage, lanes, "batch of %d ms:" % n, " ".join("%.0f" % x for x in ts), flush=True)
    # single calls on pinned input
    ts = []
    for rep in range(6):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(4):
            P.shiftable_bf(pin_in[i], params)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    print("single x4 ms:", " ".join("%.0f" % x for x in ts), flush=True)


if __name__ == "__main__":
    main()
