"""The bench's e2e leg (64 config-4 images, pinned in/out) step by step."""
import gc, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())


def main():
    import paper_1203_5128_b200 as P
    from paper_1203_5128_b200.workloads import CONFIGS, generate_many
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    host = [np.ascontiguousarray(a) for a in generate_many(4, list(range(64)))]
    devs = [torch.from_numpy(a).to(dev) for a in host]  # like the bench's device-resident leg
    pin_in = [torch.from_numpy(a).pin_memory() for a in host]
    pin_out = [torch.empty(a.shape, dtype=torch.float32, pin_memory=True) for a in host]
    p = CONFIGS[4]
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    for lanes in [int(x) for x in sys.argv[1:]] or [4, 3, 4]:
        for _ in range(2):
            P.shiftable_bf_batch(pin_in, params, lanes=lanes, out=pin_out)
        torch.cuda.synchronize()
        gc.disable()
        ts = []
        for _ in range(6):
            t = time.perf_counter()
            P.shiftable_bf_batch(pin_in, params, lanes=lanes, out=pin_out)
            ts.append((time.perf_counter() - t) * 1e3)
        gc.enable()
        print("lanes", lanes, "e2e step ms:", " ".join("%.0f" % x for x in ts), flush=True)


if __name__ == "__main__":
    main()
