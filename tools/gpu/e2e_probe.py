"""e2e variance probe: pinned H2D / D2H bandwidth and the config-4 batch call,
with and without binding to the GPU's NUMA-local cores."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.workloads import CONFIGS, generate_many

def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "none"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if mode == "bind":
        print("bound, cores:", len(bench.bind_to_gpu_numa(torch, dev) or []), "->", len(os.sched_getaffinity(0)))
    n = 16
    host = [np.ascontiguousarray(a) for a in generate_many(4, list(range(n)))]
    pin_in = [torch.from_numpy(a).pin_memory() for a in host]
    pin_out = [torch.empty_like(t).pin_memory() for t in pin_in]
    dbuf = [torch.empty_like(t, device=dev) for t in pin_in]
    def bw(direction):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(n):
            if direction == "h2d": dbuf[i].copy_(pin_in[i], non_blocking=True)
            else: pin_out[i].copy_(dbuf[i], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        return n * pin_in[0].nbytes / dt / 1e9
    for _ in range(2):
        print(mode, "H2D GB/s %.1f  D2H GB/s %.1f" % (bw("h2d"), bw("d2h")), flush=True)
    p = CONFIGS[4]
    params = P.FilterParams(sigma_s=p["sigma_s"], sigma_r=p["sigma_r"], epsilon=p["epsilon"])
    for rep in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        P.shiftable_bf_batch(pin_in, params, lanes=4, out=pin_out)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(mode, "batch of %d: %.1f ms (%.0f Mpix/s)" % (n, dt * 1e3, n * 4096 * 4096 / dt / 1e6), flush=True)
    # device-resident reference
    devs = [t.to(dev) for t in pin_in]
    outs = [torch.empty_like(t) for t in devs]
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        P.shiftable_bf_batch(devs, params, lanes=4, out=outs)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(mode, "device batch of %d: %.1f ms" % (n, dt * 1e3), flush=True)


if __name__ == "__main__":
    main()
