"""e2e A/B for the config-4 batch API: copy-engine vs SM staging, lanes."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1203_5128_b200 as P
from paper_1203_5128_b200.workloads import generate_many
def main():
    imgs = generate_many(4, range(16))
    params = P.FilterParams(sigma_s=6, sigma_r=20, epsilon=0.01)
    pin = [torch.from_numpy(a).pin_memory() for a in imgs]
    outs = [torch.empty(a.shape, dtype=torch.float32, pin_memory=True) for a in imgs]
    dev = [torch.from_numpy(a).cuda() for a in imgs]
    for stage in ("ce", "sm"):
        for lanes in (2, 3, 4):
            for _ in range(2):
                P.shiftable_bf_batch(pin, params, lanes=lanes, out=outs, stage=stage)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(3):
                P.shiftable_bf_batch(pin, params, lanes=lanes, out=outs, stage=stage)
            dt = (time.perf_counter() - t) / 3
            print(f"host {stage} lanes {lanes}: {dt*1e3:.1f} ms / 16 images -> {16*4096*4096/dt/1e6:.0f} Mpix/s", flush=True)
    for lanes in (3,):
        P.shiftable_bf_batch(dev, params, lanes=lanes)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            P.shiftable_bf_batch(dev, params, lanes=lanes)
        dt = (time.perf_counter() - t) / 3
        print(f"device lanes {lanes}: {dt*1e3:.1f} ms -> {16*4096*4096/dt/1e6:.0f} Mpix/s")
    # raw transfer rates
    x = pin[0]; y = torch.empty_like(dev[0])
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): y.copy_(x, non_blocking=True)
    torch.cuda.synchronize(); print("CE H2D GB/s", 10 * x.numel() * 4 / (time.perf_counter() - t) / 1e9)
    lib = P._lib.load()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): lib.sbf_stage_h2d(x.data_ptr(), 0, x.numel(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize(); print("SM H2D GB/s", 10 * x.numel() * 4 / (time.perf_counter() - t) / 1e9)
    o = outs[0]
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): o.copy_(y, non_blocking=True)
    torch.cuda.synchronize(); print("CE D2H GB/s", 10 * x.numel() * 4 / (time.perf_counter() - t) / 1e9)


if __name__ == "__main__":
    main()
