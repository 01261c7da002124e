"""Can a single small frame's H2D and D2H overlap? Pinned copies of a PETS
frame (1.33 MB each way) split into k bands on two streams (band i's D2H
waits for band i's H2D, as the pixelize pipeline would), timed per call."""
import json
import time

import numpy as np
import torch


def main():
    n = 576 * 768 * 3
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for k in (1, 2, 3, 4, 6, 8):
        bounds = [n * i // k for i in range(k + 1)]

        def call():
            evs = []
            for i in range(k):
                with torch.cuda.stream(s_in):
                    d[bounds[i]:bounds[i + 1]].copy_(h_in[bounds[i]:bounds[i + 1]], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s_in)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(e)
                    h_out[bounds[i]:bounds[i + 1]].copy_(d[bounds[i]:bounds[i + 1]], non_blocking=True)
            s_out.synchronize()
        for _ in range(30):
            call()
        ts = []
        for _ in range(300):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        res[f"bands_{k}_us"] = round(float(np.median(ts)) * 1e6, 1)
    # one direction alone
    def h2d():
        d.copy_(h_in, non_blocking=True)
        torch.cuda.synchronize()
    for _ in range(30):
        h2d()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        h2d()
        ts.append(time.perf_counter() - t0)
    res["h2d_only_us"] = round(float(np.median(ts)) * 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
