"""Single-frame host-call latency (PETS 768x576 RGB uniform b16 by default):
the public host API on pinned buffers, per call, median of many calls; and the
floor of the same bytes as plain serial / overlapped pinned copies.
Run with DPPX_GRAPH=0 / DPPX_GRAPH_BANDS=k to compare paths."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04261_b200 as dp  # noqa: E402


def main():
    M, N, C, b = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (576, 768, 3, 16)))
    adaptive = len(sys.argv) > 5 and sys.argv[5] == "a"
    import torch
    ctx = dp.Context(0)
    fr = dp.pinned_empty((1, M, N, C))
    fr[:] = np.random.default_rng(0).integers(0, 256, fr.shape, dtype=np.uint8)
    mk = dp.pinned_empty((1, M, N))
    mk[:] = 1
    out = dp.pinned_empty((1, M, N, C))
    p = dp.make_privacy_params(0.5, 16, b, 4 if adaptive else 1)
    seeds = dp.plane_seeds(42, 1, C)
    call = (lambda: ctx.pixelize_adaptive(fr, mk, p, dp.NOISE_KEYED, seeds, out=out)) if adaptive else \
        (lambda: ctx.pixelize_uniform(fr, p, dp.NOISE_KEYED, seeds, out=out))
    for _ in range(50):
        call()
    ts = []
    for _ in range(500):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    # device time of the kernels inside one call (CUDA events around each launch)
    ctx.reset_stats()
    ctx.set_timing(True)
    for _ in range(50):
        call()
    st = ctx.stats()
    ctx.set_timing(False)
    dev_us = {k: round(v / 50 * 1e3, 2) for k, v in st["device_ms"].items() if v}
    # copy floors
    nbytes = M * N * C
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def serial():
        d.copy_(h, non_blocking=True)
        h2.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
    def overlapped():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
    floors = {}
    for name, fn in (("serial_copies", serial), ("overlapped_copies", overlapped)):
        for _ in range(50):
            fn()
        tt = []
        for _ in range(500):
            t0 = time.perf_counter()
            fn()
            tt.append(time.perf_counter() - t0)
        floors[name] = round(float(np.median(tt)) * 1e6, 2)
    print(json.dumps({"shape": [M, N, C], "b": b, "adaptive": adaptive,
                      "graph": os.environ.get("DPPX_GRAPH", "1"),
                      "bands": os.environ.get("DPPX_GRAPH_BANDS", "auto"),
                      "median_us": round(float(np.median(ts)) * 1e6, 2),
                      "p10_us": round(float(np.percentile(ts, 10)) * 1e6, 2),
                      "p90_us": round(float(np.percentile(ts, 90)) * 1e6, 2), **floors,
                      "kernel_us_per_call": dev_us,
                      "launches": ctx.stats()["launches"]}))


if __name__ == "__main__":
    main()
