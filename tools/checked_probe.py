#!/usr/bin/env python3
"""Where the batch runner's per-chunk call (dppx_pixelize_checked) spends its
time: 64 x 1080p gray adaptive b16 n4 from pinned host memory; wall time per
call and device time per kernel family (CUDA events)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2511_04261_b200 as dp  # noqa: E402


def main():
    F, M, N = 64, 1080, 1920
    ctx = dp.Context(0)
    fr = dp.pinned_empty((F, M, N, 1))
    fr[:] = np.random.default_rng(1).integers(0, 256, fr.shape, dtype=np.uint8)
    mk = dp.pinned_empty((F, M, N))
    mk[:] = 1
    mk[:, 300:700, 700:1200] = 0
    p = dp.make_privacy_params(0.5, 16, 16, 4)
    seeds = [42] * F
    for _ in range(3):
        ctx.pixelize_checked(fr, mk, p, "adaptive", dp.NOISE_KEYED, seeds)
    ctx.reset_stats()
    ctx.set_timing(True)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        ctx.pixelize_checked(fr, mk, p, "adaptive", dp.NOISE_KEYED, seeds)
    t1 = time.perf_counter()
    s = ctx.stats()
    ctx.set_timing(False)
    print(json.dumps({"wall_ms_per_call": round((t1 - t0) / reps * 1e3, 2),
                      "device_ms_per_call": {k: round(v / reps, 3) for k, v in s["device_ms"].items() if v},
                      "launches_per_call": {k: v / reps for k, v in s["launches"].items() if v},
                      "h2d_MB": round(s["h2d_bytes"] / reps / 1e6, 1), "d2h_MB": round(s["d2h_bytes"] / reps / 1e6, 1)}))


if __name__ == "__main__":
    main()
