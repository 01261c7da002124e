#!/usr/bin/env python3
"""Benchmark of the B200 dppix pixelization path (BASELINE.json metric).

Default workload (BASELINE.json configs[1]): region-adaptive DP pixelization,
b=16, n=4, m=16, eps=0.5, u8 fg/bg mask, a 600-frame synthetic 1920x1080 RGB
clip per GPU (weak scaling: each rank owns its own 600 frames, global frame
indices rank*600 + i, so the noise streams never repeat across ranks).

  value  -- device-resident: frames, masks and outputs live in HBM when the
            timed region starts; one step = K0 + K1 over the whole clip
            (classification, statistics, keyed Laplace noise, compact DPPX
            payloads, full reconstructed image). MP/s over all ranks.
  e2e    -- the same metric through the public host API dppx_pixelize_adaptive
            with pinned HOST buffers: every step copies that step's frames and
            masks H2D and reads payloads + reconstructed image back D2H.
  roofline   -- K1 (k_stats_tma), algorithmic bytes / CUDA-event duration.
  cpu_baseline -- the reference (oracle/_ref, compiled from /root/reference
            sources) timed on this host on a bounded sample, rank 0 only.

`--impl reference` times only the reference CPU implementation (rank 0).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec and 1080p frames/sec (adaptive DP pixelization); % of HBM roofline"

WORKLOADS = {
    # name: (M, N, C, frames_per_gpu, b, n, m, eps, adaptive, description)
    "venice": (1080, 1920, 3, 600, 16, 4, 16, 0.5, True,
               "region-adaptive DP pixelization with fg/bg mask, 600-frame synthetic "
               "1920x1080 RGB clip (Venice-2 shape), b=16 n=4 m=16 eps=0.5"),
    "pets": (576, 768, 3, 1, 16, 1, 16, 0.5, False,
             "uniform DP pixelization b=16 m=16 eps=0.5, one 768x576 RGB frame (PETS shape)"),
    "pets_clip": (576, 768, 3, 795, 16, 1, 16, 0.5, False,
                  "uniform DP pixelization b=16 m=16 eps=0.5 on a 795-frame 768x576 RGB clip "
                  "(PETS shape; the paper times 795 PETS frames, PAPER.md:593)"),
    "4k": (2160, 3840, 3, 64, 32, 8, 16, 0.5, True,
           "region-adaptive b=32 n=8 on synthetic 3840x2160 RGB images with compact store + "
           "reconstruction"),
    "celeba": (218, 178, 3, 100000, 16, 1, 16, 0.5, False,
               "uniform b=16 on a 100k-image batch of 178x218 RGB faces (CelebA shape)"),
    # one step = the 12-run sweep b in {4,8,16,32} x eps in {0.1,0.5,1} over the batch
    "sweep": (1083, 1917, 3, 60, 16, 1, 16, 0.5, False,
              "grid-size/padding sweep b in {4,8,16,32} x eps in {0.1,0.5,1}, uniform m=16, "
              "60 synthetic 1917x1083 RGB frames (non-divisible dims); value counts frame-runs"),
}
SWEEP = [(bb, ee) for bb in (4, 8, 16, 32) for ee in (0.1, 0.5, 1.0)]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="venice")
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU")
    ap.add_argument("--e2e-frames", type=int, default=0,
                    help="frames per e2e step (default: ~1 GB of input, <= frames per GPU)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU-work seconds for the reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pad-scratch", action="store_true",
                    help="never write output row padding (A/B of dppx_ctx_set_out_pad_scratch)")
    ap.add_argument("--sweep-mode", choices=["fused", "runs"], default="fused",
                    help="sweep workload: one-read K1s + per-run broadcast (fused) or 12 separate "
                         "K1 runs (runs)")
    ap.add_argument("--chunk-frames", type=int, default=0,
                    help="host pipeline frames per chunk (0 = automatic)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every ~2 ms) during the timed
    region; falls back to nvidia-smi polling when NVML is unavailable."""

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reasons_bitmask)
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._ready.set()
            while not self._stop.is_set():
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                self._stop.wait(0.002)
            nv.nvmlShutdown()
        except Exception:
            self._ready.set()
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.device),
                         "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip().split(",")
                    self.samples.append((int(out[0]), int(out[1]), int(out[2].strip(), 16)))
                except Exception:
                    pass
                self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(30)
        time.sleep(0.01)  # at least a few samples before the region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def summary(self):
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for bit, name in self.REASONS.items()
                          if s[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(s[1] for s in self.samples) if sm else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload):
    """dram read+write bytes per K1 launch from a committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def workload_config(args, wl, F, world):
    """The `config` object of BOTH arms (same keys and values, so the driver's
    same-config check compares like with like)."""
    M, N, C, _, b, n, m, eps, adaptive, desc = wl
    pitch = ((N * C + 15) // 16) * 16
    mpitch = ((N + 15) // 16) * 16
    working_set = 2 * F * M * pitch + (F * M * mpitch if adaptive else 0)
    flush_l2 = working_set < 2 * 126 * 2**20
    cfg = {"workload": desc, "frames_per_gpu": F, "shape": f"{N}x{M}x{C}",
           "b": b, "n": n, "m": m, "epsilon": eps,
           "noise": "keyed splitmix64 + inverse-CDF Laplace (reference stream), "
                    "per-(frame, channel) derived plane seeds",
           "mask": "u8 centred ellipse (0.4M x 0.2N), ~25% complex" if adaptive else None,
           "l2": (f"working set {working_set / 1e9:.4f} GB < 2 x 126 MB L2: each step timed "
                  "alone after a 512 MB write that evicts L2" if flush_l2 else
                  f"working set {working_set / 1e9:.2f} GB > 2 x 126 MB L2, no flush needed"),
           "parallelism": f"frame-parallel x{world}, no collective on the data path",
           "out_pad": ("none (N*C % 16 == 0)" if pitch == N * C else
                       "output row padding never written" if args.no_pad_scratch else
                       f"rows padded {N * C} -> {pitch} B, padding declared scratch: "
                       "stores end on whole 32-B sectors")}
    if args.workload == "sweep":
        cfg["runs"] = [f"b{bb} eps{ee}" for bb, ee in SWEEP]
    return cfg, working_set, flush_l2


# ----------------------------------------------------------------------------
# reference CPU arm (oracle/_ref = the reference compiled from its sources)
# ----------------------------------------------------------------------------
def cpu_reference_sample(M, N, C, b, n, m, eps, adaptive, seconds, frame0=0):
    import numpy as np

    import oracle
    if oracle.ref is None:
        return None
    workers = os.cpu_count() or 1
    one = oracle.synth_frames(frame0, 1, M, N, C)[0]
    mask1 = oracle.synth_masks(frame0, 1, M, N)
    planes1 = np.ascontiguousarray(one.transpose(2, 0, 1))
    t = oracle.ref.time_planes(planes1[:1], mask1, not adaptive, eps, m, b, n, 42, 1)
    per_plane = max(t, 1e-5)
    n_planes = int(max(C, min(3 * 600, seconds / per_plane)))
    n_frames = max(1, n_planes // C)
    frames = oracle.synth_frames(frame0, n_frames, M, N, C)
    masks = oracle.synth_masks(frame0, n_frames, M, N)
    # colour planes are de-interleaved upstream, untimed
    planes = np.ascontiguousarray(frames.transpose(0, 3, 1, 2)).reshape(n_frames * C, M, N)
    pmasks = np.repeat(masks, C, axis=0) if adaptive else None
    return dict(planes=planes, masks=pmasks, n_frames=n_frames, workers=workers)


def run_reference_once(sample, M, N, C, b, n, m, eps, adaptive):
    import oracle
    return oracle.ref.time_planes(sample["planes"], sample["masks"], not adaptive, eps, m, b, n,
                                  42, sample["workers"])


def reference_arm(args, wl, F, world):
    M, N, C, _, b, n, m, eps, adaptive, desc = wl
    import oracle
    if oracle.ref is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libdppix_ref.so not built (needs /root/reference)"}))
        return
    per_step = max(2.0, min(args.cpu_seconds, 20.0))
    sample = cpu_reference_sample(M, N, C, b, n, m, eps, adaptive, per_step)
    for _ in range(args.warmup):
        run_reference_once(sample, M, N, C, b, n, m, eps, adaptive)
    times = [run_reference_once(sample, M, N, C, b, n, m, eps, adaptive) for _ in range(args.steps)]
    t = statistics.median(times)  # median over the K steps (each a whole bounded sample)
    mp = sample["n_frames"] * M * N / 1e6
    value = mp / t
    cfg, _, _ = workload_config(args, wl, F, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "MP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "frames_per_sec": round(sample["n_frames"] / t, 3),
        "config": cfg,
        "cpu_baseline": {"value": round(value, 3), "unit": "MP/s", "cores": sample["workers"],
                         "kind": "reference", "cpu_model": cpu_model(),
                         "statistic": f"median of {args.steps} steps",
                         "step_seconds": [round(x, 4) for x in times],
                         "sample": f"{sample['n_frames']} frames x {C} planes of the workload per step, "
                                   f"pixelize_{'adaptive' if adaptive else 'parallel'} per plane "
                                   f"(threads=1), frame-parallel over {sample['workers']} threads "
                                   "(run_batch scheme, cli.cpp:175-213)"},
        "e2e": {"value": round(value, 3), "unit": "MP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_spawn(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with N ranks on this node (one process per GPU), the
    launch the driver itself uses; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    sys.stdout.flush()
    os.execvpe(cmd[0], cmd, env)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_spawn(args)
    if world > 1 and args.gpus != world and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} ranks",
              file=sys.stderr)
    wl = WORKLOADS[args.workload]
    M, N, C, F, b, n, m, eps, adaptive, desc = wl
    if args.frames:
        F = args.frames

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, wl, F, world)
        return

    import numpy as np
    import torch

    import paper_2511_04261_b200 as dp
    from paper_2511_04261_b200 import shard as sh

    # One process per GPU (LOCAL_RANK). DPPX_DIST_BACKEND=gloo + DPPX_FORCE_DEVICE
    # exist only to exercise the multi-rank launcher on a single test GPU (the
    # ranks never wait on each other's kernels).
    gpu = int(os.environ.get("DPPX_FORCE_DEVICE", local))
    backend = os.environ.get("DPPX_DIST_BACKEND", "nccl")
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    local = gpu
    pg = None
    if world > 1:
        import torch.distributed as tdist
        if backend == "nccl":
            # Communicator init lines (nranks) for the driver's log; NCCL carries
            # only the barrier and the end-of-run max/sum of timings.
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
        pg = tdist
    red_dev = dev if backend == "nccl" else torch.device("cpu")

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if not pg:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    ctx = dp.Context(local)
    # `out` below is the bench's own buffer: its row padding (pitch - N*C) is
    # scratch, so rows may end on whole 32-byte sectors (dppx_ctx_set_out_pad_scratch).
    ctx.set_out_pad_scratch(not args.no_pad_scratch)
    # torch's work (allocations, L2 flushes, reductions) runs on the context
    # stream: ordered with the kernels, and the _dev wrappers add no fences
    torch.cuda.set_stream(torch.cuda.ExternalStream(ctx.stream, device=dev))
    geom = dp.grid_dims(M, N, b)
    G = geom.grid_count()
    p = dp.make_privacy_params(eps, m, b, n)
    pitch = ((N * C + 15) // 16) * 16
    mpitch = ((N + 15) // 16) * 16
    d = dp._desc(M, N, C, F, pitch=pitch, mpitch=mpitch, opitch=pitch)
    my = sh.weak_shard(rank, world, F)  # global frame indices key the noise
    frame0 = my.frame0
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, mpitch), dtype=torch.uint8, device=dev) if adaptive else None
    ctx.synth_frames_dev(d, 101, frame0, img, mask)
    if adaptive:
        cap = dp.adaptive_payload_capacity(M, N, b, n)
        sstride = (cap + 15) // 16 * 16
    else:
        sstride = G
    stats = torch.zeros((F * C, sstride), dtype=torch.uint8, device=dev)
    lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
    seeds = sh.plane_seed_list(42, my, C)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, seeds)
    sweep = args.workload == "sweep"
    fused = sweep and args.sweep_mode == "fused"
    jobs = []  # (params, means buffer, G, image buffer) per run of one step
    if sweep:
        for bb, ee in SWEEP:
            gb = dp.grid_dims(M, N, bb).grid_count()
            jobs.append((dp.make_privacy_params(ee, m, bb),
                         torch.zeros((F * C, gb), dtype=torch.uint8, device=dev), gb,
                         out if not fused else torch.empty_like(img)))
    runs = len(jobs) if sweep else 1
    sweep_b = sorted({bb for bb, _ in SWEEP})
    sweep_e = sorted({ee for _, ee in SWEEP})

    def step():
        if fused:  # one read of the frames, every run's statistics + image
            ctx.pixelize_uniform_sweep_dev(d, img, sweep_b, sweep_e, m, nz, [j[1] for j in jobs],
                                           [j[3] for j in jobs])
        elif sweep:
            for pj, mj, _, oj in jobs:
                ctx.pixelize_uniform_dev(d, img, pj, nz, mj, oj)
        elif adaptive:
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, sstride, lens, out)
        else:
            ctx.pixelize_uniform_dev(d, img, p, nz, stats, out)

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    # payload bytes actually written (for the roofline's algorithmic bytes)
    payload_bytes = int(lens.sum().item()) if adaptive else F * C * G
    if sweep:
        payload_bytes = sum(F * C * j[2] for j in jobs) / runs  # mean per K1 launch
    # ---- timed region: device-resident ----
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    ctx.reset_stats()
    ctx.set_timing(True)
    barrier()
    config, working_set, flush_l2 = workload_config(args, wl, F, world)
    scratch = torch.empty(512 * 2**20, dtype=torch.uint8, device=dev) if flush_l2 else None
    with ClockSampler(local) as clk:
        if flush_l2:
            # each step timed on its own; a 512 MB write evicts L2 between steps
            ms_total = 0.0
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    scratch.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                e1.synchronize()
                ms_total += e0.elapsed_time(e1)
        else:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            ev1.synchronize()
            ms_total = ev0.elapsed_time(ev1)
    barrier()
    st = ctx.stats()
    ctx.set_timing(False)
    ms_step = allmax(ms_total / args.steps)
    frames_total = F * world * runs
    value = frames_total * M * N / 1e6 / (ms_step / 1e3)
    fps = frames_total / (ms_step / 1e3)
    # roofline of K1 (dominant kernel): algorithmic bytes / measured duration
    kfam = ("stats_tma" if st["launches"]["stats_tma"] else
            "stats_rows" if st["launches"].get("stats_rows") else "stats_generic")
    sweep_info = None
    if fused:
        # K1s reads each frame once and writes 12 means arrays; 12 broadcasts
        # (K2, write-only) produce the images. The dominant kernel is K2.
        means_bytes = sum(F * C * j[2] for j in jobs)
        s_ms = st["device_ms"]["sweep"] / max(1, st["launches"]["sweep"])
        e_ms = st["device_ms"]["expand"] / max(1, st["launches"]["expand"])
        s_bytes = F * M * N * C + means_bytes
        e_bytes = F * M * N * C + means_bytes / runs
        per_run_bytes = runs * 2 * F * M * N * C + means_bytes  # 12 separate read+write runs
        one_read_bytes = F * M * N * C * (1 + runs) + 2 * means_bytes
        step_s = ms_total / args.steps / 1e3
        pk, _ = measured_peak()
        sweep_info = {
            "k1s_ms": round(s_ms, 4), "k1s_algorithmic_bytes": int(s_bytes),
            "k1s_gbs": round(s_bytes / (s_ms / 1e3) / 1e9, 1),
            "k1s_frac": round(s_bytes / (s_ms / 1e3) / 1e9 / pk, 4),
            "k2_ms_per_run": round(e_ms, 4), "k2_algorithmic_bytes_per_run": int(e_bytes),
            "k2_frac": round(e_bytes / (e_ms / 1e3) / 1e9 / pk, 4),
            "step_bytes_one_read": int(one_read_bytes),
            "step_bytes_per_run_accounting": int(per_run_bytes),
            "step_frac_one_read": round(one_read_bytes / step_s / 1e9 / pk, 4),
            "step_frac_per_run_accounting": round(per_run_bytes / step_s / 1e9 / pk, 4),
            "note": "one read of each frame for all 12 runs (K1s), then 12 write-only broadcasts"}
        # the draws of the 4-px level overlap the other levels' broadcasts on a
        # second stream, so per-kernel durations are not separable: the roofline
        # is the whole step against the one-read algorithmic bytes
        kfam = "expand"
        k1_launches = 1
        k1_ms = ms_total / args.steps
        k1_bytes = int(one_read_bytes)
    else:
        k1_launches = max(1, st["launches"][kfam])
        k1_ms = st["device_ms"][kfam] / k1_launches
        k1_bytes = int(F * M * N * C * 2 + payload_bytes)  # read frame, write image, write stats
    k0_bytes = (F * M * N + 4 * G * C * F + 4 * F * C) if adaptive else 0
    peak, peak_src = measured_peak()
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9
    step_gbs = ((sweep_info["step_bytes_one_read"] if fused else k1_bytes * runs + k0_bytes)
                / (ms_total / args.steps / 1e3) / 1e9)
    traffic = ncu_traffic(args.workload)
    launches_timed = sum(st["launches"].values())

    # ---- standalone reconstruction (reassemble / broadcast_means): K0(payload) + K2 ----
    recon = None
    try:
        ctx.reset_stats()
        ctx.set_timing(True)
        reps = 3
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(reps + 1):
            if i == 1:
                r0.record(stream)
            if adaptive:
                ctx.reassemble_dev(d, stats, sstride, lens, b, n, out)
            else:
                ctx.broadcast_means_dev(d, stats, b, out)
        r1.record(stream)
        r1.synchronize()
        ctx.synchronize()
        rs = ctx.stats()
        ctx.set_timing(False)
        k2_ms = rs["device_ms"]["expand"] / max(1, rs["launches"]["expand"])
        k2_bytes = F * M * N * C + payload_bytes
        recon = {"ms_per_call": round(r0.elapsed_time(r1) / reps, 4),
                 "k2_ms": round(k2_ms, 4),
                 "k2_gbs": round(k2_bytes / (k2_ms / 1e3) / 1e9, 1),
                 "k2_frac": round(k2_bytes / (k2_ms / 1e3) / 1e9 / peak, 4),
                 "k2_algorithmic_bytes": k2_bytes}
    except Exception as exc:  # reported, never fatal for the headline
        recon = {"error": str(exc)[:200]}

    # ---- e2e: public host API, pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        Fe = min(F, args.e2e_frames or max(1, (1 << 30) // (M * N * (C + (1 if adaptive else 0)))))
        hbytes = Fe * M * N * C
        h_img = torch.empty((Fe, M, N, C), dtype=torch.uint8).pin_memory()
        h_img.copy_(img[:Fe, :, : N * C].reshape(Fe, M, N, C).cpu())
        h_mask = None
        if adaptive:
            h_mask = torch.empty((Fe, M, N), dtype=torch.uint8).pin_memory()
            h_mask.copy_(mask[:Fe, :, :N].cpu())
        h_out = torch.empty((Fe, M, N, C), dtype=torch.uint8).pin_memory()
        h_stats = torch.zeros((Fe * C, sstride), dtype=torch.uint8).pin_memory()
        h_lens = torch.zeros(Fe * C, dtype=torch.int32).pin_memory()
        de = dp._desc(M, N, C, Fe)
        seeds_e = dp.plane_seeds(42, Fe, C, frame0=frame0)
        nze, keep_e = dp.Context._noise(dp.NOISE_KEYED, seeds_e)
        import ctypes as Ct

        h_means = [torch.zeros((Fe * C, j[2]), dtype=torch.uint8).pin_memory() for j in jobs]

        sw_mp = (Ct.c_void_p * len(jobs))(*[hm.data_ptr() for hm in h_means])
        sw_op = (Ct.c_void_p * len(jobs))(*([h_out.data_ptr()] * len(jobs)))
        sw_b = (Ct.c_int32 * len(sweep_b))(*sweep_b) if sweep else None
        sw_e = (Ct.c_double * len(sweep_e))(*sweep_e) if sweep else None

        def e2e_step():
            if fused:  # one upload, every run's means and image back (h_out reused per run)
                ctx._check(dp._lib.dppx_pixelize_uniform_sweep(
                    ctx._h, Ct.byref(de), h_img.data_ptr(), len(sweep_b), sw_b, len(sweep_e), sw_e, m,
                    Ct.byref(nze), sw_mp, sw_op, None, None), "e2e")
                return
            if sweep:
                for (pj, _, _, _), hm in zip(jobs, h_means):
                    ctx._check(dp._lib.dppx_pixelize_uniform(ctx._h, Ct.byref(de), h_img.data_ptr(),
                                                             Ct.byref(pj), Ct.byref(nze),
                                                             hm.data_ptr(), h_out.data_ptr()), "e2e")
                return
            if adaptive:
                rc = dp._lib.dppx_pixelize_adaptive(ctx._h, Ct.byref(de), h_img.data_ptr(),
                                                    h_mask.data_ptr(), Ct.byref(p), Ct.byref(nze),
                                                    h_stats.data_ptr(), sstride,
                                                    h_lens.data_ptr(), h_out.data_ptr())
            else:
                rc = dp._lib.dppx_pixelize_uniform(ctx._h, Ct.byref(de), h_img.data_ptr(),
                                                   Ct.byref(p), Ct.byref(nze), h_stats.data_ptr(),
                                                   h_out.data_ptr())
            ctx._check(rc, "e2e")

        # link roofline: pinned copies of the same byte counts, each direction alone
        def link_gbs(nbytes, h2d):
            hb = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            for _ in range(2):
                (db.copy_(hb, non_blocking=True) if h2d else hb.copy_(db, non_blocking=True))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                (db.copy_(hb, non_blocking=True) if h2d else hb.copy_(db, non_blocking=True))
            e1.record()
            e1.synchronize()
            return 3 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9

        h2d_link = link_gbs(1 << 30, True)
        d2h_link = link_gbs(1 << 30, False)

        def duplex_gbs(nbytes):  # both directions at once, on two streams
            ha = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            hb = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            da = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                with torch.cuda.stream(s1):
                    da.copy_(ha, non_blocking=True)
                with torch.cuda.stream(s2):
                    hb.copy_(db, non_blocking=True)
            torch.cuda.synchronize()
            return 6 * nbytes / (time.perf_counter() - t0) / 1e9

        duplex_link = duplex_gbs(1 << 29)
        ctx.set_chunk_frames(args.chunk_frames)
        # small calls (a single PETS frame) are latency-bound: time many of them
        e_steps = args.e2e_steps if hbytes >= (16 << 20) else max(args.e2e_steps, 200)
        for _ in range(max(2, min(e_steps // 10, 20))):
            e2e_step()
        ctx.reset_stats()
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        t1 = time.perf_counter()
        barrier()
        es = ctx.stats()
        args.e2e_steps = e_steps  # (per-step byte counts below)
        e_ms = allmax((t1 - t0) / e_steps * 1e3)
        e2e = {"value": round(Fe * runs * world * M * N / 1e6 / (e_ms / 1e3), 3), "unit": "MP/s",
               "h2d_bytes_per_step": es["h2d_bytes"] // args.e2e_steps,
               "d2h_bytes_per_step": es["d2h_bytes"] // args.e2e_steps,
               "frames_per_step": Fe, "ms_per_step": round(e_ms, 3),
               "kernel_launches": {k: v for k, v in es["launches"].items() if v},
               "frames_per_sec": round(Fe * runs * world / (e_ms / 1e3), 3),
               "link_gbs": {"h2d": round(h2d_link, 1), "d2h": round(d2h_link, 1),
                            "duplex": round(duplex_link, 1)},
               "duplex_frac": round((es["h2d_bytes"] + es["d2h_bytes"]) / args.e2e_steps
                                    / (duplex_link * 1e9) / (e_ms / 1e3), 4),
               "link_frac": round(max(es["h2d_bytes"] / args.e2e_steps / (h2d_link * 1e9),
                                      es["d2h_bytes"] / args.e2e_steps / (d2h_link * 1e9))
                                  / (e_ms / 1e3), 4),
               "path": "dppx_pixelize_adaptive (host pointers, pinned, chunked H2D/K0/K1/D2H "
                       "pipeline on 3 streams)" if adaptive else
                       ("dppx_pixelize_uniform_sweep (one upload of the frames; every run's means "
                        "and image back to host)" if fused else
                        ("dppx_pixelize_uniform (one pinned frame: K1z reads and writes the mapped "
                         "host buffers over PCIe, no staging copies)" if es["launches"].get("stats_zerocopy")
                         else "dppx_pixelize_uniform"))}
        del h_img, h_mask, h_out, h_stats

    # ---- CPU reference baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = cpu_reference_sample(M, N, C, b, n, m, eps, adaptive, args.cpu_seconds / 3, frame0)
        if sample is not None:
            runs = sorted(run_reference_once(sample, M, N, C, b, n, m, eps, adaptive) for _ in range(3))
            t = runs[1]  # median of 3
            # single-thread reference on one frame (all C planes), as SURVEY 8(d) asks
            import oracle
            k1 = min(C, sample["planes"].shape[0])
            t1 = oracle.ref.time_planes(sample["planes"][:k1],
                                        sample["masks"][:k1] if adaptive else None, not adaptive,
                                        eps, m, b, n, 42, 1)
            cpu = {"value": round(sample["n_frames"] * M * N / 1e6 / t, 3), "unit": "MP/s",
                   "single_thread_value": round(M * N / 1e6 / (t1 * C / k1), 3),
                   "cores": sample["workers"], "kind": "reference", "cpu_model": cpu_model(),
                   "statistic": "median of 3 runs", "run_seconds": [round(x, 4) for x in runs],
                   "sample": f"{sample['n_frames']} frames x {C} planes, pixelize_"
                             f"{'adaptive' if adaptive else 'parallel'} per plane (threads=1), "
                             f"frame-parallel over {sample['workers']} threads, {t:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "MP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "frames_per_sec": round(fps, 1),
            "config": config,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic,
                         "kernel": ("sweep step: K1s (one read: level sums + draws of all 12 runs) "
                                    "and 12 broadcasts, overlapped on two streams" if fused
                                    else f"K1 {kfam}"),
                         "algorithmic_bytes_per_launch": k1_bytes,
                         "avg_launch_ms": round(k1_ms, 4), "peak_source": peak_src,
                         # context only: HGX nominal 7.7 TB/s (B200_PROFILING.md)
                         "frac_of_nominal_7700": round(achieved / 7700.0, 4),
                         "step_gbs_incl_K0": round(step_gbs, 1),
                         "step_frac_incl_K0": round(step_gbs / peak, 4),
                         "k0_ms_per_launch": round(st["device_ms"]["classify"] /
                                                   max(1, st["launches"]["classify"]), 4)},
            "cpu_baseline": cpu,
            "sweep": sweep_info,
            "reconstruct": recon,
            "e2e": e2e,
            "gpu_launches": launches_timed,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    ctx.close()
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
