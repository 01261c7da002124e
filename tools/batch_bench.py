#!/usr/bin/env python3
"""Batch runner, end to end on files: the reference's run_batch
(cli.cpp:175-213, compiled from its sources: oracle/_ref/dppix_batch_ref) vs
run_batch_gpu (include/dppix/batch.hpp: tests/cpp/batch_gpu) on the same
directory of P5 PGM frames + paired masks. Both write <stem>.pix.pgm and
<stem>.dppx and run the reconstruct check + metrics; the tool times both and
compares every output file byte for byte.

usage (GPU box): python tools/batch_bench.py [--files 64] [--height 1080] [--width 1920]
"""
import argparse
import filecmp
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode())
        f.write(img.tobytes())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--files", type=int, default=64)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--mode", default="a", choices=["a", "u"])
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--dir", default="/tmp/dppx_batch")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np

    import oracle
    M, N, F = args.height, args.width, args.files
    shutil.rmtree(args.dir, ignore_errors=True)
    d_in, d_mask = os.path.join(args.dir, "in"), os.path.join(args.dir, "masks")
    d_ref, d_gpu = os.path.join(args.dir, "out_ref"), os.path.join(args.dir, "out_gpu")
    for d in (d_in, d_mask, d_ref, d_gpu):
        os.makedirs(d)
    frames = oracle.synth_frames(0, F, M, N, 1)[..., 0]
    masks = oracle.synth_masks(0, F, M, N)
    for i in range(F):
        write_pgm(os.path.join(d_in, f"f{i:05d}.pgm"), frames[i])
        write_pgm(os.path.join(d_mask, f"f{i:05d}.pgm"), (masks[i] * 255).astype(np.uint8))
    n = args.n if args.mode == "a" else 1
    common = [args.mode, d_mask, "0.5", "16", str(args.b), str(n), "42"]
    threads = str(os.cpu_count() or 1)
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "dppix_batch_ref")
    gpu_bin = os.path.join(ROOT, "tests", "cpp", "batch_gpu")
    def run(cmd, reps):  # median of `reps` whole-process runs (each includes its own setup)
        outs = [json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
                for _ in range(reps)]
        outs.sort(key=lambda o: o["seconds"])
        med = dict(outs[len(outs) // 2])
        med["runs_s"] = [o["seconds"] for o in outs]
        return med
    if os.environ.get("DPPX_BATCH_TRACE"):  # per-phase trace of one GPU run (stderr)
        r = subprocess.run([gpu_bin, d_in, d_gpu] + common + ["0"], capture_output=True, text=True)
        sys.stderr.write(r.stderr)
    ref = run([ref_bin, d_in, d_ref] + common + [threads], args.reps)
    # GPU arm: one untimed warm-up process (file cache, driver), then `reps`
    subprocess.run([gpu_bin, d_in, d_gpu] + common + ["0"], check=True, capture_output=True)
    gpu = run([gpu_bin, d_in, d_gpu] + common + ["0"], args.reps)
    if os.environ.get("DPPX_BATCH_TRACE"):  # and one more after the timed runs (outputs exist now)
        r = subprocess.run([gpu_bin, d_in, d_gpu] + common + ["0"], capture_output=True, text=True)
        sys.stderr.write("after timed runs:\n" + r.stderr)
    names = sorted(os.listdir(d_ref))
    same = names == sorted(os.listdir(d_gpu)) and all(
        filecmp.cmp(os.path.join(d_ref, x), os.path.join(d_gpu, x), shallow=False) for x in names)
    mp = F * M * N / 1e6
    print(json.dumps({
        "workload": f"{F} P5 files {N}x{M} gray, {'adaptive' if args.mode == 'a' else 'uniform'} "
                    f"b{args.b} n{n} eps 0.5 m 16, same seed per file (run_batch), outputs "
                    ".pix.pgm + .dppx, reconstruct check + metrics",
        "reference": {**ref, "threads": int(threads), "MP_per_s": round(mp / ref["seconds"], 1)},
        "gpu": {**gpu, "MP_per_s": round(mp / gpu["seconds"], 1)},
        "speedup": round(ref["seconds"] / gpu["seconds"], 2), "statistic": f"median of {args.reps} runs",
        "outputs_identical": same, "output_files": len(names)}))
    shutil.rmtree(args.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
