#!/usr/bin/env python3
"""Generate tests/golden/*.npz|json from the REFERENCE itself.

The reference (/root/reference/proj/src, unmodified) is compiled by
oracle/Makefile into oracle/_ref/libdppix_ref.so; this script calls it through
oracle/ref_shim.cpp and stores inputs (when small) and outputs. /root/reference
does not exist on the GPU box: the committed fixtures are what travels.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

ref = oracle.ref
assert ref is not None, "oracle/_ref not built (needs /root/reference)"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def noise_vectors():
    rng = np.random.default_rng(2511)
    out = []
    for i in range(96):
        seed = int(rng.integers(0, 2**63)) if i else 42
        k = [int(x) for x in rng.integers(0, 2**20, 4)]
        sigma = float(rng.choice([1.0, 31.875, 510.0, 2550.0]))
        bits = ref.keyed_bits(seed, *k)
        u = ref.uniform_from_bits(bits)
        lap = ref.laplace_at(seed, *k, sigma)
        out.append({"seed": str(seed), "key": k, "sigma": sigma, "bits": str(bits),
                    "u": u.hex(), "laplace": lap.hex()})
    # the uniform clamp endpoints (noise.cpp:99-104)
    ends = {"u_of_0": ref.uniform_from_bits(0).hex(),
            "u_of_max": ref.uniform_from_bits(2**64 - 1).hex()}
    json.dump({"source": "reference noise.cpp via oracle/_ref", "draws": out, "ends": ends},
              open(os.path.join(HERE, "noise.json"), "w"), indent=0)


def small_cases():
    """Random small gray images: inputs stored, outputs from the reference."""
    rng = np.random.default_rng(4261)
    cases = {}
    n_case = 0
    while n_case < 40:
        M, N = int(rng.integers(1, 48)), int(rng.integers(1, 48))
        b = int(rng.integers(1, min(max(M, N), 12) + 1))
        g = oracle.grid_dims(M, N, b)
        if (g.pad_rows or g.pad_cols) and (g.pad_rows >= M or g.pad_cols >= N):
            continue
        n = int(rng.choice([d for d in range(1, b + 1) if b % d == 0]))
        eps = float(rng.choice([0.1, 0.5, 1.0, 2.0]))
        m = int(rng.integers(1, 32))
        seed = int(rng.integers(0, 2**63)) if n_case % 5 else None
        img = rng.integers(0, 256, (M, N), dtype=np.uint8)
        mask = rng.integers(0, 2, (M, N), dtype=np.uint8)
        uimg, umeans = ref.pixelize_parallel(img, eps, m, b, seed)
        aimg, payload = ref.pixelize_adaptive(img, mask, eps, m, b, n, seed)
        k = f"c{n_case:02d}"
        cases[f"{k}_img"] = img
        cases[f"{k}_mask"] = mask
        cases[f"{k}_params"] = np.array([M, N, b, n, m, -1 if seed is None else 0], np.int64)
        cases[f"{k}_eps"] = np.array([eps])
        cases[f"{k}_seed"] = np.array([seed or 0], np.uint64)
        cases[f"{k}_umeans"] = umeans
        cases[f"{k}_uimg"] = uimg
        cases[f"{k}_payload"] = np.frombuffer(payload, np.uint8)
        cases[f"{k}_aimg"] = aimg
        cases[f"{k}_refimg"] = ref.pixelize_reference(img, eps, m, b, seed)  # Algorithm 1
        n_case += 1
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **cases)


def shaped_cases():
    """BASELINE shapes on one gray plane of the deterministic synthetic frame
    (oracle.synth_frames, reproduced bit for bit by the device generator):
    outputs (means / payloads) stored, images by sha256."""
    out = {}
    specs = [
        ("pets_uniform_b16", 576, 768, 16, 1, 16, 0.5, False),
        ("venice_adaptive_b16n4", 1080, 1920, 16, 4, 16, 0.5, True),
        ("sweep_uniform_b4_eps0.1", 1083, 1917, 4, 1, 16, 0.1, False),
        ("sweep_uniform_b32_eps1", 1083, 1917, 32, 1, 16, 1.0, False),
        ("celeba_adaptive_b16n4", 218, 178, 16, 4, 16, 0.5, True),
    ]
    for name, M, N, b, n, m, eps, adaptive in specs:
        frame = oracle.synth_frames(3, 1, M, N, 3)[0]
        mask = oracle.synth_masks(3, 1, M, N)[0]
        for ch in range(3):
            plane = np.ascontiguousarray(frame[:, :, ch])
            seed = oracle.derive_plane_seed(42, 3, ch)
            key = f"{name}_ch{ch}"
            if adaptive:
                img, payload = ref.pixelize_adaptive(plane, mask, eps, m, b, n, seed)
                out[f"{key}_payload"] = np.frombuffer(payload, np.uint8)
            else:
                img, means = ref.pixelize_parallel(plane, eps, m, b, seed)
                out[f"{key}_means"] = means
            out[f"{key}_imgsha"] = np.frombuffer(bytes.fromhex(sha(img)), np.uint8)
        out[f"{name}_spec"] = np.array([M, N, b, n, m], np.int64)
        out[f"{name}_eps"] = np.array([eps])
        out[f"{name}_inputsha"] = np.frombuffer(bytes.fromhex(sha(frame)), np.uint8)
        out[f"{name}_masksha"] = np.frombuffer(bytes.fromhex(sha(mask)), np.uint8)
    np.savez_compressed(os.path.join(HERE, "shaped_cases.npz"), **out)


def records():
    """Complete .dppx records from the reference's encode (record.cpp:124-175)."""
    recs = {}
    img = np.ascontiguousarray(oracle.synth_frames(0, 1, 576, 768, 1)[0, :, :, 0])
    recs["pets_uniform_b16"] = ref.encode_uniform(img, 0.5, 16, 16, 11)
    mask = oracle.synth_masks(0, 1, 576, 768)[0]
    recs["pets_adaptive_b16n4"] = ref.encode_adaptive(img, mask, 0.5, 16, 16, 4, 11)
    np.savez_compressed(os.path.join(HERE, "records.npz"),
                        **{k: np.frombuffer(v, np.uint8) for k, v in recs.items()})


def config_digests():
    """Every BASELINE config and every kernel family's grid side, RGB, pinned
    to the reference by sha256 (payload / means bytes and image per plane):
    config 4 (4K adaptive b32 n8), all 12 sweep runs of config 3, CelebA
    uniform + adaptive, and the paper's other grid sides at 1080p (b = 12, 24,
    30, 40, 64, 128 with n up to 32). Inputs are the deterministic synthetic
    frames (oracle.synth_frames / synth_masks, frame 5), plane seeds derived
    from (42, frame 5, channel)."""
    specs = [("4k_adaptive_b32n8", 2160, 3840, 32, 8, 16, 0.5, True)]
    for b in (4, 8, 16, 32):
        for eps in (0.1, 0.5, 1.0):
            specs.append((f"sweep_b{b}_eps{eps}", 1083, 1917, b, 1, 16, eps, False))
    specs += [("celeba_uniform_b16", 218, 178, 16, 1, 16, 0.5, False),
              ("pets_adaptive_b16n4", 576, 768, 16, 4, 16, 0.5, True)]
    for b, n in ((12, 1), (12, 3), (24, 4), (24, 8), (30, 1), (30, 5), (30, 10), (40, 4), (40, 8),
                 (64, 16), (64, 8), (128, 8), (128, 16), (128, 32), (16, 8), (20, 5), (2, 2), (7, 1)):
        specs.append((f"1080p_b{b}n{n}", 1080, 1920, b, n, 16, 0.5, n > 1 or b in (30, 128)))
    out = {}
    frames = {}
    for name, M, N, b, n, m, eps, adaptive in specs:
        if (M, N) not in frames:
            frames[(M, N)] = (oracle.synth_frames(5, 1, M, N, 3)[0], oracle.synth_masks(5, 1, M, N)[0])
        frame, mask = frames[(M, N)]
        ent = {"M": M, "N": N, "b": b, "n": n, "m": m, "eps": eps, "adaptive": adaptive,
               "input_sha": sha(frame), "mask_sha": sha(mask), "planes": []}
        for ch in range(3):
            plane = np.ascontiguousarray(frame[:, :, ch])
            seed = oracle.derive_plane_seed(42, 5, ch)
            if adaptive:
                img, payload = ref.pixelize_adaptive(plane, mask, eps, m, b, n, seed)
                stats = np.frombuffer(payload, np.uint8)
            else:
                img, stats = ref.pixelize_parallel(plane, eps, m, b, seed)
            ent["planes"].append({"stats_len": int(stats.size), "stats_sha": sha(stats),
                                  "image_sha": sha(img)})
        out[name] = ent
    json.dump({"source": "reference pixelize_parallel / pixelize_adaptive via oracle/_ref",
               "frame": 5, "seed": 42, "cases": out},
              open(os.path.join(HERE, "config_digests.json"), "w"), indent=1)


if __name__ == "__main__":
    noise_vectors()
    small_cases()
    shaped_cases()
    records()
    config_digests()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
