"""Multi-GPU paths on one B200 (the pool gives one GPU per call): the C++
device-group runner (dppx_group_*: one host thread + ctx per listed device;
here the same device listed several times) and the multi-rank bench launch
(one process per rank, gloo for the plumbing, every rank on GPU 0). Both are
checked byte-for-byte against a single context over the whole batch: noise is
keyed per plane / global frame, never by device or rank."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

import paper_2511_04261_b200 as dp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workers", [2, 3])
@pytest.mark.parametrize("M,N,C,b,n", [(72, 136, 3, 16, 4), (218, 178, 3, 16, 4), (61, 253, 3, 30, 5)])
def test_group_matches_single_context(ctx, workers, M, N, C, b, n):
    F = 7  # uneven blocks over 2 and 3 workers
    frames = oracle.synth_frames(11, F, M, N, C)
    masks = oracle.synth_masks(11, F, M, N)
    g = dp.Group([0] * workers)
    try:
        assert g.devices == [0] * workers
        p = dp.make_privacy_params(0.5, 16, b, n)
        seeds = dp.plane_seeds(42, F, C)
        G = dp.grid_dims(M, N, b).grid_count()
        inj = np.random.default_rng(1).laplace(0, 20, (F * C, G * n * n))
        for kind, sd, injected in ((dp.NOISE_KEYED, seeds, None), (dp.NOISE_PHILOX, [99], None),
                                   (dp.NOISE_INJECTED, None, inj), (dp.NOISE_NONE, None, None)):
            pa, ia = g.pixelize_adaptive(frames, masks, p, kind, sd, frame_base=5, injected=injected)
            pb, ib = ctx.pixelize_adaptive(frames, masks, p, kind, sd, frame_base=5, injected=injected)
            assert pa == pb and np.array_equal(ia, ib), kind
        back = g.reassemble(pa, M, N, b, n, channels=C, frames=F)
        assert np.array_equal(back, ia)
        pu = dp.make_privacy_params(0.5, 16, b)
        ma, ua = g.pixelize_uniform(frames, pu, dp.NOISE_KEYED, seeds)
        mb, ub = ctx.pixelize_uniform(frames, pu, dp.NOISE_KEYED, seeds)
        assert np.array_equal(ma, mb) and np.array_equal(ua, ub)
        assert np.array_equal(g.broadcast_means(ma, M, N, b, channels=C, frames=F), ua)
        st = g.stats()
        assert st["launches"]["classify"] >= workers  # every worker ran kernels
        # errors keep the reference taxonomy
        bad = [bytes(len(pa[0]))] * (F * C)
        with pytest.raises(dp.RecordError):
            g.reassemble(bad, M, N, b, n, channels=C, frames=F)
        with pytest.raises(ValueError):
            g.pixelize_uniform(frames, dp.make_privacy_params(0.5, 16, b, n) if n > 1 else
                               dp.make_privacy_params(0.5, 16, 4 * max(M, N)), dp.NOISE_KEYED, seeds)
    finally:
        g.close()


def _run(cmd, env_extra, timeout=600):
    env = dict(os.environ, **env_extra)
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_two_rank_shards_byte_identical_on_gpu(tmp_path):
    """tools/shard_check.py under torchrun: 2 ranks (gloo plumbing, both on GPU
    0 -- the ranks never wait on each other's kernels) each pixelize their
    strong shard of a 9-frame clip through the GPU path; rank 0 gathers the
    digests and compares them with a 1-rank run of the whole clip."""
    out = tmp_path / "shard.json"
    r = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
              "--master-addr=127.0.0.1", "--master-port=29517", "tools/shard_check.py", str(out)],
             {"DPPX_DIST_BACKEND": "gloo", "DPPX_FORCE_DEVICE": "0"})
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["world"] == 2 and res["identical"], res
    assert res["frames"] == [5, 4]


def test_bench_self_spawns_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself with 2 ranks and
    reports n_gpus = 2 (weak scaling: each rank owns its frames)."""
    r = _run([sys.executable, "bench.py", "--gpus", "2", "--frames", "24", "--steps", "3",
              "--warmup", "3", "--no-cpu-baseline", "--e2e-frames", "8", "--e2e-steps", "1"],
             {"DPPX_DIST_BACKEND": "gloo", "DPPX_FORCE_DEVICE": "0"})
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["frames_per_gpu"] == 24


def _write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode())
        f.write(img.tobytes())


@pytest.mark.parametrize("mode", ["a", "u"])
def test_batch_runner_multi_worker_equals_reference_run_batch(tmp_path, mode):
    """run_batch_gpu (dppix::run_batch) with its chunks spread over 1 and 3
    workers (DPPX_BATCH_DEVICES=0 / 0,0,0: one host thread + ctx each) writes
    the same .pix.pgm / .dppx bytes as the reference's own run_batch
    (oracle/_ref/dppix_batch_ref, cli.cpp:175-213, compiled from its sources)."""
    import filecmp
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "dppix_batch_ref")
    gpu_bin = os.path.join(ROOT, "tests", "cpp", "batch_gpu")
    if not os.path.exists(gpu_bin):
        pytest.skip("tests/cpp/batch_gpu not built")
    d_in, d_mask = tmp_path / "in", tmp_path / "masks"
    d_in.mkdir()
    d_mask.mkdir()
    k = 0
    for (M, N, F) in ((64, 96, 7), (72, 136, 5), (218, 178, 4)):
        frames = oracle.synth_frames(k, F, M, N, 1)[..., 0]
        masks = oracle.synth_masks(k, F, M, N)
        for i in range(F):
            _write_pgm(str(d_in / f"f{k:03d}.pgm"), frames[i])
            _write_pgm(str(d_mask / f"f{k:03d}.pgm"), (masks[i] * 255).astype(np.uint8))
            k += 1
    n = "4" if mode == "a" else "1"
    common = [mode, str(d_mask), "0.5", "16", "16", n, "42", "0", "2"]  # 2 frames per call: 9 chunks
    outs = {}
    for devs in ("0", "0,0,0"):
        d_out = tmp_path / f"out_{devs.replace(',', '')}"
        r = _run([gpu_bin, str(d_in), str(d_out)] + common, {"DPPX_BATCH_DEVICES": devs})
        assert r.returncode == 0, r.stderr[-2000:]
        assert json.loads(r.stdout)["failures"] == 0
        outs[devs] = d_out
    names = sorted(os.listdir(outs["0"]))
    assert len(names) == 2 * k
    for x in names:
        assert filecmp.cmp(outs["0"] / x, outs["0,0,0"] / x, shallow=False), x
    if os.path.exists(ref_bin):
        d_ref = tmp_path / "out_ref"
        r = subprocess.run([ref_bin, str(d_in), str(d_ref)] + common[:-2] + ["4"], capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert sorted(os.listdir(d_ref)) == names
        for x in names:
            assert filecmp.cmp(outs["0,0,0"] / x, d_ref / x, shallow=False), x


def test_batch_runner_bad_inputs_and_stale_outputs_match_reference(tmp_path):
    """Header-first ingest (rasters read straight into the chunk buffers) and
    in-place output rewrites: a batch mixing good files with a truncated
    raster, a P2 file, a header whose comments run past the 4 KB peek, a mask
    of the wrong size and a missing mask -- written over stale, LONGER output
    files -- gives the same failure count and byte-identical outputs as the
    reference's run_batch (cli.cpp:175-213)."""
    import filecmp
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "dppix_batch_ref")
    gpu_bin = os.path.join(ROOT, "tests", "cpp", "batch_gpu")
    if not os.path.exists(gpu_bin) or not os.path.exists(ref_bin):
        pytest.skip("batch binaries not built")
    d_in, d_mask = tmp_path / "in", tmp_path / "masks"
    d_in.mkdir()
    d_mask.mkdir()
    M, N = 40, 56
    frames = oracle.synth_frames(5, 6, M, N, 1)[..., 0]
    masks = oracle.synth_masks(5, 6, M, N)
    for i in range(6):
        _write_pgm(str(d_in / f"g{i}.pgm"), frames[i])
        _write_pgm(str(d_mask / f"g{i}.pgm"), (masks[i] * 255).astype(np.uint8))
    with open(d_in / "g1.pgm", "r+b") as f:  # truncated raster
        f.truncate(f.seek(0, 2) - 7)
    (d_in / "g2.pgm").write_bytes(b"P2\n2 2\n255\n1 2 3 4\n")
    long_comment = b"#" + b"x" * 5000 + b"\n"  # header longer than the peek
    (d_in / "g3.pgm").write_bytes(b"P5\n" + long_comment + f"{N} {M}\n255\n".encode() + frames[3].tobytes())
    _write_pgm(str(d_mask / "g4.pgm"), np.zeros((M, N + 1), np.uint8))  # mask size mismatch
    os.remove(d_mask / "g5.pgm")  # missing mask
    _write_pgm(str(d_in / "g6.pgm"), frames[0])
    _write_pgm(str(d_mask / "g6.pgm"), (masks[0] * 255).astype(np.uint8))
    common = ["a", str(d_mask), "0.5", "16", "8", "4", "42"]
    d_gpu, d_ref = tmp_path / "out_gpu", tmp_path / "out_ref"
    d_gpu.mkdir()
    for stem in ("g0", "g3", "g6"):  # stale outputs, longer than the new ones
        (d_gpu / f"{stem}.pix.pgm").write_bytes(b"\xff" * (M * N * 3))
        (d_gpu / f"{stem}.dppx").write_bytes(b"\xee" * 300000)
    r = _run([gpu_bin, str(d_in), str(d_gpu)] + common + ["0"], {})
    rr = subprocess.run([ref_bin, str(d_in), str(d_ref)] + common + ["4"], capture_output=True, text=True,
                        timeout=600)
    assert r.stdout and rr.stdout, (r.stderr[-2000:], rr.stderr[-2000:])
    g, ref = json.loads(r.stdout), json.loads(rr.stdout)
    assert g["files"] == ref["files"] == 7 and g["failures"] == ref["failures"] == 4, (g, ref)
    names = sorted(os.listdir(d_ref))
    assert names == sorted(os.listdir(d_gpu)) and len(names) == 6
    for x in names:
        assert filecmp.cmp(d_gpu / x, d_ref / x, shallow=False), x
