"""CPU oracle for the dppix pixelization path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both used only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu-baseline / ``--impl reference`` legs, never by the
product package (``paper_2511_04261_b200``):

* ``liboracle.so`` -- ``dppx_oracle.c``, a plain-C restatement of the
  reference algorithm (every function cites /root/reference/proj file:line).
* ``_ref/libdppix_ref.so`` -- the UNMODIFIED reference library compiled from
  /root/reference/proj/src by ``oracle/Makefile`` plus ``ref_shim.cpp``
  (extern "C" wrappers). Present in this container and shipped to the GPU box;
  ``ref`` is None when it was not built.

Parity of the restatement is pinned against the reference's own known-answer
tests (tests/test_oracle_kats.py), live against ``_ref`` (tests/test_oracle_vs_ref.py)
and against committed fixtures made from ``_ref`` (tests/golden/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NOISE_NONE, NOISE_KEYED, NOISE_PHILOX, NOISE_INJECTED = 0, 1, 2, 3
_NOISE_KIND = {"none": 0, "keyed": 1, "philox": 2, "injected": 3}

u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)
u32p = C.POINTER(C.c_uint32)


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    return C.CDLL(path)


_lib_path = os.path.join(HERE, "liboracle.so")
if not os.path.exists(_lib_path):
    build()
lib = _load(_lib_path)


class Geom(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("b", "grid_rows", "grid_cols", "pad_rows", "pad_cols")]


class Params(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("m", C.c_int), ("b", C.c_int), ("n", C.c_int),
                ("subgrid_side", C.c_int), ("delta", C.c_double), ("sigma", C.c_double),
                ("delta_sub", C.c_double), ("sigma_sub", C.c_double)]


lib.or_grid_dims.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(Geom)]
lib.or_make_privacy_params.argtypes = [C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(Params)]
lib.or_keyed_bits.restype = C.c_uint64
lib.or_keyed_bits.argtypes = [C.c_uint64] + [C.c_uint32] * 4
lib.or_uniform_from_bits.restype = C.c_double
lib.or_uniform_from_bits.argtypes = [C.c_uint64]
lib.or_laplace_from_uniform.restype = C.c_double
lib.or_laplace_from_uniform.argtypes = [C.c_double, C.c_double]
lib.or_laplace_at.restype = C.c_double
lib.or_laplace_at.argtypes = [C.c_uint64] + [C.c_uint32] * 4 + [C.c_double]
lib.or_derive_plane_seed.restype = C.c_uint64
lib.or_derive_plane_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
lib.or_philox_bits.restype = C.c_uint64
lib.or_philox_bits.argtypes = [C.c_uint64] + [C.c_uint32] * 6
lib.or_pixelize_uniform_plane.argtypes = [u8p, C.c_int, C.c_int, C.c_long, C.c_int, C.c_int,
                                          C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_uint32,
                                          f64p, u8p, u8p, C.c_long]
lib.or_adaptive_payload_capacity.restype = C.c_size_t
lib.or_adaptive_payload_capacity.argtypes = [C.c_int] * 4
lib.or_pixelize_adaptive_plane.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_long, C.c_long,
                                           C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_double, C.c_int, C.c_uint64, C.c_uint32, f64p,
                                           u8p, u32p, u8p, C.c_long]
lib.or_reassemble_plane.argtypes = [u8p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, u8p, C.c_long]
lib.or_broadcast_plane.argtypes = [u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u8p,
                                   C.c_long]
lib.or_pixelize_reference.argtypes = [u8p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.c_uint64, u8p]
lib.or_synth_frames.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_long, C.c_long, u8p]
lib.or_classify_variance.argtypes = [u8p, C.c_int, C.c_int, C.c_long, C.c_int, C.c_int,
                                     C.c_double, C.POINTER(C.c_float)]
lib.or_pixelize_adaptive_plane_mm.argtypes = [u8p, C.POINTER(C.c_float), C.c_int, C.c_int, C.c_long,
                                              C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                              C.c_double, C.c_int, C.c_uint64, C.c_uint32, f64p,
                                              u8p, u32p, u8p, C.c_long]
lib.or_mse.restype = C.c_double
lib.or_mse.argtypes = [u8p, u8p, C.c_long]
lib.or_ssim.restype = C.c_double
lib.or_ssim.argtypes = [u8p, u8p, C.c_int, C.c_int]
lib.or_synth_masks.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, u8p]


def _p(a, t=u8p):
    return None if a is None else a.ctypes.data_as(t)


class OracleError(ValueError):
    pass


def grid_dims(M, N, b):
    g = Geom()
    if lib.or_grid_dims(M, N, b, C.byref(g)) != 0:
        raise OracleError("grid_dims: invalid")
    return g


def make_privacy_params(eps, m, b, n=1):
    p = Params()
    if lib.or_make_privacy_params(eps, m, b, n, C.byref(p)) != 0:
        raise OracleError("make_privacy_params: invalid")
    return p


def keyed_bits(seed, r, c, sr=0, sc=0):
    return lib.or_keyed_bits(seed, r, c, sr, sc)


def uniform_from_bits(bits):
    return lib.or_uniform_from_bits(bits)


def laplace_from_uniform(u, sigma):
    return lib.or_laplace_from_uniform(u, sigma)


def laplace_at(seed, r, c, sr, sc, sigma):
    return lib.or_laplace_at(seed, r, c, sr, sc, sigma)


def derive_plane_seed(seed, frame, channel):
    return lib.or_derive_plane_seed(seed, frame, channel)


def philox_bits(seed, frame, channel, r, c, sr=0, sc=0):
    return lib.or_philox_bits(seed, frame, channel, r, c, sr, sc)


def _planes(img):
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim == 2:
        return img, 1
    return img, img.shape[2]


def pixelize_uniform(img, b, sigma, noise="none", seeds=None, frame=0, injected=None,
                     want_image=True):
    """Uniform (Algorithm 2) per channel plane. Returns (means[C, G], image).

    seeds: per-channel plane seeds (keyed/philox). injected: [C, G] doubles.
    """
    img, Cn = _planes(img)
    M, N = img.shape[:2]
    g = grid_dims(M, N, b)
    G = g.grid_rows * g.grid_cols
    means = np.zeros((Cn, G), np.uint8)
    out = np.zeros_like(img) if want_image else None
    kind = _NOISE_KIND[noise]
    for ch in range(Cn):
        inj = None
        if kind == NOISE_INJECTED:
            inj = np.ascontiguousarray(np.asarray(injected, np.float64).reshape(Cn, -1)[ch])
        rc = lib.or_pixelize_uniform_plane(
            _p(img), M, N, N * Cn, Cn, ch, b, sigma, kind,
            int(seeds[ch]) if seeds is not None else 0, frame, _p(inj, f64p),
            means[ch].ctypes.data_as(u8p), _p(out), N * Cn)
        if rc != 0:
            raise OracleError(f"pixelize_uniform: rc={rc}")
    return means, out


def pixelize_adaptive(img, mask, b, n, sigma, sigma_sub, noise="none", seeds=None, frame=0,
                      injected=None, want_image=True):
    """Adaptive (Algorithm 3) per channel plane. Returns (payloads: list[bytes], image).

    Each payload is the DPPX v1 adaptive payload of that plane (record.hpp:48-54).
    injected: [C, G*n*n] doubles indexed (g*n + sr)*n + sc.
    """
    img, Cn = _planes(img)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    M, N = img.shape[:2]
    cap = lib.or_adaptive_payload_capacity(M, N, b, n)
    if cap == 0:
        raise OracleError("pixelize_adaptive: invalid geometry")
    out = np.zeros_like(img) if want_image else None
    kind = _NOISE_KIND[noise]
    payloads = []
    for ch in range(Cn):
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint32(0)
        inj = None
        if kind == NOISE_INJECTED:
            inj = np.ascontiguousarray(np.asarray(injected, np.float64).reshape(Cn, -1)[ch])
        rc = lib.or_pixelize_adaptive_plane(
            _p(img), _p(mask), M, N, N * Cn, N, Cn, ch, b, n, sigma, sigma_sub, kind,
            int(seeds[ch]) if seeds is not None else 0, frame, _p(inj, f64p), _p(buf),
            C.byref(ln), _p(out), N * Cn)
        if rc != 0:
            raise OracleError(f"pixelize_adaptive: rc={rc}")
        payloads.append(bytes(buf[: ln.value]))
    return payloads, out


def classify_variance(img, b, tau):
    """EXTENSION: per-cell mask means 1.0 (simple) / 0.0 (variance >= tau)."""
    img, Cn = _planes(img)
    M, N = img.shape[:2]
    g = grid_dims(M, N, b)
    mm = np.zeros(g.grid_rows * g.grid_cols, np.float32)
    if lib.or_classify_variance(_p(img), M, N, N * Cn, Cn, b, tau,
                                mm.ctypes.data_as(C.POINTER(C.c_float))) != 0:
        raise OracleError("classify_variance: invalid")
    return mm


def pixelize_adaptive_variance(img, b, n, sigma, sigma_sub, tau, noise="none", seeds=None,
                               frame=0):
    """EXTENSION: adaptive pixelization with the variance classification."""
    img, Cn = _planes(img)
    M, N = img.shape[:2]
    mm = classify_variance(img, b, tau)
    cap = lib.or_adaptive_payload_capacity(M, N, b, n)
    out = np.zeros_like(img)
    payloads = []
    for ch in range(Cn):
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint32(0)
        rc = lib.or_pixelize_adaptive_plane_mm(
            _p(img), mm.ctypes.data_as(C.POINTER(C.c_float)), M, N, N * Cn, Cn, ch, b, n, sigma,
            sigma_sub, _NOISE_KIND[noise], int(seeds[ch]) if seeds is not None else 0, frame,
            None, _p(buf), C.byref(ln), _p(out), N * Cn)
        if rc != 0:
            raise OracleError(f"pixelize_adaptive_variance: rc={rc}")
        payloads.append(bytes(buf[: ln.value]))
    return payloads, out


def reassemble(payload: bytes, M, N, b, n):
    out = np.zeros((M, N), np.uint8)
    buf = np.frombuffer(payload, np.uint8).copy()
    rc = lib.or_reassemble_plane(_p(buf), len(payload), M, N, b, n, 1, 0, _p(out), N)
    if rc != 0:
        raise OracleError(f"reassemble: rc={rc}")
    return out


def broadcast_means(means, M, N, b):
    out = np.zeros((M, N), np.uint8)
    m = np.ascontiguousarray(means, np.uint8)
    if lib.or_broadcast_plane(_p(m), M, N, b, 1, 0, _p(out), N) != 0:
        raise OracleError("broadcast: invalid")
    return out


def pixelize_reference(img, b, sigma, seed=None):
    img = np.ascontiguousarray(img, np.uint8)
    M, N = img.shape
    out = np.zeros_like(img)
    rc = lib.or_pixelize_reference(_p(img), M, N, b, sigma, NOISE_KEYED if seed is not None
                                   else NOISE_NONE, seed or 0, _p(out))
    if rc != 0:
        raise OracleError("pixelize_reference: invalid")
    return out


def synth_frames(f0, F, M, N, Cn, data_seed=101):
    out = np.zeros((F, M, N, Cn), np.uint8)
    lib.or_synth_frames(data_seed, f0, F, M, N, Cn, N * Cn, M * N * Cn, _p(out))
    return out


def synth_masks(f0, F, M, N):
    out = np.zeros((F, M, N), np.uint8)
    lib.or_synth_masks(f0, F, M, N, N, M * N, _p(out))
    return out


def mse(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    return lib.or_mse(_p(a), _p(b), a.size)


def ssim(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    return lib.or_ssim(_p(a), _p(b), a.shape[0], a.shape[1])


def parse_adaptive_payload(payload: bytes, G, n):
    """Split a DPPX adaptive payload into (mask_means f32[G], S, simple, complex)."""
    mm = np.frombuffer(payload[: 4 * G], "<f4")
    S = int.from_bytes(payload[4 * G: 4 * G + 4], "little")
    simple = np.frombuffer(payload[4 * G + 4: 4 * G + 4 + S], np.uint8)
    cplx = np.frombuffer(payload[4 * G + 4 + S:], np.uint8)
    return mm, S, simple, cplx


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref), when built.
# ---------------------------------------------------------------------------
class _Ref:
    def __init__(self, path):
        self.path = path
        L = self.lib = _load(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_keyed_bits.restype = C.c_uint64
        L.ref_keyed_bits.argtypes = [C.c_uint64] + [C.c_uint32] * 4
        L.ref_uniform_from_bits.restype = C.c_double
        L.ref_uniform_from_bits.argtypes = [C.c_uint64]
        L.ref_laplace_at.restype = C.c_double
        L.ref_laplace_at.argtypes = [C.c_uint64] + [C.c_uint32] * 4 + [C.c_double]
        L.ref_make_privacy_params.argtypes = [C.c_double, C.c_int, C.c_int, C.c_int, f64p,
                                              C.POINTER(C.c_int)]
        L.ref_grid_dims.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_pixelize_parallel.argtypes = [u8p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                            C.c_int, C.c_uint64, C.c_int, u8p, u8p]
        L.ref_pixelize_reference.argtypes = [u8p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                             C.c_int, C.c_uint64, u8p]
        L.ref_pixelize_adaptive.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_double, C.c_int,
                                            C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, u8p,
                                            u8p, u32p]
        L.ref_reconstruct_adaptive.argtypes = [u8p, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                               C.c_int, u8p]
        L.ref_encode_adaptive.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_double, C.c_int,
                                          C.c_int, C.c_int, C.c_int, C.c_uint64, u8p, C.c_uint32,
                                          u32p]
        L.ref_encode_uniform.argtypes = [u8p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                         C.c_int, C.c_uint64, u8p, C.c_uint32, u32p]
        L.ref_mse.restype = C.c_double
        L.ref_mse.argtypes = [u8p, u8p, C.c_int, C.c_int]
        L.ref_ssim.restype = C.c_double
        L.ref_ssim.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_int]
        L.ref_time_planes.restype = C.c_double
        L.ref_time_planes.argtypes = [u8p, u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]

    def _check(self, rc, who):
        if rc == -1:
            raise ValueError(f"{who}: {self.lib.ref_last_error().decode()}")
        if rc == -2:
            raise RuntimeError(f"{who}: RecordError: {self.lib.ref_last_error().decode()}")
        if rc != 0:
            raise RuntimeError(f"{who}: {self.lib.ref_last_error().decode()}")

    def keyed_bits(self, seed, r, c, sr=0, sc=0):
        return self.lib.ref_keyed_bits(seed, r, c, sr, sc)

    def uniform_from_bits(self, bits):
        return self.lib.ref_uniform_from_bits(bits)

    def laplace_at(self, seed, r, c, sr, sc, sigma):
        return self.lib.ref_laplace_at(seed, r, c, sr, sc, sigma)

    def make_privacy_params(self, eps, m, b, n=1):
        out = (C.c_double * 5)()
        ss = C.c_int(0)
        self._check(self.lib.ref_make_privacy_params(eps, m, b, n, out, C.byref(ss)),
                    "make_privacy_params")
        return dict(epsilon=out[0], delta=out[1], sigma=out[2], delta_sub=out[3],
                    sigma_sub=out[4], subgrid_side=ss.value)

    def grid_dims(self, M, N, b):
        out = (C.c_int * 5)()
        self._check(self.lib.ref_grid_dims(M, N, b, out), "grid_dims")
        return tuple(out)

    def pixelize_parallel(self, img, eps, m, b, seed=None, threads=1):
        img = np.ascontiguousarray(img, np.uint8)
        M, N = img.shape
        g = grid_dims(M, N, b) if b <= max(M, N) else None
        out = np.zeros_like(img)
        means = np.zeros(g.grid_rows * g.grid_cols if g else 1, np.uint8)
        self._check(self.lib.ref_pixelize_parallel(_p(img), M, N, eps, m, b, seed is not None,
                                                   seed or 0, threads, _p(out), _p(means)),
                    "pixelize_parallel")
        return out, means

    def pixelize_reference(self, img, eps, m, b, seed=None):
        img = np.ascontiguousarray(img, np.uint8)
        M, N = img.shape
        out = np.zeros_like(img)
        self._check(self.lib.ref_pixelize_reference(_p(img), M, N, eps, m, b, seed is not None,
                                                    seed or 0, _p(out)), "pixelize_reference")
        return out

    def pixelize_adaptive(self, img, mask, eps, m, b, n, seed=None, threads=1):
        img = np.ascontiguousarray(img, np.uint8)
        mask = np.ascontiguousarray(mask, np.uint8)
        M, N = img.shape
        cap = max(1, lib.or_adaptive_payload_capacity(M, N, b, n))
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint32(0)
        out = np.zeros_like(img)
        self._check(self.lib.ref_pixelize_adaptive(_p(img), _p(mask), M, N, eps, m, b, n,
                                                   seed is not None, seed or 0, threads, _p(out),
                                                   _p(buf), C.byref(ln)), "pixelize_adaptive")
        return out, bytes(buf[: ln.value])

    def reconstruct_adaptive(self, payload, M, N, b, n):
        buf = np.frombuffer(payload, np.uint8).copy()
        out = np.zeros((M, N), np.uint8)
        self._check(self.lib.ref_reconstruct_adaptive(_p(buf), len(payload), M, N, b, n,
                                                      _p(out)), "reconstruct")
        return out

    def encode_adaptive(self, img, mask, eps, m, b, n, seed=None):
        img = np.ascontiguousarray(img, np.uint8)
        mask = np.ascontiguousarray(mask, np.uint8)
        M, N = img.shape
        cap = 64 + lib.or_adaptive_payload_capacity(M, N, b, n)
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint32(0)
        self._check(self.lib.ref_encode_adaptive(_p(img), _p(mask), M, N, eps, m, b, n,
                                                 seed is not None, seed or 0, _p(buf), cap,
                                                 C.byref(ln)), "encode_adaptive")
        return bytes(buf[: ln.value])

    def encode_uniform(self, img, eps, m, b, seed=None):
        img = np.ascontiguousarray(img, np.uint8)
        M, N = img.shape
        cap = 64 + M * N
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint32(0)
        self._check(self.lib.ref_encode_uniform(_p(img), M, N, eps, m, b, seed is not None,
                                                seed or 0, _p(buf), cap, C.byref(ln)),
                    "encode_uniform")
        return bytes(buf[: ln.value])

    def mse(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        return self.lib.ref_mse(_p(a), _p(b), a.shape[0], a.shape[1])

    def ssim(self, a, b, threads=1):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        return self.lib.ref_ssim(_p(a), _p(b), a.shape[0], a.shape[1], threads)

    def time_planes(self, planes, masks, uniform, eps, m, b, n, seed, workers):
        planes = np.ascontiguousarray(planes, np.uint8)
        P, M, N = planes.shape
        mk = None if masks is None else np.ascontiguousarray(masks, np.uint8)
        t = self.lib.ref_time_planes(_p(planes), _p(mk), P, M, N, int(uniform), eps, m, b, n,
                                     seed, workers)
        if t < 0:
            raise RuntimeError("ref_time_planes failed")
        return t


_ref_path = os.path.join(HERE, "_ref", "libdppix_ref.so")
ref = _Ref(_ref_path) if os.path.exists(_ref_path) else None


lib.or_log1p_glibc.restype = C.c_double
lib.or_log1p_glibc.argtypes = [C.c_double]
lib.or_log1p_glibc_mismatches.restype = C.c_long
lib.or_log1p_glibc_mismatches.argtypes = [C.c_void_p, C.c_long, C.POINTER(C.c_double)]


def log1p_glibc(x: float) -> float:
    """Restatement of glibc 2.39's FMA-variant log1p (see or_log1p_glibc)."""
    return lib.or_log1p_glibc(x)


def log1p_glibc_mismatches(xs) -> tuple:
    """(count, first mismatching x) of or_log1p_glibc vs the host libm's log1p."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    first = C.c_double(0.0)
    n = lib.or_log1p_glibc_mismatches(xs.ctypes.data, xs.size, C.byref(first))
    return n, first.value
