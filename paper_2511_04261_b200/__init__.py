"""B200-native dppix pixelization path (arXiv 2511.04261), Python host side.

This package binds ``lib/libdppx_gpu.so`` (the C ABI declared in
``include/dppx_gpu.h``; sm_100a kernels in ``csrc/``) with ctypes and mirrors
the reference's ``dppix::`` interface (/root/reference/proj/include/dppix):

    reference (C++)                         here
    make_privacy_params  noise.hpp:55       make_privacy_params
    grid_dims            image.hpp:86       grid_dims
    pixelize_parallel    pixelize.hpp:55    pixelize_parallel
    pixelize_adaptive    adaptive.hpp:70    pixelize_adaptive
    broadcast_means      pixelize.hpp:62    broadcast_means
    reassemble           adaptive.hpp:78    reassemble
    classify_regions     adaptive.hpp:45    classify_regions

Errors keep the reference's taxonomy: ``std::invalid_argument`` -> ValueError,
``RecordError(corrupt_record)`` -> RecordError. Batched multi-frame / RGB entry
points live on :class:`Context`. There is no CPU fallback: the compute entry
points raise :class:`DeviceUnavailable` when no sm_100 GPU is usable.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import sys
import threading
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DPPX_LIB") or os.path.join(_HERE, "lib", "libdppx_gpu.so")  # A/B override
DROPIN_PATH = os.path.join(_HERE, "lib", "libdppix_gpu.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_2511_04261_b200` "
        "(or __graft_entry__.build()); there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)

OK, ERR_INVALID, ERR_CORRUPT, ERR_CUDA, ERR_OOM, ERR_NO_DEVICE = range(6)
ERR_NOT_A_RECORD, ERR_UNSUPPORTED_VERSION, ERR_CORRUPTION = 6, 7, 8
NOISE_NONE, NOISE_KEYED, NOISE_PHILOX, NOISE_INJECTED = range(4)
K_CLASSIFY, K_STATS, K_GENERIC, K_EXPAND, K_AUX, K_ROWS, K_SWEEP, K_ZEROCOPY, K_COUNT = range(9)
SMALL_AUTO, SMALL_GRAPH, SMALL_ZEROCOPY, SMALL_STAGED = 0, 1, 2, 3
SMALL_AUTO_ZEROCOPY = ("u", "a")  # modes SMALL_AUTO sends through the zero-copy kernels

KERNEL_FAMILIES = ("classify", "stats_tma", "stats_generic", "expand", "aux", "stats_rows", "sweep",
                   "stats_zerocopy")


class Geometry(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("b", "grid_rows", "grid_cols", "pad_rows", "pad_cols")]

    def grid_count(self):
        return self.grid_rows * self.grid_cols

    def __eq__(self, o):
        return all(getattr(self, n) == getattr(o, n) for n, _ in self._fields_)

    def __repr__(self):
        return "GridGeometry(" + ", ".join(f"{n}={getattr(self, n)}" for n, _ in self._fields_) + ")"


class PrivacyParams(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("m", C.c_int32), ("b", C.c_int32), ("n", C.c_int32),
                ("subgrid_side", C.c_int32), ("delta", C.c_double), ("sigma", C.c_double),
                ("delta_sub", C.c_double), ("sigma_sub", C.c_double)]


class FramesDesc(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("channels", C.c_int32),
                ("frames", C.c_int32), ("pitch", C.c_int64), ("frame_stride", C.c_int64),
                ("mask_pitch", C.c_int64), ("mask_frame_stride", C.c_int64),
                ("out_pitch", C.c_int64), ("out_frame_stride", C.c_int64)]


class Noise(C.Structure):
    _fields_ = [("kind", C.c_int32), ("frame_base", C.c_uint32),
                ("plane_seeds", C.POINTER(C.c_uint64)), ("injected", C.POINTER(C.c_double))]


class RecordInfo(C.Structure):
    _fields_ = [("height", C.c_int32), ("width", C.c_int32), ("b", C.c_int32), ("n", C.c_int32),
                ("mode", C.c_int32), ("payload_offset", C.c_uint32), ("payload_len", C.c_uint32)]


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_uint64 * K_COUNT), ("device_ms", C.c_double * K_COUNT),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p
_ctxp = C.c_void_p
_descp = C.POINTER(FramesDesc)
_pp = C.POINTER(PrivacyParams)
_np = C.POINTER(Noise)

# Every symbol of include/dppx_gpu.h with its ctypes signature.
ABI = {
    "dppx_version": (C.c_char_p, []),
    "dppx_grid_dims": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(Geometry)]),
    "dppx_make_privacy_params": (C.c_int, [C.c_double, C.c_int32, C.c_int32, C.c_int32, _pp]),
    "dppx_sensitivity": (C.c_double, [C.c_int32, C.c_int32]),
    "dppx_keyed_bits": (C.c_uint64, [C.c_uint64] + [C.c_uint32] * 4),
    "dppx_uniform_from_bits": (C.c_double, [C.c_uint64]),
    "dppx_laplace_at": (C.c_double, [C.c_uint64] + [C.c_uint32] * 4 + [C.c_double]),
    "dppx_derive_plane_seed": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint32]),
    "dppx_adaptive_payload_capacity": (C.c_size_t, [C.c_int32] * 4),
    "dppx_adaptive_payload_length": (C.c_size_t, [C.c_int32] * 4 + [C.c_uint32]),
    "dppx_ctx_create": (C.c_int, [C.c_int32, C.POINTER(_ctxp)]),
    "dppx_ctx_destroy": (None, [_ctxp]),
    "dppx_ctx_last_error": (C.c_char_p, [_ctxp]),
    "dppx_ctx_stream": (_vp, [_ctxp]),
    "dppx_ctx_set_stream": (C.c_int, [_ctxp, _vp]),
    "dppx_ctx_synchronize": (C.c_int, [_ctxp]),
    "dppx_ctx_set_timing": (C.c_int, [_ctxp, C.c_int32]),
    "dppx_ctx_get_stats": (C.c_int, [_ctxp, C.POINTER(KernelStats)]),
    "dppx_ctx_reset_stats": (C.c_int, [_ctxp]),
    "dppx_ctx_set_chunk_frames": (C.c_int, [_ctxp, C.c_int32]),
    "dppx_ctx_set_exact_noise": (C.c_int, [_ctxp, C.c_int32]),
    "dppx_ctx_set_out_pad_scratch": (C.c_int, [_ctxp, C.c_int32]),
    "dppx_ctx_set_small_frame_path": (C.c_int, [_ctxp, C.c_int32]),
    "dppx_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "dppx_host_free": (None, [_vp]),
    "dppx_pixelize_uniform_dev": (C.c_int, [_ctxp, _descp, _vp, _pp, _np, _vp, _vp]),
    "dppx_pixelize_adaptive_dev": (C.c_int, [_ctxp, _descp, _vp, _vp, _pp, _np, _vp, C.c_int64,
                                             _vp, _vp]),
    "dppx_broadcast_means_dev": (C.c_int, [_ctxp, _descp, _vp, C.c_int32, _vp]),
    "dppx_reassemble_dev": (C.c_int, [_ctxp, _descp, _vp, C.c_int64, _vp, C.c_int32, C.c_int32,
                                      _vp]),
    "dppx_synth_frames_dev": (C.c_int, [_ctxp, _descp, C.c_uint32, C.c_uint32, _vp, _vp]),
    "dppx_pixelize_uniform_sweep_dev": (C.c_int, [_ctxp, _descp, _vp, C.c_int32, C.POINTER(C.c_int32),
                                                  C.c_int32, C.POINTER(C.c_double), C.c_int32, _np,
                                                  C.POINTER(_vp), C.POINTER(_vp)]),
    "dppx_pixelize_uniform": (C.c_int, [_ctxp, _descp, _vp, _pp, _np, _vp, _vp]),
    "dppx_pixelize_adaptive": (C.c_int, [_ctxp, _descp, _vp, _vp, _pp, _np, _vp, C.c_int64, _vp,
                                         _vp]),
    "dppx_broadcast_means": (C.c_int, [_ctxp, _descp, _vp, C.c_int32, _vp]),
    "dppx_pixelize_adaptive_variance": (C.c_int, [_ctxp, _descp, _vp, C.c_double, _pp, _np, _vp,
                                                  C.c_int64, _vp, _vp]),
    "dppx_pixelize_adaptive_variance_dev": (C.c_int, [_ctxp, _descp, _vp, C.c_double, _pp, _np,
                                                      _vp, C.c_int64, _vp, _vp]),
    "dppx_pixelize_reference": (C.c_int, [_ctxp, _descp, _vp, _pp, _np, _vp, _vp]),
    "dppx_reassemble": (C.c_int, [_ctxp, _descp, _vp, C.c_int64, _vp, C.c_int32, C.c_int32, _vp]),
    "dppx_classify_regions": (C.c_int, [_ctxp, _descp, _vp, C.c_int32, _vp]),
    "dppx_mse": (C.c_int, [_ctxp, _descp, _vp, _vp, _vp]),
    "dppx_ssim": (C.c_int, [_ctxp, _descp, _vp, _vp, _vp]),
    "dppx_metrics": (C.c_int, [_ctxp, _descp, _vp, _vp, _vp, _vp]),
    "dppx_mse_dev": (C.c_int, [_ctxp, _descp, _vp, _vp, _vp]),
    "dppx_ssim_dev": (C.c_int, [_ctxp, _descp, _vp, _vp, _vp]),
    "dppx_crc32": (C.c_uint32, [C.c_uint32, _vp, C.c_size_t]),
    "dppx_record_size": (C.c_size_t, [C.c_size_t]),
    "dppx_encode_record": (C.c_int, [C.c_int32] * 5 + [_vp, C.c_size_t, _vp, C.c_size_t,
                                                       C.POINTER(C.c_size_t)]),
    "dppx_decode_record": (C.c_int, [_vp, C.c_size_t, C.POINTER(RecordInfo)]),
    "dppx_reconstruct_record": (C.c_int, [_ctxp, _vp, C.c_size_t, _vp, C.c_size_t]),
    "dppx_debug_device_laplace": (C.c_int, [_ctxp, C.c_uint64, _vp, C.c_int32, C.c_double, _vp]),
    "dppx_debug_lg2_max_error": (C.c_int, [_ctxp, C.POINTER(C.c_double)]),
    "dppx_pixelize_uniform_sweep": (C.c_int, [_ctxp, _descp, _vp, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                              C.POINTER(C.c_double), C.c_int32, _np, C.POINTER(_vp),
                                              C.POINTER(_vp), _vp, _vp]),
    "dppx_pixelize_checked": (C.c_int, [_ctxp, C.c_int32, _descp, _vp, _vp, _pp, _np, _vp, C.c_int64, _vp,
                                        _vp, _vp, _vp, _vp]),
    "dppx_pixelize_checked_reserve": (C.c_int, [_ctxp, C.c_int32, _descp, _pp]),
    "dppx_group_create": (C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.POINTER(_vp)]),
    "dppx_group_destroy": (None, [_vp]),
    "dppx_group_size": (C.c_int32, [_vp]),
    "dppx_group_device": (C.c_int32, [_vp, C.c_int32]),
    "dppx_group_ctx": (_ctxp, [_vp, C.c_int32]),
    "dppx_group_last_error": (C.c_char_p, [_vp]),
    "dppx_group_run": (C.c_int, [_vp, C.c_int32, _vp, _vp]),
    "dppx_group_pixelize_uniform": (C.c_int, [_vp, _descp, _vp, _pp, _np, _vp, _vp]),
    "dppx_group_pixelize_adaptive": (C.c_int, [_vp, _descp, _vp, _vp, _pp, _np, _vp, C.c_int64,
                                               _vp, _vp]),
    "dppx_group_broadcast_means": (C.c_int, [_vp, _descp, _vp, C.c_int32, _vp]),
    "dppx_group_reassemble": (C.c_int, [_vp, _descp, _vp, C.c_int64, _vp, C.c_int32, C.c_int32,
                                        _vp]),
    "dppx_group_get_stats": (C.c_int, [_vp, C.POINTER(KernelStats)]),
}
for _name, (_res, _args) in ABI.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class RecordError(RuntimeError):
    """dppix::RecordError (errors.hpp:37-55); ``kind`` is 'corrupt_record' here."""

    def __init__(self, msg, kind="corrupt_record"):
        super().__init__(msg)
        self.kind = kind


class DeviceUnavailable(RuntimeError):
    """No usable sm_100 device: the GPU path cannot run and nothing falls back."""


class CudaError(RuntimeError):
    pass


def _raise(rc, msg):
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_CORRUPT:
        raise RecordError(msg)
    if rc == ERR_NOT_A_RECORD:
        raise RecordError(msg, "not_a_record")
    if rc == ERR_UNSUPPORTED_VERSION:
        raise RecordError(msg, "unsupported_version")
    if rc == ERR_CORRUPTION:
        raise RecordError(msg, "corruption")
    if rc == ERR_OOM:
        raise MemoryError(msg)
    if rc == ERR_NO_DEVICE:
        raise DeviceUnavailable(msg)
    raise CudaError(msg)


# ---------------------------------------------------------------- parameters
def grid_dims(height: int, width: int, b: int) -> Geometry:
    """grid_dims (image.cpp:48-72)."""
    if height < 1 or width < 1:
        raise ValueError("grid_dims: dimensions must be >= 1")
    if b < 1:
        raise ValueError("grid_dims: grid side b must be >= 1")
    g = Geometry()
    if _lib.dppx_grid_dims(height, width, b, C.byref(g)) != OK:
        raise ValueError("grid_dims: grid side b exceeds both image dimensions")
    return g


def make_privacy_params(epsilon: float, m: int, b: int, n: int = 1) -> PrivacyParams:
    """make_privacy_params (noise.cpp:39-68): sigma = 255 m / (b^2 eps), sigma_sub = sigma n^2."""
    if not epsilon > 0.0:
        raise ValueError("make_privacy_params: epsilon must be > 0")
    if m < 1:
        raise ValueError("make_privacy_params: m must be >= 1")
    if b < 1:
        raise ValueError("make_privacy_params: b must be >= 1")
    if n < 1:
        raise ValueError("make_privacy_params: n must be >= 1")
    if b % n:
        raise ValueError("make_privacy_params: n must divide b")
    p = PrivacyParams()
    _lib.dppx_make_privacy_params(epsilon, m, b, n, C.byref(p))
    return p


def sensitivity(b: int, m: int) -> float:
    if b < 1 or m < 1:
        raise ValueError("sensitivity: b and m must be >= 1")
    return _lib.dppx_sensitivity(b, m)


def keyed_bits(seed: int, r: int, c: int, sr: int = 0, sc: int = 0) -> int:
    return _lib.dppx_keyed_bits(seed, r, c, sr, sc)


def laplace_at(seed: int, r: int, c: int, sr: int, sc: int, sigma: float) -> float:
    if not sigma > 0.0:
        raise ValueError("laplace_at: sigma must be > 0")
    return _lib.dppx_laplace_at(seed, r, c, sr, sc, sigma)


def derive_plane_seed(seed: int, frame: int, channel: int) -> int:
    return _lib.dppx_derive_plane_seed(seed, frame, channel)


def adaptive_payload_capacity(height, width, b, n) -> int:
    return _lib.dppx_adaptive_payload_capacity(height, width, b, n)


def plane_seeds(seed: int, frames: int, channels: int, frame0: int = 0, mode: str = "derived"):
    """Per-plane seeds: 'derived' = derive_plane_seed(seed, f, k); 'shared' = the
    reference's run_batch behaviour (same seed for every file, cli.cpp:200-201)."""
    if mode == "shared":
        return np.full(frames * channels, seed, np.uint64)
    return np.array([derive_plane_seed(seed, frame0 + f, k)
                     for f in range(frames) for k in range(channels)], np.uint64)


# ---------------------------------------------------------------- context
def _ptr(a):
    """Address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def _desc(M, N, Cn, F, pitch=None, fstride=None, mpitch=None, mfstride=None, opitch=None,
          ofstride=None):
    d = FramesDesc()
    d.height, d.width, d.channels, d.frames = M, N, Cn, F
    d.pitch = pitch if pitch is not None else N * Cn
    d.frame_stride = fstride if fstride is not None else d.pitch * M
    d.mask_pitch = mpitch if mpitch is not None else N
    d.mask_frame_stride = mfstride if mfstride is not None else d.mask_pitch * M
    d.out_pitch = opitch if opitch is not None else N * Cn
    d.out_frame_stride = ofstride if ofstride is not None else d.out_pitch * M
    return d


def _frames_shape(img):
    """(F, M, N, C) of a [M,N], [M,N,C], [F,M,N] (with channels=1) or [F,M,N,C] array."""
    s = tuple(img.shape)
    if len(s) == 2:
        return 1, s[0], s[1], 1
    if len(s) == 3:
        return 1, s[0], s[1], s[2]
    return s[0], s[1], s[2], s[3]


def pinned_empty(shape, dtype=np.uint8) -> np.ndarray:
    """Page-locked host array (torch's pinned allocator; the array keeps the
    tensor alive). Host calls on pinned buffers DMA directly; pageable ones are
    staged through the context's pinned buffers by host threads."""
    import torch
    t = torch.empty(tuple(shape), dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
    a = t.numpy()
    holder = _PinnedArray(a)
    holder._tensor = t
    return holder


class _PinnedArray(np.ndarray):
    def __new__(cls, a):
        return np.asarray(a).view(cls)


def _out_image(frames, out, want_image):
    if out is None:
        return np.zeros_like(frames) if want_image else None
    if out.shape != frames.shape or out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous uint8 array of the frames' shape")
    return out


class Context:
    """One dppx_ctx: a device, its streams, scratch and pinned staging.

    Methods with ``_dev`` take torch CUDA tensors (device-resident, async on the
    context stream); the others take host numpy arrays and run the pinned
    H2D -> kernels -> D2H pipeline.
    """

    def __init__(self, device: int = 0):
        h = _ctxp()
        rc = _lib.dppx_ctx_create(device, C.byref(h))
        if rc != OK:
            _raise(rc, f"dppx_ctx_create(device={device}) failed with status {rc}")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            _lib.dppx_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, who):
        if rc != OK:
            _raise(rc, f"{who}: {self._last_error()}")

    def _last_error(self) -> str:
        return _lib.dppx_ctx_last_error(self._h).decode()

    @staticmethod
    def _api(name):  # host entry point of one context (Group: of a device group)
        return getattr(_lib, "dppx_" + name)

    # ---- plumbing
    @property
    def stream(self) -> int:
        return _lib.dppx_ctx_stream(self._h) or 0

    def set_stream(self, stream_handle: Optional[int]):
        self._check(_lib.dppx_ctx_set_stream(self._h, stream_handle), "set_stream")

    def synchronize(self):
        self._check(_lib.dppx_ctx_synchronize(self._h), "synchronize")

    def set_timing(self, on: bool):
        _lib.dppx_ctx_set_timing(self._h, 1 if on else 0)

    def set_chunk_frames(self, frames: int):
        self._check(_lib.dppx_ctx_set_chunk_frames(self._h, frames), "set_chunk_frames")

    def set_exact_noise(self, on: bool):
        """Force the f64 reference arithmetic for every statistic (testing)."""
        self._check(_lib.dppx_ctx_set_exact_noise(self._h, 1 if on else 0), "set_exact_noise")

    def set_small_frame_path(self, path: int):
        """SMALL_AUTO / SMALL_GRAPH / SMALL_ZEROCOPY / SMALL_STAGED (dppx_ctx_set_small_frame_path)."""
        self._check(_lib.dppx_ctx_set_small_frame_path(self._h, path), "set_small_frame_path")

    def set_out_pad_scratch(self, on: bool):
        """Declare output pitch padding scratch: rows may end on whole 32-byte sectors."""
        self._check(_lib.dppx_ctx_set_out_pad_scratch(self._h, 1 if on else 0), "set_out_pad_scratch")

    def lg2_max_error(self) -> float:
        v = C.c_double()
        self._check(_lib.dppx_debug_lg2_max_error(self._h, C.byref(v)), "lg2_max_error")
        return v.value

    def stats(self) -> dict:
        s = KernelStats()
        _lib.dppx_ctx_get_stats(self._h, C.byref(s))
        return {"launches": {k: int(s.launches[i]) for i, k in enumerate(KERNEL_FAMILIES)},
                "device_ms": {k: float(s.device_ms[i]) for i, k in enumerate(KERNEL_FAMILIES)},
                "h2d_bytes": int(s.h2d_bytes), "d2h_bytes": int(s.d2h_bytes)}

    def reset_stats(self):
        _lib.dppx_ctx_reset_stats(self._h)

    @staticmethod
    def _noise(kind, seeds, frame_base=0, injected=None):
        nz = Noise()
        nz.kind = kind
        nz.frame_base = frame_base
        keep = []
        if seeds is not None:
            arr = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
            keep.append(arr)
            nz.plane_seeds = arr.ctypes.data_as(C.POINTER(C.c_uint64))
        if injected is not None:
            if isinstance(injected, np.ndarray):
                inj = np.ascontiguousarray(injected, dtype=np.float64)
                keep.append(inj)
                nz.injected = inj.ctypes.data_as(_f64p)
            else:  # torch tensor on device
                keep.append(injected)
                nz.injected = C.cast(C.c_void_p(injected.data_ptr()), _f64p)
        return nz, keep

    # ---- host entry points (numpy in / numpy out)
    def pixelize_uniform(self, frames, params: PrivacyParams, noise=NOISE_NONE, seeds=None,
                         frame_base=0, injected=None, want_image=True, out=None, stats_out=None):
        """frames: uint8 [F,M,N,C] (or [M,N], [M,N,C]). Returns (means[F*C, G], image).
        `out` (optional, frames' shape) receives the image, e.g. a pinned_empty buffer;
        `stats_out` (optional, uint8 [F*C, G], e.g. pinned) receives the means."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        g = grid_dims(M, N, params.b)
        means = np.zeros((F * Cn, g.grid_count()), np.uint8) if stats_out is None else stats_out
        assert means.shape == (F * Cn, g.grid_count()) and means.dtype == np.uint8 and means.flags.c_contiguous
        out = _out_image(frames, out, want_image)
        nz, keep = self._noise(noise, seeds, frame_base, injected)
        d = _desc(M, N, Cn, F)
        self._check(self._api("pixelize_uniform")(self._h, C.byref(d), _ptr(frames), C.byref(params),
                                               C.byref(nz), _ptr(means), _ptr(out)),
                    "pixelize_uniform")
        del keep
        return means, out

    def pixelize_adaptive(self, frames, masks, params: PrivacyParams, noise=NOISE_NONE,
                          seeds=None, frame_base=0, injected=None, want_image=True, out=None,
                          stats_out=None):
        """frames uint8 [F,M,N,C], masks uint8 [F,M,N]. Returns (payloads: list of bytes per
        plane (f*C + c), image). `out` as in pixelize_uniform; `stats_out` (optional,
        uint8 [F*C, stride], stride >= the payload capacity rounded up to 4) holds the slots."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        masks = np.ascontiguousarray(masks, dtype=np.uint8).reshape(F, M, N)
        cap = adaptive_payload_capacity(M, N, params.b, params.n)
        stride = (cap + 3) & ~3 if stats_out is None else stats_out.shape[1]
        buf = np.zeros((F * Cn, stride), np.uint8) if stats_out is None else stats_out
        assert buf.shape[0] == F * Cn and buf.dtype == np.uint8 and buf.flags.c_contiguous
        lens = np.zeros(F * Cn, np.uint32)
        out = _out_image(frames, out, want_image)
        nz, keep = self._noise(noise, seeds, frame_base, injected)
        d = _desc(M, N, Cn, F)
        self._check(self._api("pixelize_adaptive")(self._h, C.byref(d), _ptr(frames), _ptr(masks),
                                                C.byref(params), C.byref(nz), _ptr(buf), stride,
                                                _ptr(lens), _ptr(out)), "pixelize_adaptive")
        del keep
        return [bytes(buf[i, : lens[i]]) for i in range(F * Cn)], out

    def pixelize_reference(self, frames, params: PrivacyParams, noise=NOISE_NONE, seeds=None,
                           frame_base=0):
        """Algorithm 1 (pixelize.cpp:50-84). Returns (means[F*C, G], image)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        g = grid_dims(M, N, params.b)
        means = np.zeros((F * Cn, g.grid_count()), np.uint8)
        out = np.zeros_like(frames)
        nz, keep = self._noise(noise, seeds, frame_base, None)
        d = _desc(M, N, Cn, F)
        self._check(_lib.dppx_pixelize_reference(self._h, C.byref(d), _ptr(frames), C.byref(params),
                                                 C.byref(nz), _ptr(means), _ptr(out)),
                    "pixelize_reference")
        del keep
        return means, out

    def pixelize_adaptive_variance(self, frames, tau: float, params: PrivacyParams,
                                   noise=NOISE_NONE, seeds=None, frame_base=0):
        """EXTENSION: adaptive pixelization where a cell is complex iff the
        variance of its C*b*b samples is >= tau (the classification is derived
        from the private frames and is not covered by epsilon)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        cap = adaptive_payload_capacity(M, N, params.b, params.n)
        stride = (cap + 3) & ~3
        buf = np.zeros((F * Cn, stride), np.uint8)
        lens = np.zeros(F * Cn, np.uint32)
        out = np.zeros_like(frames)
        nz, keep = self._noise(noise, seeds, frame_base, None)
        d = _desc(M, N, Cn, F)
        self._check(_lib.dppx_pixelize_adaptive_variance(self._h, C.byref(d), _ptr(frames), tau,
                                                         C.byref(params), C.byref(nz), _ptr(buf),
                                                         stride, _ptr(lens), _ptr(out)),
                    "pixelize_adaptive_variance")
        del keep
        return [bytes(buf[i, : lens[i]]) for i in range(F * Cn)], out

    def pixelize_uniform_sweep(self, frames, b_list, eps_list, m, noise=NOISE_NONE, seeds=None,
                               want_images=True, metrics=False):
        """dppx_pixelize_uniform_sweep (host buffers): one upload, every (b, eps) run.
        Returns (means list, images list or None, mse [runs, F*C] or None, ssim or None)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        nb, ne = len(b_list), len(eps_list)
        means = [np.zeros((F * Cn, grid_dims(M, N, b).grid_count()), np.uint8) for b in b_list for _ in eps_list]
        imgs = [np.zeros_like(frames) for _ in range(nb * ne)] if want_images else None
        mse = np.zeros((nb * ne, F * Cn)) if metrics else None
        ssim = np.zeros((nb * ne, F * Cn)) if metrics and M >= 7 and N >= 7 else None
        nz, keep = self._noise(noise, seeds)
        d = _desc(M, N, Cn, F)
        mp = (_vp * (nb * ne))(*[x.ctypes.data for x in means])
        op = (_vp * (nb * ne))(*[x.ctypes.data for x in imgs]) if want_images else None
        self._check(_lib.dppx_pixelize_uniform_sweep(
            self._h, C.byref(d), _ptr(frames), nb, (C.c_int32 * nb)(*b_list), ne, (C.c_double * ne)(*eps_list),
            m, C.byref(nz), mp, op, _ptr(mse), _ptr(ssim)), "pixelize_uniform_sweep")
        del keep
        return means, imgs, mse, ssim

    def pixelize_checked_reserve(self, shape, params: PrivacyParams, mode="adaptive"):
        """dppx_pixelize_checked_reserve: size the buffers of a later
        pixelize_checked call on frames of `shape` (F, M, N[, C])."""
        F, M, N = shape[:3]
        Cn = shape[3] if len(shape) > 3 else 1
        m = {"uniform": 0, "adaptive": 1, "reference": 2}[mode]
        d = _desc(M, N, Cn, F)
        self._check(_lib.dppx_pixelize_checked_reserve(self._h, m, C.byref(d), C.byref(params)),
                    "pixelize_checked_reserve")

    def pixelize_checked(self, frames, masks, params: PrivacyParams, mode="adaptive",
                         noise=NOISE_NONE, seeds=None):
        """dppx_pixelize_checked: pixelize + on-device reconstruct check + mse / ssim
        from one upload. Returns (stats, lens, image, recon_ok, mse, ssim)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        F, M, N, Cn = _frames_shape(frames)
        m = {"uniform": 0, "adaptive": 1, "reference": 2}[mode]
        g = grid_dims(M, N, params.b)
        stride = ((adaptive_payload_capacity(M, N, params.b, params.n) + 3) & ~3) if m == 1 else g.grid_count()
        stats = np.zeros((F * Cn, stride), np.uint8)
        lens = np.zeros(F * Cn, np.uint32)
        out = np.zeros_like(frames)
        ok = np.zeros(F, np.uint8)
        mse = np.zeros(F * Cn, np.float64)
        ssim = np.zeros(F * Cn, np.float64)
        mk = None if m != 1 else np.ascontiguousarray(masks, dtype=np.uint8).reshape(F, M, N)
        nz, keep = self._noise(noise, seeds)
        d = _desc(M, N, Cn, F)
        self._check(_lib.dppx_pixelize_checked(self._h, m, C.byref(d), _ptr(frames), _ptr(mk), C.byref(params),
                                               C.byref(nz), _ptr(stats), stride, _ptr(lens), _ptr(out),
                                               _ptr(ok), _ptr(mse), _ptr(ssim) if M >= 7 and N >= 7 else None),
                    "pixelize_checked")
        del keep
        return stats, lens, out, ok, mse, ssim

    def reconstruct_record(self, record: bytes) -> np.ndarray:
        """dppx_reconstruct_record: decode a .dppx record and expand it on the GPU."""
        info = RecordInfo()
        buf = np.frombuffer(record, np.uint8).copy()
        rc = _lib.dppx_decode_record(_ptr(buf), buf.size, C.byref(info))
        if rc != OK:
            raise RecordError(f"decode: status {rc}")
        out = np.zeros((info.height, info.width), np.uint8)
        self._check(_lib.dppx_reconstruct_record(self._h, _ptr(buf), buf.size, _ptr(out), out.size),
                    "reconstruct_record")
        return out

    def broadcast_means(self, means, M, N, b, channels=1, frames=1):
        means = np.ascontiguousarray(means, dtype=np.uint8)
        out = np.zeros((frames, M, N, channels), np.uint8)
        d = _desc(M, N, channels, frames)
        self._check(self._api("broadcast_means")(self._h, C.byref(d), _ptr(means), b, _ptr(out)),
                    "broadcast_means")
        return out

    def reassemble(self, payloads: Sequence[bytes], M, N, b, n, channels=1, frames=1,
                   check_lengths=True):
        P = frames * channels
        stride = max(16, (max(len(p) for p in payloads) + 15) & ~15)
        buf = np.zeros((P, stride), np.uint8)
        for i, p in enumerate(payloads):
            buf[i, : len(p)] = np.frombuffer(p, np.uint8)
        lens = np.array([len(p) for p in payloads], np.uint32)
        out = np.zeros((frames, M, N, channels), np.uint8)
        d = _desc(M, N, channels, frames)
        self._check(self._api("reassemble")(self._h, C.byref(d), _ptr(buf), stride,
                                         _ptr(lens) if check_lengths else None, b, n, _ptr(out)),
                    "reassemble")
        return out

    def classify_regions(self, masks, b):
        masks = np.ascontiguousarray(masks, dtype=np.uint8)
        if masks.ndim == 2:
            masks = masks[None]
        F, M, N = masks.shape
        g = grid_dims(M, N, b)
        mm = np.zeros((F, g.grid_count()), np.float32)
        d = _desc(M, N, 1, F)
        self._check(_lib.dppx_classify_regions(self._h, C.byref(d), _ptr(masks), b, _ptr(mm)),
                    "classify_regions")
        return mm

    def metrics(self, a, b, which="ssim"):
        """mse / ssim per channel plane of two frame batches ([F,M,N,C] or [M,N]);
        which="both" returns (mse, ssim) from one upload (dppx_metrics)."""
        a = np.ascontiguousarray(a, dtype=np.uint8)
        b = np.ascontiguousarray(b, dtype=np.uint8)
        if a.shape != b.shape:
            raise ValueError(f"{which}: images must share dimensions")
        F, M, N, Cn = _frames_shape(a)
        out = np.zeros(F * Cn, np.float64)
        d = _desc(M, N, Cn, F)
        if which == "both":
            out2 = np.zeros(F * Cn, np.float64)
            self._check(_lib.dppx_metrics(self._h, C.byref(d), _ptr(a), _ptr(b), _ptr(out),
                                          _ptr(out2)), which)
            return out, out2
        fn = _lib.dppx_ssim if which == "ssim" else _lib.dppx_mse
        self._check(fn(self._h, C.byref(d), _ptr(a), _ptr(b), _ptr(out)), which)
        return out

    def device_laplace(self, seed, keys, sigma):
        keys = np.ascontiguousarray(np.asarray(keys, np.uint32).reshape(-1, 4))
        out = np.zeros(len(keys), np.float64)
        self._check(_lib.dppx_debug_device_laplace(self._h, seed, _ptr(keys), len(keys), sigma,
                                                   _ptr(out)), "device_laplace")
        return out

    # ---- device entry points (torch CUDA tensors, async on self.stream)
    def pixelize_adaptive_dev(self, desc: FramesDesc, img, mask, params, noise_struct, payload,
                              payload_stride, payload_len=None, out=None):
        self._check(_lib.dppx_pixelize_adaptive_dev(
            self._h, C.byref(desc), _ptr(img), _ptr(mask), C.byref(params), C.byref(noise_struct),
            _ptr(payload), payload_stride, _ptr(payload_len), _ptr(out)), "pixelize_adaptive_dev")

    def pixelize_uniform_dev(self, desc: FramesDesc, img, params, noise_struct, means, out=None):
        self._check(_lib.dppx_pixelize_uniform_dev(
            self._h, C.byref(desc), _ptr(img), C.byref(params), C.byref(noise_struct),
            _ptr(means), _ptr(out)), "pixelize_uniform_dev")

    def pixelize_adaptive_variance_dev(self, desc: FramesDesc, img, tau, params, noise_struct,
                                       payload, payload_stride, payload_len=None, out=None):
        self._check(_lib.dppx_pixelize_adaptive_variance_dev(
            self._h, C.byref(desc), _ptr(img), tau, C.byref(params), C.byref(noise_struct),
            _ptr(payload), payload_stride, _ptr(payload_len), _ptr(out)),
            "pixelize_adaptive_variance_dev")

    def reassemble_dev(self, desc, payload, payload_stride, payload_len, b, n, out):
        self._check(_lib.dppx_reassemble_dev(self._h, C.byref(desc), _ptr(payload),
                                             payload_stride, _ptr(payload_len), b, n, _ptr(out)),
                    "reassemble_dev")

    def broadcast_means_dev(self, desc, means, b, out):
        self._check(_lib.dppx_broadcast_means_dev(self._h, C.byref(desc), _ptr(means), b,
                                                  _ptr(out)), "broadcast_means_dev")

    def pixelize_uniform_sweep_dev(self, desc: FramesDesc, img, b_list, eps_list, m, noise_struct,
                                   means, out=None):
        """One read of the frames for every (b, eps) run of a uniform sweep
        (dppx_pixelize_uniform_sweep_dev). means / out: sequences of device
        tensors in run order (i * len(eps_list) + j); out entries may be None."""
        nb, ne = len(b_list), len(eps_list)
        bl = (C.c_int32 * nb)(*b_list)
        el = (C.c_double * ne)(*eps_list)
        mp = (_vp * (nb * ne))(*[t.data_ptr() for t in means])
        op = None if out is None else (_vp * (nb * ne))(*[None if t is None else t.data_ptr() for t in out])
        self._check(_lib.dppx_pixelize_uniform_sweep_dev(self._h, C.byref(desc), _ptr(img), nb, bl, ne, el, m,
                                                         C.byref(noise_struct), mp, op),
                    "pixelize_uniform_sweep_dev")

    def synth_frames_dev(self, desc, data_seed, f0, img, mask=None):
        self._check(_lib.dppx_synth_frames_dev(self._h, C.byref(desc), data_seed, f0, _ptr(img),
                                               _ptr(mask)), "synth_frames_dev")


_tls = threading.local()


class Group(Context):
    """A multi-GPU runner (dppx_group_*): one persistent host thread and one
    context per device; the host entry points of :class:`Context`
    (pixelize_uniform / pixelize_adaptive / broadcast_means / reassemble)
    split their frames into contiguous per-device blocks with no collective.
    Results are byte-identical to one Context (noise is keyed per plane).
    ``devices=None``: every visible sm_100 device; a device may repeat."""

    def __init__(self, devices=None):
        h = _vp()
        if devices is None:
            rc = _lib.dppx_group_create(None, 0, C.byref(h))
        else:
            arr = (C.c_int32 * len(devices))(*devices)
            rc = _lib.dppx_group_create(arr, len(devices), C.byref(h))
        if rc != OK:
            _raise(rc, f"dppx_group_create({devices}) failed with status {rc}")
        self._g = h
        self._h = h  # the entry points take the group handle in the ctx position
        self.devices = [_lib.dppx_group_device(h, i) for i in range(_lib.dppx_group_size(h))]
        self.device = self.devices[0]

    def close(self):
        if getattr(self, "_g", None):
            _lib.dppx_group_destroy(self._g)
            self._g = self._h = None

    def _last_error(self) -> str:
        return _lib.dppx_group_last_error(self._g).decode()

    @staticmethod
    def _api(name):
        return getattr(_lib, "dppx_group_" + name)

    def worker_context(self, i: int) -> "Context":
        """Non-owning view of worker i's context (configure it between group calls)."""
        c = Context.__new__(Context)
        c._h = _lib.dppx_group_ctx(self._g, i)
        c.device = self.devices[i]
        c.close = lambda: None
        return c

    def stats(self) -> dict:
        s = KernelStats()
        _lib.dppx_group_get_stats(self._g, C.byref(s))
        return {"launches": {k: int(s.launches[i]) for i, k in enumerate(KERNEL_FAMILIES)},
                "device_ms": {k: float(s.device_ms[i]) for i, k in enumerate(KERNEL_FAMILIES)},
                "h2d_bytes": int(s.h2d_bytes), "d2h_bytes": int(s.d2h_bytes)}

    def reset_stats(self):
        for i in range(len(self.devices)):
            _lib.dppx_ctx_reset_stats(_lib.dppx_group_ctx(self._g, i))

    def synchronize(self):
        for i in range(len(self.devices)):
            self._check(_lib.dppx_ctx_synchronize(_lib.dppx_group_ctx(self._g, i)), "synchronize")

    def set_timing(self, on: bool):
        for i in range(len(self.devices)):
            _lib.dppx_ctx_set_timing(_lib.dppx_group_ctx(self._g, i), 1 if on else 0)


def _torch_ordered(fn):
    """Orders a ``_dev`` call with torch: the context stream first waits for
    torch's current stream (tensors just allocated / filled by torch are ready),
    and torch's current stream then waits for the context stream (torch ops on
    the outputs see the results). Two stream-event pairs, no host sync; skipped
    when torch's current stream already is the context stream."""
    def wrapped(self, *a, **k):
        t = sys.modules.get("torch")
        if t is None or not t.cuda.is_available():
            return fn(self, *a, **k)
        h = self.stream
        cur = t.cuda.current_stream(self.device)
        if h == 0 or cur.cuda_stream == h:
            return fn(self, *a, **k)
        ours = t.cuda.ExternalStream(h, device=self.device)
        ours.wait_stream(cur)
        r = fn(self, *a, **k)
        cur.wait_stream(ours)
        return r
    wrapped.__name__, wrapped.__doc__ = fn.__name__, fn.__doc__
    return wrapped


for _name in [x for x in vars(Context) if x.endswith("_dev")]:
    setattr(Context, _name, _torch_ordered(getattr(Context, _name)))


def _group_unsupported(name):
    def f(self, *a, **k):
        raise NotImplementedError(f"Group.{name}: use worker_context(i).{name} (per-device call)")
    return f


for _name in ("stream", "set_stream", "set_chunk_frames", "set_exact_noise", "set_out_pad_scratch",
              "set_small_frame_path",
              "lg2_max_error", "pixelize_reference", "pixelize_adaptive_variance",
              "reconstruct_record", "classify_regions", "metrics", "device_laplace", "pixelize_checked",
              "pixelize_uniform_sweep",
              "pixelize_adaptive_dev", "pixelize_uniform_dev", "pixelize_adaptive_variance_dev",
              "pixelize_uniform_sweep_dev",
              "reassemble_dev", "broadcast_means_dev", "synth_frames_dev"):
    setattr(Group, _name, property(lambda self, _n=_name: _group_unsupported(_n).__get__(self))
            if _name == "stream" else _group_unsupported(_name))


def default_context() -> Context:
    """Per-thread context on device $DPPX_DEVICE (default 0)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context(int(os.environ.get("DPPX_DEVICE", "0")))
    return ctx


# ---------------------------------------------------------------- reference-shaped API
@dataclasses.dataclass
class GridMeans:
    geometry: Geometry
    values: np.ndarray


@dataclasses.dataclass
class UniformResult:
    image: np.ndarray
    means: GridMeans


@dataclasses.dataclass
class RegionClassification:
    geometry: Geometry
    mask_means: np.ndarray
    is_simple: np.ndarray

    def simple_count(self) -> int:
        return int((self.is_simple == 1).sum())


@dataclasses.dataclass
class AdaptiveMeans:
    geometry: Geometry
    n: int
    classification: RegionClassification
    simple_means: np.ndarray
    complex_submeans: np.ndarray

    def payload(self) -> bytes:
        """DPPX v1 adaptive payload (record.hpp:52-54)."""
        mm = np.asarray(self.classification.mask_means, "<f4").tobytes()
        S = len(self.simple_means)
        return (mm + int(S).to_bytes(4, "little") + bytes(self.simple_means)
                + bytes(self.complex_submeans))


@dataclasses.dataclass
class AdaptiveResult:
    image: np.ndarray
    means: AdaptiveMeans


def _check_gray(img, who):
    img = np.asarray(img)
    if img.ndim != 2 or img.shape[0] < 1 or img.shape[1] < 1:
        raise ValueError(f"{who}: malformed image")
    return np.ascontiguousarray(img, dtype=np.uint8)


def parse_adaptive_payload(payload: bytes, geom: Geometry, n: int) -> AdaptiveMeans:
    G = geom.grid_count()
    mm = np.frombuffer(payload[: 4 * G], "<f4").copy()
    S = int.from_bytes(payload[4 * G: 4 * G + 4], "little")
    simple = np.frombuffer(payload[4 * G + 4: 4 * G + 4 + S], np.uint8).copy()
    cplx = np.frombuffer(payload[4 * G + 4 + S:], np.uint8).copy()
    cls = RegionClassification(geom, mm, (mm > np.float32(0.5)).astype(np.uint8))
    return AdaptiveMeans(geom, n, cls, simple, cplx)


def pixelize_parallel(img, params: PrivacyParams, seed: Optional[int] = None,
                      threads: int = 0) -> UniformResult:
    """pixelize_parallel (pixelize.cpp:86-124) on the GPU; `threads` is ignored."""
    img = _check_gray(img, "pixelize_parallel")
    if params.n != 1:
        raise ValueError("pixelize_parallel: requires n == 1")
    geom = grid_dims(img.shape[0], img.shape[1], params.b)
    ctx = default_context()
    means, out = ctx.pixelize_uniform(img, params, NOISE_KEYED if seed is not None else NOISE_NONE,
                                      [seed] if seed is not None else None)
    return UniformResult(out, GridMeans(geom, means[0]))


def pixelize_adaptive(img, mask, params: PrivacyParams, seed: Optional[int] = None,
                      threads: int = 0) -> AdaptiveResult:
    """pixelize_adaptive (adaptive.cpp:88-179) on the GPU; `threads` is ignored."""
    img = _check_gray(img, "pixelize_adaptive")
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    if mask.shape != img.shape:
        raise ValueError("pixelize_adaptive: mask dimensions do not match image")
    if params.n < 1 or params.b % params.n or params.subgrid_side * params.n != params.b:
        raise ValueError("pixelize_adaptive: invalid subgrid factor")
    geom = grid_dims(img.shape[0], img.shape[1], params.b)
    ctx = default_context()
    payloads, out = ctx.pixelize_adaptive(img, mask, params,
                                          NOISE_KEYED if seed is not None else NOISE_NONE,
                                          [seed] if seed is not None else None)
    return AdaptiveResult(out, parse_adaptive_payload(payloads[0], geom, params.n))


def pixelize_reference(img, params: PrivacyParams, seed: Optional[int] = None) -> np.ndarray:
    """pixelize_reference, Algorithm 1 (pixelize.cpp:50-84), on the GPU."""
    img = _check_gray(img, "pixelize_reference")
    if params.n != 1:
        raise ValueError("pixelize_reference: requires n == 1")
    _, out = default_context().pixelize_reference(
        img, params, NOISE_KEYED if seed is not None else NOISE_NONE,
        [seed] if seed is not None else None)
    return out


def broadcast_means(means: GridMeans, height: int, width: int) -> np.ndarray:
    """broadcast_means (pixelize.cpp:126-150)."""
    if height < 1 or width < 1:
        raise ValueError("broadcast_means: dimensions must be >= 1")
    expected = grid_dims(height, width, means.geometry.b)
    if not (means.geometry == expected) or len(means.values) != expected.grid_count():
        raise ValueError("broadcast_means: means do not fit the target dimensions")
    return default_context().broadcast_means(means.values, height, width, means.geometry.b)[0, :, :, 0]


def reassemble(means: AdaptiveMeans, height: int, width: int) -> np.ndarray:
    """reassemble (adaptive.cpp:181-245), with its RecordError(corrupt_record) checks."""
    if height < 1 or width < 1:
        raise ValueError("reassemble: dimensions must be >= 1")
    geom = means.geometry
    if not (geom == grid_dims(height, width, geom.b)):
        raise ValueError("reassemble: geometry does not match the target dimensions")
    n = means.n
    if n < 1 or geom.b % n:
        raise RecordError("reassemble: subgrid factor does not divide grid side")
    G = geom.grid_count()
    cls = means.classification
    if len(cls.mask_means) != G or len(cls.is_simple) != G:
        raise RecordError("reassemble: classification length mismatch")
    S = cls.simple_count()
    if len(means.simple_means) != S or len(means.complex_submeans) != (G - S) * n * n:
        raise RecordError("reassemble: mean array length mismatch")
    mm = np.asarray(cls.mask_means, np.float32).copy()
    flags = np.asarray(cls.is_simple) != 0
    disagree = (mm > np.float32(0.5)) != flags
    mm[disagree] = np.where(flags[disagree], 1.0, 0.0)
    payload = (mm.astype("<f4").tobytes() + int(S).to_bytes(4, "little")
               + bytes(np.asarray(means.simple_means, np.uint8))
               + bytes(np.asarray(means.complex_submeans, np.uint8)))
    return default_context().reassemble([payload], height, width, geom.b, n)[0, :, :, 0]


def mse(a, b) -> float:
    """mse (metrics.cpp:26-37) on the GPU."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.ndim != 2 or a.size == 0:
        raise ValueError("mse: images must share valid dimensions")
    return float(default_context().metrics(a, b, "mse")[0])


def ssim(a, b, threads: int = 0) -> float:
    """ssim (metrics.cpp:73-183) on the GPU; `threads` is ignored."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape or a.ndim != 2:
        raise ValueError("ssim: images must share dimensions")
    return float(default_context().metrics(a, b, "ssim")[0])


def classify_regions(mask, geom: Geometry) -> RegionClassification:
    """classify_regions (adaptive.cpp:34-65) on the GPU."""
    mask = np.asarray(mask)
    if mask.ndim != 2 or mask.shape[0] < 1 or mask.shape[1] < 1:
        raise ValueError("classify_regions: malformed mask")
    if not (geom == grid_dims(mask.shape[0], mask.shape[1], geom.b)):
        raise ValueError("classify_regions: geometry does not match mask dimensions")
    mm = default_context().classify_regions(mask, geom.b)[0]
    return RegionClassification(geom, mm, (mm > np.float32(0.5)).astype(np.uint8))


# ---------------------------------------------------------------- .dppx records
def crc32(data: bytes, crc: int = 0) -> int:
    buf = np.frombuffer(data, np.uint8)
    return _lib.dppx_crc32(crc, buf.ctypes.data if len(buf) else None, len(buf))


def encode_record(height: int, width: int, b: int, n: int, payload: bytes,
                  adaptive: bool) -> bytes:
    """encode (record.cpp:124-175) around a statistics plane (the compact store)."""
    buf = np.frombuffer(payload, np.uint8)
    out = np.zeros(_lib.dppx_record_size(len(buf)), np.uint8)
    n_out = C.c_size_t(0)
    rc = _lib.dppx_encode_record(height, width, b, n, 2 if adaptive else 1,
                                 buf.ctypes.data if len(buf) else None, len(buf),
                                 out.ctypes.data, len(out), C.byref(n_out))
    if rc != OK:
        _raise(rc, "encode: payload or header fields inconsistent")
    return out.tobytes()


@dataclasses.dataclass
class PixelRecord:
    """dppix::PixelRecord (record.hpp:37-46): dims plus GridMeans or AdaptiveMeans."""
    height: int
    width: int
    payload: object  # GridMeans | AdaptiveMeans

    def mode(self) -> int:
        return 1 if isinstance(self.payload, GridMeans) else 2


def encode(record: PixelRecord) -> bytes:
    p = record.payload
    if isinstance(p, GridMeans):
        return encode_record(record.height, record.width, p.geometry.b, 1,
                             bytes(np.asarray(p.values, np.uint8)), False)
    return encode_record(record.height, record.width, p.geometry.b, p.n, p.payload(), True)


def decode(data: bytes) -> PixelRecord:
    """decode (record.cpp:177-278) with the reference's RecordError taxonomy."""
    buf = np.frombuffer(data, np.uint8)
    info = RecordInfo()
    rc = _lib.dppx_decode_record(buf.ctypes.data if len(buf) else None, len(buf), C.byref(info))
    if rc != OK:
        _raise(rc, f"decode: status {rc}")
    body = bytes(buf[info.payload_offset: info.payload_offset + info.payload_len])
    geom = grid_dims(info.height, info.width, info.b)
    if info.mode == 1:
        return PixelRecord(info.height, info.width, GridMeans(geom, np.frombuffer(body, np.uint8).copy()))
    return PixelRecord(info.height, info.width, parse_adaptive_payload(body, geom, info.n))


def reconstruct(record: PixelRecord) -> np.ndarray:
    """reconstruct (record.cpp:280-286) on the GPU."""
    if isinstance(record.payload, GridMeans):
        return broadcast_means(record.payload, record.height, record.width)
    return reassemble(record.payload, record.height, record.width)


__all__ = [
    "mse", "ssim", "crc32", "encode_record", "encode", "decode", "reconstruct", "PixelRecord", "RecordInfo",
    "Context", "default_context", "grid_dims", "make_privacy_params", "sensitivity", "keyed_bits",
    "laplace_at", "derive_plane_seed", "plane_seeds", "adaptive_payload_capacity",
    "pixelize_parallel", "pixelize_adaptive", "pixelize_reference", "broadcast_means", "reassemble", "classify_regions",
    "parse_adaptive_payload", "GridMeans", "UniformResult", "AdaptiveMeans", "AdaptiveResult",
    "RegionClassification", "RecordError", "DeviceUnavailable", "PrivacyParams", "Geometry",
    "FramesDesc", "Noise", "ABI", "LIB_PATH", "DROPIN_PATH",
    "NOISE_NONE", "NOISE_KEYED", "NOISE_PHILOX", "NOISE_INJECTED",
]
