/*
 * dppx_gpu.h -- C ABI of the B200-native dppix pixelization path.
 *
 * Drop-in boundary for the reference's static C++ library API
 * (/root/reference/proj/include/dppix). The reference exposes value-semantics
 * C++ functions; this ABI exposes the same operations over plain pointers and
 * sizes so that any host language can bind it (see INTEGRATION.md for the
 * ctypes binding shipped in paper_2511_04261_b200/ and for the C++ shim that
 * re-creates the exact dppix:: signatures, include/dppix/).
 *
 *   reference symbol (file:line)                         replaced by
 *   dppix::grid_dims            image.hpp:86             dppx_grid_dims
 *   dppix::make_privacy_params  noise.hpp:55             dppx_make_privacy_params
 *   dppix::keyed_bits           noise.hpp:69             dppx_keyed_bits
 *   dppix::laplace_at           noise.hpp:80             dppx_laplace_at (host diagnostic)
 *   dppix::pixelize_parallel    pixelize.hpp:55-58       dppx_pixelize_uniform[_dev]
 *   dppix::pixelize_adaptive    adaptive.hpp:70-73       dppx_pixelize_adaptive[_dev]
 *   dppix::pixelize_reference   pixelize.hpp:45-46       dppx_pixelize_reference (Algorithm 1)
 *   dppix::broadcast_means      pixelize.hpp:62          dppx_broadcast_means[_dev]
 *   dppix::reassemble           adaptive.hpp:78          dppx_reassemble[_dev]
 *   dppix::reconstruct          record.hpp:63            dppx_reassemble / dppx_broadcast_means
 *   dppix::classify_regions     adaptive.hpp:45-46       dppx_classify_regions
 *   dppix::encode / decode      record.hpp:55-61         dppx_encode_record / dppx_decode_record
 *   dppix::mse / ssim           metrics.hpp:27-37        dppx_mse / dppx_ssim
 *   RecordError / invalid_argument  errors.hpp:22-55     dppx_status codes
 *
 * Conventions
 *  - Caller-owned buffers. Images are row-major uint8 with C interleaved
 *    channels (C = 1 is the reference's GrayImage; C = 3 is RGB, every channel
 *    plane processed with the reference's per-plane semantics).
 *  - A batch holds F frames with the same geometry; plane (f, c) is channel c
 *    of frame f and gets its own noise seed (plane_seeds[f*C + c]).
 *  - Uniform statistics: F*C planes of G = grid_rows*grid_cols bytes, plane
 *    (f, c) at means + (f*C + c)*G (the DPPX v1 uniform payload, record.hpp:52).
 *  - Adaptive statistics: F*C slots of `payload_stride` bytes, each holding the
 *    DPPX v1 adaptive payload (record.hpp:52-54): G f32 mask means, u32 simple
 *    count S, S simple means, (G-S)*n*n complex submeans. payload_stride must be
 *    >= dppx_adaptive_payload_capacity() and a multiple of 4.
 *  - *_dev entry points take DEVICE pointers and are asynchronous on the ctx
 *    stream (dppx_ctx_stream); errors detected on the device are returned by
 *    the next dppx_ctx_synchronize. Host entry points take HOST pointers, run
 *    a pinned double-buffered H2D -> kernels -> D2H pipeline and return when
 *    results are in host memory.
 *  - A ctx is bound to one device and used by one host thread at a time
 *    (the reference functions are reentrant; use one ctx per thread).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns DPPX_ERR_NO_DEVICE.
 */
#ifndef DPPX_GPU_H_
#define DPPX_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPPX_ABI_VERSION 1

typedef enum {
  DPPX_OK = 0,
  DPPX_ERR_INVALID = 1,   /* std::invalid_argument in the reference            */
  DPPX_ERR_CORRUPT = 2,   /* RecordError(corrupt_record) (adaptive.cpp:192-210) */
  DPPX_ERR_CUDA = 3,      /* std::runtime_error: CUDA failure                  */
  DPPX_ERR_OOM = 4,       /* std::bad_alloc                                    */
  DPPX_ERR_NO_DEVICE = 5, /* no sm_100 device / kernels not loadable           */
  DPPX_ERR_NOT_A_RECORD = 6,        /* RecordError(not_a_record)             */
  DPPX_ERR_UNSUPPORTED_VERSION = 7, /* RecordError(unsupported_version)      */
  DPPX_ERR_CORRUPTION = 8           /* RecordError(corruption): CRC mismatch */
} dppx_status;

typedef enum {
  DPPX_NOISE_NONE = 0,     /* std::nullopt seed: no noise                                */
  DPPX_NOISE_KEYED = 1,    /* reference stream: splitmix64 keyed_bits + inverse-CDF      */
                           /* Laplace (noise.cpp:76-117), seed per plane                 */
  DPPX_NOISE_PHILOX = 2,   /* Philox4x32-10 keyed (seed, frame, channel, cell) extension */
  DPPX_NOISE_INJECTED = 3  /* caller-supplied noise doubles (parity testing)             */
} dppx_noise_kind;

/* GridGeometry, image.hpp:71-82. */
typedef struct {
  int32_t b, grid_rows, grid_cols, pad_rows, pad_cols;
} dppx_geometry;

/* PrivacyParams, noise.hpp:41-51. */
typedef struct {
  double epsilon;
  int32_t m, b, n, subgrid_side;
  double delta, sigma, delta_sub, sigma_sub;
} dppx_privacy_params;

/* A batch of F frames of one geometry. Strides are in bytes. */
typedef struct {
  int32_t height, width, channels, frames; /* M, N, C (1..4), F */
  int64_t pitch, frame_stride;             /* input image               */
  int64_t mask_pitch, mask_frame_stride;   /* adaptive region mask (u8) */
  int64_t out_pitch, out_frame_stride;     /* reconstructed image       */
} dppx_frames_desc;

typedef struct {
  int32_t kind;                /* dppx_noise_kind                                        */
  uint32_t frame_base;         /* PHILOX: global index of frame 0 of this batch          */
  const uint64_t* plane_seeds; /* KEYED: F*C host seeds, (f, c) at f*C + c.              */
                               /* PHILOX: plane_seeds[0] is the base seed.               */
  const double* injected;      /* INJECTED: per plane G*n*n doubles,                      */
                               /* ((f*C + c)*G + g)*n*n + sr*n + sc. Device memory for    */
                               /* *_dev entry points, host memory otherwise.              */
} dppx_noise;

/* Per kernel-family launch counts and (when timing is on) summed device ms. */
typedef enum {
  DPPX_K_CLASSIFY = 0, /* K0: mask -> per-cell classification + slot scan */
  DPPX_K_STATS = 1,    /* K1: TMA-staged fused stats/noise/store/reconstruct  */
                       /*     (b in {4,8,12,16,20,24,32,40,64}, C in {1,3})     */
  DPPX_K_GENERIC = 2,  /* K1g: Algorithm 1 and shapes K1r cannot hold          */
  DPPX_K_EXPAND = 3,   /* K2: statistics -> pixels                            */
  DPPX_K_AUX = 4,      /* synthetic generator, payload checks                 */
  DPPX_K_ROWS = 5,     /* K1r: row-streaming stats for other grid sides        */
  DPPX_K_SWEEP = 6,    /* K1s: one-read statistics of a grid-size x eps sweep  */
  DPPX_K_ZEROCOPY = 7, /* K1z: small host frames read / written over PCIe     */
  DPPX_K_COUNT = 8
} dppx_kernel_family;

typedef struct {
  uint64_t launches[DPPX_K_COUNT];
  double device_ms[DPPX_K_COUNT];
  uint64_t h2d_bytes, d2h_bytes;
} dppx_kernel_stats;

typedef struct dppx_ctx dppx_ctx;

/* ---- host-side parameter helpers (no device needed) --------------------- */
const char* dppx_version(void);
int dppx_grid_dims(int32_t height, int32_t width, int32_t b, dppx_geometry* out);
int dppx_make_privacy_params(double epsilon, int32_t m, int32_t b, int32_t n,
                             dppx_privacy_params* out);
double dppx_sensitivity(int32_t b, int32_t m); /* < 0 on invalid input */
uint64_t dppx_keyed_bits(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc);
double dppx_uniform_from_bits(uint64_t bits);
double dppx_laplace_at(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc,
                       double sigma);
/* Seed of plane (frame, channel) for multi-frame / multi-channel batches:
 * keyed_bits(seed, {frame, channel, 0xFFFFFFFF, 0xFFFFFFFF}). */
uint64_t dppx_derive_plane_seed(uint64_t seed, uint32_t frame, uint32_t channel);
size_t dppx_adaptive_payload_capacity(int32_t height, int32_t width, int32_t b, int32_t n);
size_t dppx_adaptive_payload_length(int32_t height, int32_t width, int32_t b, int32_t n,
                                    uint32_t simple_count);

/* ---- context ------------------------------------------------------------- */
int dppx_ctx_create(int32_t device, dppx_ctx** out);
void dppx_ctx_destroy(dppx_ctx* ctx);
const char* dppx_ctx_last_error(const dppx_ctx* ctx);
void* dppx_ctx_stream(dppx_ctx* ctx); /* cudaStream_t */
int dppx_ctx_set_stream(dppx_ctx* ctx, void* stream); /* NULL restores the ctx's own */
int dppx_ctx_synchronize(dppx_ctx* ctx);
int dppx_ctx_set_timing(dppx_ctx* ctx, int32_t on);
int dppx_ctx_get_stats(dppx_ctx* ctx, dppx_kernel_stats* out);
int dppx_ctx_reset_stats(dppx_ctx* ctx);
/* 1: evaluate every statistic with the reference's f64 arithmetic (no bounded
 * f32 fast path); the bytes produced are identical either way. */
int dppx_ctx_set_exact_noise(dppx_ctx* ctx, int32_t on);
/* Output row padding, bytes [N*C, out_pitch), of the device entry points.
 * Default 0: every kernel stores exactly the bytes [0, N*C) of each row, so
 * the output may be a window of a larger image (neighbouring bytes are never
 * touched; tests/test_gpu_parity.py::test_default_stores_are_window_safe).
 * 1: the caller declares the padding scratch; stores may end every row on a
 * whole 32-byte sector, [0, min(out_pitch, round_up(N*C, 32))), removing
 * partial-sector DRAM writes. Pixels [0, N*C) are identical either way. The
 * host entry points always use it on their own staging buffers. */
int dppx_ctx_set_out_pad_scratch(dppx_ctx* ctx, int32_t on);
/* How the host entry points move ONE small frame (< 4 MB, pinned buffers):
 *   DPPX_SMALL_AUTO      default: zero-copy where the shape allows it, else graph
 *   DPPX_SMALL_GRAPH     H2D, kernels and D2H replayed as one CUDA graph
 *   DPPX_SMALL_ZEROCOPY  the kernels read / write the mapped pinned buffers
 *                        over PCIe themselves (uniform: K1z; adaptive: K0 + K1r)
 *   DPPX_SMALL_STAGED    the ordinary staged pipeline
 * Results are identical on every path. */
enum { DPPX_SMALL_AUTO = 0, DPPX_SMALL_GRAPH = 1, DPPX_SMALL_ZEROCOPY = 2, DPPX_SMALL_STAGED = 3 };
int dppx_ctx_set_small_frame_path(dppx_ctx* ctx, int32_t path);
/* Frames per pipeline chunk of the host entry points (0 = automatic). */
int dppx_ctx_set_chunk_frames(dppx_ctx* ctx, int32_t frames);

int dppx_host_alloc(size_t bytes, void** out); /* pinned */
void dppx_host_free(void* p);

/* ---- device-resident entry points (async on the ctx stream) -------------- */
int dppx_pixelize_uniform_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                              const dppx_privacy_params* params, const dppx_noise* noise,
                              uint8_t* means, uint8_t* out /* nullable */);
int dppx_pixelize_adaptive_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                               const uint8_t* mask, const dppx_privacy_params* params,
                               const dppx_noise* noise, uint8_t* payload, int64_t payload_stride,
                               uint32_t* payload_len /* nullable, F*C */,
                               uint8_t* out /* nullable */);
int dppx_broadcast_means_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* means,
                             int32_t b, uint8_t* out);
/* payload_len: nullable; when given, each plane's length is checked. */
int dppx_reassemble_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* payload,
                        int64_t payload_stride, const uint32_t* payload_len, int32_t b,
                        int32_t n, uint8_t* out);
/* Synthetic workload (bench / tests): frames f0..f0+F-1, see oracle/dppx_oracle.c. */
int dppx_synth_frames_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, uint32_t data_seed,
                          uint32_t f0, uint8_t* img, uint8_t* mask /* nullable */);

/* One HBM read of the frames for every run of a uniform grid-size x epsilon
 * sweep (run_sweep cli.cpp:231-288 / SURVEY 8(d) config 3). Run (i, j) is
 * pixelize_parallel with grid side b_list[i] and epsilon eps_list[j] (m and
 * noise shared): statistics at means[i*ne + j] (F*C planes of G_i bytes, as
 * dppx_pixelize_uniform_dev) and, if out != NULL and out[i*ne + j] != NULL, its
 * reconstructed image there (desc out_pitch / out_frame_stride). Bytes are
 * identical to separate dppx_pixelize_uniform_dev calls. Grid sides in
 * {4, 8, 16, 32} (KEYED / PHILOX / NONE noise, C in {1, 3}, 16-byte aligned
 * frames): one statistics kernel reads each frame once -- 4-px cell sums over
 * the largest padded extent aggregate exactly to the larger sides, and the
 * keyed bits and Laplace magnitude of a cell are drawn once for all eps --
 * then one broadcast per run writes the images. Other lists run per b. */
int dppx_pixelize_uniform_sweep_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                                    int32_t nb, const int32_t* b_list, int32_t ne,
                                    const double* eps_list, int32_t m, const dppx_noise* noise,
                                    uint8_t* const* means, uint8_t* const* out /* nullable */);

/* Host-pointer form of the sweep (run_sweep's caller shape): one upload of the
 * F frames, the runs as in dppx_pixelize_uniform_sweep_dev, then for every
 * run (i*ne + j) its statistics to means[r] (F*C planes of G_i bytes), its
 * image to out[r] (if out and out[r] are non-NULL; desc out_pitch /
 * out_frame_stride) and, computed on the device against the input,
 * mse_out[r*F*C + plane] / ssim_out[...] (each may be NULL; no ssim below 7x7). */
int dppx_pixelize_uniform_sweep(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img, int32_t nb,
                                const int32_t* b_list, int32_t ne, const double* eps_list, int32_t m,
                                const dppx_noise* noise, uint8_t* const* means, uint8_t* const* out,
                                double* mse_out, double* ssim_out);

/* EXTENSION (north-star "per-region complexity measure"; no reference
 * counterpart -- the reference takes external masks): cell
 * (r, c) is complex iff the variance of its C*b*b mirror-padded samples,
 * (n*S2 - S1^2)/n^2 from exact integer sums, is >= var_tau. Mask means are
 * stored as 1.0f / 0.0f so records decode to the same classification.
 * PRIVACY: the classification is computed from the private frames and is NOT
 * covered by the epsilon guarantee; use only where that is acceptable. */
int dppx_pixelize_adaptive_variance_dev(dppx_ctx* ctx, const dppx_frames_desc* desc,
                                        const uint8_t* img, double var_tau,
                                        const dppx_privacy_params* params, const dppx_noise* noise,
                                        uint8_t* payload, int64_t payload_stride,
                                        uint32_t* payload_len, uint8_t* out /* nullable */);

/* ---- host entry points (pinned pipeline; synchronous) -------------------- */
int dppx_pixelize_uniform(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                          const dppx_privacy_params* params, const dppx_noise* noise,
                          uint8_t* means, uint8_t* out /* nullable */);
int dppx_pixelize_adaptive(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                           const uint8_t* mask, const dppx_privacy_params* params,
                           const dppx_noise* noise, uint8_t* payload, int64_t payload_stride,
                           uint32_t* payload_len /* nullable */, uint8_t* out /* nullable */);
int dppx_pixelize_adaptive_variance(dppx_ctx* ctx, const dppx_frames_desc* desc,
                                    const uint8_t* img, double var_tau,
                                    const dppx_privacy_params* params, const dppx_noise* noise,
                                    uint8_t* payload, int64_t payload_stride,
                                    uint32_t* payload_len, uint8_t* out /* nullable */);
int dppx_broadcast_means(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* means,
                         int32_t b, uint8_t* out);
/* Algorithm 1 (pixelize.cpp:50-84): no padding, border cells average their real
 * h x w pixels; means has one byte per cell like dppx_pixelize_uniform. */
int dppx_pixelize_reference(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* img,
                            const dppx_privacy_params* params, const dppx_noise* noise,
                            uint8_t* means, uint8_t* out /* nullable */);
int dppx_reassemble(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* payload,
                    int64_t payload_stride, const uint32_t* payload_len, int32_t b, int32_t n,
                    uint8_t* out);

/* ---- multi-GPU runner (one host thread + one ctx per device) -------------
 * The reference's multi-image parallelism is run_batch's file-level
 * parallel_for (cli.cpp:194-211). A group owns one persistent host thread and
 * one dppx_ctx per listed device; dppx_group_* entry points take the same
 * arguments as the host entry points above, split the F frames into
 * contiguous blocks (one per device) and run them concurrently. There is no
 * collective on the data path: noise is keyed per plane / global frame, never
 * by device, so results are byte-identical to one ctx over the whole batch.
 * devices == NULL: every visible sm_100 device (at most `count` if count > 0).
 * A device may be listed twice (two contexts, e.g. to test the runner on one GPU). */
typedef struct dppx_group dppx_group;
int dppx_group_create(const int32_t* devices, int32_t count, dppx_group** out);
void dppx_group_destroy(dppx_group* group);
int32_t dppx_group_size(const dppx_group* group);
int32_t dppx_group_device(const dppx_group* group, int32_t worker);
/* The worker's context (for configuration between group calls only). */
dppx_ctx* dppx_group_ctx(dppx_group* group, int32_t worker);
const char* dppx_group_last_error(const dppx_group* group);
/* Dynamic parallel-for over the workers: each task runs once, on whichever
 * worker thread claims it next, with that worker's ctx. Returns the status of
 * the lowest-numbered failing task (its message in dppx_group_last_error). */
int dppx_group_run(dppx_group* group, int32_t tasks,
                   int (*fn)(dppx_ctx* ctx, int32_t worker, int32_t task, void* user), void* user);
int dppx_group_pixelize_uniform(dppx_group* group, const dppx_frames_desc* desc,
                                const uint8_t* img, const dppx_privacy_params* params,
                                const dppx_noise* noise, uint8_t* means, uint8_t* out);
int dppx_group_pixelize_adaptive(dppx_group* group, const dppx_frames_desc* desc,
                                 const uint8_t* img, const uint8_t* mask,
                                 const dppx_privacy_params* params, const dppx_noise* noise,
                                 uint8_t* payload, int64_t payload_stride, uint32_t* payload_len,
                                 uint8_t* out);
int dppx_group_broadcast_means(dppx_group* group, const dppx_frames_desc* desc,
                               const uint8_t* means, int32_t b, uint8_t* out);
int dppx_group_reassemble(dppx_group* group, const dppx_frames_desc* desc, const uint8_t* payload,
                          int64_t payload_stride, const uint32_t* payload_len, int32_t b,
                          int32_t n, uint8_t* out);
/* Launch counts and transfer bytes summed over the workers; device_ms is the max. */
int dppx_group_get_stats(dppx_group* group, dppx_kernel_stats* out);

/* The batch runner's per-file work (run_single, cli.cpp:93-173) for F frames
 * on ONE upload: pixelize (mode 0 uniform / 1 adaptive / 2 Algorithm 1), then,
 * where both images already live, the reconstruct check -- the statistics just
 * produced, expanded again (broadcast_means / reassemble), must equal the
 * emitted frames: recon_ok[f] = 1 / 0 (always 1 for mode 2, which keeps no
 * statistics) -- and mse / ssim of input vs emitted frames (ssim_out may be
 * NULL; frames smaller than 7 x 7 get no ssim). Outputs as the host entry
 * points above (stats / lens / out; stats may be NULL for mode 2). */
int dppx_pixelize_checked(dppx_ctx* ctx, int32_t mode, const dppx_frames_desc* desc, const uint8_t* img,
                          const uint8_t* mask, const dppx_privacy_params* params, const dppx_noise* noise,
                          uint8_t* stats, int64_t payload_stride, uint32_t* payload_len, uint8_t* out,
                          uint8_t* recon_ok, double* mse_out, double* ssim_out);
/* Sizes everything dppx_pixelize_checked would allocate for (mode, desc,
 * params) -- device buffers, scratch, the pinned staging pieces -- without
 * running anything, so a batch runner can pay for it while it still reads its
 * inputs. Optional: dppx_pixelize_checked grows the same buffers itself. */
int dppx_pixelize_checked_reserve(dppx_ctx* ctx, int32_t mode, const dppx_frames_desc* desc,
                                  const dppx_privacy_params* params);

/* classify_regions (adaptive.cpp:34-65) of F masks (desc mask fields; channels
 * ignored): per-frame G float mask means at mask_means + f*G. */
int dppx_classify_regions(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* mask,
                          int32_t b, float* mask_means);

/* ---- .dppx records (record.hpp:48-71, record.cpp:124-278; host only) ------ */
/* Decoded header of a record; the payload is bytes[payload_offset, +payload_len). */
typedef struct {
  int32_t height, width, b, n, mode; /* mode 1 = uniform, 2 = adaptive */
  uint32_t payload_offset, payload_len;
} dppx_record_info;

uint32_t dppx_crc32(uint32_t crc, const uint8_t* data, size_t len); /* zlib-compatible */
size_t dppx_record_size(size_t payload_len);                         /* 20 + payload + 4 */
/* Header + payload (a statistics plane as the kernels wrote it) + CRC32.
 * DPPX_ERR_INVALID mirrors encode's std::invalid_argument (record.cpp:124-150). */
int dppx_encode_record(int32_t height, int32_t width, int32_t b, int32_t n, int32_t mode,
                       const uint8_t* payload, size_t payload_len, uint8_t* out, size_t cap,
                       size_t* out_len);
/* decode's checks in order: NOT_A_RECORD, CORRUPT (truncated header), CORRUPTION
 * (CRC), UNSUPPORTED_VERSION, CORRUPT (mode/reserved/dims/fields/lengths/count). */
int dppx_decode_record(const uint8_t* bytes, size_t len, dppx_record_info* info);
/* reconstruct(decode(bytes)) (record.hpp:63, record.cpp:280-286): decodes the
 * record with the checks above, then expands it on the GPU (broadcast_means
 * for uniform, reassemble for adaptive) into out (height x width bytes, dense;
 * out_cap >= height * width). Status codes as dppx_decode_record / the expanders. */
int dppx_reconstruct_record(dppx_ctx* ctx, const uint8_t* bytes, size_t len, uint8_t* out,
                            size_t out_cap);

/* ---- utility metrics (metrics.hpp:27-37, metrics.cpp:26-183) ------------- */
/* Per channel plane (f, c) of frame batches a (pitch, frame_stride) and b
 * (out_pitch, out_frame_stride); out[f*C + c]. Bit-identical to the reference:
 * exact integer sums, the reference's f64 operation order, rows summed in order. */
int dppx_mse(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* a, const uint8_t* b,
             double* out);
int dppx_ssim(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* a, const uint8_t* b,
              double* out); /* 7x7 uniform window, C1 = 6.5025, C2 = 58.5225 */
/* Both metrics from one upload of a and b (the batch runner's per-file
 * mse + ssim, cli.cpp:164-171); either output may be NULL. */
int dppx_metrics(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* a, const uint8_t* b,
                 double* mse_out, double* ssim_out);
int dppx_mse_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* a, const uint8_t* b,
                 double* out);
int dppx_ssim_dev(dppx_ctx* ctx, const dppx_frames_desc* desc, const uint8_t* a, const uint8_t* b,
                  double* out);

/* Diagnostics for parity tests: the device noise of `count` keys
 * (keys[4*i..4*i+3] = r, c, sr, sc) for one plane seed at scale sigma. */
int dppx_debug_device_laplace(dppx_ctx* ctx, uint64_t seed, const uint32_t* keys, int32_t count,
                              double sigma, double* out);
/* Max |lg2.approx(m) - log2(m)| over all f32 mantissas (fast-path error bound). */
int dppx_debug_lg2_max_error(dppx_ctx* ctx, double* out);

#ifdef __cplusplus
}
#endif

#endif /* DPPX_GPU_H_ */
