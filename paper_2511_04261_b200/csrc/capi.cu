// capi.cu -- host runtime behind include/dppx_gpu.h: context (device, streams,
// scratch, pinned staging), argument validation with the reference's error
// semantics, kernel selection, and the pinned double-buffered
// H2D -> K0/K1 -> D2H pipeline of the host entry points.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <map>
#include <utility>
#include <vector>

#include "../../include/dppx_gpu.h"
#include "dppx_params.h"
#include "dppx_device.cuh"
#include "maskpack.h"

namespace dppx {
using StatsKernel = void (*)(const CUtensorMap, const CUtensorMap, const StatsArgs);
StatsKernel select_stats_kernel(int C, int b, int n, bool adaptive, bool packed);
StatsKernel select_stats_kernel_var(int C, int b, int n);
StatsKernel select_uniform_b4_rows2(int C);
cudaError_t launch_gather_stage(const GatherArgs& a, cudaStream_t s);
int rows_smem_bytes(const BatchGeom& g);
cudaError_t launch_stats_rows(const StatsArgs& a, size_t smem, cudaStream_t s);
cudaError_t launch_stats_zc(const StatsArgs& a, int unit_target, int ctas, int sms, cudaStream_t s, bool* launched,
                            bool dry_run);
cudaError_t launch_expand_rows(const ExpandArgs& a, size_t smem, cudaStream_t s);
int stats_threads();
int stats_tile_px();
int stats_tile_px_for(int b, bool adaptive);
int expand_packed_tile_px();
int stats_max_stages();
cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t s);
cudaError_t launch_stats_tma(StatsKernel k, const CUtensorMap& tin, const CUtensorMap& tout,
                             const StatsArgs& a, int grid, size_t smem, cudaStream_t s);
cudaError_t launch_stats_generic(const StatsArgs& a, cudaStream_t s);
cudaError_t launch_stats_px(const StatsArgs& a, cudaStream_t s);
cudaError_t launch_expand(const ExpandArgs& a, cudaStream_t s);
cudaError_t launch_expand_px(const ExpandArgs& a, cudaStream_t s);
using ExpandKernel = void (*)(const CUtensorMap, const ExpandArgs);
ExpandKernel select_expand_kernel(int C, int b, int n, bool adaptive, bool packed, int split);
cudaError_t launch_expand_tma(ExpandKernel k, const CUtensorMap& tout, const ExpandArgs& a,
                              int grid, size_t smem, cudaStream_t s);
cudaError_t launch_synth(const BatchGeom& g, uint32_t seed, uint32_t f0, uint8_t* img,
                         int64_t pitch, int64_t fstride, uint8_t* mask, int64_t mpitch,
                         int64_t mfstride, cudaStream_t s);
cudaError_t launch_debug_lg2(unsigned int* out, cudaStream_t s);
struct MetricArgs {
  int M, N, C, F;
  const uint8_t* a;
  int64_t pitch, fstride;
  const uint8_t* b;
  int64_t bpitch, bfstride;
  unsigned long long* sums;
  double* row_sums;
};
cudaError_t launch_metrics(const MetricArgs& m, bool ssim, cudaStream_t s);
cudaError_t launch_repitch(uint8_t* dst, int64_t dpitch, const uint8_t* src, int64_t spitch,
                           int64_t width, int64_t rows, cudaStream_t s);
cudaError_t launch_frames_equal(const uint8_t* a, const uint8_t* b, int64_t pitch, int64_t fstride,
                                int64_t width, int rows, int frames, uint32_t* eq, cudaStream_t s);
cudaError_t launch_debug_laplace(uint64_t mixed, const uint32_t* keys, int count, double sigma,
                                 double* out, cudaStream_t s);
constexpr int kSweepMaxLevels = 4;
constexpr int kSweepMaxEps = 4;
struct SweepLevels {  // sweep.cu
  int nlev;
  int ne;
  uint32_t active;
  int GR[kSweepMaxLevels], GC[kSweepMaxLevels];
  int64_t G[kSweepMaxLevels];
  double area[kSweepMaxLevels];
  double sigma[kSweepMaxLevels][kSweepMaxEps];
  float sln2[kSweepMaxLevels][kSweepMaxEps];  // f32(sigma * ln 2)
  float margin[kSweepMaxLevels][kSweepMaxEps];
  uint8_t* means[kSweepMaxLevels][kSweepMaxEps];
  void* sums[kSweepMaxLevels];
  int srows[kSweepMaxLevels], scols[kSweepMaxLevels];
  int64_t item0[kSweepMaxLevels + 1];
  int64_t item_begin, item_end;
  int groups[kSweepMaxLevels];
  FastDiv div_groups[kSweepMaxLevels], div_rows[kSweepMaxLevels];
  int planes;
};
using SweepSumsKernel = void (*)(const CUtensorMap, const StatsArgs, const SweepLevels);
SweepSumsKernel select_sweep_kernel(int C, int nlev);
cudaError_t launch_sweep_sums(SweepSumsKernel k, const CUtensorMap& tin, const StatsArgs& a,
                              const SweepLevels& L, int grid, size_t smem, cudaStream_t s);
cudaError_t launch_sweep_draw(const StatsArgs& a, const SweepLevels& L, int max_grid, cudaStream_t s);
int sweep_draw_threads();
}  // namespace dppx

using namespace dppx;

namespace {

// ---- host mirrors of the reference's scalar helpers ------------------------
uint64_t mix64_h(uint64_t z) {  // noise.cpp:77-82
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t keyed_bits_h(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc) {
  uint64_t s = mix64_h(seed);  // noise.cpp:86-91
  s = mix64_h(s ^ ((static_cast<uint64_t>(r) << 32) | c));
  return mix64_h(s ^ ((static_cast<uint64_t>(sr) << 32) | sc));
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

struct PendingTiming {
  int family;
  cudaEvent_t start, stop;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct dppx_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // compute stream (own or user's)
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaStream_t s_meta = nullptr;  // payload lengths D2H, ahead of the image copies on s_out
  std::string err;
  // scratch
  DevBuf cellinfo, rowcnt, rowprefix, totals, counters, status, seeds, keys, dbl, work, met_a, met_b, met_out;
  uint64_t* seeds_pinned = nullptr;
  size_t seeds_pinned_n = 0;
  cudaEvent_t seeds_ev = nullptr;
  // host-pipeline staging (2 slots)
  DevBuf img[2], mask[2], out[2], stats[2], lens[2], inj[2], sd[2], dense[2], dense_out[2],
      dense_mask[2];  // dense (input) and dense_out never alias: chunk ci+2's H2D may run
                      // while chunk ci's D2H is still reading its output
  DevBuf var_flags, var_stage;  // fused variance classification staging
  DevBuf sweep_sums[4];         // K1s level sums (one-read sweep)
  DevBuf check_img, check_eq;   // dppx_pixelize_checked: rebuilt frames, per-frame flags
  uint64_t* sd_pinned[2] = {nullptr, nullptr};
  size_t sd_pinned_n[2] = {0, 0};
  cudaEvent_t in_done[2] = {}, comp_done[2] = {}, out_done[2] = {};
  // written-length payload D2H: per slot, the chunk's lengths land in pinned
  // memory first (lens_ev), then only the written bytes of the payloads move
  uint32_t* lens_pinned[2] = {nullptr, nullptr};
  size_t lens_pinned_n[2] = {0, 0};
  cudaEvent_t lens_ev[2] = {};
  static constexpr int kMaxBands = 8;
  cudaEvent_t band_in[kMaxBands] = {}, band_comp[kMaxBands] = {};  // single-frame row bands
  int chunk_frames = 0;
  bool exact_noise = false;
  bool out_pad_scratch = false;  // dppx_ctx_set_out_pad_scratch
  bool force_rows = false;       // zero-copy calls: row-streaming kernels (plain loads/stores)
  int small_path = -1;           // DPPX_SMALL_*; -1: from the environment on first use
  double var_tau = 0.0;  // AdaptiveVariance host calls
  // bit-packed mask transport (maskpack.h): pinned staging per slot + packer pool
  dppx::MaskPacker* packer = nullptr;
  uint32_t* mbits_pinned[2] = {nullptr, nullptr};
  size_t mbits_pinned_n[2] = {0, 0};
  int mask_bits_mode = -1;  // -1 unset (env DPPX_MASK_BITS, default on), 0 off, 1 on
  // pageable caller buffers: pinned staging per slot, filled / drained by host threads
  uint8_t* stg_in[2] = {nullptr, nullptr};
  uint8_t* stg_out[2] = {nullptr, nullptr};
  size_t stg_in_n[2] = {0, 0}, stg_out_n[2] = {0, 0};
  cudaEvent_t stg_ev[2] = {};
  uint8_t* piece[2] = {nullptr, nullptr};  // h2d_frames pieces
  size_t piece_n[2] = {0, 0};
  cudaEvent_t piece_ev[2] = {};
  // single-frame host calls replayed as CUDA graphs (host_single_graph)
  struct FrameGraph;
  std::vector<FrameGraph*> graphs;
  // Bumped whenever a ctx buffer is (re)allocated: a captured graph holds the
  // addresses of the ctx buffers it touches, so graphs older than the last
  // (re)allocation are dropped, never replayed.
  uint64_t alloc_gen = 0;
  uint64_t graph_tick = 0;  // LRU clock of the graph cache
  uint64_t* gseeds_pinned = nullptr;  // mixed plane seeds of the next replay
  DevBuf gseeds;
  uint8_t* gstats_pinned = nullptr;   // statistics / lengths land here, then the caller's buffers
  size_t gstats_pinned_n = 0;
  // stats
  bool timing = false;
  std::vector<PendingTiming> pending;
  std::vector<cudaEvent_t> event_pool;
  dppx_kernel_stats kstats{};
  std::map<std::pair<const void*, size_t>, int> occupancy;  // (TMA kernel, smem) -> CTAs/SM
};

// A single-frame host call captured once per (operation, geometry, privacy
// parameters, noise kind, band count) and replayed: H2D row bands, K0, K1 row
// bands and D2H row bands as one graph launch. Per replay only the caller's
// host pointers (memcpy node parameters) and the mixed plane seeds (a pinned
// buffer the graph copies from) change.
struct dppx_ctx::FrameGraph {
  int op, M, N, C, b, n, kind, exact, nb, want_out;
  double sigma, sigma_sub;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  struct Copy {
    cudaGraphNode_t node;
    cudaMemcpy3DParms p;
    int which;        // 0: image source, 1: mask source, 2: image destination
    int64_t offset;   // bytes from the caller's base pointer
  };
  std::vector<Copy> copies;
  const void* cur[3] = {nullptr, nullptr, nullptr};
  uint64_t launches[DPPX_K_COUNT] = {};
  uint64_t h2d = 0, d2h = 0;
  uint64_t last_use = 0;
  uint64_t gen = 0;  // ctx->alloc_gen when captured
  ~FrameGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

namespace {

int set_err(dppx_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? DPPX_ERR_OOM : DPPX_ERR_CUDA,  \
                     "%s: %s", #expr, cudaGetErrorString(e_));                             \
    }                                                                                      \
  } while (0)

int ensure(dppx_ctx* ctx, DevBuf& b, size_t bytes, bool zero = false) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return DPPX_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  ++ctx->alloc_gen;  // (invalidates captured graphs, see host_single_graph)
  const size_t sz = std::max(bytes, static_cast<size_t>(256));
  CUDA_TRY(ctx, cudaMalloc(&b.p, sz));
  b.bytes = sz;
  if (zero) CUDA_TRY(ctx, cudaMemset(b.p, 0, sz));
  return DPPX_OK;
}

cudaEvent_t get_event(dppx_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void timing_begin(dppx_ctx* ctx, int family, PendingTiming* pt) {
  ctx->kstats.launches[family] += 1;
  pt->family = family;
  pt->start = pt->stop = nullptr;
  if (!ctx->timing) return;
  pt->start = get_event(ctx);
  pt->stop = get_event(ctx);
  cudaEventRecord(pt->start, ctx->stream);
}

void timing_end(dppx_ctx* ctx, PendingTiming* pt) {
  if (!pt->start) return;
  cudaEventRecord(pt->stop, ctx->stream);
  ctx->pending.push_back(*pt);
}

void collect_timings(dppx_ctx* ctx) {
  for (auto& pt : ctx->pending) {
    float ms = 0.f;
    cudaEventSynchronize(pt.stop);
    if (cudaEventElapsedTime(&ms, pt.start, pt.stop) == cudaSuccess)
      ctx->kstats.device_ms[pt.family] += ms;
    ctx->event_pool.push_back(pt.start);
    ctx->event_pool.push_back(pt.stop);
  }
  ctx->pending.clear();
}

// ---- TMA tensor maps ---------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// F frames x M rows x (row_bytes / 8) u64 elements, box (box_bytes / 8) x rows x 1.
bool encode_frames_map(CUtensorMap* m, const void* base, int64_t row_bytes, int M, int F,
                       int64_t pitch, int64_t fstride, int box_bytes, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc || row_bytes < 16) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(row_bytes / 8), static_cast<cuuint64_t>(M),
                              static_cast<cuuint64_t>(F)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(fstride)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_bytes / 8), static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output rows for the TMA store maps: N*C bytes rounded down to 16 (the < 16
// byte tail is stored by threads; the TMA unit moves whole 16-byte granules,
// so an extent that ends mid-granule -- an odd number of 8-byte elements --
// would let a box store write up to 8 bytes past the row: measured, and
// pinned by tests/test_gpu_parity.py::test_default_stores_are_window_safe),
// or, when the caller declared the pitch
// padding scratch (dppx_ctx_set_out_pad_scratch), N*C rounded up to whole
// 32-byte sectors within the pitch: every row then ends in a full sector, with
// no partial-sector DRAM writes and no thread-stored tail (CelebA 178 x 218:
// K2 3.38 -> 1.63 ms, K1 80 -> 98 % of measured HBM; profiles/r01m_*).
int64_t out_map_row_bytes(const dppx_ctx* ctx, int64_t row_bytes, int64_t opitch) {
  if (ctx->out_pad_scratch) {
    const int64_t r = std::min<int64_t>(opitch, (row_bytes + 31) / 32 * 32) / 16 * 16;
    if (r >= row_bytes) return r;
  }
  // (DPPX_TAIL32=1: A/B knob, extent down to whole 32-byte sectors so the
  // row's last, partial sector is written by threads alone)
  static const bool tail32 = std::getenv("DPPX_TAIL32") && std::getenv("DPPX_TAIL32")[0] == '1';
  if (tail32 && row_bytes >= 32) return row_bytes / 32 * 32;
  return row_bytes / 16 * 16;
}

// ---- validation mirroring the reference's throws ----------------------------
int geometry(dppx_ctx* ctx, int M, int N, int C, int F, int b, int n, BatchGeom* g,
             bool check_pad) {
  if (M < 1 || N < 1) return set_err(ctx, DPPX_ERR_INVALID, "malformed image (dimensions < 1)");
  if (C < 1 || C > 4) return set_err(ctx, DPPX_ERR_INVALID, "channels must be 1..4");
  if (F < 0) return set_err(ctx, DPPX_ERR_INVALID, "frames must be >= 0");
  dppx_geometry gg;
  if (dppx_grid_dims(M, N, b, &gg) != DPPX_OK)  // image.cpp:48-58
    return set_err(ctx, DPPX_ERR_INVALID,
                   b < 1 ? "grid_dims: grid side b must be >= 1"
                         : "grid_dims: grid side b exceeds both image dimensions");
  if (check_pad && (gg.pad_rows != 0 || gg.pad_cols != 0) &&
      (gg.pad_rows >= M || gg.pad_cols >= N))  // image.cpp:94-98
    return set_err(ctx, DPPX_ERR_INVALID,
                   "mirror_pad: padding exceeds image size, reflection source out of range "
                   "(use b <= min(M, N))");
  if (n < 1 || b % n != 0)
    return set_err(ctx, DPPX_ERR_INVALID, "invalid subgrid factor");
  if (static_cast<int64_t>(gg.grid_rows) * gg.grid_cols > 0x7FFFFFFFll)
    return set_err(ctx, DPPX_ERR_INVALID, "image too large: more than 2^31 - 1 grids per plane");
  g->M = M;
  g->N = N;
  g->C = C;
  g->F = F;
  g->b = b;
  g->n = n;
  g->sb = b / n;
  g->GR = gg.grid_rows;
  g->GC = gg.grid_cols;
  g->G = gg.grid_rows * gg.grid_cols;
  g->PR = gg.pad_rows;
  g->PC = gg.pad_cols;
  return DPPX_OK;
}

int check_desc(dppx_ctx* ctx, const dppx_frames_desc* d, bool need_mask, bool need_out) {
  if (!d) return set_err(ctx, DPPX_ERR_INVALID, "null frames descriptor");
  const int64_t row = static_cast<int64_t>(d->width) * d->channels;
  if (d->pitch < row || d->frame_stride < d->pitch * d->height)
    return set_err(ctx, DPPX_ERR_INVALID, "image pitch/frame_stride too small");
  if (need_mask && (d->mask_pitch < d->width || d->mask_frame_stride < d->mask_pitch * d->height))
    return set_err(ctx, DPPX_ERR_INVALID, "mask pitch/frame_stride too small");
  if (need_out && (d->out_pitch < row || d->out_frame_stride < d->out_pitch * d->height))
    return set_err(ctx, DPPX_ERR_INVALID, "out pitch/frame_stride too small");
  return DPPX_OK;
}

// Upload per-plane noise parameters; returns the device NoiseArgs.
int prepare_noise(dppx_ctx* ctx, const dppx_noise* nz, int planes, const double* dev_injected,
                  const BatchGeom& g, const dppx_privacy_params* pp, NoiseArgs* out,
                  cudaStream_t stream, DevBuf& dev_seeds, uint64_t*& pinned, size_t& pinned_n,
                  cudaEvent_t guard, bool record_guard) {
  out->kind = nz ? nz->kind : DPPX_NOISE_NONE;
  out->frame_base = nz ? nz->frame_base : 0;
  out->mixed_seeds = nullptr;
  out->injected = dev_injected;
  out->inline_count = 0;
  if (out->kind == DPPX_NOISE_NONE) return DPPX_OK;
  if (out->kind < 0 || out->kind > DPPX_NOISE_INJECTED)
    return set_err(ctx, DPPX_ERR_INVALID, "unknown noise kind");
  if (out->kind == DPPX_NOISE_INJECTED) {
    if (!dev_injected) return set_err(ctx, DPPX_ERR_INVALID, "injected noise pointer is null");
    return DPPX_OK;
  }
  // laplace_at: sigma must be > 0 (noise.cpp:112-116).
  if (!(pp->sigma > 0.0) || (g.n > 1 && !(pp->sigma_sub > 0.0)))
    return set_err(ctx, DPPX_ERR_INVALID, "laplace_at: sigma must be > 0");
  if (!nz->plane_seeds) return set_err(ctx, DPPX_ERR_INVALID, "plane_seeds is null");
  const size_t cnt = out->kind == DPPX_NOISE_KEYED ? static_cast<size_t>(planes) : 1;
  out->inline_count = 0;
  if (cnt <= static_cast<size_t>(kInlineSeeds)) {  // small batches: seeds in the params
    for (size_t i = 0; i < cnt; ++i)
      out->inline_seeds[i] =
          out->kind == DPPX_NOISE_KEYED ? mix64_h(nz->plane_seeds[i]) : nz->plane_seeds[i];
    out->inline_count = static_cast<int>(cnt);
    return DPPX_OK;
  }
  if (guard) cudaEventSynchronize(guard);  // previous upload from `pinned` has executed
  if (pinned_n < cnt) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_n = 0;
    CUDA_TRY(ctx, cudaMallocHost(reinterpret_cast<void**>(&pinned), cnt * sizeof(uint64_t) + 64));
    pinned_n = cnt;
  }
  for (size_t i = 0; i < cnt; ++i)
    pinned[i] = out->kind == DPPX_NOISE_KEYED ? mix64_h(nz->plane_seeds[i]) : nz->plane_seeds[i];
  if (int rc = ensure(ctx, dev_seeds, cnt * sizeof(uint64_t))) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(dev_seeds.p, pinned, cnt * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, stream));
  if (guard && record_guard) cudaEventRecord(guard, stream);
  out->mixed_seeds = static_cast<const uint64_t*>(dev_seeds.p);
  return DPPX_OK;
}

int ensure_scratch(dppx_ctx* ctx, const BatchGeom& g, int planes) {
  const size_t P = static_cast<size_t>(std::max(planes, 1));
  if (int rc = ensure(ctx, ctx->cellinfo, P * g.G * 4)) return rc;
  if (int rc = ensure(ctx, ctx->rowcnt, P * g.GR * 4)) return rc;
  if (int rc = ensure(ctx, ctx->rowprefix, P * g.GR * 4)) return rc;
  if (int rc = ensure(ctx, ctx->totals, P * 4)) return rc;
  if (int rc = ensure(ctx, ctx->counters, P * 4, /*zero=*/true)) return rc;
  if (int rc = ensure(ctx, ctx->status, 16, true)) return rc;
  return DPPX_OK;
}

struct VarianceSource {  // extension: classify cells by the frames' own variance
  const uint8_t* img = nullptr;
  int64_t pitch = 0, fstride = 0;
  double tau = 0.0;
};

int classify(dppx_ctx* ctx, const BatchGeom& g, int planes, bool from_payload, const uint8_t* mask,
             int64_t mpitch, int64_t mfstride, uint8_t* payload, const uint8_t* payload_in,
             int64_t pstride, uint32_t* payload_len, const uint32_t* in_len,
             const VarianceSource* var = nullptr, bool mask_bits = false,
             int64_t plen_limit = -1) {
  ClassifyArgs a{};
  a.g = g;
  a.planes = planes;
  a.from_payload = from_payload ? 1 : 0;
  if (var) {
    a.from_payload = 2;
    a.img = var->img;
    a.pitch = var->pitch;
    a.fstride = var->fstride;
    a.var_tau = var->tau;
    a.img_vec4 = (reinterpret_cast<uintptr_t>(var->img) & 3) == 0 && var->pitch % 4 == 0 &&
                 var->fstride % 4 == 0 && (g.b * g.C) % 4 == 0;
  }
  a.mask = mask;
  a.mpitch = mpitch;
  a.mfstride = mfstride;
  a.vec = 1;
  a.mask_bits = mask_bits ? 1 : 0;
  a.band = 0;
  if (!from_payload && !var && mask_bits && g.b >= 48) a.band = 2;  // bits, large b: per-(cell, row) popc
  if (!from_payload && !var && !mask_bits) {
    const bool al16 = aligned16(mask) && mpitch % 16 == 0 && mfstride % 16 == 0;
    if (g.b % 16 == 0 && al16) a.vec = 16;
    else if (g.b % 4 == 0 && (reinterpret_cast<uintptr_t>(mask) & 3) == 0 && mpitch % 4 == 0 &&
             mfstride % 4 == 0)
      a.vec = 4;
    // Grid sides without a per-cell vector path: band column sums.
    const bool per_cell_vec = (a.vec == 16 && (g.b == 16 || g.b == 32)) ||
                              (a.vec == 4 && (g.b == 4 || g.b == 8));
    if (!per_cell_vec && g.b >= 4 && g.b <= 257 &&
        static_cast<int64_t>(g.GC) * g.b * 4 <= 160 * 1024) {
      a.band = 1;
      a.vec = al16 ? 16 : 1;
    }
  }
  a.payload = payload;
  a.payload_in = payload_in;
  a.pstride = pstride;
  a.plen_limit = plen_limit < 0 ? pstride : plen_limit;
  a.payload_len = payload_len;
  a.in_len = in_len;
  a.cellinfo = static_cast<uint32_t*>(ctx->cellinfo.p);
  a.rowcnt = static_cast<uint32_t*>(ctx->rowcnt.p);
  a.rowprefix = static_cast<uint32_t*>(ctx->rowprefix.p);
  a.totals = static_cast<uint32_t*>(ctx->totals.p);
  a.counters = static_cast<uint32_t*>(ctx->counters.p);
  a.status = static_cast<int*>(ctx->status.p);
  a.area = static_cast<double>(g.b) * g.b;
  a.inv_area_pow2 = (g.b & (g.b - 1)) == 0 ? 1.0 / a.area : 0.0;  // exact: b = 2^k
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_CLASSIFY, &pt);
  CUDA_TRY(ctx, launch_classify(a, ctx->stream));
  timing_end(ctx, &pt);
  return DPPX_OK;
}

constexpr int kNoFusedPath = -1;  // internal: fused variance K1 not applicable

// K0 mode 3: the fused variance K1's per-cell flags -> slots, S, lengths and
// the 1.0f / 0.0f mask means of every channel payload.
int classify_flags(dppx_ctx* ctx, const BatchGeom& g, const uint8_t* flags, uint8_t* payload,
                   int64_t pstride, uint32_t* payload_len) {
  ClassifyArgs a{};
  a.g = g;
  a.planes = g.F;
  a.from_payload = 3;
  a.flags = flags;
  a.vec = 1;
  a.payload = payload;
  a.pstride = pstride;
  a.payload_len = payload_len;
  a.cellinfo = static_cast<uint32_t*>(ctx->cellinfo.p);
  a.rowcnt = static_cast<uint32_t*>(ctx->rowcnt.p);
  a.rowprefix = static_cast<uint32_t*>(ctx->rowprefix.p);
  a.totals = static_cast<uint32_t*>(ctx->totals.p);
  a.counters = static_cast<uint32_t*>(ctx->counters.p);
  a.status = static_cast<int*>(ctx->status.p);
  a.area = static_cast<double>(g.b) * g.b;
  a.inv_area_pow2 = (g.b & (g.b - 1)) == 0 ? 1.0 / a.area : 0.0;  // exact: b = 2^k
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_CLASSIFY, &pt);
  CUDA_TRY(ctx, launch_classify(a, ctx->stream));
  timing_end(ctx, &pt);
  return DPPX_OK;
}

// K1 (fast, TMA-staged) when the geometry and alignment allow, else K1g.
// With a.var_flags set (fused variance), only the staged VAR kernel qualifies:
// returns kNoFusedPath without launching anything when it does not apply.
int run_stats(dppx_ctx* ctx, StatsArgs& a) {
  const BatchGeom& g = a.g;
  if (a.row_count == 0 || g.F == 0) return DPPX_OK;
  StatsKernel k = nullptr;
  const bool aligned = aligned16(a.img) && a.pitch % 16 == 0 && a.fstride % 16 == 0 &&
                       (!a.out || (aligned16(a.out) && a.opitch % 16 == 0 && a.ofstride % 16 == 0));
  PendingTiming pt;
  CUtensorMap tin{}, tout{};
  const int tile = stats_tile_px_for(g.b, a.adaptive != 0);
  const int64_t row_bytes = static_cast<int64_t>(g.N) * g.C;
  // Narrow frames: pack several padded frame rows side by side in one tile.
  const int padded_px = g.GC * g.b;
  const int64_t stage_bytes = static_cast<int64_t>(g.b) * tile * g.C;
  a.pack = 1;
  a.slot_px = tile;
  const bool var = a.var_flags != nullptr;
  // (slots are whole 16-byte granules wide: a padded row of 184 px x 3 takes a
  // 192-px slot; the lanes past the last cell idle, the TMA box's bytes past
  // the row are zero-filled on load and clipped on store)
  static const bool slot16 = !(std::getenv("DPPX_SLOT16") && std::getenv("DPPX_SLOT16")[0] == '0');
  const int slot_w = (padded_px * g.C) % 16 == 0 ? padded_px : (slot16 ? round_up(padded_px, 16) : 0);
  if (!var && slot_w > 0 && 2 * slot_w <= tile) {
    const int64_t stride = round_up(static_cast<int64_t>(g.b) * slot_w * g.C, 128);
    const int pk = static_cast<int>(std::min<int64_t>(tile / slot_w, stage_bytes / stride));
    if (pk >= 2) {
      a.pack = pk;
      a.slot_px = slot_w;
    }
  }
  a.slot_stride = static_cast<int>(round_up(static_cast<int64_t>(g.b) * a.slot_px * g.C, 128));
  k = var ? select_stats_kernel_var(g.C, g.b, g.n)
          : select_stats_kernel(g.C, g.b, g.n, a.adaptive != 0, a.pack > 1);
  if (!k && a.pack > 1) {  // no packed instantiation for this (b, n): one frame per tile
    a.pack = 1;
    a.slot_px = tile;
    a.slot_stride = static_cast<int>(round_up(static_cast<int64_t>(g.b) * a.slot_px * g.C, 128));
    k = select_stats_kernel(g.C, g.b, g.n, a.adaptive != 0, false);
  }
  // Uniform b = 4 on wide frames: two cell rows (an 8-row band) per unit.
  static const bool rows2_off = std::getenv("DPPX_NO_ROWS2") != nullptr;  // A/B knob
  int rpu = 1;
  if (k && !var && !a.adaptive && g.b == 4 && a.pack == 1 && a.row_begin == 0 && a.row_count == g.GR &&
      g.M >= 16 && !rows2_off && !a.partial_borders) {
    if (StatsKernel k2 = select_uniform_b4_rows2(g.C)) {
      k = k2;
      rpu = 2;
    }
  }
  if (ctx->force_rows) {  // zero-copy call: k1z when the shape allows, else K1r
    if (!var) {
      static const int zc_unit = std::getenv("DPPX_ZC_UNIT") ? std::atoi(std::getenv("DPPX_ZC_UNIT")) : 6144;
      static const int zc_ctas = std::getenv("DPPX_ZC_CTAS") ? std::atoi(std::getenv("DPPX_ZC_CTAS")) : 0;
      bool ok = false;
      CUDA_TRY(ctx, launch_stats_zc(a, zc_unit, zc_ctas, ctx->sms, ctx->stream, &ok, true));
      if (ok) {
        timing_begin(ctx, DPPX_K_ZEROCOPY, &pt);
        CUDA_TRY(ctx, launch_stats_zc(a, zc_unit, zc_ctas, ctx->sms, ctx->stream, &ok, false));
        timing_end(ctx, &pt);
        return DPPX_OK;
      }
    }
    k = nullptr;
  }
  a.row_slack = a.pitch >= round_up(row_bytes, 16) ? 1 : 0;
  const int box_bytes = a.slot_px * g.C;
  // Input rows: the tensor's inner extent is rounded UP to 8 bytes when the
  // pitch has slack (the stray bytes past N*C are overwritten by the mirror
  // fill), so no row tail has to be gathered from global memory.
  // (Whole 16-byte granules, like the output maps: a load extent ending
  // mid-granule could touch up to 8 bytes past the row.)
  const int64_t in_row = a.row_slack ? round_up(row_bytes, 16) : row_bytes / 16 * 16;
  bool maps = k && aligned && g.F > 0 && box_bytes / 8 <= 256 && g.b <= 256 &&
              (a.pack == 1 || static_cast<int64_t>(a.pack) * a.slot_stride <= stage_bytes) &&
              encode_frames_map(&tin, a.img, in_row, g.M, g.F, a.pitch, a.fstride, box_bytes, g.b * rpu);
  if (maps && a.out)
    maps = encode_frames_map(&tout, a.out, out_map_row_bytes(ctx, row_bytes, a.opitch), g.M, g.F, a.opitch, a.ofstride,
                              box_bytes, g.b * rpu);
  if (maps && !a.out) tout = tin;
  if (maps) {
    a.tensor_in_bytes = static_cast<int>(in_row);
    a.tensor_out_bytes = static_cast<int>(a.out ? out_map_row_bytes(ctx, row_bytes, a.opitch) : row_bytes / 16 * 16);
    a.tiles_per_row = a.pack > 1 ? 1 : (padded_px + tile - 1) / tile;
    const int64_t groups = (g.F + a.pack - 1) / a.pack;
    const int64_t bands = (a.row_count + rpu - 1) / rpu;  // units per frame column (rpu cell rows each)
    const int64_t units = groups * bands * a.tiles_per_row;
    if (units > 0x7FFFFFFF) return set_err(ctx, DPPX_ERR_INVALID, "batch too large for one launch");
    a.units = static_cast<int>(units);
    a.div_tiles = make_fastdiv(static_cast<uint32_t>(a.tiles_per_row));
    a.div_rows = make_fastdiv(static_cast<uint32_t>(bands));
    // (128-byte aligned stages: equal to b * tile * C for every b % 4 == 0 kernel)
    const size_t stage = static_cast<size_t>(round_up(static_cast<int64_t>(g.b) * rpu * tile * g.C, 128));
    // Two stages: measured best for every shape on B200 (a 2-deep ring per CTA
    // with 4 CTAs/SM at b = 16 beats 3-4 deep rings with fewer CTAs; see
    // profiles/r01_stage_sweep.md).
    // (uniform b = 4 with two-row units: 12 KB stages, a 3-deep ring measured
    // best -- 0.354 -> 0.329 ms per 120 x 1080p RGB, profiles/r02dd_b4_stages.txt)
    int S = rpu > 1 ? 3 : 2;
    if (const char* env = std::getenv("DPPX_STAGES"))  // tuning knob (2..4)
      S = std::max(2, std::min(stats_max_stages(), std::atoi(env)));
    a.stages = S;
    const size_t smem = stage * S;
    const auto key = std::make_pair(reinterpret_cast<const void*>(k), smem);
    auto it = ctx->occupancy.find(key);
    int per_sm = 0;
    if (it == ctx->occupancy.end()) {
      CUDA_TRY(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
      CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, stats_threads(),
                                                                  smem));
      ctx->occupancy[key] = per_sm;
    } else {
      per_sm = it->second;
    }
    const int grid = static_cast<int>(std::min<int64_t>(units, static_cast<int64_t>(std::max(per_sm, 1)) * ctx->sms));
    // Zeroed once at allocation; each launch's last producer resets it.
    if (int rc = ensure(ctx, ctx->work, 16, /*zero=*/true)) return rc;
    a.work_counter = static_cast<int*>(ctx->work.p);
    timing_begin(ctx, DPPX_K_STATS, &pt);
    CUDA_TRY(ctx, launch_stats_tma(k, tin, tout, a, grid, smem, ctx->stream));
  } else {
    if (var) return kNoFusedPath;  // caller takes the 2-pass variance path
    // Other grid sides (b = 12, 24, 30, 40, 64, 128 ...): row-streaming K1r.
    const int rsm = a.partial_borders ? 0 : rows_smem_bytes(g);
    const int64_t units = static_cast<int64_t>(g.F) * a.row_count;
    static const bool no_px = std::getenv("DPPX_NO_K1P") != nullptr;
    if (g.b <= 2 && (g.C == 1 || g.C == 3) && !a.partial_borders && !no_px) {
      // b = 1, 2: K1p, one thread per cell, all loops compile-time
      timing_begin(ctx, DPPX_K_GENERIC, &pt);
      if (g.F > 0) CUDA_TRY(ctx, launch_stats_px(a, ctx->stream));
    } else if (rsm > 0 && units <= 0x7FFFFFFF && !std::getenv("DPPX_NO_ROWS")) {
      a.units = static_cast<int>(units);
      a.div_rows = make_fastdiv(static_cast<uint32_t>(a.row_count));
      timing_begin(ctx, DPPX_K_ROWS, &pt);
      CUDA_TRY(ctx, launch_stats_rows(a, static_cast<size_t>(rsm), ctx->stream));
    } else {
      timing_begin(ctx, DPPX_K_GENERIC, &pt);
      if (g.F > 0) CUDA_TRY(ctx, launch_stats_generic(a, ctx->stream));
    }
  }
  timing_end(ctx, &pt);
  return DPPX_OK;
}

int check_ctx(dppx_ctx* ctx) {
  if (!ctx) return DPPX_ERR_INVALID;
  CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  return DPPX_OK;
}

int check_params(dppx_ctx* ctx, const dppx_privacy_params* p, bool adaptive) {
  if (!p) return set_err(ctx, DPPX_ERR_INVALID, "null privacy params");
  if (!adaptive && p->n != 1)
    return set_err(ctx, DPPX_ERR_INVALID, "pixelize_parallel: requires n == 1");
  if (adaptive && (p->n < 1 || p->b % p->n != 0 || p->subgrid_side * p->n != p->b))
    return set_err(ctx, DPPX_ERR_INVALID, "pixelize_adaptive: invalid subgrid factor");
  return DPPX_OK;
}

// Less common options of pixelize_dev.
struct PixOpts {
  bool partial = false;          // Algorithm 1 (pixelize_reference)
  double var_tau = std::nan("");  // set: variance classification (extension)
  bool mask_bits = false;        // mask rows are packed bits (host pipeline transport)
  int row_begin = 0;             // grid rows [row_begin, row_begin + row_count) only
  int row_count = -1;            // -1: all rows
  bool classify = true;          // adaptive: run K0 (false: a previous band already did)
  const uint64_t* seeds_dev = nullptr;  // KEYED: mixed plane seeds already in device memory
                                        // (graph replays: nothing baked into kernel params)
};

// Device-pointer core of both pixelize entry points.
int pixelize_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img, const uint8_t* mask,
                 const dppx_privacy_params* pp, const dppx_noise* nz, const double* dev_injected,
                 uint8_t* stats, int64_t sstride, uint32_t* payload_len, uint8_t* out,
                 bool adaptive, DevBuf& dev_seeds, uint64_t*& pinned, size_t& pinned_n,
                 cudaEvent_t guard, bool record_guard, const PixOpts& o = PixOpts()) {
  const bool partial = o.partial;
  const double var_tau = o.var_tau;
  const bool mask_bits = o.mask_bits;
  BatchGeom g;
  if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, pp->b,
                        adaptive ? pp->n : 1, &g, !partial))
    return rc;
  if (d->frames == 0) return DPPX_OK;
  const bool by_variance = adaptive && !std::isnan(var_tau);
  if (!img || !stats || (adaptive && !mask && !by_variance))
    return set_err(ctx, DPPX_ERR_INVALID, "null image/statistics/mask pointer");
  if (by_variance && !(var_tau >= 0.0))
    return set_err(ctx, DPPX_ERR_INVALID, "variance threshold must be >= 0");
  if (adaptive) {
    const size_t cap = dppx_adaptive_payload_capacity(g.M, g.N, g.b, g.n);
    if (sstride < static_cast<int64_t>(cap) || sstride % 4 != 0)
      return set_err(ctx, DPPX_ERR_INVALID, "payload_stride must be >= %zu and a multiple of 4",
                     cap);
  }
  StatsArgs a{};
  a.g = g;
  a.adaptive = adaptive ? 1 : 0;
  a.img = img;
  a.pitch = d->pitch;
  a.fstride = d->frame_stride;
  a.out = out;
  a.opitch = d->out_pitch;
  a.ofstride = d->out_frame_stride;
  a.stats = stats;
  a.sstride = sstride;
  a.area = static_cast<double>(g.b) * g.b;
  a.sub_area = static_cast<double>(g.sb) * g.sb;
  a.sigma = pp->sigma;
  a.sigma_sub = adaptive ? pp->sigma_sub : pp->sigma;
  a.exact_noise = ctx->exact_noise ? 1 : 0;
  a.partial_borders = partial ? 1 : 0;
  a.row_begin = o.row_count < 0 ? 0 : o.row_begin;
  a.row_count = o.row_count < 0 ? g.GR : o.row_count;
  if (a.row_begin < 0 || a.row_count < 0 || a.row_begin + a.row_count > g.GR)
    return set_err(ctx, DPPX_ERR_INVALID, "row band out of range");
  if (o.seeds_dev && nz && nz->kind == DPPX_NOISE_KEYED) {
    if (!(pp->sigma > 0.0) || (g.n > 1 && !(pp->sigma_sub > 0.0)))
      return set_err(ctx, DPPX_ERR_INVALID, "laplace_at: sigma must be > 0");
    a.noise = NoiseArgs{};
    a.noise.kind = DPPX_NOISE_KEYED;
    a.noise.mixed_seeds = o.seeds_dev;
  } else if (int rc = prepare_noise(ctx, nz, g.F * g.C, dev_injected, g, pp, &a.noise, ctx->stream,
                                    dev_seeds, pinned, pinned_n, guard, record_guard)) {
    return rc;
  }
  const char* fused_env = std::getenv("DPPX_VAR_FUSED");  // A/B knob: "0" = 2-pass path
  if (by_variance && !partial && !(fused_env && fused_env[0] == '0')) {
    // Fused: K1 classifies each cell by its own variance while summing (one
    // read of the frames), stages the statistics per cell; K0 (mode 3) turns
    // the flags into slots and k_gather_stage compacts the payloads.
    if (int rc = ensure_scratch(ctx, g, g.F)) return rc;
    const int64_t nn = static_cast<int64_t>(g.n) * g.n;
    const int64_t stage_cx = round_up(static_cast<int64_t>(g.G), 16);
    const int64_t stage_stride = round_up(stage_cx + static_cast<int64_t>(g.G) * nn, 16);
    if (int rc = ensure(ctx, ctx->var_flags, static_cast<size_t>(g.F) * g.G)) return rc;
    if (int rc = ensure(ctx, ctx->var_stage, static_cast<size_t>(stage_stride) * g.F * g.C)) return rc;
    StatsArgs v = a;
    v.var_tau = var_tau;
    v.var_flags = static_cast<uint8_t*>(ctx->var_flags.p);
    v.stage = static_cast<uint8_t*>(ctx->var_stage.p);
    v.stage_stride = stage_stride;
    v.stage_cx = stage_cx;
    const int rc = run_stats(ctx, v);
    if (rc != kNoFusedPath) {
      if (rc) return rc;
      if (int rc2 = classify_flags(ctx, g, v.var_flags, stats, sstride, payload_len)) return rc2;
      GatherArgs ga{};
      ga.g = g;
      ga.stage = v.stage;
      ga.stage_stride = stage_stride;
      ga.stage_cx = stage_cx;
      ga.cellinfo = static_cast<const uint32_t*>(ctx->cellinfo.p);
      ga.rowprefix = static_cast<const uint32_t*>(ctx->rowprefix.p);
      ga.totals = static_cast<const uint32_t*>(ctx->totals.p);
      ga.payload = stats;
      ga.pstride = sstride;
      PendingTiming pt;
      timing_begin(ctx, DPPX_K_AUX, &pt);
      CUDA_TRY(ctx, launch_gather_stage(ga, ctx->stream));
      timing_end(ctx, &pt);
      return DPPX_OK;
    }
  }
  if (adaptive && !o.classify) {  // a previous row band of this call ran K0
    a.cellinfo = static_cast<const uint32_t*>(ctx->cellinfo.p);
    a.rowprefix = static_cast<const uint32_t*>(ctx->rowprefix.p);
    a.totals = static_cast<const uint32_t*>(ctx->totals.p);
  } else if (adaptive) {
    if (int rc = ensure_scratch(ctx, g, g.F)) return rc;
    VarianceSource vs{img, d->pitch, d->frame_stride, var_tau};
    if (int rc = classify(ctx, g, g.F, false, mask, d->mask_pitch, d->mask_frame_stride, stats,
                          nullptr, sstride, payload_len, nullptr, by_variance ? &vs : nullptr,
                          mask_bits))
      return rc;
    a.cellinfo = static_cast<const uint32_t*>(ctx->cellinfo.p);
    a.rowprefix = static_cast<const uint32_t*>(ctx->rowprefix.p);
    a.totals = static_cast<const uint32_t*>(ctx->totals.p);
  }
  if (partial) {  // Algorithm 1 has no staged fast path (a bench/oracle row)
    PendingTiming pt;
    timing_begin(ctx, DPPX_K_GENERIC, &pt);
    CUDA_TRY(ctx, launch_stats_generic(a, ctx->stream));
    timing_end(ctx, &pt);
    return DPPX_OK;
  }
  return run_stats(ctx, a);
}

int expand_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* stats, int64_t sstride,
               const uint32_t* in_len, int b, int n, uint8_t* out, bool adaptive,
               int64_t caller_stride = -1) {
  if (caller_stride < 0) caller_stride = sstride;
  BatchGeom g;
  if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, b, adaptive ? n : 1, &g,
                        false)) {
    // reassemble reports a bad subgrid factor as RecordError(corrupt_record)
    // (adaptive.cpp:188-191); dimension problems stay invalid_argument.
    if (adaptive && (n < 1 || (b >= 1 && b % n != 0)) && b >= 1 &&
        b <= std::max(d->height, d->width))
      return set_err(ctx, DPPX_ERR_CORRUPT, "reassemble: subgrid factor does not divide grid side");
    return rc;
  }
  if (d->frames == 0) return DPPX_OK;
  if (!stats || !out) return set_err(ctx, DPPX_ERR_INVALID, "null statistics/output pointer");
  ExpandArgs e{};
  e.g = g;
  e.adaptive = adaptive ? 1 : 0;
  e.stats = stats;
  e.sstride = sstride;
  e.out = out;
  e.opitch = d->out_pitch;
  e.ofstride = d->out_frame_stride;
  if (adaptive) {
    if (sstride < 4ll * g.G + 4 || sstride % 4 != 0)
      return set_err(ctx, DPPX_ERR_INVALID, "payload_stride too small or not a multiple of 4");
    // The shortest valid payload (every cell simple) is 5G + 4 bytes: a slot
    // that cannot hold it holds no valid payload (adaptive.cpp:192-210).
    if (caller_stride < 5ll * g.G + 4)
      return set_err(ctx, DPPX_ERR_CORRUPT, "reassemble: payload shorter than its mask means imply");
    const int P = g.F * g.C;
    if (int rc = ensure_scratch(ctx, g, P)) return rc;
    if (int rc = classify(ctx, g, P, true, nullptr, 0, 0, nullptr, stats, sstride, nullptr, in_len,
                          nullptr, false, caller_stride))
      return rc;
    e.cellinfo = static_cast<const uint32_t*>(ctx->cellinfo.p);
    e.rowprefix = static_cast<const uint32_t*>(ctx->rowprefix.p);
    e.totals = static_cast<const uint32_t*>(ctx->totals.p);
  }
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_EXPAND, &pt);
  // Fast path: staged tile, TMA box stores (aligned output, the K1 grid sides,
  // C in {1,3}); narrow frames packed side by side.
  int tile = stats_tile_px_for(g.b, adaptive);
  const int64_t row_bytes = static_cast<int64_t>(g.N) * g.C;
  const int padded_px = g.GC * g.b;
  int64_t stage_bytes = static_cast<int64_t>(g.b) * tile * g.C;
  e.pack = 1;
  e.slot_px = tile;
  const int tile0 = tile;
  const int64_t stage0 = stage_bytes;
  // (slots of whole 16-byte granules, as K1: 184 px x 3 -> 192-px slots)
  static const bool slot16 = !(std::getenv("DPPX_SLOT16") && std::getenv("DPPX_SLOT16")[0] == '0');
  const int slot_w = (padded_px * g.C) % 16 == 0 ? padded_px : (slot16 ? static_cast<int>(round_up(padded_px, 16)) : 0);
  if (tile == stats_tile_px() && slot_w > 0 && 2 * slot_w <= expand_packed_tile_px()) {
    // Narrow frames: frame slots side by side in a wider (1024-px) tile.
    const int ptile = expand_packed_tile_px();
    const int64_t pstage = static_cast<int64_t>(g.b) * ptile * g.C;
    const int64_t stride = round_up(static_cast<int64_t>(g.b) * slot_w * g.C, 128);
    const int pk = static_cast<int>(std::min<int64_t>(ptile / slot_w, pstage / stride));
    if (pk >= 2) {
      e.pack = pk;
      e.slot_px = slot_w;
      tile = ptile;
      stage_bytes = pstage;
    }
  }
  e.slot_stride = static_cast<int>(round_up(static_cast<int64_t>(g.b) * e.slot_px * g.C, 128));
  // b = 32 / 64 wide frames: each band split into units of b/split rows (a
  // fraction of the smem per CTA, so more CTAs per SM hide the statistics
  // loads; DPPX_K2_SPLIT=1 disables, 2 / 4 force a split)
  // Measured (tools/k2_split_sweep.sh, profiles/r02ii_k2_split.txt): 16-row
  // units are best for every b = 32 / 64 case but b = 32 n = 4 (8 rows).
  static const int split_env = std::getenv("DPPX_K2_SPLIT") ? std::atoi(std::getenv("DPPX_K2_SPLIT")) : 0;
  ExpandKernel k = nullptr;
  int unit_rows = g.b;
  if (e.pack == 1 && (g.b == 32 || g.b == 64)) {
    const int want = split_env > 0 ? split_env : (g.b == 32 && g.n == 4 ? 4 : g.b / 16);
    for (int sp : {want, 2})
      if (!k && sp > 1 && (k = select_expand_kernel(g.C, g.b, g.n, adaptive, false, sp))) unit_rows = g.b / sp;
  }
  if (!k) k = select_expand_kernel(g.C, g.b, g.n, adaptive, e.pack > 1, 1);
  if (!k && e.pack > 1) {  // no packed instantiation for this (b, n): one frame per tile
    e.pack = 1;
    e.slot_px = tile0;
    tile = tile0;
    stage_bytes = stage0;
    e.slot_stride = static_cast<int>(round_up(static_cast<int64_t>(g.b) * e.slot_px * g.C, 128));
    k = select_expand_kernel(g.C, g.b, g.n, adaptive, false, 1);
  }
  if (unit_rows != g.b) stage_bytes = static_cast<int64_t>(unit_rows) * tile * g.C;
  e.stage_bytes = static_cast<int>(round_up(stage_bytes, 128));
  CUtensorMap tout{};
  const bool aligned = aligned16(out) && e.opitch % 16 == 0 && e.ofstride % 16 == 0;
  const int box_bytes = e.slot_px * g.C;
  if (k && aligned && box_bytes / 8 <= 256 &&
      encode_frames_map(&tout, out, out_map_row_bytes(ctx, row_bytes, e.opitch), g.M, g.F, e.opitch, e.ofstride,
                        box_bytes, unit_rows)) {
    e.tiles_per_row = e.pack > 1 ? 1 : (padded_px + tile - 1) / tile;
    e.tensor_out_bytes = static_cast<int>(out_map_row_bytes(ctx, row_bytes, e.opitch));
    e.div_tiles = make_fastdiv(static_cast<uint32_t>(e.tiles_per_row));
    e.div_rows = make_fastdiv(static_cast<uint32_t>(g.GR));
    const int64_t groups = (g.F + e.pack - 1) / e.pack;
    const int64_t units = groups * g.GR * e.tiles_per_row * (g.b / unit_rows);
    if (units > 0x7FFFFFFF) return set_err(ctx, DPPX_ERR_INVALID, "batch too large for one launch");
    e.units = static_cast<int>(units);
    // One unit per CTA (many short CTAs hide the statistics-load latency
    // better than a persistent double-buffered loop: measured 0.69 vs 0.88 ms
    // on 600 x 1080p); the kernel loops only if the grid is capped.
    const size_t smem = static_cast<size_t>(e.stage_bytes);
    const auto key = std::make_pair(reinterpret_cast<const void*>(k), smem);
    auto it = ctx->occupancy.find(key);
    int per_sm = 0;
    if (it == ctx->occupancy.end()) {
      CUDA_TRY(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
      CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, stats_tile_px() / 4, smem));
      ctx->occupancy[key] = per_sm;
    } else {
      per_sm = it->second;
    }
    (void)per_sm;
    CUDA_TRY(ctx, launch_expand_tma(k, tout, e, e.units, smem, ctx->stream));
  } else if (g.b <= 2 && (g.C == 1 || g.C == 3) && !std::getenv("DPPX_NO_K2P")) {
    CUDA_TRY(ctx, launch_expand_px(e, ctx->stream));  // b = 1, 2: K2p
  } else if (const int rsm = rows_smem_bytes(g);
             rsm > 0 && static_cast<int64_t>(g.F) * g.GR <= 0x7FFFFFFF && !std::getenv("DPPX_NO_ROWS")) {
    CUDA_TRY(ctx, launch_expand_rows(e, static_cast<size_t>(rsm), ctx->stream));
  } else {
    CUDA_TRY(ctx, launch_expand(e, ctx->stream));
  }
  timing_end(ctx, &pt);
  return DPPX_OK;
}

int read_status(dppx_ctx* ctx) {
  if (!ctx->status.p) return DPPX_OK;
  int st = 0;
  CUDA_TRY(ctx, cudaMemcpy(&st, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (st != 0) {
    CUDA_TRY(ctx, cudaMemset(ctx->status.p, 0, sizeof(int)));
    return set_err(ctx, st, "reassemble: payload inconsistent (simple count or length mismatch)");
  }
  return DPPX_OK;
}

// ---- host pipeline -----------------------------------------------------------
// Copy Fk frames of M rows x width bytes between pitched layouts with as few
// copy operations as the strides allow (one linear copy when both sides are
// dense, one 2-D copy when frames are row-contiguous, else one per frame).
cudaError_t copy_frames(void* dst, int64_t dpitch, int64_t dfs, const void* src, int64_t spitch,
                        int64_t sfs, int64_t width, int M, int Fk, cudaMemcpyKind kind,
                        cudaStream_t st) {
  auto* d = static_cast<uint8_t*>(dst);
  const auto* s = static_cast<const uint8_t*>(src);
  if (dpitch == width && spitch == width && dfs == width * M && sfs == width * M)
    return cudaMemcpyAsync(d, s, static_cast<size_t>(width) * M * Fk, kind, st);
  if (dfs == dpitch * M && sfs == spitch * M)
    return cudaMemcpy2DAsync(d, dpitch, s, spitch, width, static_cast<size_t>(M) * Fk, kind, st);
  for (int f = 0; f < Fk; ++f) {
    const cudaError_t e =
        cudaMemcpy2DAsync(d + f * dfs, dpitch, s + f * sfs, spitch, width, M, kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

enum class HostOp { Uniform, Adaptive, Broadcast, Reassemble, Reference, AdaptiveVariance };

// Page-locked (or device / managed) memory the DMA engines can read directly.
bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type != cudaMemoryTypeUnregistered;
}

int grow_pinned(dppx_ctx* ctx, uint8_t*& buf, size_t& have, size_t need) {
  if (have >= need) return DPPX_OK;
  if (buf) CUDA_TRY(ctx, cudaFreeHost(buf));
  buf = nullptr;
  have = 0;
  CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&buf), need, cudaHostAllocDefault));
  have = need;
  return DPPX_OK;
}

// Rows per pinned piece of a pageable transfer: ~4 MB (DPPX_PIECE_MB). Small
// enough that the two pieces cost little to pin on a context's first pageable
// call (2 x 16 MB took 14.6 ms, most of a batch runner's device setup), large
// enough that a piece's DMA (~80 us) dwarfs its copy and event overheads.
int64_t piece_rows(int64_t pitch) {
  static const int64_t bytes = [] {
    const char* e = std::getenv("DPPX_PIECE_MB");
    const long mb = e ? std::strtol(e, nullptr, 10) : 0;
    return (mb > 0 ? static_cast<int64_t>(mb) : int64_t{4}) << 20;
  }();
  return std::max<int64_t>(1, bytes / pitch);
}

// Host -> device copy of F frames (rows of `row` bytes). A pinned source is one
// DMA; a pageable one is cut into ~4 MB pieces of whole rows that host threads
// copy into two pinned buffers in turn, so the host copies overlap the DMA.
int h2d_frames(dppx_ctx* ctx, uint8_t* dst, int64_t dpitch, int64_t dfs, const uint8_t* src,
               int64_t spitch, int64_t sfs, int64_t row, int M, int F, cudaStream_t st) {
  if (host_pinned(src)) {
    CUDA_TRY(ctx, copy_frames(dst, dpitch, dfs, src, spitch, sfs, row, M, F, cudaMemcpyHostToDevice, st));
    return DPPX_OK;
  }
  if (!ctx->packer) ctx->packer = dppx::mask_packer_create(0);
  const int64_t rows = static_cast<int64_t>(F) * M;
  const int64_t per = piece_rows(dpitch);
  const bool linear = dfs == static_cast<int64_t>(M) * dpitch;  // dst row r at r * dpitch
  for (int s = 0; s < 2; ++s) {
    if (int rc = grow_pinned(ctx, ctx->piece[s], ctx->piece_n[s], static_cast<size_t>(per * dpitch)))
      return rc;
    if (!ctx->piece_ev[s]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->piece_ev[s], cudaEventDisableTiming));
  }
  int64_t r0 = 0;
  for (int k = 0; r0 < rows; ++k) {
    int64_t r1 = std::min(rows, r0 + per);
    if (!linear) r1 = std::min(r1, (r0 / M + 1) * M);  // pieces stay inside one frame
    const int s = k & 1;
    // the buffer's previous DMA (this call's piece k-2, or an earlier call's)
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->piece_ev[s]));
    uint8_t* buf = ctx->piece[s];
    dppx::pool_for(ctx->packer, r1 - r0, [&](int64_t a, int64_t b) {
      for (int64_t r = r0 + a; r < r0 + b; ++r)
        std::memcpy(buf + (r - r0) * dpitch, src + (r / M) * sfs + (r % M) * spitch, static_cast<size_t>(row));
    });
    uint8_t* d0 = dst + (r0 / M) * dfs + (r0 % M) * dpitch;
    const size_t bytes = static_cast<size_t>(r1 - r0 - 1) * dpitch + row;
    CUDA_TRY(ctx, cudaMemcpyAsync(d0, buf, bytes, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->piece_ev[s], st));
    r0 = r1;
  }
  return DPPX_OK;
}

// Device -> host copy of F frames into a caller buffer: one DMA when the
// destination is pinned; otherwise ~4 MB pieces land in the ctx's two pinned
// piece buffers in turn and host threads copy each piece out while the next
// one is in flight.
int d2h_frames(dppx_ctx* ctx, uint8_t* dst, int64_t dpitch, int64_t dfs, const uint8_t* src,
               int64_t spitch, int64_t sfs, int64_t row, int M, int F, cudaStream_t st) {
  if (host_pinned(dst)) {
    CUDA_TRY(ctx, copy_frames(dst, dpitch, dfs, src, spitch, sfs, row, M, F, cudaMemcpyDeviceToHost, st));
    return DPPX_OK;
  }
  if (!ctx->packer) ctx->packer = dppx::mask_packer_create(0);
  const int64_t rows = static_cast<int64_t>(F) * M;
  const int64_t per = piece_rows(spitch);
  for (int s = 0; s < 2; ++s) {
    if (int rc = grow_pinned(ctx, ctx->piece[s], ctx->piece_n[s], static_cast<size_t>(per * spitch))) return rc;
    if (!ctx->piece_ev[s]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->piece_ev[s], cudaEventDisableTiming));
  }
  const bool linear = sfs == static_cast<int64_t>(M) * spitch;
  int64_t pending_r0[2] = {-1, -1}, pending_r1[2] = {0, 0};
  auto drain = [&](int s) -> int {
    if (pending_r0[s] < 0) return DPPX_OK;
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->piece_ev[s]));
    const int64_t a0 = pending_r0[s], a1 = pending_r1[s];
    const uint8_t* buf = ctx->piece[s];
    dppx::pool_for(ctx->packer, a1 - a0, [&](int64_t x, int64_t y) {
      for (int64_t r = a0 + x; r < a0 + y; ++r)
        std::memcpy(dst + (r / M) * dfs + (r % M) * dpitch, buf + (r - a0) * spitch, static_cast<size_t>(row));
    });
    pending_r0[s] = -1;
    return DPPX_OK;
  };
  int64_t r0 = 0;
  for (int k = 0; r0 < rows; ++k) {
    int64_t r1 = std::min(rows, r0 + per);
    if (!linear) r1 = std::min(r1, (r0 / M + 1) * M);
    const int s = k & 1;
    if (int rc = drain(s)) return rc;  // the piece buffer's previous rows leave first
    const uint8_t* s0 = src + (r0 / M) * sfs + (r0 % M) * spitch;
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->piece[s], s0, static_cast<size_t>(r1 - r0 - 1) * spitch + row,
                                  cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaEventRecord(ctx->piece_ev[s], st));
    pending_r0[s] = r0;
    pending_r1[s] = r1;
    r0 = r1;
  }
  for (int k = 0; k < 2; ++k)
    if (int rc = drain(k)) return rc;
  return DPPX_OK;
}

// Single-frame host calls: there is no second frame to overlap with, so the
// frame is split into bands of grid rows. Band i's rows are copied in while
// band i-1 is computed and band i-2 is copied out (H2D, K1, D2H on three
// streams). Adaptive frames ship the whole mask first (K0 classifies the frame
// once, before band 0's K1); the statistics are copied out after the last
// band. Bands are in order on the input stream, so the mirrored rows a last
// band reads from its predecessor are always resident.
int host_pipeline_bands(dppx_ctx* ctx, bool adaptive, const dppx_frames_desc* d,
                        const BatchGeom& g, const uint8_t* img, const uint8_t* mask,
                        const dppx_privacy_params* pp, const dppx_noise* nz, uint8_t* stats,
                        int64_t sstride, uint32_t* lens, uint8_t* out, int nb) {
  const int C = g.C, M = g.M, N = g.N, b = g.b;
  const int64_t row = static_cast<int64_t>(N) * C;
  const int64_t dpitch = round_up(row, 16), dfs = dpitch * M;
  const int64_t dmpitch = round_up(N, 16), dmfs = dmpitch * M;
  const size_t cap = adaptive ? dppx_adaptive_payload_capacity(M, N, b, g.n) : g.G;
  const int64_t dstride = adaptive ? round_up(static_cast<int64_t>(cap), 16) : g.G;
  if (ensure(ctx, ctx->img[0], static_cast<size_t>(dfs))) return DPPX_ERR_OOM;
  if (out && ensure(ctx, ctx->out[0], static_cast<size_t>(dfs))) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->stats[0], static_cast<size_t>(dstride) * C)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->lens[0], sizeof(uint32_t) * C)) return DPPX_ERR_OOM;
  uint8_t* dimg = static_cast<uint8_t*>(ctx->img[0].p);
  uint8_t* dout = static_cast<uint8_t*>(ctx->out[0].p);
  uint8_t* dstats = static_cast<uint8_t*>(ctx->stats[0].p);
  uint32_t* dlens = static_cast<uint32_t*>(ctx->lens[0].p);
  cudaStream_t comp = ctx->stream;
  // The previous call's copies out of these buffers must be done.
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_in, ctx->out_done[0], 0));
  bool bits = false;
  uint8_t* dmask = nullptr;
  int64_t mp = dmpitch, mfs = dmfs;
  // The mask ships right after band 0's rows: packing it overlaps that copy.
  auto ship_mask = [&]() -> int {
    if (ensure(ctx, ctx->mask[0], static_cast<size_t>(dmfs))) return DPPX_ERR_OOM;
    dmask = static_cast<uint8_t*>(ctx->mask[0].p);
    if (ctx->mask_bits_mode == 1) {
      const int64_t wpr = dppx::mask_words_per_row(N);
      const size_t bytes = static_cast<size_t>(wpr) * 4 * M;
      if (!ctx->packer) ctx->packer = dppx::mask_packer_create(0);
      if (ctx->mbits_pinned_n[0] < bytes) {
        CUDA_TRY(ctx, cudaStreamSynchronize(ctx->s_in));
        if (ctx->mbits_pinned[0]) CUDA_TRY(ctx, cudaFreeHost(ctx->mbits_pinned[0]));
        ctx->mbits_pinned[0] = nullptr;
        ctx->mbits_pinned_n[0] = 0;
        CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->mbits_pinned[0]), bytes,
                                    cudaHostAllocDefault));
        ctx->mbits_pinned_n[0] = bytes;
      }
      CUDA_TRY(ctx, cudaEventSynchronize(ctx->in_done[0]));  // staging buffer free
      bits = dppx::pack_mask_bits(ctx->packer, mask, d->mask_pitch, d->mask_frame_stride, M, N, 1,
                                  ctx->mbits_pinned[0], wpr);
      if (bits) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dmask, ctx->mbits_pinned[0], bytes, cudaMemcpyHostToDevice,
                                      ctx->s_in));
        ctx->kstats.h2d_bytes += bytes;
        mp = wpr * 4;
        mfs = static_cast<int64_t>(bytes);
      }
    }
    if (!bits) {
      CUDA_TRY(ctx, cudaMemcpy2DAsync(dmask, dmpitch, mask, d->mask_pitch, N, M,
                                      cudaMemcpyHostToDevice, ctx->s_in));
      ctx->kstats.h2d_bytes += static_cast<uint64_t>(N) * M;
    }
    return DPPX_OK;
  };
  if (adaptive && ensure(ctx, ctx->mask[0], static_cast<size_t>(dmfs))) return DPPX_ERR_OOM;
  // Band sizes in grid rows (the last band keeps >= 2 rows for its reflections).
  int sizes[dppx_ctx::kMaxBands];
  {
    int left = g.GR;
    for (int i = 0; i < nb; ++i) {
      sizes[i] = left / (nb - i);
      left -= sizes[i];
    }
  }
  dppx_frames_desc dd = *d;
  dd.pitch = dpitch;
  dd.frame_stride = dfs;
  dd.mask_pitch = mp;
  dd.mask_frame_stride = mfs;
  dd.out_pitch = dpitch;
  dd.out_frame_stride = dfs;
  // DPPX_BAND_TRACE=1: print when each band's copies / kernels finished (timing events).
  static const bool trace = std::getenv("DPPX_BAND_TRACE") != nullptr;
  cudaEvent_t tr[3 * dppx_ctx::kMaxBands + 1];
  if (trace) {
    for (auto& e : tr) cudaEventCreate(&e);
    cudaEventRecord(tr[3 * nb], ctx->s_in);
  }
  int r0 = 0;
  for (int i = 0; i < nb; ++i) {
    const int r1 = r0 + sizes[i];
    const int y0 = r0 * b, y1 = std::min(r1 * b, M);
    CUDA_TRY(ctx, copy_frames(dimg + y0 * dpitch, dpitch, dpitch * (y1 - y0), img + y0 * d->pitch,
                              d->pitch, d->pitch * (y1 - y0), row, y1 - y0, 1,
                              cudaMemcpyHostToDevice, ctx->s_in));
    ctx->kstats.h2d_bytes += static_cast<uint64_t>(row) * (y1 - y0);
    if (i == 0 && adaptive) {
      if (int rc = ship_mask()) return rc;
      dd.mask_pitch = mp;
      dd.mask_frame_stride = mfs;
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->band_in[i], ctx->s_in));
    if (trace) cudaEventRecord(tr[3 * i], ctx->s_in);
    CUDA_TRY(ctx, cudaStreamWaitEvent(comp, ctx->band_in[i], 0));
    PixOpts po;
    po.mask_bits = bits;
    po.row_begin = r0;
    po.row_count = r1 - r0;
    po.classify = i == 0;
    if (int rc = pixelize_dev(ctx, &dd, dimg, dmask, pp, nz, nullptr, dstats, dstride,
                              adaptive ? dlens : nullptr, out ? dout : nullptr, adaptive, ctx->sd[0],
                              ctx->sd_pinned[0], ctx->sd_pinned_n[0], ctx->comp_done[0], false, po))
      return rc;
    CUDA_TRY(ctx, cudaEventRecord(ctx->band_comp[i], comp));
    if (trace) cudaEventRecord(tr[3 * i + 1], comp);
    if (out) {
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_out, ctx->band_comp[i], 0));
      CUDA_TRY(ctx, copy_frames(out + y0 * d->out_pitch, d->out_pitch, d->out_pitch * (y1 - y0),
                                dout + y0 * dpitch, dpitch, dpitch * (y1 - y0), row, y1 - y0, 1,
                                cudaMemcpyDeviceToHost, ctx->s_out));
      ctx->kstats.d2h_bytes += static_cast<uint64_t>(row) * (y1 - y0);
    }
    if (trace) cudaEventRecord(tr[3 * i + 2], ctx->s_out);
    r0 = r1;
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->in_done[0], ctx->s_in));
  CUDA_TRY(ctx, cudaEventRecord(ctx->comp_done[0], comp));
  CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_out, ctx->comp_done[0], 0));
  CUDA_TRY(ctx, cudaMemcpy2DAsync(stats, sstride, dstats, dstride, cap, C, cudaMemcpyDeviceToHost,
                                  ctx->s_out));
  ctx->kstats.d2h_bytes += static_cast<uint64_t>(cap) * C;
  if (adaptive && lens) {
    CUDA_TRY(ctx, cudaMemcpyAsync(lens, dlens, sizeof(uint32_t) * C, cudaMemcpyDeviceToHost,
                                  ctx->s_out));
    ctx->kstats.d2h_bytes += sizeof(uint32_t) * C;
  }
  CUDA_TRY(ctx, cudaEventRecord(ctx->out_done[0], ctx->s_out));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->s_out));
  CUDA_TRY(ctx, cudaStreamSynchronize(comp));
  if (trace) {
    for (int i = 0; i < nb; ++i) {
      float a = 0, k = 0, o = 0;
      cudaEventElapsedTime(&a, tr[3 * nb], tr[3 * i]);
      cudaEventElapsedTime(&k, tr[3 * nb], tr[3 * i + 1]);
      cudaEventElapsedTime(&o, tr[3 * nb], tr[3 * i + 2]);
      std::fprintf(stderr, "band %d rows %d: in %.1f us, k1 %.1f us, out %.1f us\n", i, sizes[i],
                   a * 1e3f, k * 1e3f, o * 1e3f);
    }
    for (auto& e : tr) cudaEventDestroy(e);
  }
  if (ctx->timing) collect_timings(ctx);
  return DPPX_OK;
}

// Device-accessible alias of a page-locked host buffer (nullptr if none).
void* mapped_alias(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost) return nullptr;
  return at.devicePointer;
}

// Single small frame, zero-copy: the kernels read the caller's page-locked
// frame (and mask) and write the reconstructed frame straight over PCIe --
// no staging copies, so no per-copy latency. The row-streaming kernels (plain
// 16-byte loads / stores) are used; statistics land in the ctx's mapped
// pinned staging and are copied to the caller's buffers on the host.
int host_single_zerocopy(dppx_ctx* ctx, bool adaptive, const dppx_frames_desc* d, const BatchGeom& g,
                         const uint8_t* img, const uint8_t* mask, const dppx_privacy_params* pp,
                         const dppx_noise* nz, uint8_t* stats, int64_t sstride, uint32_t* lens,
                         uint8_t* out, bool* used, bool k1z_only) {
  *used = false;
  const int C = g.C;
  // K1z (uniform): whole cells only, 16-byte rows; it reads exactly the frame.
  // (adaptive: K0 reads the mapped mask, then the adaptive K1z)
  const bool k1z = g.PR == 0 && g.PC == 0 && (C == 1 || C == 3) && g.b <= 64 &&
                   (static_cast<int64_t>(g.N) * C) % 16 == 0 && d->pitch % 16 == 0 &&
                   (!out || d->out_pitch % 16 == 0) && (!adaptive || d->mask_pitch >= g.N);
  if (k1z_only && !k1z) return DPPX_OK;
  // K1r: only shapes whose loads never touch a byte past the frame (no padding
  // columns, 16-byte rows): a read past a host allocation would fault.
  if (!k1z && (g.PC != 0 || (static_cast<int64_t>(g.N) * C) % 16 != 0 || g.N % 16 != 0 ||
               d->pitch != static_cast<int64_t>(g.N) * C || (out && d->out_pitch != d->pitch) ||
               (adaptive && d->mask_pitch != g.N)))
    return DPPX_OK;
  const size_t G = static_cast<size_t>(g.G);
  const size_t cap = adaptive ? dppx_adaptive_payload_capacity(g.M, g.N, g.b, g.n) : G;
  const int64_t dstride = adaptive ? round_up(static_cast<int64_t>(cap), 16) : static_cast<int64_t>(G);
  const size_t gst = static_cast<size_t>(dstride) * C + 16;
  if (ctx->gstats_pinned_n < gst) {
    if (ctx->gstats_pinned) CUDA_TRY(ctx, cudaFreeHost(ctx->gstats_pinned));
    ++ctx->alloc_gen;
    ctx->gstats_pinned = nullptr;
    ctx->gstats_pinned_n = 0;
    CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->gstats_pinned), gst, cudaHostAllocMapped));
    ctx->gstats_pinned_n = gst;
  }
  uint8_t* dimg = static_cast<uint8_t*>(mapped_alias(img));
  uint8_t* dout = out ? static_cast<uint8_t*>(mapped_alias(out)) : nullptr;
  uint8_t* dmask = adaptive ? static_cast<uint8_t*>(mapped_alias(mask)) : nullptr;
  uint8_t* dst = static_cast<uint8_t*>(mapped_alias(ctx->gstats_pinned));
  if (!dimg || (out && !dout) || (adaptive && !dmask) || !dst) return DPPX_OK;  // not mapped: other path
  *used = true;
  uint32_t* dlens = reinterpret_cast<uint32_t*>(dst + static_cast<size_t>(dstride) * C);
  struct Restore {
    dppx_ctx* c;
    ~Restore() { c->force_rows = false; }
  } restore{ctx};
  ctx->force_rows = true;
  // Statistics straight into the caller's buffer when it is page-locked too
  // (no host copy afterwards); else into the ctx's mapped staging.
  uint8_t* dcaller = static_cast<uint8_t*>(mapped_alias(stats));
  const int64_t cstride = adaptive ? sstride : static_cast<int64_t>(G);
  if (int rc = pixelize_dev(ctx, d, dimg, dmask, pp, nz, nullptr, dcaller ? dcaller : dst,
                            dcaller ? cstride : dstride, adaptive ? dlens : nullptr, dout, adaptive, ctx->sd[0],
                            ctx->sd_pinned[0], ctx->sd_pinned_n[0], ctx->comp_done[0], true))
    return rc;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->timing) collect_timings(ctx);
  ctx->kstats.h2d_bytes += static_cast<uint64_t>(g.M) * g.N * C + (adaptive ? static_cast<uint64_t>(g.M) * g.N : 0);
  ctx->kstats.d2h_bytes += (out ? static_cast<uint64_t>(g.M) * g.N * C : 0);
  const uint8_t* st = ctx->gstats_pinned;
  const uint32_t* ln = reinterpret_cast<const uint32_t*>(st + static_cast<size_t>(dstride) * C);
  for (int c = 0; c < C; ++c) {
    const size_t w = adaptive ? std::min<size_t>(ln[c], cap) : G;
    if (!dcaller) std::memcpy(stats + static_cast<int64_t>(c) * cstride, st + static_cast<int64_t>(c) * dstride, w);
    if (adaptive && lens) lens[c] = ln[c];
    ctx->kstats.d2h_bytes += w;
  }
  return DPPX_OK;
}

// Single-frame host call as a replayed CUDA graph (see dppx_ctx::FrameGraph).
// Preconditions (host_pipeline checks): one frame, pinned dense image / mask /
// output buffers with N*C % 16 == 0 (the device layout), KEYED or no noise.
int host_single_graph(dppx_ctx* ctx, bool adaptive, const dppx_frames_desc* d, const BatchGeom& g,
                      const uint8_t* img, const uint8_t* mask, const dppx_privacy_params* pp,
                      const dppx_noise* nz, uint8_t* stats, int64_t sstride, uint32_t* lens,
                      uint8_t* out) {
  const int C = g.C, M = g.M, N = g.N, b = g.b;
  const int64_t row = static_cast<int64_t>(N) * C;
  const int64_t dfs = row * M, dmfs = static_cast<int64_t>(N) * M;
  const size_t G = static_cast<size_t>(g.G);
  const size_t cap = adaptive ? dppx_adaptive_payload_capacity(M, N, b, g.n) : G;
  const int64_t dstride = adaptive ? round_up(static_cast<int64_t>(cap), 16) : static_cast<int64_t>(G);
  const int kind = nz ? nz->kind : DPPX_NOISE_NONE;
  // Row bands: the H2D of band i+1, K1 of band i and D2H of band i-1 overlap.
  // (one band measured fastest for a PETS frame: every extra copy node adds
  // more latency than its overlap saves, r02k_latency.txt)
  int nb = 1;
  if (const char* env = std::getenv("DPPX_GRAPH_BANDS")) nb = std::max(1, std::atoi(env));
  nb = std::max(1, std::min({nb, g.GR / 2 > 0 ? g.GR / 2 : 1, dppx_ctx::kMaxBands}));
  dppx_ctx::FrameGraph* fgp = nullptr;
  if (!ctx->graphs.empty() && ctx->graphs.front()->gen != ctx->alloc_gen) {
    for (auto* c : ctx->graphs) delete c;  // buffers they reference were reallocated
    ctx->graphs.clear();
  }
  for (auto* c : ctx->graphs)
    if (c->op == (adaptive ? 1 : 0) && c->M == M && c->N == N && c->C == C && c->b == b && c->n == g.n &&
        c->kind == kind && c->exact == (ctx->exact_noise ? 1 : 0) && c->nb == nb &&
        c->want_out == (out ? 1 : 0) && c->sigma == pp->sigma && c->sigma_sub == pp->sigma_sub)
      fgp = c;
  cudaStream_t comp = ctx->stream;
  if (!fgp) {
    // ---- capture ----
    if (ensure(ctx, ctx->img[0], static_cast<size_t>(dfs))) return DPPX_ERR_OOM;
    if (out && ensure(ctx, ctx->out[0], static_cast<size_t>(dfs))) return DPPX_ERR_OOM;
    if (adaptive && ensure(ctx, ctx->mask[0], static_cast<size_t>(dmfs))) return DPPX_ERR_OOM;
    if (ensure(ctx, ctx->stats[0], static_cast<size_t>(dstride) * C)) return DPPX_ERR_OOM;
    if (ensure(ctx, ctx->lens[0], sizeof(uint32_t) * C)) return DPPX_ERR_OOM;
    if (ensure(ctx, ctx->gseeds, sizeof(uint64_t) * C)) return DPPX_ERR_OOM;
    if (adaptive)
      if (int rc = ensure_scratch(ctx, g, 1)) return rc;
    if (int rc = ensure(ctx, ctx->work, 16, /*zero=*/true)) return rc;
    if (!ctx->gseeds_pinned)
      CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->gseeds_pinned), 8 * 4, cudaHostAllocDefault));
    const size_t gst = static_cast<size_t>(dstride) * C + 16;
    if (ctx->gstats_pinned_n < gst) {
      if (ctx->gstats_pinned) CUDA_TRY(ctx, cudaFreeHost(ctx->gstats_pinned));
      ++ctx->alloc_gen;
      ctx->gstats_pinned = nullptr;
      ctx->gstats_pinned_n = 0;
      CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->gstats_pinned), gst, cudaHostAllocMapped));
      ctx->gstats_pinned_n = gst;
    }
    // A graph owns device buffer addresses: drop the cache when it is full.
    if (ctx->graphs.size() >= 8) {
      auto old = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                  [](auto* x, auto* y) { return x->last_use < y->last_use; });
      delete *old;
      ctx->graphs.erase(old);
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(comp));
    const bool timing = ctx->timing;
    const dppx_kernel_stats saved = ctx->kstats;
    ctx->timing = false;
    ctx->kstats = dppx_kernel_stats{};
    uint8_t* dimg = static_cast<uint8_t*>(ctx->img[0].p);
    uint8_t* dout = static_cast<uint8_t*>(ctx->out[0].p);
    uint8_t* dmask = static_cast<uint8_t*>(ctx->mask[0].p);
    uint8_t* dstats = static_cast<uint8_t*>(ctx->stats[0].p);
    uint32_t* dlens = static_cast<uint32_t*>(ctx->lens[0].p);
    cudaEvent_t fork = get_event(ctx), join_in = get_event(ctx), join_out = get_event(ctx);
    int rc = DPPX_OK;
    auto fail = [&](int code) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(comp, &junk);
      if (junk) cudaGraphDestroy(junk);
      cudaGetLastError();
      ctx->timing = timing;
      ctx->kstats = saved;
      return code;
    };
    CUDA_TRY(ctx, cudaStreamBeginCapture(comp, cudaStreamCaptureModeRelaxed));
    uint64_t h2d = 0, d2h = 0;
    if (cudaEventRecord(fork, comp) != cudaSuccess || cudaStreamWaitEvent(ctx->s_in, fork, 0) != cudaSuccess ||
        cudaStreamWaitEvent(ctx->s_out, fork, 0) != cudaSuccess)
      return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: fork failed"));
    if (kind == DPPX_NOISE_KEYED &&
        cudaMemcpyAsync(ctx->gseeds.p, ctx->gseeds_pinned, sizeof(uint64_t) * C, cudaMemcpyHostToDevice,
                        ctx->s_in) != cudaSuccess)
      return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: seeds copy"));
    int sizes[dppx_ctx::kMaxBands];
    {
      int left = g.GR;
      for (int i = 0; i < nb; ++i) {
        sizes[i] = left / (nb - i);
        left -= sizes[i];
      }
    }
    dppx_frames_desc dd = *d;
    dd.pitch = row;
    dd.frame_stride = dfs;
    dd.mask_pitch = N;
    dd.mask_frame_stride = dmfs;
    dd.out_pitch = row;
    dd.out_frame_stride = dfs;
    dppx_noise gn{};
    if (nz) gn = *nz;
    int r0 = 0;
    for (int i = 0; i < nb && rc == DPPX_OK; ++i) {
      const int r1 = r0 + sizes[i];
      const int y0 = r0 * b, y1 = std::min(r1 * b, M);
      if (cudaMemcpyAsync(dimg + y0 * row, img + y0 * row, static_cast<size_t>(row) * (y1 - y0),
                          cudaMemcpyHostToDevice, ctx->s_in) != cudaSuccess)
        return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: image copy"));
      h2d += static_cast<uint64_t>(row) * (y1 - y0);
      if (i == 0 && adaptive) {
        if (cudaMemcpyAsync(dmask, mask, static_cast<size_t>(dmfs), cudaMemcpyHostToDevice, ctx->s_in) != cudaSuccess)
          return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: mask copy"));
        h2d += static_cast<uint64_t>(dmfs);
      }
      if (cudaEventRecord(ctx->band_in[i], ctx->s_in) != cudaSuccess ||
          cudaStreamWaitEvent(comp, ctx->band_in[i], 0) != cudaSuccess)
        return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: band order"));
      PixOpts po;
      po.row_begin = r0;
      po.row_count = r1 - r0;
      po.classify = i == 0;
      po.seeds_dev = static_cast<const uint64_t*>(ctx->gseeds.p);
      rc = pixelize_dev(ctx, &dd, dimg, dmask, pp, nz ? &gn : nullptr, nullptr, dstats, dstride,
                        adaptive ? dlens : nullptr, out ? dout : nullptr, adaptive, ctx->sd[0],
                        ctx->sd_pinned[0], ctx->sd_pinned_n[0], nullptr, false, po);
      if (rc) return fail(rc);
      if (out) {
        if (cudaEventRecord(ctx->band_comp[i], comp) != cudaSuccess ||
            cudaStreamWaitEvent(ctx->s_out, ctx->band_comp[i], 0) != cudaSuccess ||
            cudaMemcpyAsync(out + y0 * row, dout + y0 * row, static_cast<size_t>(row) * (y1 - y0),
                            cudaMemcpyDeviceToHost, ctx->s_out) != cudaSuccess)
          return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: output copy"));
        d2h += static_cast<uint64_t>(row) * (y1 - y0);
      }
      r0 = r1;
    }
    // statistics (+ lengths) into the ctx's pinned staging after the last band
    if (cudaMemcpyAsync(ctx->gstats_pinned, dstats, static_cast<size_t>(dstride) * C, cudaMemcpyDeviceToHost,
                        comp) != cudaSuccess ||
        (adaptive && cudaMemcpyAsync(ctx->gstats_pinned + static_cast<size_t>(dstride) * C, dlens,
                                     sizeof(uint32_t) * C, cudaMemcpyDeviceToHost, comp) != cudaSuccess))
      return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: statistics copy"));
    d2h += static_cast<uint64_t>(adaptive ? cap : G) * C + (adaptive ? 4 * C : 0);
    if (cudaEventRecord(join_in, ctx->s_in) != cudaSuccess || cudaEventRecord(join_out, ctx->s_out) != cudaSuccess ||
        cudaStreamWaitEvent(comp, join_in, 0) != cudaSuccess || cudaStreamWaitEvent(comp, join_out, 0) != cudaSuccess)
      return fail(set_err(ctx, DPPX_ERR_CUDA, "graph capture: join failed"));
    cudaGraph_t graph = nullptr;
    CUDA_TRY(ctx, cudaStreamEndCapture(comp, &graph));
    ctx->event_pool.push_back(fork);
    ctx->event_pool.push_back(join_in);
    ctx->event_pool.push_back(join_out);
    auto* ng = new dppx_ctx::FrameGraph();
    ng->op = adaptive ? 1 : 0;
    ng->M = M;
    ng->N = N;
    ng->C = C;
    ng->b = b;
    ng->n = g.n;
    ng->kind = kind;
    ng->exact = ctx->exact_noise ? 1 : 0;
    ng->nb = nb;
    ng->want_out = out ? 1 : 0;
    ng->sigma = pp->sigma;
    ng->sigma_sub = pp->sigma_sub;
    ng->graph = graph;
    for (int k = 0; k < DPPX_K_COUNT; ++k) ng->launches[k] = ctx->kstats.launches[k];
    ng->h2d = h2d;
    ng->d2h = d2h;
    ctx->timing = timing;
    ctx->kstats = saved;
    // memcpy nodes that touch the caller's buffers (re-pointed per replay)
    size_t nn = 0;
    CUDA_TRY(ctx, cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CUDA_TRY(ctx, cudaGraphGetNodes(graph, nodes.data(), &nn));
    auto inside = [](const void* p, const void* base, int64_t bytes) {
      return base && p >= base && static_cast<const uint8_t*>(p) < static_cast<const uint8_t*>(base) + bytes;
    };
    for (cudaGraphNode_t node : nodes) {
      cudaGraphNodeType ty;
      CUDA_TRY(ctx, cudaGraphNodeGetType(node, &ty));
      if (ty != cudaGraphNodeTypeMemcpy) continue;
      dppx_ctx::FrameGraph::Copy c{};
      c.node = node;
      CUDA_TRY(ctx, cudaGraphMemcpyNodeGetParams(node, &c.p));
      const void* src = c.p.srcPtr.ptr;
      const void* dst = c.p.dstPtr.ptr;
      if (inside(src, img, dfs)) {
        c.which = 0;
        c.offset = static_cast<const uint8_t*>(src) - img;
      } else if (adaptive && inside(src, mask, dmfs)) {
        c.which = 1;
        c.offset = static_cast<const uint8_t*>(src) - mask;
      } else if (out && inside(dst, out, dfs)) {
        c.which = 2;
        c.offset = static_cast<const uint8_t*>(dst) - out;
      } else {
        continue;
      }
      ng->copies.push_back(c);
    }
    const cudaError_t ie = cudaGraphInstantiate(&ng->exec, graph, 0);
    if (ie != cudaSuccess) {
      delete ng;
      return set_err(ctx, DPPX_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
    }
    ng->cur[0] = img;
    ng->cur[1] = mask;
    ng->cur[2] = out;
    // every buffer the graph references was allocated before the capture; if
    // the capture itself had to grow one, older graphs are stale now
    if (!ctx->graphs.empty() && ctx->graphs.front()->gen != ctx->alloc_gen) {
      for (auto* c : ctx->graphs) delete c;
      ctx->graphs.clear();
    }
    ng->gen = ctx->alloc_gen;
    ctx->graphs.push_back(ng);
    fgp = ng;
  }
  // ---- replay ----
  fgp->last_use = ++ctx->graph_tick;
  const void* want[3] = {img, mask, out};
  for (auto& c : fgp->copies) {
    if (fgp->cur[c.which] == want[c.which]) continue;
    cudaMemcpy3DParms p = c.p;
    if (c.which == 2)
      p.dstPtr.ptr = static_cast<uint8_t*>(const_cast<void*>(want[2])) + c.offset;
    else
      p.srcPtr.ptr = const_cast<uint8_t*>(static_cast<const uint8_t*>(want[c.which])) + c.offset;
    CUDA_TRY(ctx, cudaGraphExecMemcpyNodeSetParams(fgp->exec, c.node, &p));
  }
  for (int k = 0; k < 3; ++k) fgp->cur[k] = want[k];
  if (kind == DPPX_NOISE_KEYED)
    for (int c = 0; c < C; ++c) ctx->gseeds_pinned[c] = mix64_h(nz->plane_seeds[c]);
  CUDA_TRY(ctx, cudaGraphLaunch(fgp->exec, comp));
  CUDA_TRY(ctx, cudaStreamSynchronize(comp));
  for (int k = 0; k < DPPX_K_COUNT; ++k) ctx->kstats.launches[k] += fgp->launches[k];
  ctx->kstats.h2d_bytes += fgp->h2d;
  ctx->kstats.d2h_bytes += fgp->d2h;
  const uint8_t* st = ctx->gstats_pinned;
  const uint32_t* ln = reinterpret_cast<const uint32_t*>(st + static_cast<size_t>(dstride) * C);
  for (int c = 0; c < C; ++c) {
    const size_t w = adaptive ? std::min<size_t>(ln[c], cap) : G;
    std::memcpy(stats + static_cast<int64_t>(c) * (adaptive ? sstride : static_cast<int64_t>(G)),
                st + static_cast<int64_t>(c) * dstride, w);
    if (adaptive && lens) lens[c] = ln[c];
  }
  return DPPX_OK;
}

int host_pipeline(dppx_ctx* ctx, HostOp op, const dppx_frames_desc* d, const uint8_t* img,
                  const uint8_t* mask, const dppx_privacy_params* pp, const dppx_noise* nz,
                  uint8_t* stats, int64_t sstride, uint32_t* lens, const uint32_t* in_lens,
                  int b_arg, int n_arg, uint8_t* out) {
  static const bool trace = std::getenv("DPPX_PIPE_TRACE") != nullptr;
  const auto tp0 = std::chrono::steady_clock::now();
  auto tp_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
  };
  const bool pix = op == HostOp::Uniform || op == HostOp::Adaptive || op == HostOp::Reference ||
                   op == HostOp::AdaptiveVariance;
  const bool adaptive = op == HostOp::Adaptive || op == HostOp::Reassemble ||
                        op == HostOp::AdaptiveVariance;
  if (!d) return set_err(ctx, DPPX_ERR_INVALID, "null frames descriptor");
  const int b = pix ? (pp ? pp->b : 0) : b_arg;
  const int n = pix ? (pp ? pp->n : 1) : n_arg;
  if (pix) {
    if (int rc = check_params(ctx, pp, adaptive)) return rc;
  }
  BatchGeom g;
  if (op == HostOp::Reassemble) {
    if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, b, 1, &g, false))
      return rc;
    if (n < 1 || b % n != 0)
      return set_err(ctx, DPPX_ERR_CORRUPT, "reassemble: subgrid factor does not divide grid side");
    g.n = n;
    g.sb = b / n;
  } else if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, b,
                               adaptive ? n : 1, &g, pix && op != HostOp::Reference)) {
    return rc;
  }
  if (int rc = check_desc(ctx, d, op == HostOp::Adaptive, !pix || out != nullptr)) return rc;
  const int F = d->frames, C = g.C, M = g.M, N = g.N;
  if (F == 0) return DPPX_OK;
  if (pix && !img) return set_err(ctx, DPPX_ERR_INVALID, "null image pointer");
  if (op == HostOp::Adaptive && !mask) return set_err(ctx, DPPX_ERR_INVALID, "null mask pointer");
  if (!stats) return set_err(ctx, DPPX_ERR_INVALID, "null statistics pointer");
  if (!pix && !out) return set_err(ctx, DPPX_ERR_INVALID, "null output pointer");
  const size_t G = static_cast<size_t>(g.G);
  int64_t dstride;  // device statistics bytes per plane
  if (adaptive) {
    const size_t cap = dppx_adaptive_payload_capacity(M, N, b, n);
    dstride = round_up(static_cast<int64_t>(cap), 16);
    if (sstride < (op != HostOp::Reassemble ? static_cast<int64_t>(cap) : 4ll * g.G + 4))
      return set_err(ctx, DPPX_ERR_INVALID, "payload_stride too small");
    if (op == HostOp::Reassemble) dstride = round_up(std::max<int64_t>(sstride, 16), 16);
  } else {
    dstride = static_cast<int64_t>(G);
    sstride = static_cast<int64_t>(G);
  }
  if (ctx->mask_bits_mode < 0) {
    const char* env = std::getenv("DPPX_MASK_BITS");
    ctx->mask_bits_mode = env && env[0] == '0' ? 0 : 1;
  }
  {
    // One small frame (below the row-band threshold): zero-copy kernels or a
    // replayed CUDA graph (dppx_ctx_set_small_frame_path; environment
    // defaults DPPX_ZEROCOPY=0/1, DPPX_GRAPH=0).
    if (ctx->small_path < 0) {
      const char* zc = std::getenv("DPPX_ZEROCOPY");
      const char* gr = std::getenv("DPPX_GRAPH");
      ctx->small_path = zc && zc[0] == '1'   ? DPPX_SMALL_ZEROCOPY
                        : zc && zc[0] == '0' ? (gr && gr[0] == '0' ? DPPX_SMALL_STAGED : DPPX_SMALL_GRAPH)
                        : gr && gr[0] == '0' ? DPPX_SMALL_STAGED
                                             : DPPX_SMALL_AUTO;
    }
    const int64_t row = static_cast<int64_t>(N) * C;
    const bool small = static_cast<int64_t>(M) * row < (4ll << 20);
    // auto: zero-copy (K1z streams the frame over PCIe with the reads and
    // writes overlapped; adaptive: K0 on the mapped mask first, K1z launched
    // as its programmatic dependent): PETS 59 / 97 us per call against 88 /
    // 122 us for the graph (profiles/r02_zerocopy.txt)
    const bool zc_try = ctx->small_path == DPPX_SMALL_ZEROCOPY || ctx->small_path == DPPX_SMALL_AUTO;
    const bool graphs_on = ctx->small_path == DPPX_SMALL_AUTO || ctx->small_path == DPPX_SMALL_GRAPH;
    if (zc_try && F == 1 && small && (op == HostOp::Uniform || op == HostOp::Adaptive) &&
        (!nz || nz->kind != DPPX_NOISE_INJECTED)) {
      bool used = false;
      const int rc = host_single_zerocopy(ctx, op == HostOp::Adaptive, d, g, img, mask, pp, nz, stats, sstride,
                                          lens, out, &used, ctx->small_path == DPPX_SMALL_AUTO);
      if (rc || used) return rc;
    }
    if (graphs_on && F == 1 && small && (op == HostOp::Uniform || op == HostOp::Adaptive) &&
        (!nz || nz->kind == DPPX_NOISE_NONE || nz->kind == DPPX_NOISE_KEYED) && row % 16 == 0 &&
        d->pitch == row && (!out || d->out_pitch == row) && (op != HostOp::Adaptive || d->mask_pitch == N) &&
        host_pinned(img) && (!out || host_pinned(out)) && (op != HostOp::Adaptive || host_pinned(mask)))
      return host_single_graph(ctx, op == HostOp::Adaptive, d, g, img, mask, pp, nz, stats, sstride, lens, out);
  }
  {
    // One frame: pipeline row bands instead of frames (DPPX_BANDS=0 disables).
    const char* env = std::getenv("DPPX_BANDS");
    const bool bands_ok = !(env && env[0] == '0');
    const int64_t frame_bytes = static_cast<int64_t>(M) * N * C;
    const bool inj_any = nz && nz->kind == DPPX_NOISE_INJECTED;
    // >= 2 MB per band: a band's copies must outlast the ~20 us of host work
    // that issues it (measured: smaller bands make the pipeline issue-bound).
    const int nb = static_cast<int>(std::min<int64_t>(
        {static_cast<int64_t>(dppx_ctx::kMaxBands), g.GR / 2, frame_bytes >> 21}));
    if (bands_ok && F == 1 && (op == HostOp::Uniform || op == HostOp::Adaptive) && !inj_any &&
        nb >= 2 && host_pinned(img) && (!out || host_pinned(out)))
      return host_pipeline_bands(ctx, adaptive, d, g, img, mask, pp, nz, stats, sstride, lens, out, nb);
  }
  const int64_t dpitch = round_up(static_cast<int64_t>(N) * C, 16);
  const int64_t dmpitch = round_up(N, 16);
  const int64_t dfs = dpitch * M, dmfs = dmpitch * M;
  const int64_t per_frame = (pix ? dfs : 0) + (op == HostOp::Adaptive ? dmfs : 0) +
                            (out ? dfs : 0) + dstride * C;
  // ~10 chunks per call keeps pipeline fill + drain small; 8..192 MB per chunk
  // (measured: 12-frame 1080p chunks beat 6-frame ones by ~2% end to end).
  const int64_t target = std::min<int64_t>(192ll << 20, std::max<int64_t>(8ll << 20, per_frame * F / 10));
  int K = ctx->chunk_frames > 0 ? ctx->chunk_frames
                                : static_cast<int>(std::max<int64_t>(1, target / per_frame));
  K = std::max(1, std::min(K, F));
  // Chunk schedule: 1, 2, 4, ... ramp up, K-frame chunks, mirrored ramp down, so
  // the first H2D and the last D2H (the unoverlapped fill and drain) are small.
  std::vector<int> sizes;
  {
    std::vector<int> up;
    int sum_up = 0;
    for (int c = 1; c < K && 2 * (sum_up + c) < F; c *= 2) {
      up.push_back(c);
      sum_up += c;
    }
    const int rem = F - 2 * sum_up;
    const int mid = (rem + K - 1) / K;
    sizes = up;
    for (int i = 0; i < mid; ++i) sizes.push_back(rem / mid + (i < rem % mid ? 1 : 0));
    sizes.insert(sizes.end(), up.rbegin(), up.rend());
  }
  const int chunks = static_cast<int>(sizes.size());
  const bool inj = pix && nz && nz->kind == DPPX_NOISE_INJECTED;
  const size_t inj_plane = G * static_cast<size_t>(adaptive ? n * n : 1);
  const int64_t row = static_cast<int64_t>(N) * C;
  // Dense linear PCIe transfers + on-device re-pitch when the kernels' 16-byte
  // pitch differs from a dense host layout (e.g. 178 x 3 = 534-byte rows).
  // Pageable caller buffers: host threads copy rows into / out of pinned
  // staging in the device layout, so the DMA runs at pinned speed (the
  // driver's own pageable path is serial and several times slower).
  const bool stage_in = pix && !host_pinned(img);
  const bool stage_out = out && !host_pinned(out);
  const bool dense_in = !stage_in && pix && dpitch != row && d->pitch == row && d->frame_stride == row * M;
  const bool dense_mask = op == HostOp::Adaptive && dmpitch != N && d->mask_pitch == N &&
                          d->mask_frame_stride == static_cast<int64_t>(N) * M;
  const bool dense_out = !stage_out && out && dpitch != row && d->out_pitch == row &&
                         d->out_frame_stride == row * M;
  // Bit-packed mask transport: 1/8 of the mask's PCIe bytes (maskpack.h).
  const bool try_bits = op == HostOp::Adaptive && ctx->mask_bits_mode == 1;
  // Adaptive payloads leave the device with their written length (4G + 4 + S +
  // (G - S) n^2 per plane, known once K0 has run), not the slot capacity: each
  // chunk's lengths go D2H on s_meta right after its kernels, and the chunk's
  // payloads are copied one chunk later (DPPX_EXACT_PAYLOAD=0: copy whole
  // slots, for A/B runs).
  static const bool exact_env = !(std::getenv("DPPX_EXACT_PAYLOAD") &&
                                  std::getenv("DPPX_EXACT_PAYLOAD")[0] == '0');
  const bool exact_payload = pix && adaptive && exact_env;
  const int64_t wpr = dppx::mask_words_per_row(N);
  const size_t bits_frame = static_cast<size_t>(wpr) * 4 * M;
  if ((try_bits || stage_in || stage_out) && !ctx->packer) ctx->packer = dppx::mask_packer_create(0);
  for (int s = 0; s < 2 && s < chunks; ++s) {
    if (stage_in)
      if (int rc = grow_pinned(ctx, ctx->stg_in[s], ctx->stg_in_n[s], static_cast<size_t>(dfs) * K)) return rc;
    if (stage_out)
      if (int rc = grow_pinned(ctx, ctx->stg_out[s], ctx->stg_out_n[s], static_cast<size_t>(dfs) * K)) return rc;
    if (stage_out && !ctx->stg_ev[s])
      CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->stg_ev[s], cudaEventDisableTiming));
    if (pix && ensure(ctx, ctx->img[s], static_cast<size_t>(dfs) * K)) return DPPX_ERR_OOM;
    if (op == HostOp::Adaptive && ensure(ctx, ctx->mask[s], static_cast<size_t>(dmfs) * K))
      return DPPX_ERR_OOM;
    if (out && ensure(ctx, ctx->out[s], static_cast<size_t>(dfs) * K)) return DPPX_ERR_OOM;
    if (ensure(ctx, ctx->stats[s], static_cast<size_t>(dstride) * C * K)) return DPPX_ERR_OOM;
    if (ensure(ctx, ctx->lens[s], sizeof(uint32_t) * C * K)) return DPPX_ERR_OOM;
    if (inj && ensure(ctx, ctx->inj[s], sizeof(double) * inj_plane * C * K)) return DPPX_ERR_OOM;
    if (dense_in && ensure(ctx, ctx->dense[s], static_cast<size_t>(row) * M * K))
      return DPPX_ERR_OOM;
    if (dense_out && ensure(ctx, ctx->dense_out[s], static_cast<size_t>(row) * M * K))
      return DPPX_ERR_OOM;
    if (dense_mask && ensure(ctx, ctx->dense_mask[s], static_cast<size_t>(N) * M * K))
      return DPPX_ERR_OOM;
    if (exact_payload && ctx->lens_pinned_n[s] < static_cast<size_t>(C) * K) {
      if (ctx->lens_pinned[s]) CUDA_TRY(ctx, cudaFreeHost(ctx->lens_pinned[s]));
      ctx->lens_pinned[s] = nullptr;
      ctx->lens_pinned_n[s] = 0;
      CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->lens_pinned[s]),
                                  sizeof(uint32_t) * C * K, cudaHostAllocDefault));
      ctx->lens_pinned_n[s] = static_cast<size_t>(C) * K;
    }
    if (try_bits && ctx->mbits_pinned_n[s] < bits_frame * K) {
      if (ctx->mbits_pinned[s]) CUDA_TRY(ctx, cudaFreeHost(ctx->mbits_pinned[s]));
      ctx->mbits_pinned[s] = nullptr;
      ctx->mbits_pinned_n[s] = 0;
      CUDA_TRY(ctx, cudaHostAlloc(reinterpret_cast<void**>(&ctx->mbits_pinned[s]), bits_frame * K,
                                  cudaHostAllocDefault));
      ctx->mbits_pinned_n[s] = bits_frame * K;
    }
  }
  cudaStream_t comp = ctx->stream;
  if (trace)
    std::fprintf(stderr, "pipe: op %d F %d K %d chunks %d stage_in %d stage_out %d setup %.2f ms\n",
                 static_cast<int>(op), F, K, chunks, stage_in, stage_out, tp_ms());
  // Row copies between a caller frame range and pinned staging (device layout).
  auto stage_rows = [&](uint8_t* dst, int64_t dp, int64_t dfst, const uint8_t* src, int64_t sp,
                        int64_t sfs, int Fk) {
    dppx::pool_for(ctx->packer, static_cast<int64_t>(Fk) * M, [&](int64_t r0, int64_t r1) {
      for (int64_t r = r0; r < r1; ++r) {
        const int64_t f = r / M, i = r % M;
        std::memcpy(dst + f * dfst + i * dp, src + f * sfs + i * sp, static_cast<size_t>(row));
      }
    });
  };
  int pend_f0[2] = {-1, -1}, pend_fk[2] = {0, 0};
  auto drain = [&](int s) -> int {  // staged output of slot s -> caller buffer
    if (pend_f0[s] < 0) return DPPX_OK;
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->stg_ev[s]));
    stage_rows(out + static_cast<int64_t>(pend_f0[s]) * d->out_frame_stride, d->out_pitch,
               d->out_frame_stride, ctx->stg_out[s], dpitch, dfs, pend_fk[s]);
    pend_f0[s] = -1;
    return DPPX_OK;
  };
  std::vector<int> chunk_f0(chunks, 0);
  const size_t cap_plane = adaptive ? dppx_adaptive_payload_capacity(M, N, b, n) : G;
  // D2H of chunk cj's payloads (its lengths are in lens_pinned): one 2-D copy
  // of the chunk's longest written payload per plane slot -- the planes of a
  // chunk share their masks frame by frame, so this is within a few bytes of
  // the written total -- then the slot's out_done (chunk cj's image and
  // payload copies are queued).
  auto issue_payload = [&](int cj) -> int {
    const int sj = cj & 1, Fj = sizes[cj];
    CUDA_TRY(ctx, cudaEventSynchronize(ctx->lens_ev[sj]));
    const uint32_t* ln = ctx->lens_pinned[sj];
    if (lens) std::memcpy(lens + static_cast<int64_t>(chunk_f0[cj]) * C, ln, sizeof(uint32_t) * Fj * C);
    size_t w = 0;
    for (int q = 0; q < Fj * C; ++q) w = std::max<size_t>(w, ln[q]);
    w = std::min(w, cap_plane);  // (a corrupt length never over-reads the slot)
    CUDA_TRY(ctx, cudaMemcpy2DAsync(stats + static_cast<int64_t>(chunk_f0[cj]) * C * sstride, sstride,
                                    ctx->stats[sj].p, dstride, w, static_cast<size_t>(Fj) * C,
                                    cudaMemcpyDeviceToHost, ctx->s_out));
    ctx->kstats.d2h_bytes += static_cast<uint64_t>(w) * Fj * C;
    CUDA_TRY(ctx, cudaEventRecord(ctx->out_done[sj], ctx->s_out));
    return DPPX_OK;
  };
  int f0 = 0;
  for (int ci = 0; ci < chunks; ++ci) {
    const int s = ci & 1;
    const int Fk = sizes[ci];
    // ---- H2D (input stream): wait until chunk ci-2 released this slot ----
    if (ci >= 2) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_in, ctx->comp_done[s], 0));
    uint8_t* dimg = static_cast<uint8_t*>(ctx->img[s].p);
    uint8_t* dmask = static_cast<uint8_t*>(ctx->mask[s].p);
    uint8_t* dout = static_cast<uint8_t*>(ctx->out[s].p);
    uint8_t* dstats = static_cast<uint8_t*>(ctx->stats[s].p);
    uint32_t* dlens = static_cast<uint32_t*>(ctx->lens[s].p);
    uint8_t* ddense = static_cast<uint8_t*>(ctx->dense[s].p);
    uint8_t* ddense_out = static_cast<uint8_t*>(ctx->dense_out[s].p);
    uint8_t* ddmask = static_cast<uint8_t*>(ctx->dense_mask[s].p);
    if (pix && stage_in) {
      if (ci >= 2) CUDA_TRY(ctx, cudaEventSynchronize(ctx->in_done[s]));
      stage_rows(ctx->stg_in[s], dpitch, dfs, img + static_cast<int64_t>(f0) * d->frame_stride, d->pitch,
                 d->frame_stride, Fk);
      CUDA_TRY(ctx, cudaMemcpyAsync(dimg, ctx->stg_in[s], static_cast<size_t>(dfs) * Fk,
                                    cudaMemcpyHostToDevice, ctx->s_in));
      ctx->kstats.h2d_bytes += static_cast<uint64_t>(Fk) * M * row;
    } else if (pix) {
      if (dense_in)
        CUDA_TRY(ctx, cudaMemcpyAsync(ddense, img + static_cast<int64_t>(f0) * d->frame_stride,
                                      static_cast<size_t>(row) * M * Fk, cudaMemcpyHostToDevice,
                                      ctx->s_in));
      else
        CUDA_TRY(ctx, copy_frames(dimg, dpitch, dfs, img + static_cast<int64_t>(f0) * d->frame_stride,
                                  d->pitch, d->frame_stride, row, M, Fk, cudaMemcpyHostToDevice,
                                  ctx->s_in));
      ctx->kstats.h2d_bytes += static_cast<uint64_t>(Fk) * M * row;
    }
    bool bits = false;
    if (try_bits) {
      // The slot's staging buffer is free once chunk ci-2's copies finished.
      if (ci >= 2) CUDA_TRY(ctx, cudaEventSynchronize(ctx->in_done[s]));
      bits = dppx::pack_mask_bits(ctx->packer, mask + static_cast<int64_t>(f0) * d->mask_frame_stride,
                                  d->mask_pitch, d->mask_frame_stride, M, N, Fk,
                                  ctx->mbits_pinned[s], wpr);
      if (bits) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dmask, ctx->mbits_pinned[s], bits_frame * Fk,
                                      cudaMemcpyHostToDevice, ctx->s_in));
        ctx->kstats.h2d_bytes += static_cast<uint64_t>(bits_frame) * Fk;
      }
    }
    if (op == HostOp::Adaptive && !bits) {
      if (dense_mask)
        CUDA_TRY(ctx, cudaMemcpyAsync(ddmask, mask + static_cast<int64_t>(f0) * d->mask_frame_stride,
                                      static_cast<size_t>(N) * M * Fk, cudaMemcpyHostToDevice,
                                      ctx->s_in));
      else
        CUDA_TRY(ctx, copy_frames(dmask, dmpitch, dmfs,
                                  mask + static_cast<int64_t>(f0) * d->mask_frame_stride,
                                  d->mask_pitch, d->mask_frame_stride, N, M, Fk,
                                  cudaMemcpyHostToDevice, ctx->s_in));
      ctx->kstats.h2d_bytes += static_cast<uint64_t>(Fk) * M * N;
    }
    if (!pix) {
      CUDA_TRY(ctx, cudaMemcpy2DAsync(dstats, dstride, stats + static_cast<int64_t>(f0) * C * sstride,
                                      sstride, static_cast<size_t>(std::min(sstride, dstride)),
                                      static_cast<size_t>(Fk) * C, cudaMemcpyHostToDevice, ctx->s_in));
      ctx->kstats.h2d_bytes += static_cast<uint64_t>(Fk) * C * std::min(sstride, dstride);
      if (in_lens) {
        CUDA_TRY(ctx, cudaMemcpyAsync(dlens, in_lens + static_cast<int64_t>(f0) * C,
                                      sizeof(uint32_t) * Fk * C, cudaMemcpyHostToDevice, ctx->s_in));
      }
    }
    if (inj) {
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->inj[s].p, nz->injected + static_cast<int64_t>(f0) * C * inj_plane,
                                    sizeof(double) * inj_plane * C * Fk, cudaMemcpyHostToDevice,
                                    ctx->s_in));
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->in_done[s], ctx->s_in));
    // ---- compute ----
    CUDA_TRY(ctx, cudaStreamWaitEvent(comp, ctx->in_done[s], 0));
    if (ci >= 2) CUDA_TRY(ctx, cudaStreamWaitEvent(comp, ctx->out_done[s], 0));
    if (dense_in) {
      PendingTiming pt;
      timing_begin(ctx, DPPX_K_AUX, &pt);
      CUDA_TRY(ctx, launch_repitch(dimg, dpitch, ddense, row, row, static_cast<int64_t>(M) * Fk, comp));
      timing_end(ctx, &pt);
    }
    if (dense_mask && !bits) {
      PendingTiming pt;
      timing_begin(ctx, DPPX_K_AUX, &pt);
      CUDA_TRY(ctx, launch_repitch(dmask, dmpitch, ddmask, N, N, static_cast<int64_t>(M) * Fk, comp));
      timing_end(ctx, &pt);
    }
    dppx_frames_desc dd = *d;
    dd.frames = Fk;
    dd.pitch = dpitch;
    dd.frame_stride = dfs;
    dd.mask_pitch = bits ? wpr * 4 : dmpitch;
    dd.mask_frame_stride = bits ? static_cast<int64_t>(bits_frame) : dmfs;
    dd.out_pitch = dpitch;
    dd.out_frame_stride = dfs;
    int rc;
    // dout is the ctx's own staging buffer: its pitch padding is scratch.
    struct PadScratch {
      dppx_ctx* c;
      bool prev;
      ~PadScratch() { c->out_pad_scratch = prev; }
    } pad_scope{ctx, ctx->out_pad_scratch};
    ctx->out_pad_scratch = true;
    if (pix) {
      dppx_noise cn{};
      if (nz) {
        cn = *nz;
        if (nz->kind == DPPX_NOISE_KEYED && nz->plane_seeds) cn.plane_seeds = nz->plane_seeds + static_cast<int64_t>(f0) * C;
        if (nz->kind == DPPX_NOISE_PHILOX) cn.frame_base = nz->frame_base + f0;
      }
      PixOpts po;
      po.partial = op == HostOp::Reference;
      if (op == HostOp::AdaptiveVariance) po.var_tau = ctx->var_tau;
      po.mask_bits = bits;
      rc = pixelize_dev(ctx, &dd, dimg, dmask, pp, nz ? &cn : nullptr,
                        inj ? static_cast<const double*>(ctx->inj[s].p) : nullptr, dstats, dstride,
                        adaptive ? dlens : nullptr, out ? dout : nullptr, adaptive, ctx->sd[s],
                        ctx->sd_pinned[s], ctx->sd_pinned_n[s], ctx->comp_done[s], false, po);
    } else {
      rc = expand_dev(ctx, &dd, dstats, dstride, in_lens ? dlens : nullptr, b, n, dout, adaptive,
                      sstride);
    }
    if (rc) return rc;
    if (dense_out) {
      PendingTiming pt;
      timing_begin(ctx, DPPX_K_AUX, &pt);
      CUDA_TRY(ctx, launch_repitch(ddense_out, row, dout, dpitch, row, static_cast<int64_t>(M) * Fk, comp));
      timing_end(ctx, &pt);
    }
    CUDA_TRY(ctx, cudaEventRecord(ctx->comp_done[s], comp));
    // ---- D2H (output stream) ----
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_out, ctx->comp_done[s], 0));
    if (exact_payload) {
      // this chunk's lengths, ahead of the image copies queued on s_out
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_meta, ctx->comp_done[s], 0));
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->lens_pinned[s], dlens, sizeof(uint32_t) * Fk * C,
                                    cudaMemcpyDeviceToHost, ctx->s_meta));
      CUDA_TRY(ctx, cudaEventRecord(ctx->lens_ev[s], ctx->s_meta));
      ctx->kstats.d2h_bytes += sizeof(uint32_t) * Fk * C;
      // the previous chunk's payloads go first: its slot is released
      // (out_done) before this chunk's image copy is queued behind it
      if (ci >= 1)
        if (int rc2 = issue_payload(ci - 1)) return rc2;
    } else if (pix) {
      const size_t w = adaptive ? dppx_adaptive_payload_capacity(M, N, b, n) : G;
      CUDA_TRY(ctx, cudaMemcpy2DAsync(stats + static_cast<int64_t>(f0) * C * sstride, sstride, dstats,
                                      dstride, w, static_cast<size_t>(Fk) * C, cudaMemcpyDeviceToHost,
                                      ctx->s_out));
      ctx->kstats.d2h_bytes += static_cast<uint64_t>(w) * Fk * C;
      if (adaptive && lens) {
        CUDA_TRY(ctx, cudaMemcpyAsync(lens + static_cast<int64_t>(f0) * C, dlens, sizeof(uint32_t) * Fk * C,
                                      cudaMemcpyDeviceToHost, ctx->s_out));
        ctx->kstats.d2h_bytes += sizeof(uint32_t) * Fk * C;
      }
    }
    if (out && stage_out) {
      if (int rc2 = drain(s)) return rc2;  // chunk ci-2's rows leave the slot first
      CUDA_TRY(ctx, cudaMemcpyAsync(ctx->stg_out[s], dout, static_cast<size_t>(dfs) * Fk,
                                    cudaMemcpyDeviceToHost, ctx->s_out));
      CUDA_TRY(ctx, cudaEventRecord(ctx->stg_ev[s], ctx->s_out));
      pend_f0[s] = f0;
      pend_fk[s] = Fk;
      ctx->kstats.d2h_bytes += static_cast<uint64_t>(Fk) * M * row;
    } else if (out) {
      if (dense_out)
        CUDA_TRY(ctx, cudaMemcpyAsync(out + static_cast<int64_t>(f0) * d->out_frame_stride, ddense_out,
                                      static_cast<size_t>(row) * M * Fk, cudaMemcpyDeviceToHost,
                                      ctx->s_out));
      else
        CUDA_TRY(ctx, copy_frames(out + static_cast<int64_t>(f0) * d->out_frame_stride, d->out_pitch,
                                  d->out_frame_stride, dout, dpitch, dfs, row, M, Fk,
                                  cudaMemcpyDeviceToHost, ctx->s_out));
      ctx->kstats.d2h_bytes += static_cast<uint64_t>(Fk) * M * row;
    }
    if (!exact_payload) CUDA_TRY(ctx, cudaEventRecord(ctx->out_done[s], ctx->s_out));
    chunk_f0[ci] = f0;
    f0 += Fk;
  }
  if (exact_payload && chunks > 0)
    if (int rc2 = issue_payload(chunks - 1)) return rc2;
  if (trace) std::fprintf(stderr, "pipe: issued %.2f ms\n", tp_ms());
  for (int k = 0; k < 2; ++k) {  // oldest pending slot first
    const int s = (chunks + k) & 1;
    if (int rc2 = drain(s)) return rc2;
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->s_out));
  CUDA_TRY(ctx, cudaStreamSynchronize(comp));
  if (trace) std::fprintf(stderr, "pipe: done %.2f ms\n", tp_ms());
  if (ctx->timing) collect_timings(ctx);
  if (!pix) return read_status(ctx);
  return DPPX_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* dppx_version(void) { return "dppx-b200 1 (sm_100a)"; }

int dppx_grid_dims(int32_t M, int32_t N, int32_t b, dppx_geometry* out) {
  if (!out || M < 1 || N < 1 || b < 1 || b > std::max(M, N)) return DPPX_ERR_INVALID;
  out->b = b;  // image.cpp:59-70, 64-bit intermediates
  out->grid_rows = static_cast<int32_t>((static_cast<int64_t>(M) + b - 1) / b);
  out->grid_cols = static_cast<int32_t>((static_cast<int64_t>(N) + b - 1) / b);
  out->pad_rows = static_cast<int32_t>(static_cast<int64_t>(out->grid_rows) * b - M);
  out->pad_cols = static_cast<int32_t>(static_cast<int64_t>(out->grid_cols) * b - N);
  return DPPX_OK;
}

double dppx_sensitivity(int32_t b, int32_t m) {
  if (b < 1 || m < 1) return -1.0;
  return 255.0 * m / (static_cast<double>(b) * b);  // noise.cpp:22-27
}

int dppx_make_privacy_params(double eps, int32_t m, int32_t b, int32_t n, dppx_privacy_params* p) {
  if (!p || !(eps > 0.0) || m < 1 || b < 1 || n < 1 || b % n != 0) return DPPX_ERR_INVALID;
  p->epsilon = eps;  // noise.cpp:39-68
  p->m = m;
  p->b = b;
  p->n = n;
  p->subgrid_side = b / n;
  p->delta = dppx_sensitivity(b, m);
  p->sigma = p->delta / eps;
  p->delta_sub = dppx_sensitivity(p->subgrid_side, m);
  p->sigma_sub = p->sigma * (static_cast<double>(n) * n);
  return DPPX_OK;
}

uint64_t dppx_keyed_bits(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc) {
  return keyed_bits_h(seed, r, c, sr, sc);
}

double dppx_uniform_from_bits(uint64_t bits) {  // noise.cpp:93-105
  const double k = 0x1.0p-53, half = 0.5 - k;
  const double u = static_cast<double>(bits >> 11) * k - 0.5;
  return u <= -half ? -half : (u >= half ? half : u);
}

double dppx_laplace_at(uint64_t seed, uint32_t r, uint32_t c, uint32_t sr, uint32_t sc,
                       double sigma) {
  if (!(sigma > 0.0)) return std::nan("");
  const double u = dppx_uniform_from_bits(keyed_bits_h(seed, r, c, sr, sc));
  const double sign = u < 0.0 ? -1.0 : 1.0;  // noise.cpp:107-110
  return sign * sigma * -std::log1p(-2.0 * std::fabs(u));
}

uint64_t dppx_derive_plane_seed(uint64_t seed, uint32_t frame, uint32_t channel) {
  return keyed_bits_h(seed, frame, channel, 0xFFFFFFFFu, 0xFFFFFFFFu);
}

size_t dppx_adaptive_payload_capacity(int32_t M, int32_t N, int32_t b, int32_t n) {
  dppx_geometry g;
  if (dppx_grid_dims(M, N, b, &g) != DPPX_OK || n < 1) return 0;
  const size_t G = static_cast<size_t>(g.grid_rows) * g.grid_cols;
  return 4 * G + 4 + G * static_cast<size_t>(n) * n;
}

size_t dppx_adaptive_payload_length(int32_t M, int32_t N, int32_t b, int32_t n, uint32_t S) {
  dppx_geometry g;
  if (dppx_grid_dims(M, N, b, &g) != DPPX_OK || n < 1) return 0;
  const size_t G = static_cast<size_t>(g.grid_rows) * g.grid_cols;
  if (S > G) return 0;
  return 4 * G + 4 + S + (G - S) * static_cast<size_t>(n) * n;
}

int dppx_ctx_create(int32_t device, dppx_ctx** out) {
  if (!out) return DPPX_ERR_INVALID;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return DPPX_ERR_NO_DEVICE;
  if (device < 0 || device >= count) return DPPX_ERR_INVALID;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DPPX_ERR_NO_DEVICE;
  if (prop.major != 10 || prop.minor != 0) return DPPX_ERR_NO_DEVICE;  // built for sm_100a only
  dppx_ctx* ctx = new dppx_ctx();
  ctx->device = device;
  ctx->sms = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->s_meta, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return DPPX_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  for (int s = 0; s < 2; ++s) {
    cudaEventCreateWithFlags(&ctx->in_done[s], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->comp_done[s], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->out_done[s], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->lens_ev[s], cudaEventDisableTiming);
  }
  for (int i = 0; i < dppx_ctx::kMaxBands; ++i) {
    cudaEventCreateWithFlags(&ctx->band_in[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->band_comp[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&ctx->seeds_ev, cudaEventDisableTiming);
  cudaEventRecord(ctx->seeds_ev, ctx->stream);
  // Verify that the sm_100a kernels load on this device (no silent fallback).
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(
                                     select_stats_kernel(3, 16, 4, true, false))) != cudaSuccess) {
    dppx_ctx_destroy(ctx);
    return DPPX_ERR_NO_DEVICE;
  }
  *out = ctx;
  return DPPX_OK;
}

void dppx_ctx_destroy(dppx_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&ctx->cellinfo, &ctx->rowcnt, &ctx->rowprefix, &ctx->totals, &ctx->counters,
                    &ctx->status, &ctx->seeds, &ctx->keys, &ctx->dbl, &ctx->work,
                    &ctx->met_a, &ctx->met_b, &ctx->met_out, &ctx->var_flags, &ctx->var_stage};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (DevBuf& b : ctx->sweep_sums)
    if (b.p) cudaFree(b.p);
  for (DevBuf* b : {&ctx->check_img, &ctx->check_eq})
    if (b->p) cudaFree(b->p);
  for (int s = 0; s < 2; ++s) {
    DevBuf* sb[] = {&ctx->img[s], &ctx->mask[s], &ctx->out[s], &ctx->stats[s], &ctx->lens[s],
                    &ctx->inj[s], &ctx->sd[s], &ctx->dense[s], &ctx->dense_out[s], &ctx->dense_mask[s]};
    for (DevBuf* b : sb)
      if (b->p) cudaFree(b->p);
    if (ctx->sd_pinned[s]) cudaFreeHost(ctx->sd_pinned[s]);
    if (ctx->mbits_pinned[s]) cudaFreeHost(ctx->mbits_pinned[s]);
    if (ctx->stg_in[s]) cudaFreeHost(ctx->stg_in[s]);
    if (ctx->stg_out[s]) cudaFreeHost(ctx->stg_out[s]);
    if (ctx->stg_ev[s]) cudaEventDestroy(ctx->stg_ev[s]);
    if (ctx->piece[s]) cudaFreeHost(ctx->piece[s]);
    if (ctx->piece_ev[s]) cudaEventDestroy(ctx->piece_ev[s]);
    cudaEventDestroy(ctx->in_done[s]);
    cudaEventDestroy(ctx->comp_done[s]);
    cudaEventDestroy(ctx->out_done[s]);
    cudaEventDestroy(ctx->lens_ev[s]);
    if (ctx->lens_pinned[s]) cudaFreeHost(ctx->lens_pinned[s]);
  }
  if (ctx->seeds_pinned) cudaFreeHost(ctx->seeds_pinned);
  for (auto* fgp : ctx->graphs) delete fgp;
  if (ctx->gseeds.p) cudaFree(ctx->gseeds.p);
  if (ctx->gseeds_pinned) cudaFreeHost(ctx->gseeds_pinned);
  if (ctx->gstats_pinned) cudaFreeHost(ctx->gstats_pinned);
  for (int i = 0; i < dppx_ctx::kMaxBands; ++i) {
    cudaEventDestroy(ctx->band_in[i]);
    cudaEventDestroy(ctx->band_comp[i]);
  }
  cudaEventDestroy(ctx->seeds_ev);
  dppx::mask_packer_destroy(ctx->packer);
  for (auto& pt : ctx->pending) {
    cudaEventDestroy(pt.start);
    cudaEventDestroy(pt.stop);
  }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->own_stream);
  cudaStreamDestroy(ctx->s_in);
  cudaStreamDestroy(ctx->s_out);
  cudaStreamDestroy(ctx->s_meta);
  delete ctx;
}

const char* dppx_ctx_last_error(const dppx_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void* dppx_ctx_stream(dppx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int dppx_ctx_set_stream(dppx_ctx* ctx, void* stream) {
  if (!ctx) return DPPX_ERR_INVALID;
  cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  if (next != ctx->stream) {
    // The ctx-wide scratch (work counter, cell info, row scan, seeds) may still
    // be in use by kernels on the old stream: order the new stream after them.
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    cudaEvent_t e = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(e, ctx->stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(next, e, 0));
    ctx->event_pool.push_back(e);  // reusable: the wait captured the recorded state
  }
  ctx->stream = next;
  return DPPX_OK;
}

int dppx_ctx_synchronize(dppx_ctx* ctx) {
  if (int rc = check_ctx(ctx)) return rc;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->timing) collect_timings(ctx);
  return read_status(ctx);
}

int dppx_ctx_set_timing(dppx_ctx* ctx, int32_t on) {
  if (!ctx) return DPPX_ERR_INVALID;
  ctx->timing = on != 0;
  return DPPX_OK;
}

int dppx_ctx_get_stats(dppx_ctx* ctx, dppx_kernel_stats* out) {
  if (!ctx || !out) return DPPX_ERR_INVALID;
  if (!ctx->pending.empty()) {
    cudaSetDevice(ctx->device);
    collect_timings(ctx);
  }
  *out = ctx->kstats;
  return DPPX_OK;
}

int dppx_ctx_reset_stats(dppx_ctx* ctx) {
  if (!ctx) return DPPX_ERR_INVALID;
  if (!ctx->pending.empty()) collect_timings(ctx);
  ctx->kstats = dppx_kernel_stats{};
  return DPPX_OK;
}

int dppx_ctx_set_chunk_frames(dppx_ctx* ctx, int32_t frames) {
  if (!ctx || frames < 0) return DPPX_ERR_INVALID;
  ctx->chunk_frames = frames;
  return DPPX_OK;
}

int dppx_ctx_set_out_pad_scratch(dppx_ctx* ctx, int32_t on) {
  if (!ctx) return DPPX_ERR_INVALID;
  ctx->out_pad_scratch = on != 0;
  return DPPX_OK;
}

int dppx_ctx_set_small_frame_path(dppx_ctx* ctx, int32_t path) {
  if (!ctx) return DPPX_ERR_INVALID;
  if (path < DPPX_SMALL_AUTO || path > DPPX_SMALL_STAGED)
    return set_err(ctx, DPPX_ERR_INVALID, "unknown small-frame path");
  ctx->small_path = path;
  return DPPX_OK;
}

int dppx_ctx_set_exact_noise(dppx_ctx* ctx, int32_t on) {
  if (!ctx) return DPPX_ERR_INVALID;
  ctx->exact_noise = on != 0;
  return DPPX_OK;
}

int dppx_host_alloc(size_t bytes, void** out) {
  if (!out) return DPPX_ERR_INVALID;
  return cudaMallocHost(out, bytes) == cudaSuccess ? DPPX_OK : DPPX_ERR_OOM;
}

void dppx_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int dppx_pixelize_uniform_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                              const dppx_privacy_params* pp, const dppx_noise* nz, uint8_t* means,
                              uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_params(ctx, pp, false)) return rc;
  if (int rc = check_desc(ctx, d, false, out != nullptr)) return rc;
  BatchGeom g;
  if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, pp->b, 1, &g, true))
    return rc;
  return pixelize_dev(ctx, d, img, nullptr, pp, nz, nz ? nz->injected : nullptr, means, g.G,
                      nullptr, out, false, ctx->seeds, ctx->seeds_pinned, ctx->seeds_pinned_n,
                      ctx->seeds_ev, true);
}

int dppx_pixelize_uniform_sweep_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                                    int32_t nb, const int32_t* b_list, int32_t ne, const double* eps_list,
                                    int32_t m, const dppx_noise* nz, uint8_t* const* means,
                                    uint8_t* const* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (nb < 1 || ne < 1 || !b_list || !eps_list || !means)
    return set_err(ctx, DPPX_ERR_INVALID, "sweep lists must be non-empty");
  if (int rc = check_desc(ctx, d, false, out != nullptr)) return rc;
  // Every run is a valid pixelize_parallel call (make_privacy_params, grid_dims,
  // mirror_pad checks), as run_sweep would find it.
  std::vector<dppx_privacy_params> pp(static_cast<size_t>(nb) * ne);
  for (int i = 0; i < nb; ++i) {
    BatchGeom gi;
    if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, b_list[i], 1, &gi, true)) return rc;
    for (int j = 0; j < ne; ++j)
      if (dppx_make_privacy_params(eps_list[j], m, b_list[i], 1, &pp[i * ne + j]) != DPPX_OK)
        return set_err(ctx, DPPX_ERR_INVALID, "make_privacy_params: invalid sweep parameters");
    for (int j = 0; j < ne; ++j)
      if (!means[i * ne + j]) return set_err(ctx, DPPX_ERR_INVALID, "null means pointer");
  }
  if (d->frames == 0) return DPPX_OK;
  if (!img) return set_err(ctx, DPPX_ERR_INVALID, "null image pointer");
  // Fused one-read path?
  int bmax = 0;
  uint32_t active = 0;
  bool fused = ne <= kSweepMaxEps && (d->channels == 1 || d->channels == 3) &&
               (!nz || nz->kind != DPPX_NOISE_INJECTED) && !std::getenv("DPPX_NO_SWEEP") &&
               aligned16(img) && d->pitch % 16 == 0 && d->frame_stride % 16 == 0;
  for (int i = 0; i < nb && fused; ++i) {
    const int b = b_list[i];
    const int lv = b == 4 ? 0 : b == 8 ? 1 : b == 16 ? 2 : b == 32 ? 3 : -1;
    if (lv < 0 || (active >> lv) & 1u) fused = false;
    else active |= 1u << lv;
    bmax = std::max(bmax, b);
  }
  const int nlev = bmax == 8 ? 2 : bmax == 16 ? 3 : bmax == 32 ? 4 : 0;
  SweepSumsKernel k = fused ? select_sweep_kernel(d->channels, nlev) : nullptr;
  BatchGeom g;
  if (k && geometry(ctx, d->height, d->width, d->channels, d->frames, bmax, 1, &g, true) != DPPX_OK) {
    k = nullptr;  // the largest side's padding would exceed the image: per-run path
    ctx->err.clear();
  }
  if (!k) {
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < ne; ++j)
        if (int rc = dppx_pixelize_uniform_dev(ctx, d, img, &pp[i * ne + j], nz, means[i * ne + j],
                                               out ? out[i * ne + j] : nullptr))
          return rc;
    return DPPX_OK;
  }
  StatsArgs a{};
  a.g = g;
  a.img = img;
  a.pitch = d->pitch;
  a.fstride = d->frame_stride;
  a.exact_noise = ctx->exact_noise ? 1 : 0;
  a.row_begin = 0;
  a.row_count = g.GR;
  if (int rc = prepare_noise(ctx, nz, g.F * g.C, nullptr, g, &pp[0], &a.noise, ctx->stream, ctx->seeds,
                             ctx->seeds_pinned, ctx->seeds_pinned_n, ctx->seeds_ev, true))
    return rc;
  SweepLevels L{};
  L.nlev = nlev;
  L.ne = ne;
  L.active = active;
  L.planes = g.F * g.C;
  int64_t items = 0;
  for (int lv = 0; lv < nlev; ++lv) {
    dppx_geometry gg;
    dppx_grid_dims(d->height, d->width, 4 << lv, &gg);
    L.GR[lv] = gg.grid_rows;
    L.GC[lv] = gg.grid_cols;
    L.G[lv] = static_cast<int64_t>(gg.grid_rows) * gg.grid_cols;
    L.area[lv] = static_cast<double>(4 << lv) * (4 << lv);
    // level sums over the largest side's padded extent
    L.srows[lv] = g.GR * (bmax >> (2 + lv));
    L.scols[lv] = g.GC * (bmax >> (2 + lv));
    const size_t bytes = static_cast<size_t>(L.planes) * L.srows[lv] * L.scols[lv] * (lv == 3 ? 4 : 2);
    if (int rc = ensure(ctx, ctx->sweep_sums[lv], bytes)) return rc;
    L.sums[lv] = ctx->sweep_sums[lv].p;
    L.groups[lv] = (L.GC[lv] + 3) / 4;
    L.div_groups[lv] = make_fastdiv(static_cast<uint32_t>(L.groups[lv]));
    L.div_rows[lv] = make_fastdiv(static_cast<uint32_t>(L.GR[lv]));
    L.item0[lv] = items;
    items += static_cast<int64_t>(L.planes) * L.GR[lv] * L.groups[lv];
  }
  L.item0[nlev] = items;
  if (items > 0x7FFFFFFFll) return set_err(ctx, DPPX_ERR_INVALID, "sweep batch too large for one launch");
  for (int i = 0; i < nb; ++i) {
    const int lv = b_list[i] == 4 ? 0 : b_list[i] == 8 ? 1 : b_list[i] == 16 ? 2 : 3;
    for (int j = 0; j < ne; ++j) {
      L.sigma[lv][j] = pp[i * ne + j].sigma;
      L.sln2[lv][j] = static_cast<float>(pp[i * ne + j].sigma * 0.6931471805599453);
      L.margin[lv][j] = fast_margin(pp[i * ne + j].sigma);
      L.means[lv][j] = means[i * ne + j];
    }
  }
  const int64_t row_bytes = static_cast<int64_t>(g.N) * g.C;
  const int tile = stats_tile_px();
  a.pack = 1;
  a.slot_px = tile;
  a.slot_stride = static_cast<int>(round_up(static_cast<int64_t>(g.b) * tile * g.C, 128));
  a.row_slack = a.pitch >= round_up(row_bytes, 16) ? 1 : 0;
  const int64_t in_row = a.row_slack ? round_up(row_bytes, 16) : row_bytes / 16 * 16;
  CUtensorMap tin{};
  if (!encode_frames_map(&tin, img, in_row, g.M, g.F, a.pitch, a.fstride, tile * g.C, g.b)) {
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < ne; ++j)
        if (int rc = dppx_pixelize_uniform_dev(ctx, d, img, &pp[i * ne + j], nz, means[i * ne + j],
                                               out ? out[i * ne + j] : nullptr))
          return rc;
    return DPPX_OK;
  }
  a.tensor_in_bytes = static_cast<int>(in_row);
  a.tiles_per_row = (g.GC * g.b + tile - 1) / tile;
  const int64_t units = static_cast<int64_t>(g.F) * g.GR * a.tiles_per_row;
  if (units > 0x7FFFFFFF) return set_err(ctx, DPPX_ERR_INVALID, "batch too large for one launch");
  a.units = static_cast<int>(units);
  a.div_tiles = make_fastdiv(static_cast<uint32_t>(a.tiles_per_row));
  a.div_rows = make_fastdiv(static_cast<uint32_t>(g.GR));
  a.stages = 2;  // K1s-sum is a streaming kernel: a 2-deep ring per CTA
  const size_t smem = static_cast<size_t>(round_up(static_cast<int64_t>(g.b) * tile * g.C, 128)) * 2;
  const auto key = std::make_pair(reinterpret_cast<const void*>(k), smem);
  int per_sm = 0;
  auto it = ctx->occupancy.find(key);
  if (it == ctx->occupancy.end()) {
    CUDA_TRY(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, stats_threads(), smem));
    ctx->occupancy[key] = per_sm;
  } else {
    per_sm = it->second;
  }
  const int grid = static_cast<int>(std::min<int64_t>(units, static_cast<int64_t>(std::max(per_sm, 1)) * ctx->sms));
  if (int rc = ensure(ctx, ctx->work, 16, /*zero=*/true)) return rc;
  a.work_counter = static_cast<int*>(ctx->work.p);
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_SWEEP, &pt);
  CUDA_TRY(ctx, launch_sweep_sums(k, tin, a, L, grid, smem, ctx->stream));
  // Draws, largest grid side first. The broadcasts of the larger sides
  // (write-only, HBM-bound) then run on a second stream while the 4-px level's
  // draws (compute-bound, ~3/4 of all statistics) run on the first.
  const int max_draw_grid = 8 * ctx->sms;
  auto draw_levels = [&](int lo, int hi) -> int {  // levels [lo, hi)
    SweepLevels Ld = L;
    Ld.item_begin = L.item0[lo];
    Ld.item_end = L.item0[hi];
    CUDA_TRY(ctx, launch_sweep_draw(a, Ld, max_draw_grid, ctx->stream));
    return DPPX_OK;
  };
  if (nlev > 1)
    if (int rc = draw_levels(1, nlev)) return rc;
  auto broadcast_runs = [&](bool level0) -> int {
    for (int i = 0; i < nb; ++i) {
      if ((b_list[i] == 4) != level0) continue;
      for (int j = 0; j < ne; ++j)
        if (out[i * ne + j]) {
          dppx_geometry gg;
          dppx_grid_dims(d->height, d->width, b_list[i], &gg);
          if (int rc = expand_dev(ctx, d, means[i * ne + j], static_cast<int64_t>(gg.grid_rows) * gg.grid_cols,
                                  nullptr, b_list[i], 1, out[i * ne + j], false))
            return rc;
        }
    }
    return DPPX_OK;
  };
  cudaStream_t main_stream = ctx->stream;
  cudaEvent_t big_ready = nullptr, aux_done = nullptr;
  if (out) {
    big_ready = get_event(ctx);
    aux_done = get_event(ctx);
    CUDA_TRY(ctx, cudaEventRecord(big_ready, main_stream));
    CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->s_in, big_ready, 0));
    ctx->stream = ctx->s_in;  // (the expanders launch on ctx->stream)
    const int rc = broadcast_runs(false);
    ctx->stream = main_stream;
    if (rc) return rc;
    CUDA_TRY(ctx, cudaEventRecord(aux_done, ctx->s_in));
  }
  if (active & 1u)
    if (int rc = draw_levels(0, 1)) return rc;
  timing_end(ctx, &pt);
  if (out) {
    if (int rc = broadcast_runs(true)) return rc;
    CUDA_TRY(ctx, cudaStreamWaitEvent(main_stream, aux_done, 0));  // join
    ctx->event_pool.push_back(big_ready);
    ctx->event_pool.push_back(aux_done);
  }
  return DPPX_OK;
}

namespace {
int metric_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b, bool ssim,
               double* out);
}  // namespace

int dppx_pixelize_uniform_sweep(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img, int32_t nb,
                                const int32_t* b_list, int32_t ne, const double* eps_list, int32_t m,
                                const dppx_noise* nz, uint8_t* const* means, uint8_t* const* out,
                                double* mse_out, double* ssim_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (nb < 1 || ne < 1 || !b_list || !eps_list || !means)
    return set_err(ctx, DPPX_ERR_INVALID, "sweep lists must be non-empty");
  const bool want_img = out != nullptr || mse_out != nullptr || ssim_out != nullptr;
  if (int rc = check_desc(ctx, d, false, want_img)) return rc;
  const int F = d->frames, M = d->height, N = d->width, C = d->channels;
  if (F == 0) return DPPX_OK;
  if (!img) return set_err(ctx, DPPX_ERR_INVALID, "null image pointer");
  if (C < 1 || C > 4) return set_err(ctx, DPPX_ERR_INVALID, "channels must be 1..4");
  const int runs = nb * ne;
  const int64_t row = static_cast<int64_t>(N) * C;
  const int64_t dpitch = round_up(row, 16), dfs = dpitch * M;
  std::vector<int64_t> G(static_cast<size_t>(nb));
  int64_t means_bytes = 0;
  for (int i = 0; i < nb; ++i) {
    dppx_geometry gg;
    if (dppx_grid_dims(M, N, b_list[i], &gg) != DPPX_OK)
      return set_err(ctx, DPPX_ERR_INVALID, "grid_dims: grid side b exceeds both image dimensions");
    G[i] = static_cast<int64_t>(gg.grid_rows) * gg.grid_cols;
    means_bytes += round_up(G[i] * F * C, 256) * ne;
  }
  // device: frames, every run's means and (when wanted) image
  if (ensure(ctx, ctx->img[0], static_cast<size_t>(dfs) * F)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->check_img, static_cast<size_t>(means_bytes))) return DPPX_ERR_OOM;
  if (want_img && ensure(ctx, ctx->out[0], static_cast<size_t>(dfs) * F * runs)) return DPPX_ERR_OOM;
  uint8_t* dimg = static_cast<uint8_t*>(ctx->img[0].p);
  uint8_t* dout = static_cast<uint8_t*>(ctx->out[0].p);
  std::vector<uint8_t*> dmeans(static_cast<size_t>(runs)), douts(static_cast<size_t>(runs), nullptr);
  {
    uint8_t* q = static_cast<uint8_t*>(ctx->check_img.p);
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < ne; ++j) {
        dmeans[i * ne + j] = q;
        q += round_up(G[i] * F * C, 256);
        if (want_img) douts[i * ne + j] = dout + static_cast<int64_t>(i * ne + j) * dfs * F;
      }
  }
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->s_out));
  if (int rc = h2d_frames(ctx, dimg, dpitch, dfs, img, d->pitch, d->frame_stride, row, M, F, st)) return rc;
  ctx->kstats.h2d_bytes += static_cast<uint64_t>(row) * M * F;
  dppx_frames_desc dd = *d;
  dd.pitch = dpitch;
  dd.frame_stride = dfs;
  dd.out_pitch = dpitch;
  dd.out_frame_stride = dfs;
  {
    struct PadScratch {  // the run images are the ctx's own buffers
      dppx_ctx* c;
      bool prev;
      ~PadScratch() { c->out_pad_scratch = prev; }
    } pad_scope{ctx, ctx->out_pad_scratch};
    ctx->out_pad_scratch = true;
    if (int rc = dppx_pixelize_uniform_sweep_dev(ctx, &dd, dimg, nb, b_list, ne, eps_list, m, nz, dmeans.data(),
                                                 want_img ? douts.data() : nullptr))
      return rc;
  }
  for (int r = 0; r < runs; ++r) {  // mse / ssim of every run's image, where it lives
    if (mse_out)
      if (int rc = metric_dev(ctx, &dd, dimg, douts[r], false, mse_out + static_cast<int64_t>(r) * F * C)) return rc;
    if (ssim_out && M >= 7 && N >= 7)
      if (int rc = metric_dev(ctx, &dd, dimg, douts[r], true, ssim_out + static_cast<int64_t>(r) * F * C)) return rc;
  }
  for (int r = 0; r < runs; ++r) {
    const int i = r / ne;
    if (out && out[r]) {
      if (int rc = d2h_frames(ctx, out[r], d->out_pitch, d->out_frame_stride, douts[r], dpitch, dfs, row, M, F, st))
        return rc;
      ctx->kstats.d2h_bytes += static_cast<uint64_t>(row) * M * F;
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(means[r], dmeans[r], static_cast<size_t>(G[i] * F * C), cudaMemcpyDeviceToHost, st));
    ctx->kstats.d2h_bytes += static_cast<uint64_t>(G[i]) * F * C;
  }
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (ctx->timing) collect_timings(ctx);
  return DPPX_OK;
}

int dppx_pixelize_adaptive_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                               const uint8_t* mask, const dppx_privacy_params* pp,
                               const dppx_noise* nz, uint8_t* payload, int64_t payload_stride,
                               uint32_t* payload_len, uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_params(ctx, pp, true)) return rc;
  if (int rc = check_desc(ctx, d, true, out != nullptr)) return rc;
  return pixelize_dev(ctx, d, img, mask, pp, nz, nz ? nz->injected : nullptr, payload,
                      payload_stride, payload_len, out, true, ctx->seeds, ctx->seeds_pinned,
                      ctx->seeds_pinned_n, ctx->seeds_ev, true);
}

int dppx_broadcast_means_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* means,
                             int32_t b, uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_desc(ctx, d, false, true)) return rc;
  dppx_geometry gg;
  if (dppx_grid_dims(d->height, d->width, b, &gg) != DPPX_OK)
    return set_err(ctx, DPPX_ERR_INVALID, "broadcast_means: means do not fit the target dimensions");
  return expand_dev(ctx, d, means, static_cast<int64_t>(gg.grid_rows) * gg.grid_cols, nullptr, b, 1,
                    out, false);
}

int dppx_reassemble_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* payload,
                        int64_t payload_stride, const uint32_t* payload_len, int32_t b, int32_t n,
                        uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_desc(ctx, d, false, true)) return rc;
  if (int rc = ensure(ctx, ctx->status, 16, true)) return rc;
  return expand_dev(ctx, d, payload, payload_stride, payload_len, b, n, out, true);
}

int dppx_synth_frames_dev(dppx_ctx* ctx, const dppx_frames_desc* d, uint32_t data_seed, uint32_t f0,
                          uint8_t* img, uint8_t* mask) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_desc(ctx, d, mask != nullptr, false)) return rc;
  if (!img) return set_err(ctx, DPPX_ERR_INVALID, "null image pointer");
  BatchGeom g{};
  g.M = d->height;
  g.N = d->width;
  g.C = d->channels;
  g.F = d->frames;
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_AUX, &pt);
  CUDA_TRY(ctx, launch_synth(g, data_seed, f0, img, d->pitch, d->frame_stride, mask, d->mask_pitch,
                             d->mask_frame_stride, ctx->stream));
  timing_end(ctx, &pt);
  return DPPX_OK;
}

int dppx_pixelize_uniform(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                          const dppx_privacy_params* pp, const dppx_noise* nz, uint8_t* means,
                          uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return host_pipeline(ctx, HostOp::Uniform, d, img, nullptr, pp, nz, means, 0, nullptr, nullptr, 0,
                       1, out);
}

int dppx_pixelize_adaptive(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                           const uint8_t* mask, const dppx_privacy_params* pp, const dppx_noise* nz,
                           uint8_t* payload, int64_t payload_stride, uint32_t* payload_len,
                           uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return host_pipeline(ctx, HostOp::Adaptive, d, img, mask, pp, nz, payload, payload_stride,
                       payload_len, nullptr, 0, 0, out);
}

int dppx_pixelize_reference(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                            const dppx_privacy_params* pp, const dppx_noise* nz, uint8_t* means,
                            uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (pp && pp->n != 1) return set_err(ctx, DPPX_ERR_INVALID, "pixelize_reference: requires n == 1");
  return host_pipeline(ctx, HostOp::Reference, d, img, nullptr, pp, nz, means, 0, nullptr, nullptr, 0,
                       1, out);
}

int dppx_pixelize_adaptive_variance(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* img,
                                    double var_tau, const dppx_privacy_params* pp,
                                    const dppx_noise* nz, uint8_t* payload, int64_t payload_stride,
                                    uint32_t* payload_len, uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!(var_tau >= 0.0)) return set_err(ctx, DPPX_ERR_INVALID, "variance threshold must be >= 0");
  ctx->var_tau = var_tau;
  return host_pipeline(ctx, HostOp::AdaptiveVariance, d, img, nullptr, pp, nz, payload,
                       payload_stride, payload_len, nullptr, 0, 0, out);
}

static PixOpts var_opts(double tau) {
  PixOpts o;
  o.var_tau = tau;
  return o;
}

int dppx_pixelize_adaptive_variance_dev(dppx_ctx* ctx, const dppx_frames_desc* d,
                                        const uint8_t* img, double var_tau,
                                        const dppx_privacy_params* pp, const dppx_noise* nz,
                                        uint8_t* payload, int64_t payload_stride,
                                        uint32_t* payload_len, uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_params(ctx, pp, true)) return rc;
  if (int rc = check_desc(ctx, d, false, out != nullptr)) return rc;
  if (!(var_tau >= 0.0)) return set_err(ctx, DPPX_ERR_INVALID, "variance threshold must be >= 0");
  return pixelize_dev(ctx, d, img, nullptr, pp, nz, nz ? nz->injected : nullptr, payload,
                      payload_stride, payload_len, out, true, ctx->seeds, ctx->seeds_pinned,
                      ctx->seeds_pinned_n, ctx->seeds_ev, true, var_opts(var_tau));
}

int dppx_broadcast_means(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* means, int32_t b,
                         uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (d) {
    dppx_geometry gg;
    if (dppx_grid_dims(d->height, d->width, b, &gg) != DPPX_OK)
      return set_err(ctx, DPPX_ERR_INVALID, "broadcast_means: means do not fit the target dimensions");
  }
  return host_pipeline(ctx, HostOp::Broadcast, d, nullptr, nullptr, nullptr, nullptr,
                       const_cast<uint8_t*>(means), 0, nullptr, nullptr, b, 1, out);
}

int dppx_reconstruct_record(dppx_ctx* ctx, const uint8_t* bytes, size_t len, uint8_t* out,
                            size_t out_cap) {
  if (int rc = check_ctx(ctx)) return rc;
  dppx_record_info info{};
  if (int rc = dppx_decode_record(bytes, len, &info))
    return set_err(ctx, rc, "decode: record rejected (status %d)", rc);
  const size_t need = static_cast<size_t>(info.height) * static_cast<size_t>(info.width);
  if (!out || out_cap < need) return set_err(ctx, DPPX_ERR_INVALID, "reconstruct: output too small");
  dppx_frames_desc d{};
  d.height = info.height;
  d.width = info.width;
  d.channels = 1;
  d.frames = 1;
  d.pitch = d.mask_pitch = d.out_pitch = info.width;
  d.frame_stride = d.mask_frame_stride = d.out_frame_stride = static_cast<int64_t>(need);
  const uint8_t* payload = bytes + info.payload_offset;
  if (info.mode == 1) return dppx_broadcast_means(ctx, &d, payload, info.b, out);
  const uint32_t plen = info.payload_len;
  return dppx_reassemble(ctx, &d, payload, static_cast<int64_t>((plen + 3) & ~3u), &plen, info.b,
                         info.n, out);
}

int dppx_reassemble(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* payload,
                    int64_t payload_stride, const uint32_t* payload_len, int32_t b, int32_t n,
                    uint8_t* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = ensure(ctx, ctx->status, 16, true)) return rc;
  return host_pipeline(ctx, HostOp::Reassemble, d, nullptr, nullptr, nullptr, nullptr,
                       const_cast<uint8_t*>(payload), payload_stride, nullptr, payload_len, b, n,
                       out);
}

int dppx_classify_regions(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* mask, int32_t b,
                          float* mask_means) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!d || !mask || !mask_means) return set_err(ctx, DPPX_ERR_INVALID, "null argument");
  if (d->mask_pitch < d->width || d->mask_frame_stride < d->mask_pitch * d->height)
    return set_err(ctx, DPPX_ERR_INVALID, "mask pitch/frame_stride too small");
  BatchGeom g;
  if (int rc = geometry(ctx, d->height, d->width, 1, d->frames, b, 1, &g, true)) return rc;
  if (g.F == 0) return DPPX_OK;
  const int64_t mp = round_up(g.N, 16), mfs = mp * g.M;
  const int64_t ps = round_up(4ll * g.G + 4, 16);
  if (int rc = ensure(ctx, ctx->mask[0], static_cast<size_t>(mfs) * g.F)) return rc;
  if (int rc = ensure(ctx, ctx->stats[0], static_cast<size_t>(ps) * g.F)) return rc;
  if (int rc = ensure_scratch(ctx, g, g.F)) return rc;
  for (int f = 0; f < g.F; ++f)
    CUDA_TRY(ctx, cudaMemcpy2DAsync(static_cast<uint8_t*>(ctx->mask[0].p) + f * mfs, mp,
                                    mask + static_cast<int64_t>(f) * d->mask_frame_stride,
                                    d->mask_pitch, g.N, g.M, cudaMemcpyHostToDevice, ctx->stream));
  if (int rc = classify(ctx, g, g.F, false, static_cast<const uint8_t*>(ctx->mask[0].p), mp, mfs,
                        static_cast<uint8_t*>(ctx->stats[0].p), nullptr, ps, nullptr, nullptr))
    return rc;
  CUDA_TRY(ctx, cudaMemcpy2DAsync(mask_means, 4ll * g.G, ctx->stats[0].p, ps, 4ll * g.G, g.F,
                                  cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->timing) collect_timings(ctx);
  return DPPX_OK;
}

int dppx_debug_device_laplace(dppx_ctx* ctx, uint64_t seed, const uint32_t* keys, int32_t count,
                              double sigma, double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (count <= 0 || !keys || !out) return set_err(ctx, DPPX_ERR_INVALID, "bad arguments");
  if (int rc = ensure(ctx, ctx->keys, sizeof(uint32_t) * 4 * count)) return rc;
  if (int rc = ensure(ctx, ctx->dbl, sizeof(double) * count)) return rc;
  CUDA_TRY(ctx, cudaMemcpy(ctx->keys.p, keys, sizeof(uint32_t) * 4 * count, cudaMemcpyHostToDevice));
  CUDA_TRY(ctx, launch_debug_laplace(mix64_h(seed), static_cast<const uint32_t*>(ctx->keys.p), count,
                                     sigma, static_cast<double*>(ctx->dbl.p), ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(ctx, cudaMemcpy(out, ctx->dbl.p, sizeof(double) * count, cudaMemcpyDeviceToHost));
  return DPPX_OK;
}

// ---- utility metrics (metrics.cpp:26-183) ----------------------------------
namespace {
int metric_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
               bool ssim, double* out) {
  if (!d || !a || !b || !out) return set_err(ctx, DPPX_ERR_INVALID, "null argument");
  const int M = d->height, N = d->width, C = d->channels, F = d->frames;
  if (M < 1 || N < 1 || C < 1 || C > 4 || F < 0)
    return set_err(ctx, DPPX_ERR_INVALID, ssim ? "ssim: images must share dimensions"
                                               : "mse: images must share valid dimensions");
  if (ssim && (M < 7 || N < 7))
    return set_err(ctx, DPPX_ERR_INVALID, "ssim: images smaller than the 7x7 window");
  if (F == 0) return DPPX_OK;
  MetricArgs m{M, N, C, F, a, d->pitch, d->frame_stride, b, d->out_pitch, d->out_frame_stride,
               nullptr, nullptr};
  const int64_t P = static_cast<int64_t>(F) * C;
  const int64_t pr = M - 6;
  if (int rc = ensure(ctx, ctx->met_out, static_cast<size_t>(ssim ? P * pr * 8 : P * 8))) return rc;
  if (ssim) {
    m.row_sums = static_cast<double*>(ctx->met_out.p);
  } else {
    m.sums = static_cast<unsigned long long*>(ctx->met_out.p);
    CUDA_TRY(ctx, cudaMemsetAsync(m.sums, 0, P * 8, ctx->stream));
  }
  PendingTiming pt;
  timing_begin(ctx, DPPX_K_AUX, &pt);
  CUDA_TRY(ctx, launch_metrics(m, ssim, ctx->stream));
  timing_end(ctx, &pt);
  if (ssim) {
    std::vector<double> rows(static_cast<size_t>(P * pr));
    CUDA_TRY(ctx, cudaMemcpyAsync(rows.data(), m.row_sums, rows.size() * 8, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const double positions = static_cast<double>(pr) * (N - 6);
    for (int64_t p = 0; p < P; ++p) {  // row partials summed in row order (metrics.cpp:178-182)
      double total = 0.0;
      for (int64_t i = 0; i < pr; ++i) total += rows[p * pr + i];
      out[p] = total / positions;
    }
  } else {
    std::vector<unsigned long long> sums(static_cast<size_t>(P));
    CUDA_TRY(ctx, cudaMemcpyAsync(sums.data(), m.sums, P * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    for (int64_t p = 0; p < P; ++p)
      out[p] = static_cast<double>(sums[p]) / static_cast<double>(static_cast<int64_t>(M) * N);
  }
  if (ctx->timing) collect_timings(ctx);
  return DPPX_OK;
}

int metric_host(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
                double* mse_out, double* ssim_out) {
  if (!d || !a || !b || (!mse_out && !ssim_out)) return set_err(ctx, DPPX_ERR_INVALID, "null argument");
  if (d->height < 1 || d->width < 1 || d->channels < 1 || d->channels > 4 || d->frames < 0)
    return set_err(ctx, DPPX_ERR_INVALID, "metrics: invalid dimensions");
  const int M = d->height, F = d->frames;
  const int64_t row = static_cast<int64_t>(d->width) * d->channels;
  if (d->pitch < row || d->out_pitch < row)
    return set_err(ctx, DPPX_ERR_INVALID, "metrics: pitch too small");
  const int64_t fs = row * M;
  if (int rc = ensure(ctx, ctx->met_a, static_cast<size_t>(fs * F))) return rc;
  if (int rc = ensure(ctx, ctx->met_b, static_cast<size_t>(fs * F))) return rc;
  auto* da = static_cast<uint8_t*>(ctx->met_a.p);
  auto* db = static_cast<uint8_t*>(ctx->met_b.p);
  if (int rc = h2d_frames(ctx, da, row, fs, a, d->pitch, d->frame_stride, row, M, F, ctx->stream)) return rc;
  if (int rc = h2d_frames(ctx, db, row, fs, b, d->out_pitch, d->out_frame_stride, row, M, F, ctx->stream))
    return rc;
  dppx_frames_desc dd = *d;
  dd.pitch = dd.out_pitch = row;
  dd.frame_stride = dd.out_frame_stride = fs;
  if (mse_out)
    if (int rc = metric_dev(ctx, &dd, da, db, false, mse_out)) return rc;
  if (ssim_out)
    if (int rc = metric_dev(ctx, &dd, da, db, true, ssim_out)) return rc;
  return DPPX_OK;
}
}  // namespace

int dppx_mse(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
             double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return metric_host(ctx, d, a, b, out, nullptr);
}

int dppx_ssim(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
              double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return metric_host(ctx, d, a, b, nullptr, out);
}

int dppx_metrics(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
                 double* mse_out, double* ssim_out) {
  if (int rc = check_ctx(ctx)) return rc;
  return metric_host(ctx, d, a, b, mse_out, ssim_out);
}

namespace {
// Validated geometry + the device buffers of one dppx_pixelize_checked call
// (shared with dppx_pixelize_checked_reserve, which only sizes them).
struct CheckedLayout {
  BatchGeom g;
  size_t G = 0, cap = 0;
  int64_t row = 0, dpitch = 0, dfs = 0, dmpitch = 0, dmfs = 0, dstride = 0;
  int P = 0;
};

int checked_layout(dppx_ctx* ctx, int32_t mode, const dppx_frames_desc* d, const dppx_privacy_params* pp,
                   CheckedLayout* L) {
  if (mode < 0 || mode > 2) return set_err(ctx, DPPX_ERR_INVALID, "unknown mode");
  const bool adaptive = mode == 1, reference = mode == 2;
  if (int rc = check_params(ctx, pp, adaptive)) return rc;
  if (int rc = check_desc(ctx, d, adaptive, true)) return rc;
  BatchGeom& g = L->g;
  if (int rc = geometry(ctx, d->height, d->width, d->channels, d->frames, pp->b, adaptive ? pp->n : 1, &g,
                        !reference))
    return rc;
  if (g.F > 65535) return set_err(ctx, DPPX_ERR_INVALID, "at most 65535 frames per call");
  L->G = static_cast<size_t>(g.G);
  L->cap = adaptive ? dppx_adaptive_payload_capacity(g.M, g.N, g.b, g.n) : L->G;
  L->row = static_cast<int64_t>(g.N) * g.C;
  L->dpitch = round_up(L->row, 16), L->dfs = L->dpitch * g.M;
  L->dmpitch = round_up(g.N, 16), L->dmfs = L->dmpitch * g.M;
  L->dstride = adaptive ? round_up(static_cast<int64_t>(L->cap), 16) : static_cast<int64_t>(L->G);
  L->P = g.F * g.C;
  return DPPX_OK;
}

int checked_buffers(dppx_ctx* ctx, int32_t mode, const CheckedLayout& L) {
  const bool adaptive = mode == 1, reference = mode == 2;
  const int F = L.g.F;
  if (ensure(ctx, ctx->img[0], static_cast<size_t>(L.dfs) * F)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->out[0], static_cast<size_t>(L.dfs) * F)) return DPPX_ERR_OOM;
  if (adaptive && ensure(ctx, ctx->mask[0], static_cast<size_t>(L.dmfs) * F)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->stats[0], static_cast<size_t>(L.dstride) * L.P)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->lens[0], sizeof(uint32_t) * L.P)) return DPPX_ERR_OOM;
  if (!reference && ensure(ctx, ctx->check_img, static_cast<size_t>(L.dfs) * F)) return DPPX_ERR_OOM;
  if (ensure(ctx, ctx->check_eq, sizeof(uint32_t) * F)) return DPPX_ERR_OOM;
  return DPPX_OK;
}
}  // namespace

int dppx_pixelize_checked_reserve(dppx_ctx* ctx, int32_t mode, const dppx_frames_desc* d,
                                  const dppx_privacy_params* pp) {
  if (int rc = check_ctx(ctx)) return rc;
  CheckedLayout L;
  if (int rc = checked_layout(ctx, mode, d, pp, &L)) return rc;
  if (L.g.F == 0) return DPPX_OK;
  static const bool trace = std::getenv("DPPX_CHECKED_TRACE") != nullptr;
  auto T = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "reserve: %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(t - T).count());
    T = t;
  };
  if (int rc = checked_buffers(ctx, mode, L)) return rc;
  phase("device buffers");
  // the scratch pixelize_dev sizes per call, and the two pinned pieces
  // pageable uploads / downloads go through
  if (int rc = ensure_scratch(ctx, L.g, L.P)) return rc;
  if (int rc = ensure(ctx, ctx->met_out, static_cast<size_t>(L.P) * std::max(L.g.M - 6, 1) * 8)) return rc;
  phase("scratch");
  const int64_t per = piece_rows(L.dpitch);
  for (int s = 0; s < 2; ++s) {
    if (int rc = grow_pinned(ctx, ctx->piece[s], ctx->piece_n[s], static_cast<size_t>(per * L.dpitch)))
      return rc;
    if (!ctx->piece_ev[s]) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->piece_ev[s], cudaEventDisableTiming));
  }
  phase("pinned pieces");
  return DPPX_OK;
}

int dppx_pixelize_checked(dppx_ctx* ctx, int32_t mode, const dppx_frames_desc* d, const uint8_t* img,
                          const uint8_t* mask, const dppx_privacy_params* pp, const dppx_noise* nz,
                          uint8_t* stats, int64_t stride, uint32_t* lens, uint8_t* out, uint8_t* recon_ok,
                          double* mse, double* ssim) {
  if (int rc = check_ctx(ctx)) return rc;
  CheckedLayout L;
  if (int rc = checked_layout(ctx, mode, d, pp, &L)) return rc;
  const bool adaptive = mode == 1, reference = mode == 2;
  const BatchGeom& g = L.g;
  const int F = g.F, C = g.C, M = g.M, N = g.N;
  if (F == 0) return DPPX_OK;
  if (!img || !out || !mse || (!reference && !stats) || (adaptive && !mask))
    return set_err(ctx, DPPX_ERR_INVALID, "null image/output/statistics/mask/mse pointer");
  const size_t G = L.G, cap = L.cap;
  if (adaptive && stride < static_cast<int64_t>(cap))
    return set_err(ctx, DPPX_ERR_INVALID, "payload_stride too small");
  const int64_t row = L.row, dpitch = L.dpitch, dfs = L.dfs, dmpitch = L.dmpitch, dmfs = L.dmfs,
                dstride = L.dstride;
  const int P = L.P;
  if (int rc = checked_buffers(ctx, mode, L)) return rc;
  uint8_t* dimg = static_cast<uint8_t*>(ctx->img[0].p);
  uint8_t* dout = static_cast<uint8_t*>(ctx->out[0].p);
  uint8_t* dmask = static_cast<uint8_t*>(ctx->mask[0].p);
  uint8_t* dstats = static_cast<uint8_t*>(ctx->stats[0].p);
  uint32_t* dlens = static_cast<uint32_t*>(ctx->lens[0].p);
  uint32_t* deq = static_cast<uint32_t*>(ctx->check_eq.p);
  cudaStream_t st = ctx->stream;
  // DPPX_CHECKED_TRACE=1: per-phase wall times on stderr (synchronizes).
  static const bool trace = std::getenv("DPPX_CHECKED_TRACE") != nullptr;
  auto T = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "checked: %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(t - T).count());
    T = t;
  };
  // the previous host call's copies out of the staging buffers are done
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->s_out));
  // ---- one upload of frames (and masks) ----
  if (int rc = h2d_frames(ctx, dimg, dpitch, dfs, img, d->pitch, d->frame_stride, row, M, F, st)) return rc;
  ctx->kstats.h2d_bytes += static_cast<uint64_t>(row) * M * F;
  if (adaptive) {
    if (int rc = h2d_frames(ctx, dmask, dmpitch, dmfs, mask, d->mask_pitch, d->mask_frame_stride, N, M, F, st))
      return rc;
    ctx->kstats.h2d_bytes += static_cast<uint64_t>(N) * M * F;
  }
  phase("upload");
  dppx_frames_desc dd = *d;
  dd.pitch = dpitch;
  dd.frame_stride = dfs;
  dd.mask_pitch = dmpitch;
  dd.mask_frame_stride = dmfs;
  dd.out_pitch = dpitch;
  dd.out_frame_stride = dfs;
  {
    struct PadScratch {  // dout / check_img are the ctx's own buffers
      dppx_ctx* c;
      bool prev;
      ~PadScratch() { c->out_pad_scratch = prev; }
    } pad_scope{ctx, ctx->out_pad_scratch};
    ctx->out_pad_scratch = true;
    PixOpts po;
    po.partial = reference;
    if (int rc = pixelize_dev(ctx, &dd, dimg, dmask, pp, nz, nullptr, dstats, dstride, adaptive ? dlens : nullptr,
                              dout, adaptive, ctx->seeds, ctx->seeds_pinned, ctx->seeds_pinned_n, ctx->seeds_ev,
                              true, po))
      return rc;
    // ---- reconstruct check on the device: the statistics just produced,
    // expanded again, must equal the emitted frames (cli.cpp:135-146) ----
    CUDA_TRY(ctx, cudaMemsetAsync(deq, 0xFF, sizeof(uint32_t) * F, st));
    if (!reference) {
      uint8_t* drb = static_cast<uint8_t*>(ctx->check_img.p);
      if (int rc = expand_dev(ctx, &dd, dstats, dstride, adaptive ? dlens : nullptr, g.b, g.n, drb, adaptive))
        return rc;
      CUDA_TRY(ctx, launch_frames_equal(dout, drb, dpitch, dfs, row, M, F, deq, st));
    }
  }
  phase("pixelize+check");
  // ---- mse / ssim of input vs emitted frames, both resident (cli.cpp:164-171) ----
  dppx_frames_desc dm = dd;  // a = input (pitch), b = output (out_pitch)
  if (int rc = metric_dev(ctx, &dm, dimg, dout, false, mse)) return rc;
  if (ssim && M >= 7 && N >= 7)
    if (int rc = metric_dev(ctx, &dm, dimg, dout, true, ssim)) return rc;
  phase("metrics");
  // ---- results out ----
  if (int rc = d2h_frames(ctx, out, d->out_pitch, d->out_frame_stride, dout, dpitch, dfs, row, M, F, st))
    return rc;
  phase("download frames");
  ctx->kstats.d2h_bytes += static_cast<uint64_t>(row) * M * F;
  std::vector<uint32_t> eq(static_cast<size_t>(F));
  CUDA_TRY(ctx, cudaMemcpyAsync(eq.data(), deq, sizeof(uint32_t) * F, cudaMemcpyDeviceToHost, st));
  std::vector<uint32_t> ln(static_cast<size_t>(P), static_cast<uint32_t>(G));
  if (adaptive)
    CUDA_TRY(ctx, cudaMemcpyAsync(ln.data(), dlens, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  if (!reference) {
    size_t w = 0;
    for (int q = 0; q < P; ++q) w = std::max<size_t>(w, std::min<size_t>(ln[q], cap));
    const int64_t hs = adaptive ? stride : static_cast<int64_t>(G);
    CUDA_TRY(ctx, cudaMemcpy2D(stats, hs, dstats, dstride, w, static_cast<size_t>(P), cudaMemcpyDeviceToHost));
    ctx->kstats.d2h_bytes += static_cast<uint64_t>(w) * P;
    if (adaptive && lens) std::memcpy(lens, ln.data(), sizeof(uint32_t) * P);
  }
  phase("download statistics");
  // (K0 run on the payloads just produced cannot flag them; if it ever did,
  // every frame fails the check instead of leaving the status set)
  const bool corrupt = read_status(ctx) != DPPX_OK;
  if (recon_ok)
    for (int f = 0; f < F; ++f) recon_ok[f] = (eq[f] != 0 && !corrupt) ? 1 : 0;
  if (ctx->timing) collect_timings(ctx);
  return DPPX_OK;
}

int dppx_mse_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
                 double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return metric_dev(ctx, d, a, b, false, out);
}

int dppx_ssim_dev(dppx_ctx* ctx, const dppx_frames_desc* d, const uint8_t* a, const uint8_t* b,
                  double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  return metric_dev(ctx, d, a, b, true, out);
}

int dppx_debug_lg2_max_error(dppx_ctx* ctx, double* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!out) return set_err(ctx, DPPX_ERR_INVALID, "null output");
  if (int rc = ensure(ctx, ctx->keys, 16)) return rc;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->keys.p, 0, 4, ctx->stream));
  CUDA_TRY(ctx, launch_debug_lg2(static_cast<unsigned int*>(ctx->keys.p), ctx->stream));
  unsigned int bits = 0;
  CUDA_TRY(ctx, cudaMemcpyAsync(&bits, ctx->keys.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  float f;
  std::memcpy(&f, &bits, 4);
  *out = f;
  return DPPX_OK;
}

}  // extern "C"
