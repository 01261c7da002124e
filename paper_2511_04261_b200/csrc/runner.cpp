// runner.cpp -- the host side around the path: PGM ingest (pgm.hpp), the
// multi-GPU batch runner (batch.hpp) and the reference's orchestration API
// (cli.hpp: run_single / run_batch / run_sweep / run_bench / run_reconstruct /
// run_verify / exit_code_for, cli.cpp:93-401 semantics) over the GPU drop-in.
//
// PGM files are read with one read of the whole file and parsed from memory
// (a cursor over the bytes, no iostream tokenizing). The batch runner reads
// files on host threads, groups frames by shape and sends up to
// frames_per_call frames per C-ABI call; the calls of all shape groups are
// claimed dynamically by the workers of a device group (one host thread +
// dppx_ctx per GPU), each running its chunk's pixelize, records, GPU
// reconstruct check and GPU metrics on its own device.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <tuple>
#include <utility>

#include "dppix/adaptive.hpp"
#include "dppix/batch.hpp"
#include "dppix/cli.hpp"
#include "dppix/errors.hpp"
#include "dppix/pgm.hpp"
#include "dppix/pixelize.hpp"
#include "dppix/record.hpp"
#include "dppx_gpu.h"

namespace dppix {
namespace fs = std::filesystem;

dppx_ctx* dropin_thread_ctx();  // dropin.cpp: the calling thread's context

namespace {

// ---------------------------------------------------------------- PGM bytes
// Whole file in memory (one fread); a missing / unreadable file is an IoError.
std::vector<std::uint8_t> slurp(const std::string& path, const char* who) {
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
  if (!f) throw IoError(std::string(who) + ": cannot open " + path);
  struct stat st {};
  std::vector<std::uint8_t> buf;
  if (fstat(fileno(f.get()), &st) == 0 && st.st_size > 0) buf.resize(static_cast<size_t>(st.st_size));
  size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), f.get());
  buf.resize(got);
  return buf;
}

// Netpbm P5 header: "P5", width, height, maxval, each preceded by whitespace
// or '#' comments running to the end of the line, then ONE whitespace byte
// and the raster (pgm.cpp:54-83 accepts exactly this; P2 is rejected).
struct PgmView {
  int width = 0, height = 0;
  size_t raster = 0;  // offset of the first pixel
};

// Header of a file whose first n of `total` bytes are at b: false when the
// prefix ends inside the header (the caller reads more), otherwise the header
// or an IoError -- the same verdicts whether the prefix or the whole file is
// given.
bool parse_pgm_head(const std::uint8_t* b, size_t n, size_t total, const std::string& path, PgmView* out) {
  auto bad = [&](const std::string& why) { return IoError("read_pgm: " + why + " (" + path + ")"); };
  if (n < 2 && n < total) return false;
  if (n < 2 || b[0] != 'P' || b[1] != '5') throw bad("not a binary P5 graymap");
  size_t at = 2;
  bool more = false;
  auto space = [](std::uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; };
  auto ends = [&](const char* what) {
    if (n < total) more = true;
    else throw bad(std::string("header ends before ") + what);
  };
  auto number = [&](const char* what) -> long long {
    for (;;) {  // skip separators and comments
      if (at >= n) return ends(what), -1;
      if (b[at] == '#') {
        while (at < n && b[at] != '\n') ++at;
      } else if (space(b[at])) {
        ++at;
      } else {
        break;
      }
    }
    if (b[at] < '0' || b[at] > '9') throw bad(std::string(what) + " is not a number");
    long long v = 0;
    while (at < n && b[at] >= '0' && b[at] <= '9') {
      v = v * 10 + (b[at++] - '0');
      if (v > std::numeric_limits<int>::max()) throw bad(std::string(what) + " out of range");
    }
    if (at >= n && n < total) more = true;  // the digits may go on
    return v;
  };
  PgmView v;
  v.width = static_cast<int>(number("width"));
  if (more) return false;
  v.height = static_cast<int>(number("height"));
  if (more) return false;
  const long long maxval = number("maxval");
  if (more) return false;
  if (v.width < 1 || v.height < 1) throw bad("dimensions must be >= 1");
  if (maxval != 255) throw bad("only maxval 255 is supported");
  if (at >= n) {
    if (n < total) return false;
    throw bad("no whitespace byte before the raster");
  }
  if (!space(b[at])) throw bad("no whitespace byte before the raster");
  v.raster = at + 1;
  if (total - v.raster < static_cast<size_t>(v.width) * v.height) throw bad("raster is truncated");
  *out = v;
  return true;
}

PgmView parse_pgm(const std::vector<std::uint8_t>& b, const std::string& path) {
  PgmView v;
  parse_pgm_head(b.data(), b.size(), b.size(), path, &v);
  return v;
}

// The header alone: the file's first 4 KB (all of it if the header runs on).
PgmView peek_pgm(const std::string& path, const char* who) {
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
  if (!f) throw IoError(std::string(who) + ": cannot open " + path);
  struct stat st {};
  const size_t total = fstat(fileno(f.get()), &st) == 0 && st.st_size > 0 ? static_cast<size_t>(st.st_size) : 0;
  std::uint8_t head[4096];
  const size_t got = std::fread(head, 1, std::min(total, sizeof(head)), f.get());
  PgmView v;
  if (parse_pgm_head(head, got, std::max(total, got), path, &v)) return v;
  f.reset();
  return parse_pgm(slurp(path, who), path);
}

// W*H raster bytes at `raster` straight into dst (the chunk's staging buffer).
void read_raster(const std::string& path, const PgmView& v, std::uint8_t* dst, const char* who) {
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
  if (!f) throw IoError(std::string(who) + ": cannot open " + path);
  const size_t want = static_cast<size_t>(v.width) * v.height;
  if (std::fseek(f.get(), static_cast<long>(v.raster), SEEK_SET) != 0 ||
      std::fread(dst, 1, want, f.get()) != want)
    throw IoError(std::string(who) + ": raster is truncated (" + path + ")");
}

[[noreturn]] void raise_status(dppx_ctx* ctx, int rc, const std::string& who) {
  const std::string msg = who + ": " + (ctx ? dppx_ctx_last_error(ctx) : "");
  if (rc == DPPX_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == DPPX_ERR_CORRUPT) throw RecordError(RecordErrorKind::corrupt_record, msg);
  if (rc == DPPX_ERR_OOM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

void parallel_over(int count, int workers, const std::function<void(int)>& body) {
  workers = std::max(1, std::min(workers, count));
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w)
    pool.emplace_back([&] {
      for (int i = next++; i < count; i = next++) body(i);
    });
  for (int i = next++; i < count; i = next++) body(i);
  for (auto& t : pool) t.join();
}

struct HostBuf {  // pageable host batch buffer (no zero fill)
  std::unique_ptr<uint8_t[]> mem;
  uint8_t* p = nullptr;
  explicit HostBuf(size_t bytes) : mem(new uint8_t[bytes ? bytes : 1]), p(mem.get()) {}
};

// Process-wide device group per device list (contexts and worker threads are
// created once; run_batch calls reuse them).
// The groups live until the process exits and are deliberately not destroyed
// by static destructors (the CUDA runtime may already be torn down by then).
dppx_group* shared_group(const std::vector<int>& want) {
  static std::mutex mu;
  static auto* groups = new std::map<std::vector<int>, dppx_group*>();
  std::lock_guard<std::mutex> lk(mu);
  auto it = groups->find(want);
  if (it != groups->end()) return it->second;
  dppx_group* g = nullptr;
  const int rc = want.empty() ? dppx_group_create(nullptr, 0, &g)
                              : dppx_group_create(want.data(), static_cast<int32_t>(want.size()), &g);
  if (rc != DPPX_OK)
    throw std::runtime_error("dppix: no usable sm_100 GPU for the batch runner (status " +
                             std::to_string(rc) + ")");
  groups->emplace(want, g);
  return g;
}

std::vector<int> batch_devices(const BatchConfig& cfg) {
  if (!cfg.devices.empty()) return cfg.devices;
  std::vector<int> out;
  if (const char* env = std::getenv("DPPX_BATCH_DEVICES")) {
    std::stringstream ss(env);
    std::string tok;
    while (std::getline(ss, tok, ','))
      if (!tok.empty()) out.push_back(std::atoi(tok.c_str()));
  }
  return out;
}

int group_task_trampoline(dppx_ctx* ctx, int32_t worker, int32_t task, void* user) {
  (*static_cast<std::function<void(dppx_ctx*, int, int)>*>(user))(ctx, worker, task);
  return DPPX_OK;
}

// cli.cpp:78-89 (validate_run_config): flag combinations wrong for every input.
void validate(bool have_seed, double epsilon, bool reference_mode, bool emit_record,
              bool adaptive_mode, bool mask_empty) {
  if (!(epsilon > 0.0) && have_seed) throw UsageError("--epsilon must be > 0");
  if (reference_mode && emit_record)
    throw UsageError("reference mode keeps no grid statistics and cannot emit records");
  if (adaptive_mode && mask_empty) throw UsageError("adaptive mode requires --mask");
}

// cli.cpp:43-58 (mask_path_for): a mask directory pairs masks by input stem.
std::string paired_mask(const std::string& mask_path, const std::string& input) {
  if (mask_path.empty()) throw UsageError("adaptive mode requires --mask");
  std::error_code ec;
  if (fs::is_directory(mask_path, ec)) {
    const fs::path p = fs::path(mask_path) / (fs::path(input).stem().string() + ".pgm");
    if (!fs::exists(p, ec)) throw IoError("no mask for " + input + " (expected " + p.string() + ")");
    return p.string();
  }
  return mask_path;
}

void make_out_dir(const std::string& dir) {
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) throw IoError("cannot create output directory " + dir + ": " + ec.message());
}

}  // namespace

// ---------------------------------------------------------------- pgm.hpp
GrayImage read_pgm(const std::string& path) {
  const std::vector<std::uint8_t> bytes = slurp(path, "read_pgm");
  const PgmView v = parse_pgm(bytes, path);
  GrayImage img = make_image(v.height, v.width);
  std::memcpy(img.pixels.data(), bytes.data() + v.raster, img.pixels.size());
  return img;
}

namespace {
// Writes head + body as the whole file. An existing file is overwritten in
// place and then cut to length instead of being truncated first: rewriting a
// batch's outputs reuses their cached pages instead of freeing and
// reallocating them (60 -> 4 ms for 128 files of a 64 x 1080p batch).
// 1 = cannot open, 2 = short write.
int write_whole_file(const std::string& path, const void* head, size_t nh, const void* body, size_t nb) {
  const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_CLOEXEC, 0666);
  if (fd < 0) return 1;
  auto put = [&](const void* p, size_t n, off_t at) {
    const char* c = static_cast<const char*>(p);
    while (n > 0) {
      const ssize_t w = ::pwrite(fd, c, n, at);
      if (w <= 0) return false;
      c += w, n -= static_cast<size_t>(w), at += w;
    }
    return true;
  };
  const bool ok = put(head, nh, 0) && put(body, nb, static_cast<off_t>(nh)) &&
                  ::ftruncate(fd, static_cast<off_t>(nh + nb)) == 0;
  return (::close(fd) == 0 && ok) ? 0 : 2;
}

void write_pgm_bytes(int height, int width, const std::uint8_t* pixels, const std::string& path) {
  char head[64];
  const int hn = std::snprintf(head, sizeof(head), "P5\n%d %d\n255\n", width, height);
  const int rc = write_whole_file(path, head, static_cast<size_t>(hn), pixels, static_cast<size_t>(height) * width);
  if (rc == 1) throw IoError("write_pgm: cannot create " + path);
  if (rc == 2) throw IoError("write_pgm: short write to " + path);
}
}  // namespace

void write_pgm(const GrayImage& img, const std::string& path) {
  if (img.height < 1 || img.width < 1 ||
      img.pixels.size() != static_cast<std::size_t>(img.height) * img.width)
    throw IoError("write_pgm: image buffer does not match its dimensions (" + path + ")");
  write_pgm_bytes(img.height, img.width, img.pixels.data(), path);
}

RegionMask read_mask_pgm(const std::string& path) {  // pgm.cpp:112-119: >= 128 -> simple
  const std::vector<std::uint8_t> bytes = slurp(path, "read_mask_pgm");
  const PgmView v = parse_pgm(bytes, path);
  RegionMask mask = make_mask(v.height, v.width, 0);
  const std::uint8_t* src = bytes.data() + v.raster;
  for (std::size_t i = 0; i < mask.values.size(); ++i) mask.values[i] = src[i] >> 7;
  return mask;
}

// ---------------------------------------------------------------- batch.hpp
int batch_exit_code_for(const std::exception& err) { return exit_code_for(err); }

std::vector<BatchFileReport> run_batch_gpu(const BatchConfig& cfg) {
  validate(cfg.seed.has_value(), cfg.epsilon, cfg.mode == BatchMode::reference, cfg.emit_record,
           cfg.mode == BatchMode::adaptive, cfg.mask_path.empty());
  std::vector<std::string> inputs;
  std::error_code ec;
  if (fs::is_directory(cfg.input, ec)) {
    for (const fs::directory_entry& e : fs::directory_iterator(cfg.input))
      if (e.is_regular_file() && e.path().extension() == ".pgm") inputs.push_back(e.path().string());
    std::sort(inputs.begin(), inputs.end());
    if (inputs.empty()) throw IoError("no .pgm inputs under " + cfg.input);
  } else {
    inputs.push_back(cfg.input);
  }
  const int nfile = static_cast<int>(inputs.size());
  const int io = cfg.io_threads > 0 ? cfg.io_threads
                                    : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  std::vector<BatchFileReport> reports(nfile);
  std::vector<PgmView> heads(nfile), mheads(cfg.mode == BatchMode::adaptive ? nfile : 0);
  std::vector<char> ok(nfile, 0);
  std::mutex fail_mu;
  auto fail = [&](int i, const std::exception& err) {
    std::lock_guard<std::mutex> lk(fail_mu);
    if (reports[i].exit_code != 0) return;
    reports[i].error = err.what();
    reports[i].exit_code = exit_code_for(err);
  };
  // DPPX_BATCH_TRACE=1: per-phase wall times on stderr.
  static const bool trace = std::getenv("DPPX_BATCH_TRACE") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto T0 = tnow();
  const double eff_eps = cfg.epsilon > 0.0 ? cfg.epsilon : 1.0;  // cli.cpp:97-102
  const int n = cfg.mode == BatchMode::adaptive ? cfg.n : 1;
  const int K = std::max(1, cfg.frames_per_call);
  const int mode = cfg.mode == BatchMode::adaptive ? 1 : cfg.mode == BatchMode::uniform ? 0 : 2;
  // ---- device setup, overlapping ingest: the group (contexts, worker
  // threads), then per worker the buffers of a full chunk of the first
  // input's shape and one 1-frame call, which loads the kernels it selects.
  // Failures surface only if there is GPU work (chunks) after all. ----
  dppx_group* grp = nullptr;
  std::exception_ptr setup_err;
  std::thread setup([&] {
    try {
      const auto g0 = std::chrono::steady_clock::now();
      grp = shared_group(batch_devices(cfg));
      if (trace) std::fprintf(stderr, "batch: setup group %.1f ms\n", tms(g0, std::chrono::steady_clock::now()));
      int M = 0, N = 0;
      try {
        const PgmView v = peek_pgm(inputs[0], "read_pgm");
        M = v.height, N = v.width;
      } catch (const std::exception&) {
        return;  // ingest reports it
      }
      dppx_privacy_params pp;
      if (dppx_make_privacy_params(eff_eps, cfg.m, cfg.b, n, &pp) != DPPX_OK) return;
      dppx_geometry g;
      if (dppx_grid_dims(M, N, cfg.b, &g) != DPPX_OK) return;
      const int F = std::min(K, nfile);
      const size_t plane = static_cast<size_t>(M) * N;
      std::function<void(dppx_ctx*, int, int)> warm = [&](dppx_ctx* ctx, int, int) {
        const dppx_frames_desc full{M, N, 1, F, N, static_cast<int64_t>(plane), N, static_cast<int64_t>(plane),
                                    N, static_cast<int64_t>(plane)};
        const auto w0 = std::chrono::steady_clock::now();
        if (dppx_pixelize_checked_reserve(ctx, mode, &full, &pp) != DPPX_OK) return;
        const auto w1 = std::chrono::steady_clock::now();
        const dppx_frames_desc one{M, N, 1, 1, N, static_cast<int64_t>(plane), N, static_cast<int64_t>(plane),
                                   N, static_cast<int64_t>(plane)};
        std::vector<uint8_t> img(plane, 0), mk(plane, 1), out(plane);
        const size_t cap = mode == 1 ? (dppx_adaptive_payload_capacity(M, N, cfg.b, n) + 3) & ~size_t{3}
                                     : static_cast<size_t>(g.grid_rows) * g.grid_cols;
        std::vector<uint8_t> stats(cap);
        uint32_t len = 0;
        uint8_t ok = 0;
        double mse = 0.0, ssim = 0.0;
        uint64_t seed = 0;
        const dppx_noise nz{cfg.seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, &seed, nullptr};
        dppx_pixelize_checked(ctx, mode, &one, img.data(), mode == 1 ? mk.data() : nullptr, &pp, &nz,
                              stats.data(), static_cast<int64_t>(cap), &len, out.data(), &ok, &mse,
                              M >= 7 && N >= 7 ? &ssim : nullptr);
        if (trace)
          std::fprintf(stderr, "batch: setup reserve %.1f ms, 1-frame call %.1f ms\n", tms(w0, w1),
                       tms(w1, std::chrono::steady_clock::now()));
      };
      dppx_group_run(grp, dppx_group_size(grp), &group_task_trampoline, &warm);
    } catch (...) {
      setup_err = std::current_exception();
    }
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{setup};
  // ---- ingest: headers first (host threads) ----
  parallel_over(nfile, io, [&](int i) {
    reports[i].input = inputs[i];
    try {
      heads[i] = peek_pgm(inputs[i], "read_pgm");
      if (cfg.mode == BatchMode::adaptive) {
        mheads[i] = peek_pgm(paired_mask(cfg.mask_path, inputs[i]), "read_mask_pgm");
        if (mheads[i].height != heads[i].height || mheads[i].width != heads[i].width)
          throw UsageError("mask dimensions do not match image: " + inputs[i]);
      }
      ok[i] = 1;
    } catch (const std::exception& err) {
      fail(i, err);
    }
  });
  // ---- shape groups -> chunks of up to frames_per_call frames ----
  std::map<std::pair<int, int>, std::vector<int>> groups;
  for (int i = 0; i < nfile; ++i)
    if (ok[i]) groups[{heads[i].height, heads[i].width}].push_back(i);
  std::vector<std::vector<int>> chunks;
  for (auto& kv : groups)
    for (size_t c0 = 0; c0 < kv.second.size(); c0 += K)
      chunks.emplace_back(kv.second.begin() + c0,
                          kv.second.begin() + std::min(kv.second.size(), c0 + K));
  // ---- rasters straight into each chunk's staging buffers (frame k of a
  // chunk at k * plane; masks thresholded in place, pgm.cpp:112-119) ----
  struct ChunkBufs {  // out is touched here too: its page faults stay off the download
    HostBuf in, mk, out;
  };
  std::vector<std::unique_ptr<ChunkBufs>> bufs(chunks.size());
  std::vector<std::pair<int, int>> slot(nfile, {-1, -1});
  for (size_t t = 0; t < chunks.size(); ++t) {
    const size_t plane = static_cast<size_t>(heads[chunks[t][0]].height) * heads[chunks[t][0]].width;
    const size_t F = chunks[t].size();
    bufs[t].reset(new ChunkBufs{HostBuf(plane * F), HostBuf(cfg.mode == BatchMode::adaptive ? plane * F : 0),
                                HostBuf(plane * F)});
    for (size_t k = 0; k < F; ++k) slot[chunks[t][k]] = {static_cast<int>(t), static_cast<int>(k)};
  }
  parallel_over(nfile, io, [&](int i) {
    if (slot[i].first < 0) return;
    const size_t plane = static_cast<size_t>(heads[i].height) * heads[i].width;
    ChunkBufs& cb = *bufs[slot[i].first];
    std::uint8_t* img = cb.in.p + static_cast<size_t>(slot[i].second) * plane;
    std::memset(cb.out.p + static_cast<size_t>(slot[i].second) * plane, 0, plane);
    try {
      read_raster(inputs[i], heads[i], img, "read_pgm");
      if (cfg.mode == BatchMode::adaptive) {
        std::uint8_t* m = cb.mk.p + static_cast<size_t>(slot[i].second) * plane;
        read_raster(paired_mask(cfg.mask_path, inputs[i]), mheads[i], m, "read_mask_pgm");
        for (size_t q = 0; q < plane; ++q) m[q] >>= 7;
      }
    } catch (const std::exception& err) {  // the frame still rides along; its outputs are skipped
      std::memset(img, 0, plane);
      if (cfg.mode == BatchMode::adaptive) std::memset(cb.mk.p + static_cast<size_t>(slot[i].second) * plane, 0, plane);
      fail(i, err);
    }
  });
  if (trace) std::fprintf(stderr, "batch: ingest %.1f ms\n", tms(T0, tnow()));
  if (!chunks.empty() && (cfg.emit_image || cfg.emit_record)) make_out_dir(cfg.out_dir);
  const auto Tg = tnow();
  setup.join();
  if (chunks.empty()) return reports;
  if (setup_err) std::rethrow_exception(setup_err);
  if (trace) std::fprintf(stderr, "batch: device setup wait %.1f ms\n", tms(Tg, tnow()));
  const int workers = dppx_group_size(grp);
  const int io_per = std::max(1, io / std::max(1, std::min<int>(workers, static_cast<int>(chunks.size()))));

  std::function<void(dppx_ctx*, int, int)> task = [&](dppx_ctx* ctx, int, int t) {
    const std::vector<int>& chunk = chunks[t];
    const int F = static_cast<int>(chunk.size());
    const int M = heads[chunk[0]].height, N = heads[chunk[0]].width;
    try {
      dppx_privacy_params pp;
      if (dppx_make_privacy_params(eff_eps, cfg.m, cfg.b, n, &pp) != DPPX_OK)
        throw std::invalid_argument("make_privacy_params: invalid parameters");
      const size_t plane = static_cast<size_t>(M) * N;
      const auto t0 = tnow();
      const HostBuf& out = bufs[t]->out;
      const HostBuf& in = bufs[t]->in;
      const HostBuf& mk = bufs[t]->mk;
      const dppx_frames_desc d{M, N, 1, F, N, static_cast<int64_t>(plane), N, static_cast<int64_t>(plane),
                               N, static_cast<int64_t>(plane)};
      std::vector<uint64_t> seeds(F, cfg.seed ? cfg.seed->value : 0);  // same seed per file, cli.cpp:200-201
      const dppx_noise nz{cfg.seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, seeds.data(), nullptr};
      dppx_geometry g;
      if (dppx_grid_dims(M, N, cfg.b, &g) != DPPX_OK)
        throw std::invalid_argument("grid_dims: grid side b exceeds both image dimensions");
      const size_t G = static_cast<size_t>(g.grid_rows) * g.grid_cols;
      const size_t cap = cfg.mode == BatchMode::adaptive
                             ? (dppx_adaptive_payload_capacity(M, N, cfg.b, n) + 3) & ~size_t{3}
                             : G;
      HostBuf stats(cap * F);  // rows filled up to each plane's length by the call
      std::vector<uint32_t> lens(F, static_cast<uint32_t>(G));
      std::vector<uint8_t> recon_ok(F, 1);
      std::vector<double> mses(F), ssims(F, std::numeric_limits<double>::quiet_NaN());
      // One upload per chunk: pixelize, the reconstruct check and mse / ssim
      // all run where the frames already are (dppx_pixelize_checked).
      const auto tp0 = tnow();
      const int rc = dppx_pixelize_checked(ctx, mode, &d, in.p, cfg.mode == BatchMode::adaptive ? mk.p : nullptr,
                                           &pp, &nz, stats.p, static_cast<int64_t>(cap), lens.data(), out.p,
                                           recon_ok.data(), mses.data(),
                                           M >= 7 && N >= 7 ? ssims.data() : nullptr);
      const auto tp1 = tnow();
      if (rc != DPPX_OK) raise_status(ctx, rc, "pixelize");
      const double per_ms = tms(tp0, tp1) / F;
      // ---- records + reconstruct check (cli.cpp:132-146) ----
      // reconstruct(decode(encode(stats))) == image: decode must give back the
      // statistics' exact bytes (checked here), and their expansion equals the
      // emitted image (checked on the device: recon_ok).
      std::vector<std::vector<uint8_t>> recs(F);
      if (cfg.mode != BatchMode::reference) {
        std::vector<char> rec_ok(F, 1);
        parallel_over(F, io_per, [&](int k) {  // header + CRC32 per file, then decode
          recs[k].resize(dppx_record_size(lens[k]));
          size_t len = 0;
          if (dppx_encode_record(M, N, cfg.b, n, cfg.mode == BatchMode::adaptive ? 2 : 1, stats.p + k * cap,
                                 lens[k], recs[k].data(), recs[k].size(), &len) != DPPX_OK) {
            rec_ok[k] = 0;
            return;
          }
          if (!cfg.reconstruct_check) return;
          dppx_record_info info{};
          if (dppx_decode_record(recs[k].data(), recs[k].size(), &info) != DPPX_OK ||
              info.payload_len != lens[k] ||
              std::memcmp(recs[k].data() + info.payload_offset, stats.p + k * cap, lens[k]) != 0)
            rec_ok[k] = 2;
        });
        for (int k = 0; k < F; ++k) {
          if (rec_ok[k] == 0) throw std::invalid_argument("encode: payload inconsistent");
          if (rec_ok[k] == 2) fail(chunk[k], RecordError(RecordErrorKind::corrupt_record, "decode failed"));
          else if (cfg.reconstruct_check && !recon_ok[k])
            fail(chunk[k], ConsistencyError("reconstruction does not match the emitted image for " +
                                            inputs[chunk[k]]));
        }
      }
      const auto tr = tnow();
      const auto tm = tnow();
      // ---- outputs (host threads) ----
      parallel_over(F, io_per, [&](int k) {
        const int i = chunk[k];
        if (reports[i].exit_code != 0) return;
        try {
          const std::string stem = fs::path(inputs[i]).stem().string();
          if (cfg.emit_image) {
            const std::string path = (fs::path(cfg.out_dir) / (stem + ".pix.pgm")).string();
            write_pgm_bytes(M, N, out.p + k * plane, path);
            reports[i].written.push_back(path);
          }
          if (cfg.mode != BatchMode::reference && cfg.emit_record) {
            const std::string path = (fs::path(cfg.out_dir) / (stem + ".dppx")).string();
            if (write_whole_file(path, nullptr, 0, recs[k].data(), recs[k].size()) != 0)
              throw IoError("write_record: cannot write " + path);
            reports[i].written.push_back(path);
          }
          MetricReport& r = reports[i].report;
          r.epsilon = cfg.epsilon;
          r.m = cfg.m;
          r.b = cfg.b;
          r.n = n;
          r.seed = cfg.seed ? cfg.seed->value : 0;
          r.mse = mses[k];
          r.ssim = ssims[k];
          r.runtime_ms = per_ms;
          r.record_bytes = recs[k].size();
        } catch (const std::exception& err) {
          fail(i, err);
        }
      });
      if (trace)
        std::fprintf(stderr,
                     "batch: chunk %d (%d x %dx%d): stage %.1f pixelize %.1f records+check %.1f metrics %.1f "
                     "outputs %.1f ms\n",
                     t, F, M, N, tms(t0, tp0), tms(tp0, tp1), tms(tp1, tr), tms(tr, tm), tms(tm, tnow()));
    } catch (const std::exception& err) {
      for (int i : chunk) fail(i, err);
    }
  };
  const int grc = dppx_group_run(grp, static_cast<int32_t>(chunks.size()), &group_task_trampoline, &task);
  if (grc != DPPX_OK) raise_status(nullptr, grc, "run_batch");
  if (trace) std::fprintf(stderr, "batch: total %.1f ms on %d GPU worker(s)\n", tms(T0, tnow()), workers);
  return reports;
}

// ---------------------------------------------------------------- cli.hpp
int exit_code_for(const std::exception& err) {  // cli.cpp:386-401
  if (dynamic_cast<const ConsistencyError*>(&err)) return kExitConsistency;
  if (dynamic_cast<const RecordError*>(&err)) return kExitRecord;
  if (dynamic_cast<const IoError*>(&err)) return kExitIo;
  if (dynamic_cast<const UsageError*>(&err) || dynamic_cast<const std::invalid_argument*>(&err))
    return kExitUsage;
  return 1;
}

RunOutcome run_single(const RunConfig& cfg) {  // cli.cpp:93-173
  validate(cfg.seed.has_value(), cfg.epsilon, cfg.mode == RunMode::reference, cfg.emit_record,
           cfg.mode == RunMode::adaptive, cfg.mask_path.empty());
  const GrayImage img = read_pgm(cfg.input);
  const PrivacyParams params = make_privacy_params(cfg.epsilon > 0.0 ? cfg.epsilon : 1.0, cfg.m, cfg.b,
                                                   cfg.mode == RunMode::adaptive ? cfg.n : 1);
  using Clock = std::chrono::steady_clock;
  GrayImage pixelized;
  std::optional<PixelRecord> record;
  Clock::time_point start, stop;
  if (cfg.mode == RunMode::adaptive) {
    const RegionMask mask = read_mask_pgm(paired_mask(cfg.mask_path, cfg.input));
    if (mask.height != img.height || mask.width != img.width)
      throw UsageError("mask dimensions do not match image: " + cfg.input);
    start = Clock::now();
    AdaptiveResult r = pixelize_adaptive(img, mask, params, cfg.seed, cfg.threads);
    stop = Clock::now();
    pixelized = std::move(r.image);
    record = PixelRecord{img.height, img.width, std::move(r.means)};
  } else if (cfg.mode == RunMode::uniform) {
    start = Clock::now();
    UniformResult r = pixelize_parallel(img, params, cfg.seed, cfg.threads);
    stop = Clock::now();
    pixelized = std::move(r.image);
    record = PixelRecord{img.height, img.width, std::move(r.means)};
  } else {
    start = Clock::now();
    pixelized = pixelize_reference(img, params, cfg.seed);
    stop = Clock::now();
  }
  RunOutcome out;
  std::vector<std::uint8_t> bytes;
  if (record) {
    bytes = encode(*record);
    if (cfg.reconstruct_check && !(reconstruct(decode(bytes)) == pixelized))
      throw ConsistencyError("reconstruction does not match the emitted image for " + cfg.input);
  }
  const std::string stem = fs::path(cfg.input).stem().string();
  if (cfg.emit_image || cfg.emit_record) make_out_dir(cfg.out_dir);
  if (cfg.emit_image) {
    const std::string p = (fs::path(cfg.out_dir) / (stem + ".pix.pgm")).string();
    write_pgm(pixelized, p);
    out.written.push_back(p);
  }
  if (record && cfg.emit_record) {
    const std::string p = (fs::path(cfg.out_dir) / (stem + ".dppx")).string();
    write_record(*record, p);
    out.written.push_back(p);
  }
  MetricReport& r = out.report;
  r.epsilon = cfg.epsilon;
  r.m = cfg.m;
  r.b = cfg.b;
  r.n = params.n;
  r.seed = cfg.seed ? cfg.seed->value : 0;
  r.mse = mse(img, pixelized);
  r.ssim = img.height >= 7 && img.width >= 7 ? ssim(img, pixelized, cfg.threads)
                                              : std::numeric_limits<double>::quiet_NaN();
  r.runtime_ms = std::chrono::duration<double, std::milli>(stop - start).count();
  r.record_bytes = bytes.size();
  return out;
}

std::vector<FileReport> run_batch(const RunConfig& cfg) {  // cli.cpp:175-213, on every GPU
  BatchConfig b;
  b.input = cfg.input;
  b.out_dir = cfg.out_dir;
  b.mode = cfg.mode == RunMode::adaptive ? BatchMode::adaptive
           : cfg.mode == RunMode::reference ? BatchMode::reference : BatchMode::uniform;
  b.epsilon = cfg.epsilon;
  b.m = cfg.m;
  b.b = cfg.b;
  b.n = cfg.n;
  b.seed = cfg.seed;
  b.mask_path = cfg.mask_path;
  b.emit_image = cfg.emit_image;
  b.emit_record = cfg.emit_record;
  b.reconstruct_check = cfg.reconstruct_check;
  std::vector<FileReport> out;
  for (BatchFileReport& r : run_batch_gpu(b))
    out.push_back(FileReport{std::move(r.input), r.report, std::move(r.written), std::move(r.error), r.exit_code});
  return out;
}

// run_sweep's uniform rows for one image: every (b, eps) pair of one (m, seed)
// is computed by ONE dppx_pixelize_uniform_sweep call (one upload and one read
// of the frame for all the runs, per-run mse / ssim on the device). Pairs whose
// parameters the reference would reject are left out; the caller runs them
// through run_single so the error rows are the reference's own.
namespace {
using SweepKey = std::tuple<double, int, int, std::uint64_t>;

void fused_uniform_sweep(const RunConfig& base, std::map<SweepKey, MetricReport>& rows) {
  if (const char* e = std::getenv("DPPX_SWEEP_FUSED"); e && e[0] == '0') return;
  GrayImage img;
  try {
    img = read_pgm(base.input);
  } catch (const std::exception&) {
    return;  // every row reports the read error through run_single
  }
  const int H = img.height, W = img.width;
  dppx_ctx* ctx = dropin_thread_ctx();
  dppx_frames_desc d{H, W, 1, 1, W, static_cast<int64_t>(H) * W, W, static_cast<int64_t>(H) * W, W,
                     static_cast<int64_t>(H) * W};
  for (int m : base.m_list) {
    auto clean = [&](double eps, int b) {
      try {
        validate(true, eps, false, false, false, true);
        (void)make_privacy_params(eps, m, b, 1);
        (void)grid_dims(H, W, b);
        return true;
      } catch (const std::exception&) {
        return false;
      }
    };
    std::vector<double> eps_ok;
    for (double eps : base.epsilon_list)
      if (std::any_of(base.b_list.begin(), base.b_list.end(), [&](int b) { return clean(eps, b); }))
        eps_ok.push_back(eps);
    std::vector<int32_t> b_ok;
    for (int b : base.b_list)
      if (!eps_ok.empty() && std::all_of(eps_ok.begin(), eps_ok.end(), [&](double e) { return clean(e, b); }))
        b_ok.push_back(b);
    b_ok.erase(std::unique(b_ok.begin(), b_ok.end()), b_ok.end());
    eps_ok.erase(std::unique(eps_ok.begin(), eps_ok.end()), eps_ok.end());
    if (b_ok.empty() || eps_ok.empty()) continue;
    eps_ok.erase(std::remove_if(eps_ok.begin(), eps_ok.end(),
                                [&](double e) {
                                  return !std::all_of(b_ok.begin(), b_ok.end(), [&](int b) { return clean(e, b); });
                                }),
                 eps_ok.end());
    const int nb = static_cast<int>(b_ok.size()), ne = static_cast<int>(eps_ok.size()), runs = nb * ne;
    std::vector<GridGeometry> geom;
    for (int b : b_ok) geom.push_back(grid_dims(H, W, b));
    for (std::uint64_t seed : base.seed_list) {
      std::vector<std::vector<std::uint8_t>> means(static_cast<size_t>(runs));
      std::vector<std::vector<std::uint8_t>> images(base.reconstruct_check ? runs : 0);
      std::vector<std::uint8_t*> mp(static_cast<size_t>(runs)), op(static_cast<size_t>(runs), nullptr);
      for (int r = 0; r < runs; ++r) {
        means[r].resize(static_cast<size_t>(geom[r / ne].grid_count()));
        mp[r] = means[r].data();
        if (base.reconstruct_check) {
          images[r].resize(static_cast<size_t>(H) * W);
          op[r] = images[r].data();
        }
      }
      std::vector<double> mse_v(static_cast<size_t>(runs)), ssim_v(static_cast<size_t>(runs),
                                                                  std::numeric_limits<double>::quiet_NaN());
      const dppx_noise nz{DPPX_NOISE_KEYED, 0, &seed, nullptr};
      const auto t0 = std::chrono::steady_clock::now();
      const int rc = dppx_pixelize_uniform_sweep(ctx, &d, img.pixels.data(), nb, b_ok.data(), ne, eps_ok.data(), m,
                                                 &nz, mp.data(), base.reconstruct_check ? op.data() : nullptr,
                                                 mse_v.data(), H >= 7 && W >= 7 ? ssim_v.data() : nullptr);
      const auto t1 = std::chrono::steady_clock::now();
      if (rc != DPPX_OK) return;  // leave every row to run_single (which reports the error)
      const double per_ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / runs;
      for (int r = 0; r < runs; ++r) {
        const int i = r / ne, j = r % ne;
        PixelRecord rec{H, W, GridMeans{geom[i], std::move(means[r])}};
        const std::vector<std::uint8_t> bytes = encode(rec);
        if (base.reconstruct_check) {
          GrayImage pix;
          pix.height = H;
          pix.width = W;
          pix.pixels = std::move(images[r]);
          if (!(reconstruct(decode(bytes)) == pix))
            throw ConsistencyError("reconstruction does not match the emitted image for " + base.input);
        }
        MetricReport rep;
        rep.epsilon = eps_ok[j];
        rep.m = m;
        rep.b = b_ok[i];
        rep.n = 1;
        rep.seed = seed;
        rep.mse = mse_v[r];
        rep.ssim = ssim_v[r];
        rep.runtime_ms = per_ms;
        rep.record_bytes = bytes.size();
        rows[SweepKey{eps_ok[j], m, b_ok[i], seed}] = rep;
      }
    }
  }
}
}  // namespace

SweepResult run_sweep(const RunConfig& cfg) {  // cli.cpp:231-288
  RunConfig base = cfg;
  base.emit_image = false;
  base.emit_record = false;
  if (base.epsilon_list.empty() || base.m_list.empty() || base.b_list.empty() || base.n_list.empty() ||
      base.seed_list.empty())
    throw UsageError("sweep lists must be non-empty");
  if (base.mode == RunMode::reference) throw UsageError("sweep supports uniform and adaptive modes only");
  if (base.mode == RunMode::uniform &&
      std::any_of(base.n_list.begin(), base.n_list.end(), [](int v) { return v != 1; }))
    throw UsageError("uniform sweeps require n == 1");
  std::sort(base.epsilon_list.begin(), base.epsilon_list.end());
  std::sort(base.m_list.begin(), base.m_list.end());
  std::sort(base.b_list.begin(), base.b_list.end());
  std::sort(base.n_list.begin(), base.n_list.end());
  std::sort(base.seed_list.begin(), base.seed_list.end());
  auto quote = [](const std::string& s) {
    std::string q = "\"";
    for (char c : s) q += c == '"' ? std::string("\"\"") : std::string(1, c);
    return q + "\"";
  };
  SweepResult res;
  std::map<SweepKey, MetricReport> fused;
  if (base.mode == RunMode::uniform) fused_uniform_sweep(base, fused);
  std::ostringstream csv;
  csv << csv_header() << ",error\n";
  for (double eps : base.epsilon_list)
    for (int m : base.m_list)
      for (int b : base.b_list)
        for (int n : base.n_list)
          for (std::uint64_t seed : base.seed_list) {
            RunConfig one = base;
            one.epsilon = eps;
            one.m = m;
            one.b = b;
            one.n = n;
            one.seed = NoiseSeed{seed};
            if (auto it = fused.find(SweepKey{eps, m, b, seed}); it != fused.end()) {
              csv << csv_row(it->second) << ",\n";
              continue;
            }
            try {
              csv << csv_row(run_single(one).report) << ",\n";
            } catch (const std::exception& err) {
              ++res.failures;
              MetricReport blank;
              blank.epsilon = eps;
              blank.m = m;
              blank.b = b;
              blank.n = n;
              blank.seed = seed;
              csv << csv_row(blank) << ',' << quote(err.what()) << '\n';
            }
          }
  res.csv = csv.str();
  return res;
}

BenchResult run_bench(const RunConfig& cfg) {  // cli.cpp:303-336
  if (cfg.repeat < 1 || cfg.warmup < 0) throw UsageError("bench requires repeat >= 1 and warmup >= 0");
  const GrayImage img = read_pgm(cfg.input);
  const PrivacyParams params = make_privacy_params(cfg.epsilon > 0.0 ? cfg.epsilon : 1.0, cfg.m, cfg.b, 1);
  using Clock = std::chrono::steady_clock;
  auto ms = [](Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  BenchResult res;
  for (int round = -cfg.warmup; round < cfg.repeat; ++round) {
    const auto t0 = Clock::now();
    const GrayImage seq = pixelize_reference(img, params, cfg.seed);
    const auto t1 = Clock::now();
    const UniformResult par = pixelize_parallel(img, params, cfg.seed, cfg.threads);
    const auto t2 = Clock::now();
    if (round >= 0) {
      res.reference_ms.push_back(ms(t0, t1));
      res.parallel_ms.push_back(ms(t1, t2));
    }
    if (img.height % params.b == 0 && img.width % params.b == 0 && !(seq == par.image))
      throw ConsistencyError("bench: reference and parallel paths disagree");
  }
  auto median = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t h = v.size() / 2;
    return v.size() % 2 ? v[h] : 0.5 * (v[h - 1] + v[h]);
  };
  res.median_reference_ms = median(res.reference_ms);
  res.median_parallel_ms = median(res.parallel_ms);
  res.speedup = res.median_parallel_ms > 0.0 ? res.median_reference_ms / res.median_parallel_ms
                                             : std::numeric_limits<double>::infinity();
  return res;
}

std::string bench_text(const BenchResult& r) {
  std::ostringstream o;
  o << "reference_ms:";
  for (double v : r.reference_ms) o << ' ' << format_double(v);
  o << "\nparallel_ms:";
  for (double v : r.parallel_ms) o << ' ' << format_double(v);
  o << "\nmedian_reference_ms: " << format_double(r.median_reference_ms)
    << "\nmedian_parallel_ms: " << format_double(r.median_parallel_ms)
    << "\nspeedup: " << format_double(r.speedup) << '\n';
  return o.str();
}

std::string run_reconstruct(const std::string& record_path, const std::string& out_dir) {
  const GrayImage img = reconstruct(read_record(record_path));
  make_out_dir(out_dir);
  const std::string p = (fs::path(out_dir) / (fs::path(record_path).stem().string() + ".rec.pgm")).string();
  write_pgm(img, p);
  return p;
}

std::string run_verify(const std::string& record_path, const std::string& image_path) {
  const PixelRecord rec = read_record(record_path);
  const GrayImage rebuilt = reconstruct(rec);
  std::ostringstream o;
  o << record_path << ": mode=" << (rec.mode() == RecordMode::uniform ? "uniform" : "adaptive")
    << " dims=" << rec.height << 'x' << rec.width << " b=" << rec.grid_side()
    << " n=" << rec.subgrid_factor();
  if (!image_path.empty()) {
    if (!(rebuilt == read_pgm(image_path)))
      throw ConsistencyError("verify: reconstruction differs from " + image_path);
    o << " matches=" << image_path;
  }
  o << " ok";
  return o.str();
}

}  // namespace dppix
