// ingest.cpp -- PGM ingest (pgm.cpp:26-119 semantics) and the GPU batch runner
// (run_batch cli.cpp:175-213 / run_single cli.cpp:93-173 semantics).
//
// The batch runner reads files on host threads, groups frames of one shape,
// and sends up to frames_per_call frames per C-ABI call through the pinned
// H2D -> kernels -> D2H pipeline; encode, reconstruct check (on the GPU),
// mse/ssim (on the GPU) and file writes follow per file exactly as run_single
// does. Every file gets the same seed, as the reference's run_batch does.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <thread>
#include <utility>

#include "dppix/batch.hpp"
#include "dppix/errors.hpp"
#include "dppix/pgm.hpp"
#include "dppix/record.hpp"
#include "dppx_gpu.h"

namespace dppix {
dppx_ctx* dropin_thread_ctx();  // dropin.cpp
}

namespace dppix {
namespace fs = std::filesystem;

namespace {

int header_int(std::istream& in, const std::string& path, const char* field) {
  for (;;) {  // whitespace and '#' comments before each token
    const int ch = in.peek();
    if (ch == std::char_traits<char>::eof()) throw IoError("read_pgm: truncated header in " + path);
    if (ch == '#') {
      in.ignore(std::numeric_limits<std::streamsize>::max(), '\n');
      continue;
    }
    if (std::isspace(ch)) {
      in.get();
      continue;
    }
    break;
  }
  long long v = 0;
  if (!(in >> v) || v < 0) throw IoError("read_pgm: bad " + std::string(field) + " in " + path);
  if (v > std::numeric_limits<int>::max())
    throw IoError("read_pgm: " + std::string(field) + " overflows in " + path);
  return static_cast<int>(v);
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

[[noreturn]] void raise_status(int rc, const std::string& who) {
  const std::string msg = who + ": " + dppx_ctx_last_error(dropin_thread_ctx());
  if (rc == DPPX_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == DPPX_ERR_CORRUPT) throw RecordError(RecordErrorKind::corrupt_record, msg);
  if (rc == DPPX_ERR_OOM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

struct HostBuf {  // pageable host batch buffer (no zero fill)
  std::unique_ptr<uint8_t[]> mem;
  uint8_t* p = nullptr;
  explicit HostBuf(size_t bytes) : mem(new uint8_t[bytes ? bytes : 1]), p(mem.get()) {}
};


}  // namespace

// ---------------------------------------------------------------- pgm.hpp
GrayImage read_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("read_pgm: cannot open " + path);
  char magic[2] = {0, 0};
  in.read(magic, 2);
  if (!in || magic[0] != 'P' || magic[1] != '5')
    throw IoError("read_pgm: not a binary PGM (P5): " + path);
  const int width = header_int(in, path, "width");
  const int height = header_int(in, path, "height");
  const int maxval = header_int(in, path, "maxval");
  if (width < 1 || height < 1) throw IoError("read_pgm: non-positive dimensions in " + path);
  if (maxval != 255) throw IoError("read_pgm: unsupported maxval (expected 255) in " + path);
  const int sep = in.get();  // exactly one whitespace byte before the raster
  if (sep == std::char_traits<char>::eof() || !std::isspace(sep))
    throw IoError("read_pgm: missing raster separator in " + path);
  GrayImage img = make_image(height, width);
  in.read(reinterpret_cast<char*>(img.pixels.data()), static_cast<std::streamsize>(img.pixels.size()));
  if (static_cast<std::size_t>(in.gcount()) != img.pixels.size())
    throw IoError("read_pgm: truncated pixel data in " + path);
  return img;
}

void write_pgm(const GrayImage& img, const std::string& path) {
  if (img.height < 1 || img.width < 1 ||
      img.pixels.size() != static_cast<std::size_t>(img.height) * img.width)
    throw IoError("write_pgm: malformed image for " + path);
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("write_pgm: cannot open " + path);
  out << "P5\n" << img.width << ' ' << img.height << "\n255\n";
  out.write(reinterpret_cast<const char*>(img.pixels.data()),
            static_cast<std::streamsize>(img.pixels.size()));
  out.flush();
  if (!out) throw IoError("write_pgm: write failed for " + path);
}

RegionMask read_mask_pgm(const std::string& path) {
  const GrayImage img = read_pgm(path);
  RegionMask mask = make_mask(img.height, img.width, 0);
  for (std::size_t i = 0; i < img.pixels.size(); ++i) mask.values[i] = img.pixels[i] >= 128 ? 1 : 0;
  return mask;
}

// ---------------------------------------------------------------- batch.hpp
int batch_exit_code_for(const std::exception& err) {  // cli.cpp:386-401
  if (dynamic_cast<const ConsistencyError*>(&err)) return 5;
  if (dynamic_cast<const RecordError*>(&err)) return 4;
  if (dynamic_cast<const IoError*>(&err)) return 3;
  if (dynamic_cast<const UsageError*>(&err) || dynamic_cast<const std::invalid_argument*>(&err))
    return 2;
  return 1;
}

std::vector<BatchFileReport> run_batch_gpu(const BatchConfig& cfg) {
  // validate_run_config, cli.cpp:78-89.
  if (!(cfg.epsilon > 0.0) && cfg.seed.has_value()) throw UsageError("--epsilon must be > 0");
  if (cfg.mode == BatchMode::reference && cfg.emit_record)
    throw UsageError("reference mode keeps no grid statistics and cannot emit records");
  if (cfg.mode == BatchMode::adaptive && cfg.mask_path.empty())
    throw UsageError("adaptive mode requires --mask");
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
  std::vector<GrayImage> imgs(nfile);
  std::vector<RegionMask> masks(cfg.mode == BatchMode::adaptive ? nfile : 0);
  std::vector<char> ok(nfile, 0);
  auto fail = [&](int i, const std::exception& err) {
    reports[i].error = err.what();
    reports[i].exit_code = batch_exit_code_for(err);
  };
  // DPPX_BATCH_TRACE=1: per-phase wall times on stderr.
  static const bool trace = std::getenv("DPPX_BATCH_TRACE") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto T0 = tnow();
  // ---- ingest (host threads) ----
  parallel_over(nfile, io, [&](int i) {
    reports[i].input = inputs[i];
    try {
      imgs[i] = read_pgm(inputs[i]);
      if (cfg.mode == BatchMode::adaptive) {  // mask_path_for, cli.cpp:43-58
        fs::path mpath(cfg.mask_path);
        std::error_code e2;
        if (fs::is_directory(mpath, e2)) {
          const fs::path paired = mpath / (fs::path(inputs[i]).stem().string() + ".pgm");
          if (!fs::exists(paired, e2))
            throw IoError("no mask for " + inputs[i] + " (expected " + paired.string() + ")");
          mpath = paired;
        }
        masks[i] = read_mask_pgm(mpath.string());
        if (masks[i].height != imgs[i].height || masks[i].width != imgs[i].width)
          throw UsageError("mask dimensions do not match image: " + inputs[i]);
      }
      ok[i] = 1;
    } catch (const std::exception& err) {
      fail(i, err);
    }
  });
  const auto T1 = tnow();
  if (trace) std::fprintf(stderr, "batch: ingest %.1f ms\n", tms(T0, T1));
  // ---- group by shape, GPU calls of up to frames_per_call frames ----
  std::map<std::pair<int, int>, std::vector<int>> groups;
  for (int i = 0; i < nfile; ++i)
    if (ok[i]) groups[{imgs[i].height, imgs[i].width}].push_back(i);
  const double eff_eps = cfg.epsilon > 0.0 ? cfg.epsilon : 1.0;  // cli.cpp:97-102
  const int n = cfg.mode == BatchMode::adaptive ? cfg.n : 1;
  if (cfg.emit_image || cfg.emit_record) {
    fs::create_directories(cfg.out_dir, ec);
    if (ec) throw IoError("cannot create output directory " + cfg.out_dir + ": " + ec.message());
  }
  dppx_ctx* ctx = dropin_thread_ctx();
  for (auto& [shape, members] : groups) {
    const int M = shape.first, N = shape.second;
    dppx_privacy_params pp;
    if (dppx_make_privacy_params(eff_eps, cfg.m, cfg.b, n, &pp) != DPPX_OK) {
      for (int i : members) fail(i, std::invalid_argument("make_privacy_params: invalid parameters"));
      continue;
    }
    const size_t plane = static_cast<size_t>(M) * N;
    const int K = std::max(1, cfg.frames_per_call);
    for (size_t c0 = 0; c0 < members.size(); c0 += K) {
      const int F = static_cast<int>(std::min<size_t>(K, members.size() - c0));
      const std::vector<int> chunk(members.begin() + c0, members.begin() + c0 + F);
      try {
        // Pageable batch buffers: pinning hundreds of MB per call costs more
        // than the driver-staged copies of pageable memory (measured).
        HostBuf in(plane * F), out(plane * F), mk(cfg.mode == BatchMode::adaptive ? plane * F : 0);
        parallel_over(F, io, [&](int k) {
          std::memcpy(in.p + k * plane, imgs[chunk[k]].pixels.data(), plane);
          if (cfg.mode == BatchMode::adaptive)
            std::memcpy(mk.p + k * plane, masks[chunk[k]].values.data(), plane);
        });
        dppx_frames_desc d{M, N, 1, F, N, static_cast<int64_t>(plane), N, static_cast<int64_t>(plane),
                           N, static_cast<int64_t>(plane)};
        std::vector<uint64_t> seeds(F, cfg.seed ? cfg.seed->value : 0);
        dppx_noise nz{cfg.seed ? DPPX_NOISE_KEYED : DPPX_NOISE_NONE, 0, seeds.data(), nullptr};
        dppx_geometry g;
        dppx_grid_dims(M, N, cfg.b, &g);
        const size_t G = static_cast<size_t>(g.grid_rows) * g.grid_cols;
        const size_t cap = cfg.mode == BatchMode::adaptive
                               ? (dppx_adaptive_payload_capacity(M, N, cfg.b, n) + 3) & ~size_t{3}
                               : G;
        std::vector<uint8_t> stats(cap * F);
        std::vector<uint32_t> lens(F, static_cast<uint32_t>(G));
        const auto t0 = std::chrono::steady_clock::now();
        int rc;
        if (cfg.mode == BatchMode::adaptive)
          rc = dppx_pixelize_adaptive(ctx, &d, in.p, mk.p, &pp, &nz, stats.data(),
                                      static_cast<int64_t>(cap), lens.data(), out.p);
        else if (cfg.mode == BatchMode::uniform)
          rc = dppx_pixelize_uniform(ctx, &d, in.p, &pp, &nz, stats.data(), out.p);
        else
          rc = dppx_pixelize_reference(ctx, &d, in.p, &pp, &nz, stats.data(), out.p);
        const auto t1 = std::chrono::steady_clock::now();
        if (trace) std::fprintf(stderr, "batch: pixelize %d frames %.1f ms\n", F, tms(t0, t1));
        if (rc != DPPX_OK) raise_status(rc, "pixelize");
        const double per_ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / F;
        // ---- records + reconstruct check (cli.cpp:132-146), on the GPU ----
        std::vector<std::vector<uint8_t>> recs(F);
        if (cfg.mode != BatchMode::reference) {
          std::vector<char> enc_ok(F, 1);
          parallel_over(F, io, [&](int k) {  // header + CRC32 per file, independent
            recs[k].resize(dppx_record_size(lens[k]));
            size_t len = 0;
            enc_ok[k] = dppx_encode_record(M, N, cfg.b, n, cfg.mode == BatchMode::adaptive ? 2 : 1,
                                           stats.data() + k * cap, lens[k], recs[k].data(), recs[k].size(),
                                           &len) == DPPX_OK;
          });
          for (int k = 0; k < F; ++k)
            if (!enc_ok[k]) throw std::invalid_argument("encode: payload inconsistent");
          if (cfg.reconstruct_check) {
            HostBuf rebuilt(plane * F);
            std::vector<uint8_t> payload(cap * F);
            std::vector<uint32_t> plen(F);
            for (int k = 0; k < F; ++k) {  // decode, then rebuild from the decoded payload
              dppx_record_info info{};
              const int drc = dppx_decode_record(recs[k].data(), recs[k].size(), &info);
              if (drc != DPPX_OK) throw RecordError(RecordErrorKind::corrupt_record, "decode failed");
              std::memcpy(payload.data() + k * cap, recs[k].data() + info.payload_offset, info.payload_len);
              plen[k] = info.payload_len;
            }
            const int rrc = cfg.mode == BatchMode::adaptive
                                ? dppx_reassemble(ctx, &d, payload.data(), static_cast<int64_t>(cap),
                                                  plen.data(), cfg.b, n, rebuilt.p)
                                : dppx_broadcast_means(ctx, &d, payload.data(), cfg.b, rebuilt.p);
            if (rrc != DPPX_OK) raise_status(rrc, "reconstruct");
            std::vector<char> same(F, 1);
            parallel_over(F, io, [&](int k) {
              same[k] = std::memcmp(rebuilt.p + k * plane, out.p + k * plane, plane) == 0;
            });
            for (int k = 0; k < F; ++k)
              if (!same[k]) {
                fail(chunk[k], ConsistencyError("reconstruction does not match the emitted image for " +
                                                inputs[chunk[k]]));
              }
          }
        }
        const auto t2 = tnow();
        if (trace) std::fprintf(stderr, "batch: records + reconstruct check %.1f ms\n", tms(t1, t2));
        // ---- metrics on the GPU (cli.cpp:164-171) ----
        std::vector<double> mses(F), ssims(F, std::numeric_limits<double>::quiet_NaN());
        if (dppx_metrics(ctx, &d, in.p, out.p, mses.data(), M >= 7 && N >= 7 ? ssims.data() : nullptr) !=
            DPPX_OK)
          raise_status(DPPX_ERR_CUDA, "metrics");
        const auto t3 = tnow();
        if (trace) std::fprintf(stderr, "batch: metrics %.1f ms\n", tms(t2, t3));
        // ---- outputs (host threads) ----
        parallel_over(F, io, [&](int k) {
          const int i = chunk[k];
          if (reports[i].exit_code != 0) return;
          try {
            const std::string stem = fs::path(inputs[i]).stem().string();
            if (cfg.emit_image) {
              GrayImage pix = make_image(M, N);
              std::memcpy(pix.pixels.data(), out.p + k * plane, plane);
              const std::string path = (fs::path(cfg.out_dir) / (stem + ".pix.pgm")).string();
              write_pgm(pix, path);
              reports[i].written.push_back(path);
            }
            if (cfg.mode != BatchMode::reference && cfg.emit_record) {
              const std::string path = (fs::path(cfg.out_dir) / (stem + ".dppx")).string();
              std::ofstream f(path, std::ios::binary | std::ios::trunc);
              if (!f) throw IoError("write_record: cannot open " + path);
              f.write(reinterpret_cast<const char*>(recs[k].data()),
                      static_cast<std::streamsize>(recs[k].size()));
              f.flush();
              if (!f) throw IoError("write_record: write failed for " + path);
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
        if (trace) std::fprintf(stderr, "batch: outputs %.1f ms\n", tms(t3, tnow()));
      } catch (const std::exception& err) {
        for (int i : chunk)
          if (reports[i].exit_code == 0) fail(i, err);
      }
    }
  }
  return reports;
}

}  // namespace dppix
