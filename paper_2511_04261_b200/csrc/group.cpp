// group.cpp -- multi-GPU runner behind include/dppx_gpu.h (dppx_group_*).
//
// The reference's only multi-image parallelism is run_batch's file-level
// parallel_for (cli.cpp:194-211): independent files on spawned threads. The
// B200 equivalent is one persistent host thread + one dppx_ctx (own streams,
// pinned staging ring, device scratch) per GPU. A batch of frames is split
// into contiguous blocks, one per device, with no collective: noise is keyed
// per plane (plane_seeds[f*C + c]) or by global frame index (Philox
// frame_base), never by device, so the union of the blocks is byte-identical
// to one context processing the whole batch (the multi-GPU analogue of
// acceptance criterion 9, acceptance_main.cpp:356-401).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/dppx_gpu.h"

struct dppx_group {
  struct Worker {
    int device = 0;
    dppx_ctx* ctx = nullptr;
    int create_rc = DPPX_OK;
    std::thread th;
  };
  std::vector<Worker> w;
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  uint64_t generation = 0;   // bumped per job
  int running = 0;           // workers still inside the current job
  bool quit = false;
  std::function<void(int)> job;  // body(worker index)
  std::string err;
  int ready = 0;

  void loop(int i) {
    Worker& me = w[i];
    me.create_rc = dppx_ctx_create(me.device, &me.ctx);
    uint64_t seen = 0;
    {
      std::unique_lock<std::mutex> lk(mu);
      ++ready;
      cv_done.notify_all();
    }
    for (;;) {
      std::function<void(int)> body;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_job.wait(lk, [&] { return quit || generation != seen; });
        if (quit) break;
        seen = generation;
        body = job;
      }
      body(i);
      {
        std::unique_lock<std::mutex> lk(mu);
        if (--running == 0) cv_done.notify_all();
      }
    }
    if (me.ctx) dppx_ctx_destroy(me.ctx);
    me.ctx = nullptr;
  }

  // Runs body(i) on every worker thread; returns when all are done.
  void run_all(std::function<void(int)> body) {
    std::unique_lock<std::mutex> lk(mu);
    job = std::move(body);
    running = static_cast<int>(w.size());
    ++generation;
    cv_job.notify_all();
    cv_done.wait(lk, [&] { return running == 0; });
  }
};

namespace {

// First failure of a job (lowest frame block / task wins, like parallel_for's
// first captured exception, parallel.cpp:64-89).
struct FirstError {
  std::mutex mu;
  int rc = DPPX_OK;
  int64_t key = INT64_MAX;
  std::string msg;
  void set(int64_t k, int code, const char* m) {
    std::lock_guard<std::mutex> lk(mu);
    if (code != DPPX_OK && k < key) {
      key = k;
      rc = code;
      msg = m ? m : "";
    }
  }
};

int finish(dppx_group* g, FirstError& fe) {
  g->err = fe.msg;
  return fe.rc;
}

// Contiguous frame block of worker i (strong sharding, paper_2511_04261_b200/shard.py).
void block(int F, int workers, int i, int* f0, int* fk) {
  const int base = F / workers, extra = F % workers;
  *fk = base + (i < extra ? 1 : 0);
  *f0 = i * base + std::min(i, extra);
}

// The noise of frames [f0, f0 + fk) of a batch.
dppx_noise shard_noise(const dppx_noise* nz, int f0, int C, int64_t inj_plane) {
  dppx_noise s{};
  if (!nz) return s;
  s = *nz;
  if (nz->kind == DPPX_NOISE_KEYED && nz->plane_seeds) s.plane_seeds = nz->plane_seeds + static_cast<int64_t>(f0) * C;
  if (nz->kind == DPPX_NOISE_PHILOX) s.frame_base = nz->frame_base + static_cast<uint32_t>(f0);
  if (nz->kind == DPPX_NOISE_INJECTED && nz->injected)
    s.injected = nz->injected + static_cast<int64_t>(f0) * C * inj_plane;
  return s;
}

int64_t grid_count(const dppx_frames_desc* d, int b) {
  dppx_geometry g;
  if (dppx_grid_dims(d->height, d->width, b, &g) != DPPX_OK) return 0;
  return static_cast<int64_t>(g.grid_rows) * g.grid_cols;
}

// Splits the batch's frames over the workers and runs `call` on each block.
template <class Call>
int run_frames(dppx_group* g, const dppx_frames_desc* d, Call call) {
  if (!g) return DPPX_ERR_INVALID;
  if (!d) {
    g->err = "null frames descriptor";
    return DPPX_ERR_INVALID;
  }
  const int W = static_cast<int>(g->w.size());
  if (d->frames <= 1 || W == 1) {  // one block: the first device's context
    const int rc = call(g->w[0].ctx, *d, 0);
    g->err = rc ? dppx_ctx_last_error(g->w[0].ctx) : "";
    return rc;
  }
  FirstError fe;
  g->run_all([&](int i) {
    int f0, fk;
    block(d->frames, W, i, &f0, &fk);
    if (fk == 0) return;
    dppx_frames_desc s = *d;
    s.frames = fk;
    const int rc = call(g->w[i].ctx, s, f0);
    if (rc) fe.set(f0, rc, dppx_ctx_last_error(g->w[i].ctx));
  });
  return finish(g, fe);
}

}  // namespace

extern "C" {

int dppx_group_create(const int32_t* devices, int32_t count, dppx_group** out) {
  if (!out) return DPPX_ERR_INVALID;
  *out = nullptr;
  std::vector<int> devs;
  if (devices) {
    if (count < 1) return DPPX_ERR_INVALID;
    devs.assign(devices, devices + count);
  } else {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return DPPX_ERR_NO_DEVICE;
    }
    for (int i = 0; i < n && (count <= 0 || static_cast<int>(devs.size()) < count); ++i) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10 && p.minor == 0) devs.push_back(i);
    }
    if (devs.empty()) return DPPX_ERR_NO_DEVICE;
  }
  auto* g = new dppx_group();
  g->w.resize(devs.size());
  for (size_t i = 0; i < devs.size(); ++i) g->w[i].device = devs[i];
  for (size_t i = 0; i < devs.size(); ++i) g->w[i].th = std::thread([g, i] { g->loop(static_cast<int>(i)); });
  {
    std::unique_lock<std::mutex> lk(g->mu);
    g->cv_done.wait(lk, [&] { return g->ready == static_cast<int>(g->w.size()); });
  }
  for (auto& w : g->w)
    if (w.create_rc != DPPX_OK) {
      const int rc = w.create_rc;
      dppx_group_destroy(g);
      return rc;
    }
  *out = g;
  return DPPX_OK;
}

void dppx_group_destroy(dppx_group* g) {
  if (!g) return;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->quit = true;
    g->cv_job.notify_all();
  }
  for (auto& w : g->w)
    if (w.th.joinable()) w.th.join();
  delete g;
}

int32_t dppx_group_size(const dppx_group* g) { return g ? static_cast<int32_t>(g->w.size()) : 0; }

int32_t dppx_group_device(const dppx_group* g, int32_t i) {
  return g && i >= 0 && i < static_cast<int32_t>(g->w.size()) ? g->w[i].device : -1;
}

dppx_ctx* dppx_group_ctx(dppx_group* g, int32_t i) {
  return g && i >= 0 && i < static_cast<int32_t>(g->w.size()) ? g->w[i].ctx : nullptr;
}

const char* dppx_group_last_error(const dppx_group* g) { return g ? g->err.c_str() : ""; }

int dppx_group_run(dppx_group* g, int32_t tasks,
                   int (*fn)(dppx_ctx* ctx, int32_t worker, int32_t task, void* user), void* user) {
  if (!g || !fn || tasks < 0) return DPPX_ERR_INVALID;
  std::atomic<int> next{0};
  FirstError fe;
  g->run_all([&](int i) {
    for (int t = next++; t < tasks; t = next++) {
      const int rc = fn(g->w[i].ctx, i, t, user);
      if (rc) fe.set(t, rc, dppx_ctx_last_error(g->w[i].ctx));
    }
  });
  return finish(g, fe);
}

int dppx_group_pixelize_uniform(dppx_group* g, const dppx_frames_desc* desc, const uint8_t* img,
                                const dppx_privacy_params* params, const dppx_noise* noise,
                                uint8_t* means, uint8_t* out) {
  if (!params) return DPPX_ERR_INVALID;
  const int64_t G = grid_count(desc, params->b);
  return run_frames(g, desc, [&](dppx_ctx* c, const dppx_frames_desc& s, int f0) {
    const dppx_noise nz = shard_noise(noise, f0, s.channels, G);
    return dppx_pixelize_uniform(c, &s, img ? img + f0 * s.frame_stride : nullptr, params,
                                 noise ? &nz : nullptr,
                                 means ? means + static_cast<int64_t>(f0) * s.channels * G : nullptr,
                                 out ? out + f0 * s.out_frame_stride : nullptr);
  });
}

int dppx_group_pixelize_adaptive(dppx_group* g, const dppx_frames_desc* desc, const uint8_t* img,
                                 const uint8_t* mask, const dppx_privacy_params* params,
                                 const dppx_noise* noise, uint8_t* payload, int64_t payload_stride,
                                 uint32_t* payload_len, uint8_t* out) {
  if (!params) return DPPX_ERR_INVALID;
  const int64_t inj = grid_count(desc, params->b) * params->n * params->n;
  return run_frames(g, desc, [&](dppx_ctx* c, const dppx_frames_desc& s, int f0) {
    const dppx_noise nz = shard_noise(noise, f0, s.channels, inj);
    const int64_t p0 = static_cast<int64_t>(f0) * s.channels;
    return dppx_pixelize_adaptive(c, &s, img ? img + f0 * s.frame_stride : nullptr,
                                  mask ? mask + f0 * s.mask_frame_stride : nullptr, params,
                                  noise ? &nz : nullptr, payload ? payload + p0 * payload_stride : nullptr,
                                  payload_stride, payload_len ? payload_len + p0 : nullptr,
                                  out ? out + f0 * s.out_frame_stride : nullptr);
  });
}

int dppx_group_broadcast_means(dppx_group* g, const dppx_frames_desc* desc, const uint8_t* means,
                               int32_t b, uint8_t* out) {
  const int64_t G = grid_count(desc, b);
  return run_frames(g, desc, [&](dppx_ctx* c, const dppx_frames_desc& s, int f0) {
    return dppx_broadcast_means(c, &s, means ? means + static_cast<int64_t>(f0) * s.channels * G : nullptr,
                                b, out ? out + f0 * s.out_frame_stride : nullptr);
  });
}

int dppx_group_reassemble(dppx_group* g, const dppx_frames_desc* desc, const uint8_t* payload,
                          int64_t payload_stride, const uint32_t* payload_len, int32_t b, int32_t n,
                          uint8_t* out) {
  return run_frames(g, desc, [&](dppx_ctx* c, const dppx_frames_desc& s, int f0) {
    const int64_t p0 = static_cast<int64_t>(f0) * s.channels;
    return dppx_reassemble(c, &s, payload ? payload + p0 * payload_stride : nullptr, payload_stride,
                           payload_len ? payload_len + p0 : nullptr, b, n,
                           out ? out + f0 * s.out_frame_stride : nullptr);
  });
}

int dppx_group_get_stats(dppx_group* g, dppx_kernel_stats* out) {
  if (!g || !out) return DPPX_ERR_INVALID;
  *out = dppx_kernel_stats{};
  for (auto& w : g->w) {
    dppx_kernel_stats s;
    if (int rc = dppx_ctx_get_stats(w.ctx, &s)) return rc;
    for (int k = 0; k < DPPX_K_COUNT; ++k) {
      out->launches[k] += s.launches[k];
      out->device_ms[k] = std::max(out->device_ms[k], s.device_ms[k]);
    }
    out->h2d_bytes += s.h2d_bytes;
    out->d2h_bytes += s.d2h_bytes;
  }
  return DPPX_OK;
}

}  // extern "C"
