// Mask bit packing for the host pipeline (see maskpack.h). A small persistent
// worker pool (the caller thread takes a share too) splits the rows; each row
// is packed 32 bytes -> one u32 word with AVX2 movemask where the CPU has it,
// else 8 bytes at a time with a multiply gather.
#include "maskpack.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace dppx {

namespace {

constexpr uint64_t kNotBinary = 0xFEFEFEFEFEFEFEFEull;

// Bits 56..63 of (x * kGather) are the low bits of x's eight bytes when every
// byte is 0 or 1 (the partial products land on distinct bit positions).
constexpr uint64_t kGather = 0x0102040810204080ull;

bool pack_row_portable(const uint8_t* s, int N, uint32_t* w) {
  uint64_t seen = 0;
  const int full = N / 32;
  for (int k = 0; k < full; ++k) {
    uint32_t word = 0;
    for (int q = 0; q < 4; ++q) {
      uint64_t x;
      std::memcpy(&x, s + 32 * k + 8 * q, 8);
      seen |= x;
      word |= static_cast<uint32_t>((x * kGather) >> 56) << (8 * q);
    }
    w[k] = word;
  }
  if (full * 32 < N) {
    uint32_t word = 0;
    for (int j = full * 32; j < N; ++j) {
      seen |= s[j];
      word |= static_cast<uint32_t>(s[j] & 1u) << (j & 31);
    }
    w[full] = word;
  }
  return (seen & kNotBinary) == 0;
}

__attribute__((target("avx2"))) bool pack_row_avx2(const uint8_t* s, int N, uint32_t* w) {
  __m256i seen = _mm256_setzero_si256();
  const int full = N / 32;
  for (int k = 0; k < full; ++k) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + 32 * k));
    seen = _mm256_or_si256(seen, v);
    w[k] = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_slli_epi16(v, 7)));
  }
  bool ok = _mm256_testz_si256(seen, _mm256_set1_epi8(static_cast<char>(0xFE))) != 0;
  if (full * 32 < N) {
    uint32_t word = 0, tail = 0;
    for (int j = full * 32; j < N; ++j) {
      tail |= s[j];
      word |= static_cast<uint32_t>(s[j] & 1u) << (j & 31);
    }
    w[full] = word;
    ok = ok && (tail & 0xFEu) == 0;
  }
  return ok;
}

}  // namespace

struct MaskPacker {
  int nthreads = 1;  // including the calling thread
  bool avx2 = false;
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable go, done;
  uint64_t generation = 0;
  int pending = 0;
  bool stop = false;
  std::function<void(int)> job;

  void worker(int id) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int)> f;
      {
        std::unique_lock<std::mutex> lk(mu);
        go.wait(lk, [&] { return stop || generation != seen; });
        if (stop) return;
        seen = generation;
        f = job;
      }
      f(id);
      {
        std::lock_guard<std::mutex> lk(mu);
        if (--pending == 0) done.notify_one();
      }
    }
  }

  void run(const std::function<void(int)>& f) {
    if (nthreads == 1) {
      f(0);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      job = f;
      pending = nthreads - 1;
      ++generation;
    }
    go.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu);
    done.wait(lk, [&] { return pending == 0; });
  }
};

MaskPacker* mask_packer_create(int threads) {
  auto* p = new MaskPacker;
  if (threads <= 0) {
    const char* env = std::getenv("DPPX_PACK_THREADS");
    threads = env ? std::atoi(env) : 0;
  }
  if (threads <= 0) {
    const unsigned hw = std::thread::hardware_concurrency();
    threads = static_cast<int>(std::clamp(hw / 4u, 1u, 4u));
  }
  p->nthreads = std::max(1, threads);
  __builtin_cpu_init();
  p->avx2 = __builtin_cpu_supports("avx2");
  try {
    for (int i = 1; i < p->nthreads; ++i) p->workers.emplace_back(&MaskPacker::worker, p, i);
  } catch (...) {  // no threads available: pack on the calling thread plus what started
    p->nthreads = static_cast<int>(p->workers.size()) + 1;
  }
  return p;
}

void mask_packer_destroy(MaskPacker* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    p->stop = true;
  }
  p->go.notify_all();
  for (auto& t : p->workers) t.join();
  delete p;
}

int mask_packer_threads(const MaskPacker* p) { return p ? p->nthreads : 0; }

bool pack_mask_bits(MaskPacker* p, const uint8_t* src, int64_t pitch, int64_t fstride, int M, int N,
                    int F, uint32_t* dst, int64_t wpr) {
  const int64_t rows = static_cast<int64_t>(M) * F;
  std::atomic<bool> ok{true};
  const int parts = p->nthreads;
  const bool avx2 = p->avx2;
  p->run([&](int id) {
    const int64_t r0 = rows * id / parts, r1 = rows * (id + 1) / parts;
    bool good = true;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t f = r / M, i = r % M;
      const uint8_t* s = src + f * fstride + i * pitch;
      uint32_t* w = dst + r * wpr;
      good = (avx2 ? pack_row_avx2(s, N, w) : pack_row_portable(s, N, w)) && good;
    }
    if (!good) ok.store(false, std::memory_order_relaxed);
  });
  return ok.load();
}

void pool_for(MaskPacker* p, int64_t n, const std::function<void(int64_t, int64_t)>& body) {
  const int parts = p->nthreads;
  p->run([&](int id) {
    const int64_t b0 = n * id / parts, b1 = n * (id + 1) / parts;
    if (b0 < b1) body(b0, b1);
  });
}

}  // namespace dppx
