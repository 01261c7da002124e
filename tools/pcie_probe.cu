// PCIe probe for the single-small-frame path: how fast can one PETS frame
// (768x576x3 = 1.33 MB) cross the link each way, by copy engine versus by SM
// loads / stores on mapped pinned memory (zero-copy), at several CTA counts.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/pcie_probe tools/pcie_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

// each thread: U independent 16-byte loads in flight, grid-stride
template <int U>
__global__ void k_read(const uint4* __restrict__ src, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n16 ? __ldcs(src + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_write(uint4* __restrict__ dst, size_t n16) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride)
    dst[i] = make_uint4(static_cast<unsigned>(i), 1, 2, 3);
}

template <int U>
__global__ void k_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n16 ? __ldcs(src + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n16) dst[i + u * stride] = v[u];
  }
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 768ull * 576 * 3;
  const size_t n16 = bytes / 16;
  uint8_t *h_in, *h_out, *d_buf;
  unsigned* sink;
  CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d_buf, bytes));
  CK(cudaMalloc(&sink, 4));
  for (size_t i = 0; i < bytes; ++i) h_in[i] = static_cast<uint8_t>(i * 7);
  uint8_t *m_in, *m_out;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&m_in), h_in, 0));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&m_out), h_out, 0));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto&& fn) {
    for (int i = 0; i < 20; ++i) fn();
    CK(cudaStreamSynchronize(st));
    std::vector<float> v;
    for (int r = 0; r < 200; ++r) {
      CK(cudaEventRecord(e0, st));
      fn();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      v.push_back(ms * 1e3f);
    }
    std::sort(v.begin(), v.end());
    std::printf("{\"case\": \"%s\", \"bytes\": %zu, \"median_us\": %.2f, \"p10_us\": %.2f, \"gbs\": %.1f}\n", name,
                bytes, v[v.size() / 2], v[v.size() / 10], bytes / (v[v.size() / 2] * 1e3));
  };
  timeit("copy_engine_h2d", [&] { CK(cudaMemcpyAsync(d_buf, h_in, bytes, cudaMemcpyHostToDevice, st)); });
  timeit("copy_engine_d2h", [&] { CK(cudaMemcpyAsync(h_out, d_buf, bytes, cudaMemcpyDeviceToHost, st)); });
  timeit("copy_engine_h2d_then_d2h", [&] {
    CK(cudaMemcpyAsync(d_buf, h_in, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(h_out, d_buf, bytes, cudaMemcpyDeviceToHost, st));
  });
  // both directions at once: copy engine H2D on `st`, the other direction on `st2`
  cudaStream_t st2;
  CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  cudaEvent_t fork, join;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  uint8_t* d_buf2;
  CK(cudaMalloc(&d_buf2, bytes));
  auto both = [&](auto&& other) {
    CK(cudaEventRecord(fork, st));
    CK(cudaStreamWaitEvent(st2, fork, 0));
    CK(cudaMemcpyAsync(d_buf, h_in, bytes, cudaMemcpyHostToDevice, st));
    other();
    CK(cudaEventRecord(join, st2));
    CK(cudaStreamWaitEvent(st, join, 0));
  };
  timeit("ce_h2d_parallel_ce_d2h", [&] {
    both([&] { CK(cudaMemcpyAsync(h_out, d_buf2, bytes, cudaMemcpyDeviceToHost, st2)); });
  });
  for (int blocks : {36, 148}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "ce_h2d_parallel_zc_write_b%d", blocks);
    timeit(nm, [&] {
      both([&] { k_write<<<blocks, 256, 0, st2>>>(reinterpret_cast<uint4*>(m_out), n16); });
    });
  }
  char name[96];
  for (int blocks : {36, 74, 148, 296, 592}) {
    for (int threads : {256, 512}) {
      std::snprintf(name, sizeof name, "zc_read_u4_b%d_t%d", blocks, threads);
      timeit(name, [&] {
        k_read<4><<<blocks, threads, 0, st>>>(reinterpret_cast<const uint4*>(m_in), n16, sink);
      });
      std::snprintf(name, sizeof name, "zc_read_u1_b%d_t%d", blocks, threads);
      timeit(name, [&] {
        k_read<1><<<blocks, threads, 0, st>>>(reinterpret_cast<const uint4*>(m_in), n16, sink);
      });
      std::snprintf(name, sizeof name, "zc_write_b%d_t%d", blocks, threads);
      timeit(name, [&] { k_write<<<blocks, threads, 0, st>>>(reinterpret_cast<uint4*>(m_out), n16); });
      std::snprintf(name, sizeof name, "zc_copy_u4_b%d_t%d", blocks, threads);
      timeit(name, [&] {
        k_copy<4><<<blocks, threads, 0, st>>>(reinterpret_cast<const uint4*>(m_in), reinterpret_cast<uint4*>(m_out),
                                              n16);
      });
    }
  }
  timeit("empty_kernel", [&] { k_write<<<1, 32, 0, st>>>(reinterpret_cast<uint4*>(d_buf), 0); });
  return 0;
}
