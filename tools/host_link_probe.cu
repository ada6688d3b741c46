// Host-link peaks on this box (SURVEY §8(d) "host-link peak measurement"): pinned cudaMemcpy H2D and
// D2H of 1 GiB (best of 5), and a zero-copy READ kernel over mapped pinned memory (16-B vector loads,
// every SM, best of 5) — the access pattern of the gather. Prints one JSON line.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/host_link_probe tools/host_link_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void zc_read(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {  // four 16-B loads in flight per thread
    const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc ^= src[i].x;
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 1ull << 30;
  void *h, *d;
  unsigned long long* sink;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  cudaMalloc(&sink, 8);
  for (size_t i = 0; i < bytes; i += 4096) reinterpret_cast<char*>(h)[i] = (char)i;
  void* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best_h2d = 1e9f, best_d2h = 1e9f, best_zc = 1e9f, ms;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    best_h2d = ms < best_h2d ? ms : best_h2d;
    cudaEventRecord(a);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    best_d2h = ms < best_d2h ? ms : best_d2h;
    cudaEventRecord(a);
    zc_read<<<nsm * 4, 256>>>(reinterpret_cast<const uint4*>(hd), bytes / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    best_zc = ms < best_zc ? ms : best_zc;
  }
  const cudaError_t e = cudaGetLastError();
  printf("{\"bytes\": %zu, \"h2d_memcpy_gbs\": %.2f, \"d2h_memcpy_gbs\": %.2f, \"zero_copy_read_gbs\": %.2f, "
         "\"sms\": %d, \"status\": \"%s\"}\n",
         bytes, bytes / (best_h2d / 1e3) / 1e9, bytes / (best_d2h / 1e3) / 1e9, bytes / (best_zc / 1e3) / 1e9, nsm,
         cudaGetErrorString(e));
  return 0;
}
