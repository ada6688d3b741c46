// kvm.store_cache(k_t, v_t, 'decode') — P:123 [§4.2 Decode stage], P:266-273 [Alg. 1].
//
// Per (b, owned kv-head) instance, one CTA of 128 threads (thread e owns dimension e):
//   1. if this step is a boundary (flag) and the open segment is non-empty, seal it
//      (push (start, len) onto the sealed FIFO); force-seal when it reached max_open_segment
//      (reading R-AMB13);
//   2. append (k_t, v_t) to the local ring buffer;
//   3. while the buffer holds more than W tokens and a sealed segment exists, evict the oldest
//      sealed segment (FIFO): centroid = fp32 sequential sum of its keys in time order / len
//      (bit-identical to the oracle's recipe), bf16 copy, unit table entry (id = k + eviction
//      index), and the K/V rows written to the pinned host pool (zero-copy stores over the host
//      link, "Offload (K_seg, V_seg) to CPU memory pool").
// The open segment is never evicted.
#include "lkv_append_dev.cuh"

namespace lkv {

__global__ void __launch_bounds__(128) append_kernel(AppendArgs a) {
  pdl_wait_trigger();
  append_one(a, blockIdx.x, a.flag ? a.flag[blockIdx.x / a.hn] : 0);
}

// standalone gather of the pending jobs (unfused API path): grid (instances, row slices)
__global__ void __launch_bounds__(256) gather_kernel(AppendArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.x;
  const GatherJob J = a.jobs[li];
  const int per = (J.n_rows + gridDim.y - 1) / gridDim.y;
  const int r0 = blockIdx.y * per, r1 = min(J.n_rows, r0 + per);
  if (r0 < r1) gather_rows(a, li, J, r0, r1);
}

__global__ void clear_jobs_kernel(GatherJob* jobs, int n) {
  pdl_wait_trigger();
  for (int i = threadIdx.x; i < n; i += blockDim.x) jobs[i].n_rows = 0;
}

// full-cache layer: append (k_t, v_t) at row P + t - 1 of every (b, head) and commit the
// layer's step counter; one CTA so the read of t and its commit cannot race.
__global__ void __launch_bounds__(256) full_step_kernel(const bf16* k_t, const bf16* v_t, int64_t stride_b, int n,
                                                        int hn, bf16* full, int64_t full_cap, int64_t P, int* step,
                                                        int* error) {
  pdl_wait_trigger();
  const int t = *step + 1;
  const int64_t pos = P + t - 1;
  if (pos >= full_cap) {
    if (threadIdx.x == 0) *error = 1;
  } else {
    for (int i = threadIdx.x; i < n * 32; i += blockDim.x) {
      const int li = i >> 5, lane = i & 31, b = li / hn, h = li % hn;
      bf16* K = full + (int64_t)li * 2 * full_cap * D;
      bf16* V = K + full_cap * D;
      const bf16* src = (lane < 16 ? k_t : v_t) + (int64_t)b * stride_b + (int64_t)h * D;
      bf16* dst = (lane < 16 ? K : V) + pos * D;
      reinterpret_cast<uint4*>(dst)[lane & 15] = reinterpret_cast<const uint4*>(src)[lane & 15];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *step = t;
}

cudaError_t launch_append(const AppendArgs& a, cudaStream_t st) {
  const int gy = a.budget >= 64 ? a.budget / 64 : 1;
  launch_k(gather_kernel, dim3(a.batch * a.hn, gy), dim3(256), 0, st, a);
  launch_k(clear_jobs_kernel, dim3(1), dim3(256), 0, st, a.jobs, a.batch * a.hn);
  launch_k(append_kernel, dim3(a.batch * a.hn), dim3(128), 0, st, a);
  return cudaGetLastError();
}

cudaError_t launch_full_step(const bf16* k_t, const bf16* v_t, int64_t stride_b, int batch, int hn, bf16* full,
                             int64_t full_cap, int64_t P, int* step, int* error, cudaStream_t st) {
  launch_k(full_step_kernel, dim3(1), dim3(256), 0, st, k_t, v_t, stride_b, batch * hn, hn, full, full_cap, P, step, error);
  return cudaGetLastError();
}

}  // namespace lkv
