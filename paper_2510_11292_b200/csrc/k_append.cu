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
#include "lkv_internal.cuh"

namespace lkv {

__global__ void __launch_bounds__(128) append_kernel(AppendArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.x;
  const int b = li / a.hn;
  const int tid = threadIdx.x;
  InstState* S = a.inst + li;
  const int flag = a.flag ? a.flag[b] : 0;
  const int dec = *a.step - 1;  // decode index of this token (device step counter)
  const int cap = a.ring_cap;
  int2* fifo = a.fifo + (int64_t)li * cap;
  bf16* ringK = a.ring + (int64_t)li * 2 * cap * D;
  bf16* ringV = ringK + (int64_t)cap * D;

  __shared__ InstState s;
  if (tid == 0) {
    s = *S;
    if ((flag && s.open_len > 0) || s.open_len >= a.max_open) {
      fifo[(s.fifo_head + s.fifo_count) % cap] = make_int2(s.open_start, s.open_len);
      s.fifo_count++;
      s.open_len = 0;
    }
    if (s.open_len == 0) s.open_start = dec;
    if (s.buffered == 0) s.ring_head = dec;
    s.open_len++;
    s.buffered++;
  }
  // append the token's K and V rows
  const int slot = dec % cap;
  if (tid < 16) {
    const uint4* src = reinterpret_cast<const uint4*>(a.k_t + (int64_t)b * a.stride_b + (int64_t)(li % a.hn) * D);
    reinterpret_cast<uint4*>(ringK + (int64_t)slot * D)[tid] = src[tid];
  } else if (tid < 32) {
    const uint4* src = reinterpret_cast<const uint4*>(a.v_t + (int64_t)b * a.stride_b + (int64_t)(li % a.hn) * D);
    reinterpret_cast<uint4*>(ringV + (int64_t)slot * D)[tid - 16] = src[tid - 16];
  }
  __syncthreads();

  float* cent = a.cent + (int64_t)li * a.Umax * D;
  uint16_t* centb = reinterpret_cast<uint16_t*>(a.centb) + (int64_t)li * a.Umax * D;
  uint8_t* pool = a.pool + (int64_t)li * a.pool_inst_bytes;
  int32_t* ppos = a.pool_pos + (int64_t)li * a.pool_rows_cap;
  while (s.buffered > a.W && s.fifo_count > 0 && !s.error) {
    const int2 seg = fifo[s.fifo_head];
    const int start = seg.x, len = seg.y;
    const int uid = s.n_units;
    const int64_t prow = s.pool_rows;
    if (uid >= a.Umax || prow + len > a.pool_rows_cap) {
      __syncthreads();
      if (tid == 0) s.error = 1;
      __syncthreads();
      break;
    }
    // centroid: sequential fp32 sum in time order, then one RN division (recipe)
    {
      float sum = 0.0f;
      const uint16_t* rk = reinterpret_cast<const uint16_t*>(ringK);
      for (int i = 0; i < len; ++i) sum = __fadd_rn(sum, bf2f(rk[(int64_t)((start + i) % cap) * D + tid]));
      const float c = __fdiv_rn(sum, (float)len);
      cent[(int64_t)uid * D + tid] = c;
      centb[(int64_t)uid * D + tid] = f2bf_rne(c);
    }
    // offload rows: unit-major span [K rows | V rows] at pool row offset prow
    uint4* dst = reinterpret_cast<uint4*>(pool + prow * POOL_ROW_BYTES);
    for (int c = tid; c < 2 * len * 16; c += blockDim.x) {
      const int isV = c >= len * 16;
      const int cc = isV ? c - len * 16 : c;
      const int i = cc >> 4, sub = cc & 15;
      const bf16* src = (isV ? ringV : ringK) + (int64_t)((start + i) % cap) * D;
      dst[(int64_t)(isV ? len + i : i) * 16 + sub] = reinterpret_cast<const uint4*>(src)[sub];
    }
    for (int i = tid; i < len; i += blockDim.x) ppos[prow + i] = s.prompt_len + start + i;
    __syncthreads();
    if (tid == 0) {
      a.usize[(int64_t)li * a.Umax + uid] = len;
      a.uoff[(int64_t)li * a.Umax + uid] = prow;
      a.ufirst[(int64_t)li * a.Umax + uid] = s.prompt_len + start;
      a.sel[(int64_t)li * a.Umax + uid] = 0;
      s.n_units++;
      s.pool_rows += len;
      s.buffered -= len;
      s.ring_head += len;
      s.fifo_head = (s.fifo_head + 1) % cap;
      s.fifo_count--;
      atomicAdd(&a.stats->segments_evicted, 1ull);
      atomicAdd(&a.stats->bytes_d2h, (unsigned long long)len * POOL_ROW_BYTES);
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) *S = s;
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
  launch_k(append_kernel, dim3(a.batch * a.hn), dim3(128), 0, st, a);
  return cudaGetLastError();
}

cudaError_t launch_full_step(const bf16* k_t, const bf16* v_t, int64_t stride_b, int batch, int hn, bf16* full,
                             int64_t full_cap, int64_t P, int* step, int* error, cudaStream_t st) {
  launch_k(full_step_kernel, dim3(1), dim3(256), 0, st, k_t, v_t, stride_b, batch * hn, hn, full, full_cap, P, step, error);
  return cudaGetLastError();
}

}  // namespace lkv
