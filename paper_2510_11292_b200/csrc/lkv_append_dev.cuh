// Shared device code of kvm.store_cache(k_t, v_t, 'decode'): used by the standalone
// append kernel and by the clustered append+attention kernel.
#pragma once
#include "lkv_internal.cuh"

namespace lkv {

// Row-granular gather of instance li's pending job, rows [r0, r1) by this CTA: 16 lanes x 16 B
// per row, two rows in flight per thread; new units are read zero-copy from the pinned host pool,
// kept units device-to-device.
__device__ __forceinline__ void gather_rows(const AppendArgs& a, int li, const GatherJob& J, int r0, int r1) {
  const RowSrc* R = a.rows + (int64_t)li * a.budget;
  const int sub = threadIdx.x & 15;
  const int rpp = blockDim.x >> 4;
  uint4* dK = reinterpret_cast<uint4*>(J.dstK);
  uint4* dV = reinterpret_cast<uint4*>(J.dstV);
  for (int r = r0 + (threadIdx.x >> 4); r < r1; r += 2 * rpp) {
    const int r2 = r + rpp;
    const RowSrc s0 = R[r];
    const uint4 k0 = load_row_piece(s0.k, sub), v0 = load_row_piece(s0.v, sub);
    uint4 k1 = k0, v1 = v0;
    if (r2 < r1) {
      const RowSrc s1 = R[r2];
      k1 = load_row_piece(s1.k, sub);
      v1 = load_row_piece(s1.v, sub);
    }
    dK[(int64_t)r * (D / 8) + sub] = k0;
    dV[(int64_t)r * (D / 8) + sub] = v0;
    if (r2 < r1) {
      dK[(int64_t)r2 * (D / 8) + sub] = k1;
      dV[(int64_t)r2 * (D / 8) + sub] = v1;
    }
  }
}

// Called by every thread of one CTA (blockDim >= 128: thread e < 128 owns dimension e of the
// centroid); `flag` = this step's trigger decision. The token's decode index is the instance's
// completed-step count, which this call commits (+1); leaves the post-append state in global memory.
// pre: optional copy of the instance state already in shared memory (else loaded from global).
// The working-set fields (ws_cur, ws_rows) belong to the retrieval and are not written here.
// row_written: the caller already stored (k_t, v_t) into the ring slot of this token (decode index
// = pre->step) — the layer kernel does so from registers right after its inputs arrive.
__device__ __forceinline__ void append_one(const AppendArgs& a, const int li, const int flag,
                                           const InstState* pre = nullptr, const bool row_written = false) {
  const int b = li / a.hn;
  const int tid = threadIdx.x;
  InstState* S = a.inst + li;
  const int cap = a.ring_cap;
  int2* fifo = a.fifo + (int64_t)li * cap;
  bf16* ringK = a.ring + (int64_t)li * 2 * cap * D;
  bf16* ringV = ringK + (int64_t)cap * D;

  __shared__ InstState s;  // (function-scope shared: one instance per CTA)
  __shared__ int s_dec;
  if (tid == 0) {
    s = pre ? *pre : *S;
    const int dec = s.step;  // decode index (0-based) of this token
    s_dec = dec;
    s.step = dec + 1;
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
  __syncthreads();
  // append the token's K and V rows
  const int slot = s_dec % cap;
  if (row_written) {
  } else if (tid < 16) {
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
      if (tid < D) {
        for (int i = 0; i < len; ++i) sum = __fadd_rn(sum, bf2f(rk[(int64_t)((start + i) % cap) * D + tid]));
        const float c = __fdiv_rn(sum, (float)len);
        cent[(int64_t)uid * D + tid] = c;
        centb[(int64_t)uid * D + tid] = f2bf_rne(c);
      }
    }
    // offload rows: unit-major span [K rows | V rows] at pool row offset prow (FP8 pool: E4M3 rows)
    uint8_t* dst = pool + prow * pool_row_bytes(a.pool_fp8);
    for (int c = tid; c < 2 * len * 16; c += blockDim.x) {
      const int isV = c >= len * 16;
      const int cc = isV ? c - len * 16 : c;
      const int i = cc >> 4, sub = cc & 15;
      const bf16* src = (isV ? ringV : ringK) + (int64_t)((start + i) % cap) * D;
      const uint4 x = reinterpret_cast<const uint4*>(src)[sub];
      const int64_t drow = isV ? len + i : i;
      if (a.pool_fp8) reinterpret_cast<uint2*>(dst)[drow * 16 + sub] = bf16x8_to_e4m3x8(x);
      else reinterpret_cast<uint4*>(dst)[drow * 16 + sub] = x;
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
      atomicAdd(&a.stats->bytes_d2h, (unsigned long long)len * pool_row_bytes(a.pool_fp8));
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    S->n_units = s.n_units;
    S->pool_rows = s.pool_rows;
    S->open_len = s.open_len;
    S->open_start = s.open_start;
    S->buffered = s.buffered;
    S->ring_head = s.ring_head;
    S->fifo_head = s.fifo_head;
    S->fifo_count = s.fifo_count;
    S->error = s.error;
    S->step = s.step;
  }
}


}  // namespace lkv
