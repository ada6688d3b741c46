// Full-cache decode attention (the two full-cache layers) on tensor cores:
// o = softmax(q K^T / sqrt(d)) V over all P+t rows of one (b, kv-head) (P:63-65 [§3.1]).
//
// Split-K flash-decode, GQA-packed, mma.sync m16n8k16 bf16 -> fp32:
//   * one CTA per (instance, split), 4 warps; rows stream in 64-row chunks through a 3-stage ring
//     filled by TMA tensor copies (3-D map over the layer's cache, two 64-dim SWIZZLE_128B boxes for
//     K and two for V: 32 KB per chunk, 4 copies), so ldmatrix reads are bank-conflict free;
//   * warp w owns rows [16w, 16w+16) of every chunk: S^T = Q K^T with the g query heads as the M
//     rows of the MMA (padded to 16) and the key rows as N (two 8-row tiles), 8 k-steps over
//     d = 128 (ldmatrix.x4 of K); scale into the log2 domain in fp32, online softmax per head;
//     P (bf16) reuses the accumulator layout directly as the A operand of O += P V (ldmatrix.x4
//     .trans of V, 16 n-tiles of 8 dims);
//   * warps merge through shared memory, splits merge in a fixed order by the last CTA (atomic
//     ticket), as in the SIMT kernel — deterministic.
// HBM-bound: 512 B of K+V per row; one HBM read serves the g heads.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "lkv_internal.cuh"

namespace lkv {
namespace fa {
// per-head stride of a split partial in global memory: D accumulators, max, sum, 2 pad floats (rows
// stay 16-B aligned for the cp.async merge whatever g is; g = 1 with D + 2 was not)
constexpr int PSTR = D + 4;


constexpr int THREADS = 128;
constexpr int WARPS = THREADS / 32;
constexpr int CHUNK = 64;                      // rows per stage (16 per warp)
#ifndef FA_STAGES
#define FA_STAGES 3
#endif
#ifndef FA_MINB
#define FA_MINB 2
#endif
constexpr int STAGES = FA_STAGES;
constexpr int BOX_BYTES = CHUNK * 128;         // 64 rows x 64 dims bf16
constexpr int STAGE_BYTES = 4 * BOX_BYTES;     // K lo, K hi, V lo, V hi
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*1024-B alignment of the swizzled boxes*/ + 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(su32(bar))
      : "memory");
}
// byte offset of (row r, 16-B chunk c in 0..15) inside a stage's K (or V) pair of swizzled boxes
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 3) * BOX_BYTES + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D = A (16x16 bf16, row) * B (16x8 bf16, col) + D, fp32; rows 8-15 of A are the zero padding heads
__device__ __forceinline__ void mma16816(float* d, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const uint32_t l = f2bf_rne(lo), h = f2bf_rne(hi);
  return l | (h << 16);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
// streaming variant: the full cache is read once per step (272 MB > L2), so its lines are marked
// evict-first and do not push the retrieval layers' reused data (working sets, centroids, host rows
// cached in L2) out of the 126 MB L2
__device__ __forceinline__ void cp16_stream(uint32_t dst, const void* src, bool valid, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0), "l"(pol)
               : "memory");
}

struct FullArgs {
  const bf16* full;  // layer base [n_inst][K|V][full_cap][D]
  const bf16* q_own;
  int64_t stride_b;
  int hn;
  float scale_log2;
  int64_t full_P, full_cap;
  const int* step;
  bf16* out;
  float* out_f32;
  float* part;
  int* counters;          // [n_inst] split tickets, then [1] the layer ticket of the fused step
  // fused store_cache (louiskv_decode_layer on a full-cache layer): the kernel itself appends
  // (k_t, v_t) at row P + t - 1, commits the layer's step counter and writes the layer's flags (0)
  int fused;
  const bf16* k_t;
  const bf16* v_t;
  int64_t stride_kv;
  int* error;
  uint8_t* flag_out;
  double* r_out;
  int batch;
};

// LDGSTS: the stage ring is filled by cp.async (16 B per thread-op, coalesced rows, the same 128-B
// swizzle as the TMA boxes); else by TMA tensor copies.
template <int G, bool LDGSTS>
__global__ void __launch_bounds__(THREADS, FA_MINB) attn_full_tc_kernel(const __grid_constant__ CUtensorMap tm, FullArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.x, split = blockIdx.y, nsplit = gridDim.y;
  const int b = li / a.hn, h = li % a.hn;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(128) uint8_t fa_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fa_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;

  // fused: this launch is step t = step + 1 and attends P + t rows, the last one being (k_t, v_t)
  const int t_new = a.fused ? *a.step + 1 : 0;
  const int64_t rows_all = a.full_P + (a.fused ? t_new : *a.step);
  const int n_rows = (int)(rows_all < a.full_cap ? rows_all : a.full_cap);
  const int nck = (n_rows + CHUNK - 1) / CHUNK;  // chunk-granular split
  const int c_begin = (int)((int64_t)nck * split / nsplit), c_end = (int)((int64_t)nck * (split + 1) / nsplit);
  const int n_chunks = c_end - c_begin;
  const int zk = li * 2, zv = li * 2 + 1;

  auto issue = [&](int c) {
    const int st = c % STAGES;
    uint8_t* dst = smem + st * STAGE_BYTES;
    const int y = (c_begin + c) * CHUNK;
    ptx_mbar_expect_tx(&full_bar[st], STAGE_BYTES);
    tma3(dst, &tm, &full_bar[st], 0, y, zk);
    tma3(dst + BOX_BYTES, &tm, &full_bar[st], 64, y, zk);
    tma3(dst + 2 * BOX_BYTES, &tm, &full_bar[st], 0, y, zv);
    tma3(dst + 3 * BOX_BYTES, &tm, &full_bar[st], 64, y, zv);
  };
  const bf16* kbase = a.full + (int64_t)li * 2 * a.full_cap * D;
  const bf16* vbase = kbase + a.full_cap * D;
  if (a.fused) {
    // store_cache on a full-cache layer: the split that owns the last chunk writes the
    // new row before it loads anything (CTA barrier + proxy fence: the row is then read back by this
    // CTA's own cp.async / TMA copies; no other CTA reads it)
    if (split == nsplit - 1) {
      const int64_t pos = a.full_P + t_new - 1;
      if (pos < a.full_cap) {
        if (tid < 32) {
          const bf16* src = (tid < 16 ? a.k_t : a.v_t) + (int64_t)b * a.stride_kv + (int64_t)h * D;
          bf16* dst = const_cast<bf16*>(tid < 16 ? kbase : vbase) + pos * D;
          reinterpret_cast<uint4*>(dst)[tid & 15] = reinterpret_cast<const uint4*>(src)[tid & 15];
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
      } else if (tid == 0) {
        *a.error = 1;
      }
      __syncthreads();
    }
    if (li == 0 && split == 0 && tid < a.batch) {  // full-cache layers never retrieve
      if (a.flag_out) a.flag_out[tid] = 0;
      if (a.r_out) a.r_out[tid] = 0.0;
    }
  }
#ifndef LKV_FA_NO_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  auto load = [&](int c) {  // cp.async path: every thread copies 16 of the chunk's 2048 16-B pieces
    const int st = c % STAGES;
    const uint32_t dst = su32(smem + st * STAGE_BYTES);
    const int y = (c_begin + c) * CHUNK;
#pragma unroll
    for (int k = 0; k < (2 * CHUNK * 16) / THREADS; ++k) {
      const int i = tid + k * THREADS;
      const int kv = i >> 10, r = (i >> 4) & (CHUNK - 1), j = i & 15;
      const bool ok = y + r < n_rows;
      const bf16* src = (kv ? vbase : kbase) + (int64_t)(ok ? y + r : 0) * D + j * 8;
#ifndef LKV_FA_NO_EVICT_FIRST
      cp16_stream(dst + kv * 2 * BOX_BYTES + swz(r, j), src, ok, pol);
#else
      cp16(dst + kv * 2 * BOX_BYTES + swz(r, j), src, ok);
#endif
    }
  };
  if (LDGSTS) {
    for (int c = 0; c < STAGES - 1; ++c) {
      if (c < n_chunks) load(c);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    for (int i = 0; i < STAGES; ++i) {
      ptx_mbar_init(&full_bar[i], 1);
      ptx_mbar_init(&empty_bar[i], WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int c = 0; c < n_chunks && c < STAGES; ++c) issue(c);
  }
  // Q as the MMA A operand: row = head (lane / 4 < G), k = dims; rows 8-15 are zero padding
  uint32_t qa[8][2];
  {
    const int hq = lane >> 2;
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(a.q_own + (int64_t)b * a.stride_b + (int64_t)h * G * D);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int d0 = kk * 16 + (lane & 3) * 2;
      qa[kk][0] = hq < G ? q32[(hq * D + d0) >> 1] : 0u;
      qa[kk][1] = hq < G ? q32[(hq * D + d0 + 8) >> 1] : 0u;
    }
  }
  __syncthreads();

  float m_run = -INFINITY, l_run = 0.f;  // head lane/4 (l: this lane's rows only; quad-summed at the end)
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const uint32_t sbase = su32(smem);
  // ldmatrix lane -> (row in the warp's 16-row slice, 16-B chunk parity)
  const int lr = (lane & 7) + ((lane >> 4) << 3);  // K: matrices (r0-7,c), (r0-7,c+1), (r8-15,c), (r8-15,c+1)
  const int lc = (lane >> 3) & 1;
  const int vr = (lane & 7) + (((lane >> 3) & 1) << 3);  // V^T: (r0-7,c), (r8-15,c), (r0-7,c+1), (r8-15,c+1)
  const int vc = lane >> 4;

  for (int c = 0; c < n_chunks; ++c) {
    const int st = c % STAGES;
    if (LDGSTS) {
      if (c + STAGES - 1 < n_chunks) load(c + STAGES - 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
    } else {
      ptx_mbar_wait(&full_bar[st], (uint32_t)((c / STAGES) & 1));
    }
    const uint32_t kb = sbase + st * STAGE_BYTES, vb = kb + 2 * BOX_BYTES;
    const int row0 = warp * 16;
    // ---- S^T = Q K^T for the warp's 16 rows (two n-tiles of 8 rows)
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(kb + swz(row0 + lr, 2 * kk + lc), b0, b1, b2, b3);
      mma16816(s[0], qa[kk][0], qa[kk][1], b0, b1);
      mma16816(s[1], qa[kk][0], qa[kk][1], b2, b3);
    }
    // ---- online softmax (log2 domain) for head lane/4; rows past the end are masked
    const int grow = (c_begin + c) * CHUNK + row0 + (lane & 3) * 2;
    float p[2][2];
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float v = (grow + nt * 8 + e < n_rows) ? s[nt][e] * a.scale_log2 : -INFINITY;
        p[nt][e] = v;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    float corr = 1.f;
    if (m_new == -INFINITY) {
      p[0][0] = p[0][1] = p[1][0] = p[1][1] = 0.f;
    } else {
      corr = exp2f(m_run - m_new);  // (m_run = -inf -> 0)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) p[nt][e] = exp2f(p[nt][e] - m_new);
      m_run = m_new;
    }
    l_run = l_run * corr + (p[0][0] + p[0][1] + p[1][0] + p[1][1]);
    const uint32_t pa0 = pack_bf16(p[0][0], p[0][1]), pa2 = pack_bf16(p[1][0], p[1][1]);
    // ---- O += P V over the 16 rows: 16 n-tiles of 8 dims, ldmatrix.trans pairs of tiles
#pragma unroll
    for (int dt = 0; dt < 16; dt += 2) {
      acc[dt][0] *= corr;
      acc[dt][1] *= corr;
      acc[dt + 1][0] *= corr;
      acc[dt + 1][1] *= corr;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(vb + swz(row0 + vr, dt + vc), b0, b1, b2, b3);
      mma16816(acc[dt], pa0, pa2, b0, b1);
      mma16816(acc[dt + 1], pa0, pa2, b2, b3);
    }
    if (LDGSTS) {
      __syncthreads();  // stage st fully consumed before the next iteration's copies reuse stage st-1
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[st]);
      if (tid == 0 && c + STAGES < n_chunks) {
        ptx_mbar_wait(&empty_bar[st], (uint32_t)((c / STAGES) & 1));
        issue(c + STAGES);
      }
    }
  }

  // ---- merge: quad-sum l; per-warp (m, l, acc) of the G heads -> shared memory -> CTA partial
  if (LDGSTS) asm volatile("cp.async.wait_group 0;" ::: "memory");
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();  // every warp is done with the stage ring: reuse it
  float* s_acc = reinterpret_cast<float*>(smem);           // [WARPS][G][D]
  float* s_ml = s_acc + WARPS * G * D;                      // [WARPS][G][2]
  const int hq = lane >> 2;
  if (hq < G) {
#pragma unroll
    for (int dt = 0; dt < 16; ++dt) {
      const int d0 = dt * 8 + (lane & 3) * 2;
      s_acc[(warp * G + hq) * D + d0] = acc[dt][0];
      s_acc[(warp * G + hq) * D + d0 + 1] = acc[dt][1];
    }
    if ((lane & 3) == 0) {
      s_ml[(warp * G + hq) * 2] = m_run;
      s_ml[(warp * G + hq) * 2 + 1] = l_run;
    }
  }
  __syncthreads();
  float* part = a.part + ((int64_t)li * nsplit + split) * G * PSTR;
  for (int idx = tid; idx < G * D; idx += THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, s_ml[(w * G + j) * 2]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < WARPS; ++w) {
        const float mw = s_ml[(w * G + j) * 2];
        const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
        Lsum += s_ml[(w * G + j) * 2 + 1] * sc;
        A += s_acc[(w * G + j) * D + e] * sc;
      }
    part[j * PSTR + e] = A;
    if (e == 0) {
      part[j * PSTR + D] = M;
      part[j * PSTR + D + 1] = Lsum;
    }
  }
  // ---- the last CTA of this instance merges the splits in split order
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&a.counters[li], 1) == nsplit - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* P0 = a.part + (int64_t)li * nsplit * G * PSTR;
  // the splits' partials are staged in shared memory (the idle stage ring) by cp.async in batches
  // of SB splits — one round trip per batch instead of one dependent L2 load per split and output
  constexpr int PF = G * PSTR;                      // floats per split partial (16-B multiple: PSTR = D + 4)
  constexpr int MAXS = 64;                             // (>= the host's max_splits)
  constexpr int WB = 2 * MAXS * G * 4 + 2 * G * 4;     // bytes of the per-split weights + (M, 1/L)
  constexpr int SB = (STAGES * STAGE_BYTES - WB) / (PF * 4);  // splits per staging batch
  float* s_part = reinterpret_cast<float*>(smem);      // [SB][PF]
  float* s_wt = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES - WB);  // [nsplit][G] m, then weights
  float* s_l = s_wt + MAXS * G;                        // [nsplit][G] l
  float* s_w = s_l + MAXS * G;                         // [G] M, [G] 1/L
  float accv[(G * D + THREADS - 1) / THREADS];
#pragma unroll
  for (int i = 0; i < (G * D + THREADS - 1) / THREADS; ++i) accv[i] = 0.f;
  // (m, l) of every split-head, all loads in one round (they overlap the first batch's staging)
  for (int t = tid; t < nsplit * G; t += THREADS) {
    const int y = t / G, j = t % G;
    s_wt[t] = __ldcg(P0 + y * PF + j * PSTR + D);
    s_l[t] = __ldcg(P0 + y * PF + j * PSTR + D + 1);
  }
  __syncthreads();
  if (tid < G) {  // global max and normaliser per head, split order
    const int j = tid;
    float M = -INFINITY;
    for (int y = 0; y < nsplit; ++y) M = fmaxf(M, s_wt[y * G + j]);
    float Lsum = 0.f;
    for (int y = 0; y < nsplit; ++y) {
      const float m = s_wt[y * G + j];
      Lsum += (m == -INFINITY ? 0.f : exp2f(m - M)) * s_l[y * G + j];
    }
    s_w[j] = M;
    s_w[G + j] = 1.f / Lsum;
  }
  __syncthreads();
  for (int t = tid; t < nsplit * G; t += THREADS) {  // per-split weights 2^(m - M)
    const float m = s_wt[t];
    s_wt[t] = m == -INFINITY ? 0.f : exp2f(m - s_w[t % G]);
  }
  // weighted sum of the partials, split order (deterministic)
  for (int y0 = 0; y0 < nsplit; y0 += SB) {
    const int nb = min(SB, nsplit - y0);
    __syncthreads();  // (weights written / previous batch consumed)
    const uint32_t dst = su32(s_part);
    for (int i = tid; i < nb * PF / 4; i += THREADS) cp16(dst + i * 16, P0 + (int64_t)y0 * PF + i * 4, true);
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int i = 0; i < (G * D + THREADS - 1) / THREADS; ++i) {
      const int idx = tid + i * THREADS;
      if (idx < G * D) {
        const int j = idx / D, e = idx % D;
#pragma unroll 4
        for (int y = 0; y < nb; ++y) accv[i] = fmaf(s_wt[(y0 + y) * G + j], s_part[y * PF + j * PSTR + e], accv[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < (G * D + THREADS - 1) / THREADS; ++i) {
    const int idx = tid + i * THREADS;
    if (idx < G * D) {
      const int j = idx / D, e = idx % D;
      const float A = accv[i] * s_w[G + j];
      const int64_t oi = ((int64_t)(b * a.hn + h) * G + j) * D + e;
      a.out[oi] = __float2bfloat16_rn(A);
      if (a.out_f32) a.out_f32[oi] = A;
    }
  }
  if (tid == 0) {
    a.counters[li] = 0;
    if (a.fused) {  // the last instance to finish commits the layer's step (every CTA has read it)
      __threadfence();
      const int nl = gridDim.x;
      if (atomicAdd(&a.counters[nl], 1) == nl - 1) {
        a.counters[nl] = 0;
        *const_cast<int*>(a.step) = t_new;
      }
    }
  }
}

}  // namespace fa

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // k_kmeans_tc.cu

template <int G>
static cudaError_t launch_full_tc_g(const CUtensorMap& tm, const fa::FullArgs& fa_args, int n_inst, int splits,
                                    cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  static const bool tma = getenv("LOUISKV_FA_TMA") != nullptr;  // (load-path experiment)
  cudaError_t ea = once_per_device(attr, [] {
    cudaError_t e = cudaFuncSetAttribute(fa::attn_full_tc_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
    return e != cudaSuccess ? e : cudaFuncSetAttribute(fa::attn_full_tc_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
  });
  if (ea != cudaSuccess) return ea;
  if (tma)
    return launch_k(fa::attn_full_tc_kernel<G, false>, dim3(n_inst, splits), dim3(fa::THREADS), fa::SMEM, st, tm,
                    fa_args);
  return launch_k(fa::attn_full_tc_kernel<G, true>, dim3(n_inst, splits), dim3(fa::THREADS), fa::SMEM, st, tm, fa_args);
}

// Full-cache attention on tensor cores; returns cudaErrorNotSupported when the tensor map cannot be
// built (the caller then uses the SIMT kernel).
cudaError_t launch_attn_full_tc(const AttnArgs& a, int n_inst_layer, cudaStream_t st, const FullStepArgs* fs) {
  auto enc = tensor_map_encoder();
  if (!enc || a.g > 8 || (reinterpret_cast<uintptr_t>(a.full) & 15)) return cudaErrorNotSupported;
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)a.full_cap, (cuuint64_t)n_inst_layer * 2};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)a.full_cap * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)fa::CHUNK, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)a.full, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  fa::FullArgs f;
  f.full = a.full;
  f.q_own = a.q_own;
  f.stride_b = a.stride_b;
  f.hn = a.hn;
  f.scale_log2 = a.scale_log2;
  f.full_P = a.full_P;
  f.full_cap = a.full_cap;
  f.step = a.step;
  f.out = a.out;
  f.out_f32 = a.out_f32;
  f.part = a.part;
  f.counters = a.counters;
  f.fused = fs != nullptr;
  if (fs) {
    f.k_t = fs->k_t;
    f.v_t = fs->v_t;
    f.stride_kv = fs->stride_kv;
    f.error = fs->error;
    f.flag_out = fs->flag_out;
    f.r_out = fs->r_out;
    f.batch = fs->batch;
  }
  switch (a.g) {
    case 1: return launch_full_tc_g<1>(tm, f, n_inst_layer, a.splits, st);
    case 2: return launch_full_tc_g<2>(tm, f, n_inst_layer, a.splits, st);
    case 4: return launch_full_tc_g<4>(tm, f, n_inst_layer, a.splits, st);
    case 8: return launch_full_tc_g<8>(tm, f, n_inst_layer, a.splits, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lkv
