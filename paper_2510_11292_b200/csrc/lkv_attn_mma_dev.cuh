// Tensor-core (mma.sync m16n8k16 bf16 -> fp32) CTA-level flash-decode partial over an attention set
// given as row pieces — the attention step of the single-launch layer kernel (k_layer.cu).
// o = softmax(q K_I^T / sqrt(d)) V_I (P:63-65 [§3.1]) for the g query heads of one KV head.
//
// 8 warps, 64-row chunks: warp w owns rows [8w, 8w+8) of every chunk. S^T = Q K^T with the g heads
// as the MMA's M rows (padded to 16) and the warp's 8 rows as N, 8 k-steps over d = 128; scale into
// the log2 domain in fp32, online softmax per head; P (bf16, rows 8-15 of the k extent zero) is the
// A operand of O += P V over 16 n-tiles of 8 dims. The 3-stage smem ring (K | V, each two 64-dim
// 128-B-swizzled halves, so ldmatrix is bank-conflict free) is filled by cp.async 16-B copies, which
// gather the pieces (sinks, working set, local window) in any alignment.
#pragma once
#include "lkv_attn_dev.cuh"

namespace lkv {
namespace am {

constexpr int WARPS = AT_THREADS / 32;  // 8
constexpr int CHUNK = 64;
constexpr int STAGES = AT_STAGES;        // 3
constexpr int HALF = CHUNK * 128;        // one 64-dim half of K (or V) of a chunk: 8 KB
constexpr int STAGE = 4 * HALF;          // 32 KB == AT_STAGE_BYTES
static_assert(STAGE == AT_STAGE_BYTES, "stage size");

__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 3) * HALF + r * 128 + (((c & 7) ^ (r & 7)) << 4));
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
// D += A (16x16: regs {a_lo, 0, a_hi, 0} - rows 8-15 zero) * B (16x8: regs {b_lo, b_hi})
__device__ __forceinline__ void mma16816(float* d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a_lo), "r"(0u), "r"(a_hi), "r"(0u), "r"(b_lo), "r"(b_hi));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

}  // namespace am

// q of the G heads (bf16 [G][D] at qb) as the A fragments of the S^T MMA: row = head lane/4 (< G),
// k = dims; rows 8-15 are the zero padding (not stored)
template <int G>
__device__ __forceinline__ void mma_q_frags(const uint16_t* qb, uint32_t (&qa)[8][2]) {
  const int lane = threadIdx.x & 31, hq = lane >> 2;
  const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qb);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int d0 = kk * 16 + (lane & 3) * 2;
    qa[kk][0] = hq < G ? q32[(hq * D + d0) >> 1] : 0u;
    qa[kk][1] = hq < G ? q32[(hq * D + d0 + 8) >> 1] : 0u;
  }
}

// An attention set as row pieces plus: an excluded virtual-row range [mask_lo, mask_hi) (rows loaded
// speculatively but not in the set) and one row (`new_vr`, -1: none) supplied from registers instead
// of memory — the current token, before its ring slot is written.
struct AttnPlan {
  Pieces P;
  int rows;
  int mask_lo, mask_hi;
  int new_vr;
};

// Issue chunk c of the plan into stage c % STAGES as cp.async 16-B copies: thread t copies 16-B piece
// t % 16 of rows t/16 + 16m (m < 4), K and V (rows past the end zero-filled). The new-token row is
// not copied: threads t < 32 of the owning CTA store `nv` (K piece t for t < 16, V piece t - 16) —
// the row held in registers since entry. Every thread calls; the caller commits the group.
__device__ __forceinline__ void attn_store_new_row(const AttnPlan& pl, const int c, const uint4 nv);
__device__ __forceinline__ void attn_load_chunk(const AttnPlan& pl, const int c, const uint4 nv,
                                                const bool with_new = true) {
  using namespace am;
  extern __shared__ __align__(128) uint8_t at_smem[];
  const int tid = threadIdx.x, j = tid & 15;
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(at_smem) + (c % STAGES) * STAGE;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int r = (tid >> 4) + 16 * m;
    const int vr = c * CHUNK + r;
    if (vr == pl.new_vr) continue;
    const bf16* ks = pl.P.k[0];
    const bf16* vs = pl.P.k[0];
    int bytes = 0;
    if (vr < pl.rows) {
      // piece lookup with the (at most 4) pieces kept in registers
      int off = vr;
      ks = pl.P.k[0];
      vs = pl.P.v[0];
#pragma unroll
      for (int p = 1; p < AT_PMAX; ++p)
        if (p < pl.P.np && vr >= pl.P.v0[p]) {
          off = vr - pl.P.v0[p];
          ks = pl.P.k[p];
          vs = pl.P.v[p];
        }
      ks += (int64_t)off * D + j * 8;
      vs += (int64_t)off * D + j * 8;
      bytes = 16;
    }
    cp16(dst + swz(r, j), ks, bytes);
    cp16(dst + 2 * HALF + swz(r, j), vs, bytes);
  }
  if (with_new) attn_store_new_row(pl, c, nv);
}

// The new token's row of chunk c (if it falls in it), from registers: threads t < 32 of the owning
// CTA store `nv` (K piece t for t < 16, V piece t - 16) into the chunk's stage.
__device__ __forceinline__ void attn_store_new_row(const AttnPlan& pl, const int c, const uint4 nv) {
  using namespace am;
  extern __shared__ __align__(128) uint8_t at_smem[];
  const int tid = threadIdx.x, j = tid & 15;
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(at_smem) + (c % STAGES) * STAGE;
  if (pl.new_vr >= c * CHUNK && pl.new_vr < (c + 1) * CHUNK && tid < 32) {
    const uint32_t sdst = dst + (tid >> 4) * 2 * HALF + swz(pl.new_vr - c * CHUNK, j);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sdst), "r"(nv.x), "r"(nv.y), "r"(nv.z), "r"(nv.w)
                 : "memory");
  }
}

// Returns the CTA partial in shared memory, [G][D+2] floats (unnormalised accumulator, then the
// log2-domain max and the sum), exactly as attn_partial. The first `npre` chunks (< STAGES) were
// issued and committed (one group each) by the caller. qa from mma_q_frags. All threads.
template <int G>
__device__ __forceinline__ float* attn_run_mma(const uint32_t (&qa)[8][2], const float scale_log2, const AttnPlan& pl,
                                               const int npre, const uint4 nv, unsigned long long* prof) {
  using namespace am;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(128) uint8_t at_smem[];  // (128-B aligned: the software swizzle is row-relative)
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(at_smem);
  const int rows = pl.rows;
  const int n_chunks = (rows + CHUNK - 1) / CHUNK;
  __syncthreads();  // rows this CTA just wrote (gather) are read back by other threads
#pragma unroll 1
  for (int c = npre; c < STAGES - 1; ++c) {
    if (c < n_chunks) attn_load_chunk(pl, c, nv);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float m_run = -INFINITY, l_run = 0.f;
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const int row8 = warp * 8;
#pragma unroll 1
  for (int c = 0; c < n_chunks; ++c) {
    if (c + STAGES - 1 < n_chunks) attn_load_chunk(pl, c + STAGES - 1, nv);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    __syncthreads();
    if (c == 0) prof_stamp(prof, 8);
    const uint32_t kb = sbase + (c % STAGES) * STAGE, vb = kb + 2 * HALF;
    // ---- S^T (heads x the warp's 8 rows)
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4(kb + swz(row8 + (lane & 7), 4 * k2 + (lane >> 3)), b0, b1, b2, b3);
      mma16816(s, qa[2 * k2][0], qa[2 * k2][1], b0, b1);
      mma16816(s, qa[2 * k2 + 1][0], qa[2 * k2 + 1][1], b2, b3);
    }
    // ---- online softmax of head lane/4 over rows 2(lane%4), +1
    const int vr = c * CHUNK + row8 + (lane & 3) * 2;
    const bool ok0 = vr < rows && (vr < pl.mask_lo || vr >= pl.mask_hi);
    const bool ok1 = vr + 1 < rows && (vr + 1 < pl.mask_lo || vr + 1 >= pl.mask_hi);
    float p0 = ok0 ? s[0] * scale_log2 : -INFINITY;
    float p1 = ok1 ? s[1] * scale_log2 : -INFINITY;
    float mx = fmaxf(p0, p1);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    float corr = 1.f;
    if (m_new == -INFINITY) {
      p0 = p1 = 0.f;
    } else {
      corr = exp2f(m_run - m_new);
      p0 = exp2f(p0 - m_new);
      p1 = exp2f(p1 - m_new);
      m_run = m_new;
    }
    l_run = l_run * corr + p0 + p1;
    const uint32_t pa = (uint32_t)f2bf_rne(p0) | ((uint32_t)f2bf_rne(p1) << 16);
    // ---- O += P V (k extent: the warp's 8 rows; the other 8 are zero)
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(vb + swz(row8 + (lane & 7), 4 * q4 + (lane >> 3)), b0, b1, b2, b3);
      const uint32_t bb[4] = {b0, b1, b2, b3};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float* d = acc[4 * q4 + t];
        d[0] *= corr;
        d[1] *= corr;
        mma16816(d, pa, 0u, bb[t], 0u);
      }
    }
    __syncthreads();  // stage c % STAGES fully consumed before it is refilled
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  prof_stamp(prof, 9);

  // ---- merge the 8 warps through shared memory (the ring is idle now)
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();
  float* s_acc = reinterpret_cast<float*>(at_smem);  // [WARPS][G][D]
  float* s_ml = s_acc + WARPS * G * D;                // [WARPS][G][2]
  float* part = s_ml + WARPS * G * 2;                 // [G][D+2]
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
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, s_ml[(w * G + j) * 2]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float mw = s_ml[(w * G + j) * 2];
        const float sc = mw == -INFINITY ? 0.f : exp2f(mw - M);
        Lsum += s_ml[(w * G + j) * 2 + 1] * sc;
        A += s_acc[(w * G + j) * D + e] * sc;
      }
    }
    part[j * (D + 2) + e] = A;
    if (e == 0) {
      part[j * (D + 2) + D] = M;
      part[j * (D + 2) + D + 1] = Lsum;
    }
  }
  __syncthreads();
  return part;
}

}  // namespace lkv
