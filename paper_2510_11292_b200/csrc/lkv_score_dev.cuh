// Device code of the bit-exact recipes shared by the multi-kernel retrieve path (k_retrieve.cu) and
// the single-launch layer kernel (k_layer.cu), so both take every decision in identical arithmetic.
//   R1  trigger r_t = (1/Hq) Σ_h cos(q_ref^h, q_t^h) in fp64: per head, 16 lanes each
//       sum 8 consecutive dims sequentially, then a fixed xor tree (8, 4, 2, 1); heads summed in order.
//   R2  logits l_{j,u} = fl32(fmaf chain over e = 0..127 of q_j,e * c_u,e) * fl32(1/sqrt(d))
//   R3  exp via round-to-nearest split t = x log2 e = n + f, degree-6 Horner with fl32(ln2^i / i!)
#pragma once
#include "lkv_internal.cuh"

namespace lkv {

__device__ __forceinline__ float exp_r3(float x, const float* c) {
  const float log2e = __double2float_rn(1.4426950408889634074);
  float t = __fmul_rn(x, log2e);
  if (t < -126.0f) return 0.0f;
  float n = rintf(t);
  float f = __fsub_rn(t, n);
  float p = c[6];
#pragma unroll
  for (int i = 5; i >= 0; --i) p = __fmaf_rn(p, f, c[i]);
  int ni = (int)n;
  float scale = __int_as_float((ni + 127) << 23);
  return __fmul_rn(p, scale);
}


__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
  unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return ((unsigned long long)hi << 32) | lo;
}

// R1 per-head cosines of one sequence into s_cos[Hq] (all NT threads call; two heads per warp per
// round, lanes past the last head shuffle zeros). Every round's q_ref / q_t pieces are loaded before
// any arithmetic (Hq <= 64: at most 4 rounds at NT = 256), so the loads cost one round trip, not one
// per round. Caller syncs before reading s_cos.
template <int NT>
__device__ __forceinline__ void trigger_cosines(const uint16_t* qc, const uint16_t* qr, int Hq, double* s_cos) {
  constexpr int HPR = (NT / 32) * 2;          // heads per round
  constexpr int MAXR = (64 + HPR - 1) / HPR;  // rounds for the largest Hq (64, louiskv_create)
  const int tid = threadIdx.x, l16 = tid & 15, warp = tid >> 5, lane = tid & 31;
  uint4 ua[MAXR], uc[MAXR];
#pragma unroll
  for (int it = 0; it < MAXR; ++it) {
    const int hh = warp * 2 + it * HPR + (lane >> 4);
    ua[it] = uc[it] = make_uint4(0, 0, 0, 0);
    if (hh < Hq) {
      ua[it] = reinterpret_cast<const uint4*>(qr + hh * D)[l16];
      uc[it] = reinterpret_cast<const uint4*>(qc + hh * D)[l16];
    }
  }
#pragma unroll
  for (int it = 0; it < MAXR; ++it) {
    if (warp * 2 + it * HPR >= Hq) break;  // (warp-uniform)
    const int hh = warp * 2 + it * HPR + (lane >> 4);
    const bool act = hh < Hq;
    float fa[8], fc[8];
    unpack8(ua[it], fa);
    unpack8(uc[it], fc);
    double dot = 0.0, na = 0.0, nb = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double x = (double)fa[e], y = (double)fc[e];
      dot = __dadd_rn(dot, __dmul_rn(x, y));
      na = __dadd_rn(na, __dmul_rn(x, x));
      nb = __dadd_rn(nb, __dmul_rn(y, y));
    }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
      dot = __dadd_rn(dot, __shfl_xor_sync(0xffffffffu, dot, off));
      na = __dadd_rn(na, __shfl_xor_sync(0xffffffffu, na, off));
      nb = __dadd_rn(nb, __shfl_xor_sync(0xffffffffu, nb, off));
    }
    if (act && l16 == 0) {
      double cs = 0.0;
      if (na != 0.0 && nb != 0.0) {
        cs = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
        cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
      }
      s_cos[hh] = cs;
    }
  }
}

// R1 head mean (one thread, heads in order)
__device__ __forceinline__ double trigger_mean(const double* s_cos, int Hq) {
  double sum = 0.0;
  for (int hh = 0; hh < Hq; ++hh) sum = __dadd_rn(sum, s_cos[hh]);
  return __ddiv_rn(sum, (double)Hq);
}

// R2 logits of one unit row (bf16 centroid, 256 B) against the G query heads in sq (fp32)
// (inv_sqrt_d = fl32(1 / fl64(sqrt(d))), computed on the host: RetrieveArgs::inv_sqrt_d)
template <int G>
__device__ __forceinline__ void logits_row(const float (*sq)[D], const uint4* row, const float inv_sqrt_d,
                                           float* out) {
  uint4 cr[D / 8];
#pragma unroll
  for (int c8 = 0; c8 < D / 8; ++c8) cr[c8] = __ldg(row + c8);
  float acc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) acc[j] = 0.0f;
#pragma unroll
  for (int c8 = 0; c8 < D / 8; ++c8) {
    float cf[8];
    unpack8(cr[c8], cf);
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < G; ++j) acc[j] = __fmaf_rn(sq[j][c8 * 8 + k], cf[k], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < G; ++j) out[j] = __fmul_rn(acc[j], inv_sqrt_d);
}

// logits_row with the centroid row in shared memory (same arithmetic, same order); the query
// values are read as broadcast float4s (one shared-memory wavefront per 4 FMAs per head)
template <int G>
__device__ __forceinline__ void logits_row_smem(const float (*sq)[D], const uint4* row, const float inv_sqrt_d,
                                                float* out) {
  float acc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) acc[j] = 0.0f;
#pragma unroll 2
  for (int c8 = 0; c8 < D / 8; ++c8) {
    float cf[8];
    unpack8(row[c8], cf);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float4 qa = reinterpret_cast<const float4*>(&sq[j][c8 * 8])[0];
      const float4 qb = reinterpret_cast<const float4*>(&sq[j][c8 * 8])[1];
      acc[j] = __fmaf_rn(qa.x, cf[0], acc[j]);
      acc[j] = __fmaf_rn(qa.y, cf[1], acc[j]);
      acc[j] = __fmaf_rn(qa.z, cf[2], acc[j]);
      acc[j] = __fmaf_rn(qa.w, cf[3], acc[j]);
      acc[j] = __fmaf_rn(qb.x, cf[4], acc[j]);
      acc[j] = __fmaf_rn(qb.y, cf[5], acc[j]);
      acc[j] = __fmaf_rn(qb.z, cf[6], acc[j]);
      acc[j] = __fmaf_rn(qb.w, cf[7], acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) out[j] = __fmul_rn(acc[j], inv_sqrt_d);
}

}  // namespace lkv
