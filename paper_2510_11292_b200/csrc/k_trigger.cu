// Semantic-boundary trigger (P:101-106 [§4.1 r_t], P:301 [Alg. 1 is_new_segment]).
//
// r_t = (1/H) Σ_h cos(q_ref^h, q_t^h) over ALL H query heads; flag = (t == 1) ∨ (r_t < τ).
// Arithmetic recipe R1: fp64, e ascending, multiply then add with explicit
// round-to-nearest intrinsics (no contraction), cos = dot / (sqrt(na) * sqrt(nb)), clamped
// to [-1, 1]; a zero norm gives 0; heads summed in ascending order. This makes the decision
// bit-identical to any IEEE implementation of the same recipe.
//
// One CTA for the batch; one thread per (sequence, head) (the sequential per-head dot is the recipe).
// The work is 2*H*d bf16 per (b, layer) — latency bound, a few hundred ns.
#include "lkv_internal.cuh"

namespace lkv {

// Single CTA for the whole batch: thread i computes the per-head cosines of pairs
// (b, h) = divmod(i, Hq); then thread b sums its heads in ascending order.
__global__ void __launch_bounds__(1024) trigger_kernel(const uint16_t* __restrict__ q_all, int64_t stride_b,
                                                       int batch, int Hq, uint16_t* __restrict__ q_ref,
                                                       uint8_t* flag, double* r, uint8_t* flag_out, double* r_out,
                                                       int* step, double tau, int trigger_ref) {
  extern __shared__ double cos_h[];  // [batch * Hq]
  uint8_t* s_flag = reinterpret_cast<uint8_t*>(cos_h + batch * Hq);
  const int t = *step + 1;
  for (int p = threadIdx.x; p < batch * Hq; p += blockDim.x) {
    const int b = p / Hq, h = p % Hq;
    const uint4* a4 = reinterpret_cast<const uint4*>(q_ref + ((int64_t)b * Hq + h) * D);
    const uint4* c4 = reinterpret_cast<const uint4*>(q_all + (int64_t)b * stride_b + (int64_t)h * D);
    // issue all 32 vector loads first (they do not depend on the fp64 chains)
    uint4 ua[D / 8], uc[D / 8];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      ua[i] = a4[i];
      uc[i] = c4[i];
    }
    double dot = 0.0, na = 0.0, nb = 0.0;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      float fa[8], fc[8];
      unpack8(ua[i], fa);
      unpack8(uc[i], fc);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double x = (double)fa[e], y = (double)fc[e];
        dot = __dadd_rn(dot, __dmul_rn(x, y));
        na = __dadd_rn(na, __dmul_rn(x, x));
        nb = __dadd_rn(nb, __dmul_rn(y, y));
      }
    }
    double cs = 0.0;
    if (na != 0.0 && nb != 0.0) {
      cs = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
      cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
    }
    cos_h[p] = cs;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < batch; b += blockDim.x) {
    double s = 0.0;
    for (int h = 0; h < Hq; ++h) s = __dadd_rn(s, cos_h[b * Hq + h]);
    const double rr = __ddiv_rn(s, (double)Hq);
    const int f = (t == 1) || (rr < tau);
    flag[b] = (uint8_t)f;
    r[b] = rr;
    if (flag_out) flag_out[b] = (uint8_t)f;
    if (r_out) r_out[b] = rr;
    s_flag[b] = (uint8_t)f;
  }
  __syncthreads();
  // q_ref <- q_t ("q_prev <- q_t"); LAST_RETRIEVAL keeps the last retrieval's query
  const int vec_per_b = Hq * D / 8;
  for (int i = threadIdx.x; i < batch * vec_per_b; i += blockDim.x) {
    const int b = i / vec_per_b, o = i % vec_per_b;
    if (trigger_ref == LOUISKV_TRIG_PREV_STEP || s_flag[b])
      reinterpret_cast<uint4*>(q_ref + (int64_t)b * Hq * D)[o] =
          reinterpret_cast<const uint4*>(q_all + (int64_t)b * stride_b)[o];
  }
  if (threadIdx.x == 0) *step = t;
}

__global__ void copy_flags_kernel(const uint8_t* src_flag, const double* src_r, uint8_t* flag, double* r,
                                  uint8_t* flag_out, double* r_out, int batch, int* step) {
  const int t = *step + 1;
  for (int b = threadIdx.x; b < batch; b += blockDim.x) {
    uint8_t f = src_flag ? src_flag[b] : 0;
    double rr = src_r ? src_r[b] : 0.0;
    flag[b] = f;
    r[b] = rr;
    if (flag_out) flag_out[b] = f;
    if (r_out) r_out[b] = rr;
  }
  __syncthreads();
  if (threadIdx.x == 0) *step = t;
}

cudaError_t launch_trigger(const bf16* q_all, int64_t stride_b, int batch, int Hq, bf16* q_ref, uint8_t* flag,
                           double* r, uint8_t* flag_out, double* r_out, int* step, double tau, int trigger_ref,
                           cudaStream_t st) {
  const int pairs = batch * Hq;
  const int threads = pairs >= 1024 ? 1024 : ((pairs + 31) / 32) * 32;
  const size_t smem = sizeof(double) * pairs + batch;
  if (smem > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(trigger_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
  }
  trigger_kernel<<<1, threads < 64 ? 64 : threads, smem, st>>>(
      reinterpret_cast<const uint16_t*>(q_all), stride_b, batch, Hq, reinterpret_cast<uint16_t*>(q_ref), flag, r,
      flag_out, r_out, step, tau, trigger_ref);
  return cudaGetLastError();
}

cudaError_t launch_copy_flags(const uint8_t* src_flag, const double* src_r, uint8_t* flag, double* r,
                              uint8_t* flag_out, double* r_out, int batch, int* step, cudaStream_t st) {
  copy_flags_kernel<<<1, 128, 0, st>>>(src_flag, src_r, flag, r, flag_out, r_out, batch, step);
  return cudaGetLastError();
}

}  // namespace lkv
