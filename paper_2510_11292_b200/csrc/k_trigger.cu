// Semantic-boundary trigger (P:101-106 [§4.1 r_t], P:301 [Alg. 1 is_new_segment]).
//
// r_t = (1/H) Σ_h cos(q_ref^h, q_t^h) over ALL H query heads; flag = (t == 1) ∨ (r_t < τ).
// Arithmetic recipe R1: fp64, e ascending, multiply then add with explicit
// round-to-nearest intrinsics (no contraction), cos = dot / (sqrt(na) * sqrt(nb)), clamped
// to [-1, 1]; a zero norm gives 0; heads summed in ascending order. This makes the decision
// bit-identical to any IEEE implementation of the same recipe.
//
// One CTA per sequence; one thread per head (the sequential per-head dot is the recipe).
// The work is 2*H*d bf16 per (b, layer) — latency bound, a few hundred ns.
#include "lkv_internal.cuh"

namespace lkv {

__global__ void __launch_bounds__(64) trigger_kernel(const uint16_t* __restrict__ q_all, int64_t stride_b, int Hq,
                                                     uint16_t* __restrict__ q_ref, uint8_t* flag, double* r,
                                                     uint8_t* flag_out, double* r_out, int t, double tau,
                                                     int trigger_ref) {
  extern __shared__ double cos_h[];  // [Hq]
  __shared__ int s_flag;
  const int b = blockIdx.x;
  const uint16_t* qc = q_all + (int64_t)b * stride_b;
  uint16_t* qr = q_ref + (int64_t)b * Hq * D;
  for (int h = threadIdx.x; h < Hq; h += blockDim.x) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    const uint16_t* a = qr + h * D;
    const uint16_t* c = qc + h * D;
#pragma unroll 4
    for (int e = 0; e < D; ++e) {
      double x = (double)bf2f(a[e]);
      double y = (double)bf2f(c[e]);
      dot = __dadd_rn(dot, __dmul_rn(x, y));
      na = __dadd_rn(na, __dmul_rn(x, x));
      nb = __dadd_rn(nb, __dmul_rn(y, y));
    }
    double cs = 0.0;
    if (na != 0.0 && nb != 0.0) {
      cs = __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
      cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
    }
    cos_h[h] = cs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int h = 0; h < Hq; ++h) s = __dadd_rn(s, cos_h[h]);
    double rr = __ddiv_rn(s, (double)Hq);
    int f = (t == 1) || (rr < tau);
    flag[b] = (uint8_t)f;
    r[b] = rr;
    if (flag_out) flag_out[b] = (uint8_t)f;
    if (r_out) r_out[b] = rr;
    s_flag = f;
  }
  __syncthreads();
  if (trigger_ref == LOUISKV_TRIG_PREV_STEP || s_flag) {
    // q_ref <- q_t ("q_prev <- q_t"; LAST_RETRIEVAL keeps the last retrieval's query)
    for (int i = threadIdx.x; i < Hq * D / 8; i += blockDim.x)
      reinterpret_cast<uint4*>(qr)[i] = reinterpret_cast<const uint4*>(qc)[i];
  }
}

__global__ void copy_flags_kernel(const uint8_t* src_flag, const double* src_r, uint8_t* flag, double* r,
                                  uint8_t* flag_out, double* r_out, int batch) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  uint8_t f = src_flag ? src_flag[b] : 0;
  double rr = src_r ? src_r[b] : 0.0;
  flag[b] = f;
  r[b] = rr;
  if (flag_out) flag_out[b] = f;
  if (r_out) r_out[b] = rr;
}

cudaError_t launch_trigger(const bf16* q_all, int64_t stride_b, int batch, int Hq, bf16* q_ref, uint8_t* flag,
                           double* r, uint8_t* flag_out, double* r_out, int t, double tau, int trigger_ref,
                           cudaStream_t st) {
  trigger_kernel<<<batch, 64, sizeof(double) * Hq, st>>>(
      reinterpret_cast<const uint16_t*>(q_all), stride_b, Hq, reinterpret_cast<uint16_t*>(q_ref), flag, r, flag_out,
      r_out, t, tau, trigger_ref);
  return cudaGetLastError();
}

cudaError_t launch_copy_flags(const uint8_t* src_flag, const double* src_r, uint8_t* flag, double* r,
                              uint8_t* flag_out, double* r_out, int batch, cudaStream_t st) {
  copy_flags_kernel<<<(batch + 127) / 128, 128, 0, st>>>(src_flag, src_r, flag, r, flag_out, r_out, batch);
  return cudaGetLastError();
}

}  // namespace lkv
