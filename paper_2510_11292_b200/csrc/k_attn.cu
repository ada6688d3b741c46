// Sparse decode attention — o = softmax(q K_I^T / sqrt(d)) V_I  (P:63-65 [§3.1]),
// I = sinks ∪ KV_critical ∪ KV_local (P:143, P:307 [Alg. 1 KV_attn]); the full-cache layers
// attend to all P+t rows.
//
// Split-K flash-decode, GQA-packed: one CTA per (instance, split); the g query heads of a KV
// head share every K/V row read (one HBM read serves g heads). Inside a CTA, each half-warp
// (16 lanes x 8 dims) walks rows with an online softmax in the log2 domain; half-warps merge
// through shared memory; splits merge in a fixed order by the last CTA to finish (atomic
// ticket), so the result is deterministic. HBM-bound: 512 B of K+V per row.
#include "lkv_internal.cuh"

namespace lkv {

constexpr int AT_THREADS = 128;
constexpr int AT_HW = AT_THREADS / 16;  // half-warps per CTA
constexpr int AT_MAXG = 8;

struct RowSpan {
  const bf16* k0;  // sinks
  const bf16* v0;
  int n0;
  const bf16* k1;  // working set
  const bf16* v1;
  int n1;
  const bf16* k2;  // ring
  const bf16* v2;
  int head, cap;
};

__device__ __forceinline__ void row_ptrs(const RowSpan& sp, int r, const uint4*& kp, const uint4*& vp) {
  if (r < sp.n0) {
    kp = reinterpret_cast<const uint4*>(sp.k0 + (int64_t)r * D);
    vp = reinterpret_cast<const uint4*>(sp.v0 + (int64_t)r * D);
    return;
  }
  r -= sp.n0;
  if (r < sp.n1) {
    kp = reinterpret_cast<const uint4*>(sp.k1 + (int64_t)r * D);
    vp = reinterpret_cast<const uint4*>(sp.v1 + (int64_t)r * D);
    return;
  }
  r -= sp.n1;
  const int slot = (sp.head + r) % sp.cap;
  kp = reinterpret_cast<const uint4*>(sp.k2 + (int64_t)slot * D);
  vp = reinterpret_cast<const uint4*>(sp.v2 + (int64_t)slot * D);
}

template <int G>
__global__ void __launch_bounds__(AT_THREADS) attn_kernel(AttnArgs a) {
  const int li = blockIdx.x, split = blockIdx.y;
  const int b = li / a.hn, h = li % a.hn;
  const int tid = threadIdx.x, hw = tid >> 4, sub = tid & 15;

  RowSpan sp;
  int n_rows;
  if (a.inst) {
    const InstState& S = a.inst[li];
    const int64_t gi = a.inst_global_base + li;
    sp.k0 = a.sinks + (int64_t)li * 2 * a.S * D;
    sp.v0 = sp.k0 + (int64_t)a.S * D;
    sp.n0 = S.s_eff;
    sp.k1 = a.ws + S.ws_cur * a.ws_buf_stride + gi * a.ws_inst_stride;
    sp.v1 = sp.k1 + (int64_t)a.B * D;
    sp.n1 = S.ws_rows;
    sp.k2 = a.ring + (int64_t)li * 2 * a.ring_cap * D;
    sp.v2 = sp.k2 + (int64_t)a.ring_cap * D;
    sp.head = S.ring_head;
    sp.cap = a.ring_cap;
    n_rows = sp.n0 + sp.n1 + S.buffered;
  } else {
    sp.k0 = a.full + (int64_t)li * 2 * a.full_cap * D;
    sp.v0 = sp.k0 + a.full_cap * D;
    const int64_t rows = a.full_P + *a.step;
    n_rows = (int)(rows < a.full_cap ? rows : a.full_cap);
    sp.n0 = n_rows;
    sp.n1 = 0;
    sp.k1 = sp.v1 = sp.k2 = sp.v2 = nullptr;
    sp.head = 0;
    sp.cap = 1;
  }
  const int r_begin = (int)((int64_t)n_rows * split / gridDim.y);
  const int r_end = (int)((int64_t)n_rows * (split + 1) / gridDim.y);

  // query fragment: this lane's 8 dims for each of the G heads, pre-scaled into log2 domain
  float q[G][8];
  const uint16_t* qb = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b + (int64_t)h * G * D;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    uint4 u = reinterpret_cast<const uint4*>(qb + j * D)[sub];
    unpack8(u, q[j]);
#pragma unroll
    for (int k = 0; k < 8; ++k) q[j][k] *= a.scale_log2;
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[j][k] = 0.f;
  }

  // warp-uniform loop: each warp takes 4 consecutive rows per iteration (2 per half-warp),
  // so both half-warps always execute the same shuffles.
  const int warp = tid >> 5, half = hw & 1;
  constexpr int NWARP = AT_THREADS / 32;
  for (int base = r_begin + warp * 4; base < r_end; base += 4 * NWARP) {
    const int ra = base + half, rb = base + 2 + half;
    const bool va = ra < r_end, vb = rb < r_end;
    uint4 ku0 = make_uint4(0, 0, 0, 0), vu0 = ku0, ku1 = ku0, vu1 = ku0;
    const uint4 *kp, *vp;
    if (va) {
      row_ptrs(sp, ra, kp, vp);
      ku0 = __ldg(kp + sub);
      vu0 = __ldg(vp + sub);
    }
    if (vb) {
      row_ptrs(sp, rb, kp, vp);
      ku1 = __ldg(kp + sub);
      vu1 = __ldg(vp + sub);
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const bool valid = rr ? vb : va;
      float kf[8], vf[8];
      unpack8(rr ? ku1 : ku0, kf);
      unpack8(rr ? vu1 : vu0, vf);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) s = fmaf(q[j][k], kf[k], s);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (valid) {
          const float mn = fmaxf(m[j], s);
          const float corr = exp2f(m[j] - mn);
          const float p = exp2f(s - mn);
          l[j] = l[j] * corr + p;
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[j][k] = fmaf(acc[j][k], corr, p * vf[k]);
          m[j] = mn;
        }
      }
    }
  }

  // ---- merge half-warps through shared memory
  __shared__ float s_m[AT_HW][G], s_l[AT_HW][G];
  __shared__ float s_acc[AT_HW][G][D];
  if (sub == 0) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      s_m[hw][j] = m[j];
      s_l[hw][j] = l[j];
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int k = 0; k < 8; ++k) s_acc[hw][j][sub * 8 + k] = acc[j][k];
  __syncthreads();

  float* part = a.part + ((int64_t)li * gridDim.y + split) * G * (D + 2);
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < AT_HW; ++w) M = fmaxf(M, s_m[w][j]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < AT_HW; ++w) {
        const float sc = exp2f(s_m[w][j] - M);
        Lsum += s_l[w][j] * sc;
        A += s_acc[w][j][e] * sc;
      }
    }
    part[j * (D + 2) + e] = A;
    if (e == 0) {
      part[j * (D + 2) + D] = M;
      part[j * (D + 2) + D + 1] = Lsum;
    }
  }

  // ---- last CTA of this instance merges the splits in split order
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int ticket = atomicAdd(&a.counters[li], 1);
    s_last = (ticket == (int)gridDim.y - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* P0 = a.part + (int64_t)li * gridDim.y * G * (D + 2);
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
    for (int y = 0; y < (int)gridDim.y; ++y) M = fmaxf(M, __ldcg(P0 + (y * G + j) * (D + 2) + D));
    float Lsum = 0.f, A = 0.f;
    for (int y = 0; y < (int)gridDim.y; ++y) {
      const float my = __ldcg(P0 + (y * G + j) * (D + 2) + D);
      if (my == -INFINITY) continue;
      const float sc = exp2f(my - M);
      Lsum += __ldcg(P0 + (y * G + j) * (D + 2) + D + 1) * sc;
      A += __ldcg(P0 + (y * G + j) * (D + 2) + e) * sc;
    }
    const float o = A / Lsum;
    const int64_t oi = ((int64_t)(b * a.hn + h) * G + j) * D + e;
    a.out[oi] = __float2bfloat16_rn(o);
    if (a.out_f32) a.out_f32[oi] = o;
  }
  if (tid == 0) a.counters[li] = 0;
}

cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st) {
  dim3 grid(a.batch * a.hn, a.splits);
  switch (a.g) {
    case 1: attn_kernel<1><<<grid, AT_THREADS, 0, st>>>(a); break;
    case 2: attn_kernel<2><<<grid, AT_THREADS, 0, st>>>(a); break;
    case 4: attn_kernel<4><<<grid, AT_THREADS, 0, st>>>(a); break;
    case 8: attn_kernel<8><<<grid, AT_THREADS, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lkv
