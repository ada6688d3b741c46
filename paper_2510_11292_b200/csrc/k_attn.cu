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

constexpr int AT_THREADS = 256;
constexpr int AT_HW = AT_THREADS / 16;  // half-warps per CTA

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

  // warp-uniform loop: each half-warp takes 4 rows per iteration (8 x 16-B loads in flight per
  // lane), then one block-wise online-softmax update for the 4 rows.
  const int warp = tid >> 5, half = hw & 1;
  constexpr int NWARP = AT_THREADS / 32;
  constexpr int RB = 4;
  for (int base = r_begin + warp * (2 * RB); base < r_end; base += 2 * RB * NWARP) {
    uint4 ku[RB], vu[RB];
    bool valid[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int r = base + half + 2 * i;
      valid[i] = r < r_end;
      ku[i] = make_uint4(0, 0, 0, 0);
      vu[i] = ku[i];
      if (valid[i]) {
        const uint4 *kp, *vp;
        row_ptrs(sp, r, kp, vp);
        ku[i] = __ldg(kp + sub);
        vu[i] = __ldg(vp + sub);
      }
    }
    float s[RB][G];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      float kf[8];
      unpack8(ku[i], kf);
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t = fmaf(q[j][k], kf[k], t);
        s[i][j] = t;
      }
    }
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int j = 0; j < G; ++j) {
        float t = s[i][j];
        t += __shfl_xor_sync(0xffffffffu, t, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        s[i][j] = valid[i] ? t : -INFINITY;
      }
    float vf[RB][8];
#pragma unroll
    for (int i = 0; i < RB; ++i) unpack8(vu[i], vf[i]);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      float mb = m[j];
#pragma unroll
      for (int i = 0; i < RB; ++i) mb = fmaxf(mb, s[i][j]);
      if (mb == -INFINITY) continue;  // no valid row yet for this half-warp
      const float corr = exp2f(m[j] - mb);
      float p[RB], ps = 0.f;
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        p[i] = exp2f(s[i][j] - mb);
        ps += p[i];
      }
      l[j] = fmaf(l[j], corr, ps);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float t = acc[j][k] * corr;
#pragma unroll
        for (int i = 0; i < RB; ++i) t = fmaf(p[i], vf[i][k], t);
        acc[j][k] = t;
      }
      m[j] = mb;
    }
  }

  // ---- merge the two half-warps of each warp (lane ^ 16 holds the same dims), then the warps
  // through shared memory
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const float mo = __shfl_xor_sync(0xffffffffu, m[j], 16);
    const float lo = __shfl_xor_sync(0xffffffffu, l[j], 16);
    const float M = fmaxf(m[j], mo);
    const float sa = M == -INFINITY ? 0.f : exp2f(m[j] - M);
    const float sb = M == -INFINITY ? 0.f : exp2f(mo - M);
    l[j] = l[j] * sa + lo * sb;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float ao = __shfl_xor_sync(0xffffffffu, acc[j][k], 16);
      acc[j][k] = acc[j][k] * sa + ao * sb;
    }
    m[j] = M;
  }
  constexpr int AT_W = AT_THREADS / 32;
  __shared__ float s_m[AT_W][G], s_l[AT_W][G];
  __shared__ float s_acc[AT_W][G][D];
  if ((tid & 31) < 16) {
    if (sub == 0) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        s_m[warp][j] = m[j];
        s_l[warp][j] = l[j];
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) s_acc[warp][j][sub * 8 + k] = acc[j][k];
  }
  __syncthreads();

  float* part = a.part + ((int64_t)li * gridDim.y + split) * G * (D + 2);
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < AT_W; ++w) M = fmaxf(M, s_m[w][j]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < AT_W; ++w) {
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
  const int Y = gridDim.y;
  __shared__ float s_w[64][G];  // per-split weights exp2(m_y - M) / L
  if (tid < G) {
    const int j = tid;
    float M = -INFINITY;
    for (int y = 0; y < Y; ++y) M = fmaxf(M, __ldcg(P0 + (y * G + j) * (D + 2) + D));
    float Lsum = 0.f;
    for (int y = 0; y < Y; ++y) {
      const float my = __ldcg(P0 + (y * G + j) * (D + 2) + D);
      const float w = my == -INFINITY ? 0.f : exp2f(my - M);
      s_w[y][j] = w;
      Lsum += w * __ldcg(P0 + (y * G + j) * (D + 2) + D + 1);
    }
    const float inv = 1.f / Lsum;
    for (int y = 0; y < Y; ++y) s_w[y][j] *= inv;
  }
  __syncthreads();
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float A = 0.f;
#pragma unroll 4
    for (int y = 0; y < Y; ++y) A = fmaf(s_w[y][j], __ldcg(P0 + (y * G + j) * (D + 2) + e), A);
    const int64_t oi = ((int64_t)(b * a.hn + h) * G + j) * D + e;
    a.out[oi] = __float2bfloat16_rn(A);
    if (a.out_f32) a.out_f32[oi] = A;
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
