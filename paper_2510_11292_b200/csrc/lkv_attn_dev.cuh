// Split-K flash-decode attention body shared by the attention kernels (k_attn.cu) and the
// single-launch layer kernel (k_layer.cu). o = softmax(q K_I^T / sqrt(d)) V_I (P:63-65 [§3.1]).
#pragma once
#include <cooperative_groups.h>

#include "lkv_internal.cuh"

namespace lkv {

constexpr int AT_THREADS = 256;
constexpr int AT_HW = AT_THREADS / 16;  // half-warps per CTA
constexpr int AT_CHUNK = 64;           // rows per pipeline stage
constexpr int AT_STAGES = 3;
constexpr int AT_STAGE_BYTES = AT_CHUNK * 2 * ROW_BYTES;  // K + V: 32 KB
constexpr int AT_SMEM = AT_STAGES * AT_STAGE_BYTES + 64;
constexpr int AT_CL = 8;  // cluster size of the fused append+attention launch (one cluster per instance)

struct RowSpan {
  const bf16* k0;  // sinks (or the full cache)
  const bf16* v0;
  int n0;
  const bf16* k1;  // working set
  const bf16* v1;
  int n1;
  const bf16* k2;  // ring
  const bf16* v2;
  int head, cap;
};

// Rows of an attention set as up to AT_PMAX contiguous pieces in virtual-row order.
constexpr int AT_PMAX = 4;
struct Pieces {
  int np;
  int v0[AT_PMAX], n[AT_PMAX];
  const bf16* k[AT_PMAX];
  const bf16* v[AT_PMAX];
  __device__ __forceinline__ void add(int cnt, const bf16* kb, const bf16* vb) {
    if (cnt > 0) {
      const int base = np ? v0[np - 1] + n[np - 1] : 0;
      v0[np] = base;
      n[np] = cnt;
      k[np] = kb;
      v[np] = vb;
      ++np;
    }
  }
};

// CTA-level flash-decode partial over virtual rows [r_begin, r_end) of the pieces, for the G query
// heads at qb (bf16 [G][D]). Returns the merged partial in shared memory, [G][D+2] floats:
// unnormalised accumulator (log2-domain max subtracted), then (max, sum). Every thread calls;
// the caller's subsequent reads of the result are ordered by the internal barriers.
template <int G>
__device__ __forceinline__ float* attn_partial(const uint16_t* qb, const float scale_log2, const Pieces& P,
                                               const int r_begin, const int r_end, unsigned long long* prof) {
  const int tid = threadIdx.x, hw = tid >> 4, sub = tid & 15;
  const int np = P.np;
  // query fragment: this lane's 8 dims for each of the G heads, pre-scaled into log2 domain
  float q[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    uint4 u = reinterpret_cast<const uint4*>(qb + j * D)[sub];
    unpack8(u, q[j]);
#pragma unroll
    for (int k = 0; k < 8; ++k) q[j][k] *= scale_log2;
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[j][k] = 0.f;
  }

  extern __shared__ __align__(128) uint8_t at_smem[];
  uint8_t* sKV = at_smem;  // [AT_STAGES][K 64x256 B | V 64x256 B]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(at_smem + AT_STAGES * AT_STAGE_BYTES);
  const int n_chunks = (r_end - r_begin + AT_CHUNK - 1) / AT_CHUNK;
  auto issue = [&](int c) {
    const int st = c % AT_STAGES;
    const int c0 = r_begin + c * AT_CHUNK, c1 = min(r_end, c0 + AT_CHUNK);
    uint8_t* dK = sKV + st * AT_STAGE_BYTES;
    uint8_t* dV = dK + AT_CHUNK * ROW_BYTES;
    ptx_mbar_expect_tx(&full_bar[st], (uint32_t)(c1 - c0) * 2 * ROW_BYTES);
    for (int p = 0; p < np; ++p) {
      const int lo = max(c0, P.v0[p]), hi = min(c1, P.v0[p] + P.n[p]);
      if (lo >= hi) continue;
      const uint32_t bytes = (uint32_t)(hi - lo) * ROW_BYTES;
      ptx_bulk_g2s(dK + (lo - c0) * ROW_BYTES, P.k[p] + (int64_t)(lo - P.v0[p]) * D, bytes, &full_bar[st]);
      ptx_bulk_g2s(dV + (lo - c0) * ROW_BYTES, P.v[p] + (int64_t)(lo - P.v0[p]) * D, bytes, &full_bar[st]);
    }
  };
  if (tid == 0) {
    for (int i = 0; i < AT_STAGES; ++i) ptx_mbar_init(&full_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < n_chunks && c < AT_STAGES; ++c) issue(c);

  const int warp = tid >> 5;
  constexpr int RB = 4;  // rows per half-warp per chunk (16 half-warps x 4 = 64 rows)
  for (int c = 0; c < n_chunks; ++c) {
    const int st = c % AT_STAGES;
    const int rows = min(AT_CHUNK, r_end - (r_begin + c * AT_CHUNK));
    ptx_mbar_wait(&full_bar[st], (uint32_t)((c / AT_STAGES) & 1));
    if (c == 0) prof_stamp(prof, 8);
    const uint8_t* sK = sKV + st * AT_STAGE_BYTES;
    const uint8_t* sV = sK + AT_CHUNK * ROW_BYTES;
    uint4 ku[RB], vu[RB];
    bool valid[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int r = hw + 16 * i;
      valid[i] = r < rows;
      ku[i] = valid[i] ? reinterpret_cast<const uint4*>(sK + r * ROW_BYTES)[sub] : make_uint4(0, 0, 0, 0);
      vu[i] = valid[i] ? reinterpret_cast<const uint4*>(sV + r * ROW_BYTES)[sub] : make_uint4(0, 0, 0, 0);
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
      if (mb == -INFINITY) continue;
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
    __syncthreads();  // stage st fully consumed
    if (tid == 0 && c + AT_STAGES < n_chunks) issue(c + AT_STAGES);
  }

  prof_stamp(prof, 9);
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
  __shared__ float s_m[AT_W][G], s_lw[AT_W][G];
  // the stage ring is idle after the main loop: reuse it for the cross-warp merge
  float (*s_acc)[G][D] = reinterpret_cast<float (*)[G][D]>(at_smem);
  if ((tid & 31) < 16) {
    if (sub == 0) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        s_m[warp][j] = m[j];
        s_lw[warp][j] = l[j];
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) s_acc[warp][j][sub * 8 + k] = acc[j][k];
  }
  __syncthreads();

  float* part = reinterpret_cast<float*>(at_smem + AT_W * G * D * sizeof(float));
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < AT_W; ++w) M = fmaxf(M, s_m[w][j]);
    float Lsum = 0.f, A = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < AT_W; ++w) {
        const float sc = exp2f(s_m[w][j] - M);
        Lsum += s_lw[w][j] * sc;
        A += s_acc[w][j][e] * sc;
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

// Attention of instance li, split `split` of `nsplit` (FUSED: nsplit = AT_CL ranks of one cluster,
// merged through DSMEM; else global partials merged by the last CTA). Every thread of the CTA calls.
template <int G, bool FUSED>
__device__ __forceinline__ void attn_body(const AttnArgs& a, const int li, const int split, const int nsplit,
                                          unsigned long long* prof = nullptr) {
  namespace cg = cooperative_groups;
  const int b = li / a.hn, h = li % a.hn;
  const int tid = threadIdx.x;
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
  const int r_begin = (int)((int64_t)n_rows * split / nsplit);
  const int r_end = (int)((int64_t)n_rows * (split + 1) / nsplit);

  Pieces P;
  P.np = 0;
  if (a.inst) {
    P.add(sp.n0, sp.k0, sp.v0);
    P.add(sp.n1, sp.k1, sp.v1);
    const int nb = n_rows - sp.n0 - sp.n1;
    const int h0 = sp.head % sp.cap;
    const int first = nb < sp.cap - h0 ? nb : sp.cap - h0;
    P.add(first, sp.k2 + (int64_t)h0 * D, sp.v2 + (int64_t)h0 * D);
    P.add(nb - first, sp.k2, sp.v2);
  } else {
    P.add(sp.n0, sp.k0, sp.v0);
  }
  const uint16_t* qb = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b + (int64_t)h * G * D;
  float* part_s = attn_partial<G>(qb, a.scale_log2, P, r_begin, r_end, prof);
  // per-CTA partial: own smem (cluster merge) or global scratch (split merge by the last CTA)
  float* part = part_s;
  if constexpr (!FUSED) {
    part = a.part + ((int64_t)li * nsplit + split) * G * (D + 2);
    for (int i = tid; i < G * (D + 2); i += AT_THREADS) part[i] = part_s[i];
  }

  if constexpr (FUSED) {
    // ---- rank 0 merges the AT_CL partials through distributed shared memory, in rank order
    cg::cluster_group cl = cg::this_cluster();
    prof_stamp(prof, 10);
    cl.sync();
    prof_stamp(prof, 11);
    if (split == 0) {
      __shared__ float f_w[AT_CL][G];
      __shared__ float f_l[AT_CL][G];
      for (int t = tid; t < AT_CL * G; t += AT_THREADS) {
        const int y = t / G, j = t % G;
        const float* py = cl.map_shared_rank(part, y);
        f_w[y][j] = py[j * (D + 2) + D];
        f_l[y][j] = py[j * (D + 2) + D + 1];
      }
      __syncthreads();
      if (tid < G) {
        const int j = tid;
        float M = -INFINITY;
        for (int y = 0; y < AT_CL; ++y) M = fmaxf(M, f_w[y][j]);
        float Lsum = 0.f;
        for (int y = 0; y < AT_CL; ++y) {
          const float w = f_w[y][j] == -INFINITY ? 0.f : exp2f(f_w[y][j] - M);
          f_w[y][j] = w;
          Lsum += w * f_l[y][j];
        }
        const float inv = 1.f / Lsum;
        for (int y = 0; y < AT_CL; ++y) f_w[y][j] *= inv;
      }
      __syncthreads();
      for (int idx = tid; idx < G * D; idx += AT_THREADS) {
        const int j = idx / D, e = idx % D;
        float A = 0.f;
#pragma unroll
        for (int y = 0; y < AT_CL; ++y) A = fmaf(f_w[y][j], cl.map_shared_rank(part, y)[j * (D + 2) + e], A);
        const int64_t oi = ((int64_t)(b * a.hn + h) * G + j) * D + e;
        a.out[oi] = __float2bfloat16_rn(A);
        if (a.out_f32) a.out_f32[oi] = A;
      }
    }
    prof_stamp(prof, 12);
    cl.sync();  // keep every rank's shared memory alive until rank 0 has read it
    prof_stamp(prof, 13);
    return;
  }
  // ---- last CTA of this instance merges the splits in split order
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int ticket = atomicAdd(&a.counters[li], 1);
    s_last = (ticket == nsplit - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* P0 = a.part + (int64_t)li * nsplit * G * (D + 2);
  const int Y = nsplit;
  __shared__ float s_w[64][G];  // per-split weights exp2(m_y - M) / L
  __shared__ float s_l[64][G];
  // all (split, head) statistics loaded in parallel, then the G reductions over splits
  for (int t = tid; t < Y * G; t += AT_THREADS) {
    const int y = t / G, j = t % G;
    s_w[y][j] = __ldcg(P0 + (y * G + j) * (D + 2) + D);
    s_l[y][j] = __ldcg(P0 + (y * G + j) * (D + 2) + D + 1);
  }
  __syncthreads();
  if (tid < G) {
    const int j = tid;
    float M = -INFINITY;
    for (int y = 0; y < Y; ++y) M = fmaxf(M, s_w[y][j]);
    float Lsum = 0.f;
    for (int y = 0; y < Y; ++y) {
      const float w = s_w[y][j] == -INFINITY ? 0.f : exp2f(s_w[y][j] - M);
      s_w[y][j] = w;
      Lsum += w * s_l[y][j];
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


}  // namespace lkv
