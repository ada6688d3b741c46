// kvm.store_cache(K, V, 'prefill') — P:120 [§4.2 Prefill stage: k-means of keys, centroid =
// mean of the cluster's keys, offload to the CPU pool], P:258-265 [Alg. 1], P:126 [clustering
// kernel].
//
// Per (b, owned kv-head) instance with N = P - S keys and k = ceil(N / c) clusters:
//   init      C_j = x_{floor(j N / k)}                                    (reading R-AMB8)
//   repeat iters times:
//     assign  a_i = argmax_j (x_i · bf16(C_j) - ½||C_j||²), ties -> lower j  (tcgen05 GEMM with
//             fused argmax epilogue in k_kmeans_tc.cu; SIMT fallback kernel here)
//     hist    per 1024-key chunk cluster histogram
//     scan    per-cluster exclusive prefix over chunks + cluster offsets (counting sort)
//     repair  empty clusters take the farthest keys (largest dmin, ties -> lower index) from
//             clusters with >= 2 members (reading R-AMB9); rare, one CTA per instance
//     scatter stable counting-sort scatter: perm = keys grouped by cluster, positions ascending
//     update  C_j = (sequential fp32 sum of member keys) / |j|, one warp per cluster
//   offload   KV rows permuted cluster-major and written to the pinned host pool (zero-copy
//             stores), unit table, sinks kept on the device.
#include "lkv_internal.cuh"

namespace lkv {

constexpr int KM_CHUNK = 1024;
constexpr int KM_TASK = 32;  // members per centroid-update task

// -½||c||² folded into the tensor-core GEMM as a 9th K-step: three bf16 parts whose sum equals the
// fp32 half-norm to within fp32 rounding (h = hi + mid + lo exactly up to the last ~2^-24 of h)
__device__ __forceinline__ void write_bext(const KmArgs& a, int li, int j, float h) {
  const uint16_t hi = f2bf_rne(h);
  const float r1 = h - bf2f(hi);
  const uint16_t mid = f2bf_rne(r1);
  const uint16_t lo = f2bf_rne(r1 - bf2f(mid));
  uint4 v;
  v.x = (uint32_t)(hi ^ 0x8000u) | ((uint32_t)(mid ^ 0x8000u) << 16);  // negated (sign flip)
  v.y = (uint32_t)(lo ^ 0x8000u);
  v.z = 0u;
  v.w = 0u;
  reinterpret_cast<uint4*>(a.bext)[(int64_t)li * a.Umax + j] = v;
}

__device__ __forceinline__ const bf16* xrow(const KmArgs& a, int li, int i) {
  const int b = li / a.hn, h = li % a.hn;
  return a.k + (int64_t)b * a.sb + (int64_t)(a.S + i) * a.st + (int64_t)h * a.sh;
}
__device__ __forceinline__ const bf16* vrow(const KmArgs& a, int li, int i) {
  const int b = li / a.hn, h = li % a.hn;
  return a.v + (int64_t)b * a.sb + (int64_t)(a.S + i) * a.st + (int64_t)h * a.sh;
}

// ---- init: C_j = x_{floor(j N / k)}; bf16 copy; ½||C_j||²  (warp per cluster)
__global__ void km_init_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + warp;
  if (j >= a.kc) return;
  const int src = (int)(((int64_t)j * a.N) / a.kc);
  const uint2 u = reinterpret_cast<const uint2*>(xrow(a, li, src))[lane];
  float c[4] = {__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                __uint_as_float(u.y & 0xFFFF0000u)};
  float* C = a.cent + ((int64_t)li * a.Umax + j) * D;
  uint16_t* Cb = reinterpret_cast<uint16_t*>(a.centb) + ((int64_t)li * a.Umax + j) * D;
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    C[lane * 4 + e] = c[e];
    Cb[lane * 4 + e] = f2bf_rne(c[e]);
    ss = fmaf(c[e], c[e], ss);
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    a.half[(int64_t)li * a.hstride + j] = 0.5f * ss;
    write_bext(a, li, j, 0.5f * ss);
  }
}

// ---- +inf half-norms (-inf GEMM extension) for the padded centroid columns [kc, hstride)
__global__ void km_half_pad_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  for (int j = a.kc + threadIdx.x; j < a.hstride; j += blockDim.x) {
    a.half[(int64_t)li * a.hstride + j] = INFINITY;
    if (j < a.Umax) reinterpret_cast<uint4*>(a.bext)[(int64_t)li * a.Umax + j] = make_uint4(0xFF80u, 0u, 0u, 0u);
  }
}

// ---- SIMT assignment (correctness reference path; the tcgen05 kernel is the fast path)
constexpr int AS_TILE = 32;
__global__ void __launch_bounds__(128) km_assign_simt_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int i = blockIdx.x * 128 + threadIdx.x;
  __shared__ uint32_t sc[AS_TILE][D / 2];
  __shared__ float sh[AS_TILE];
  float x[D];
  float xn = 0.f;
  if (i < a.N) {
    const uint4* r = reinterpret_cast<const uint4*>(xrow(a, li, i));
#pragma unroll
    for (int c = 0; c < D / 8; ++c) unpack8(r[c], x + c * 8);
#pragma unroll
    for (int e = 0; e < D; ++e) xn = fmaf(x[e], x[e], xn);
  }
  float best = -INFINITY;
  int bi = 0;
  const uint32_t* Cb = reinterpret_cast<const uint32_t*>(a.centb + (int64_t)li * a.Umax * D);
  const float* half = a.half + (int64_t)li * a.hstride;
  for (int j0 = 0; j0 < a.kc; j0 += AS_TILE) {
    __syncthreads();
    for (int t = threadIdx.x; t < AS_TILE * D / 2; t += 128) {
      const int jj = t / (D / 2);
      sc[jj][t % (D / 2)] = (j0 + jj < a.kc) ? Cb[(int64_t)(j0 + jj) * (D / 2) + t % (D / 2)] : 0u;
    }
    if (threadIdx.x < AS_TILE) sh[threadIdx.x] = (j0 + threadIdx.x < a.kc) ? half[j0 + threadIdx.x] : INFINITY;
    __syncthreads();
    const int jn = min(AS_TILE, a.kc - j0);
    for (int jj = 0; jj < jn; ++jj) {
      float dot = 0.f;
#pragma unroll
      for (int e2 = 0; e2 < D / 2; ++e2) {
        const uint32_t w = sc[jj][e2];
        dot = fmaf(x[2 * e2], __uint_as_float(w << 16), dot);
        dot = fmaf(x[2 * e2 + 1], __uint_as_float(w & 0xFFFF0000u), dot);
      }
      const float s = dot - sh[jj];
      if (s > best) {
        best = s;
        bi = j0 + jj;
      }
    }
  }
  if (i < a.N) {
    a.assign[(int64_t)li * a.Nmax + i] = bi;
    a.dmin[(int64_t)li * a.Nmax + i] = fmaf(-2.f, best, xn);
  }
}

// ---- per-chunk histogram
__global__ void __launch_bounds__(256) km_hist_kernel(KmArgs a, int nchunk) {
  pdl_wait_trigger();
  extern __shared__ int hist[];
  const int li = blockIdx.y, c = blockIdx.x;
  for (int j = threadIdx.x; j < a.kc; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  const int i0 = c * KM_CHUNK, i1 = min(a.N, i0 + KM_CHUNK);
  const int32_t* as = a.assign + (int64_t)li * a.Nmax;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) atomicAdd(&hist[as[i]], 1);
  __syncthreads();
  // chunk counts, chunk-major cc[inst][chunk][cluster]: one coalesced row per chunk (the column
  // scan walks the chunks per cluster with one thread per cluster, coalesced too)
  int32_t* cc = a.cc + ((int64_t)li * a.nchunk_max + c) * a.kmax;
  for (int j = threadIdx.x; j < a.kc; j += blockDim.x) cc[j] = hist[j];
}

// column scan of cc + cluster offsets; one 1024-thread CTA per instance
__device__ int km_block_excl_scan(int v, int& total) {
  __shared__ int s_w[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < nw ? s_w[lane] : 0;
    int wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) s_w[lane] = wi - w;
    if (lane == 31) s_w[32] = wi;
  }
  __syncthreads();
  const int r = s_w[warp] + incl - v;
  total = s_w[32];
  __syncthreads();
  return r;
}

// column scan: one thread per cluster walks the chunks in order (coalesced over clusters): the
// cluster's exclusive prefix per chunk -> ccT[inst][chunk][cluster] (the scatter's bases), count
__global__ void __launch_bounds__(256) km_colscan_kernel(KmArgs a, int nchunk, int only_dirty) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  if (only_dirty && a.flags[li] != 2) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.kc) return;
  const int32_t* cc = a.cc + (int64_t)li * a.nchunk_max * a.kmax + j;
  int32_t* ccT = a.ccT + (int64_t)li * a.nchunk_max * a.kmax + j;
  int run = 0;
  for (int c0 = 0; c0 < nchunk; c0 += 8) {
    int v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = c0 + q < nchunk ? cc[(int64_t)(c0 + q) * a.kmax] : 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (c0 + q < nchunk) {
        ccT[(int64_t)(c0 + q) * a.kmax] = run;
        run += v[q];
      }
  }
  a.cnt[(int64_t)li * a.kmax + j] = run;
}

// cluster offsets and update-task offsets from the counts (one CTA per instance)
__global__ void __launch_bounds__(1024) km_offsets_kernel(KmArgs a, int only_dirty) {
  pdl_wait_trigger();
  const int li = blockIdx.x;
  if (only_dirty && a.flags[li] != 2) return;
  const int32_t* cnt = a.cnt + (int64_t)li * a.kmax;
  int32_t* off = a.off + (int64_t)li * (a.kmax + 1);
  int32_t* toff = a.toff + (int64_t)li * (a.kmax + 1);
  int4* tcl = a.tcl + (int64_t)li * a.task_max;
  const int per = (a.kc + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * per, j1 = min(a.kc, j0 + per);
  int local = 0, tloc = 0, empty = 0;
  for (int j = j0; j < j1; ++j) {
    const int c = cnt[j];
    local += c;
    tloc += (c + KM_TASK - 1) / KM_TASK;
    empty |= c == 0;
  }
  int total, ttotal;
  int run = km_block_excl_scan(local, total);
  int trun = km_block_excl_scan(tloc, ttotal);
  const int any_empty = __syncthreads_or(empty);
  for (int j = j0; j < j1; ++j) {
    off[j] = run;
    toff[j] = trun;
    {  // the update tasks of cluster j: (cluster, first member, end member, tasks of the cluster)
      const int nt = (cnt[j] + KM_TASK - 1) / KM_TASK;
      for (int q = 0; q < nt; ++q)
        tcl[trun + q] = make_int4(j, run + q * KM_TASK, min(run + cnt[j], run + (q + 1) * KM_TASK), nt);
      trun += nt;
    }
    run += cnt[j];
  }
  if (threadIdx.x == 0) {
    off[a.kc] = a.N;
    toff[a.kc] = ttotal;
    a.flags[li] = any_empty;
  }
}

// empty-cluster repair (reading R-AMB9), then recount; only instances with an empty cluster.
// Sequential rule: for each empty id ascending, the donor is the key with the largest dmin (ties ->
// lower index) among clusters that still have >= 2 members. Eligibility only decreases, so the
// donors are the first eligible keys of ONE list sorted by (dmin desc, index asc). Exact fast
// path: radix-select a dmin threshold admitting ~1.5E statically eligible keys, compact and
// bitonic-sort them in shared memory, walk them once with cluster counts in shared memory.
// If the walk runs out of candidates (many ineligible), the slow per-empty scan finishes the job.
constexpr int RP_CAND = 2048;
constexpr int RP_SMEM_MAX = 200 * 1024;
__host__ __device__ inline size_t repair_smem_base(int kc) {
  return sizeof(int) * (2 * (size_t)kc) + RP_CAND * (sizeof(unsigned long long) + sizeof(int));
}
// the eligible-donor keys of all N points are kept in shared memory when they fit (one pass over
// global memory instead of five: the four threshold passes and the compaction read them on chip)
__host__ __device__ inline bool repair_keys_in_smem(int kc, int N) {
  return repair_smem_base(kc) + sizeof(unsigned) * (size_t)N <= RP_SMEM_MAX;
}
__global__ void __launch_bounds__(1024) km_repair_kernel(KmArgs a, int nchunk) {
  pdl_wait_trigger();
  const int li = blockIdx.x;
  if (!a.flags[li]) return;
  extern __shared__ int rp_smem[];
  int* s_cnt = rp_smem;                                                   // [kc]
  int* s_empty = s_cnt + a.kc;                                            // [kc]
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(s_empty + a.kc + (a.kc & 1 ? 0 : 0));  // [RP_CAND] (2*kc ints: 8-B aligned)
  int* s_cl = reinterpret_cast<int*>(s_key + RP_CAND);                    // [RP_CAND]
  unsigned* s_dk = reinterpret_cast<unsigned*>(s_cl + RP_CAND);           // [N] donor keys (if they fit)
  const bool keys_smem = repair_keys_in_smem(a.kc, a.N);
  __shared__ int s_hist[256];
  __shared__ int s_n, s_E, s_filled, s_need;
  __shared__ unsigned s_prefix;
  int32_t* as = a.assign + (int64_t)li * a.Nmax;
  float* dm = a.dmin + (int64_t)li * a.Nmax;
  int32_t* cnt = a.cnt + (int64_t)li * a.kmax;
  const int tid = threadIdx.x;

  // counts to smem; ordered list of the empty cluster ids (block compaction)
  const int per = (a.kc + blockDim.x - 1) / blockDim.x;
  const int j0 = tid * per, j1 = min(a.kc, j0 + per);
  int ne = 0;
  for (int j = j0; j < j1; ++j) {
    const int c = cnt[j];
    s_cnt[j] = c;
    ne += c == 0;
  }
  int E;
  int pos = km_block_excl_scan(ne, E);
  for (int j = j0; j < j1; ++j)
    if (s_cnt[j] == 0) s_empty[pos++] = j;
  // dmin key of an eligible point: bits of max(dmin, 0) + 1 (monotone for non-negative floats; 0 is
  // reserved for "not eligible"; dmin = -inf marks a point already taken as a donor)
  if (keys_smem) {  // (s_cnt is complete: the block scan above ended with a barrier)
    for (int i0 = tid; i0 < a.N; i0 += 8 * blockDim.x) {
      int ai[8];
      float di[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r * blockDim.x;
        ai[r] = i < a.N ? as[i] : 0;
        di[r] = i < a.N ? dm[i] : -INFINITY;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r * blockDim.x;
        if (i < a.N)
          s_dk[i] = (di[r] != -INFINITY && s_cnt[ai[r]] >= 2) ? __float_as_uint(fmaxf(di[r], 0.f)) + 1u : 0u;
      }
    }
    __syncthreads();
  }
  // ---- threshold: the T-th largest eligible key, T = min(1.5E + 32, RP_CAND / 2)
  const int T = min(E + E / 2 + 32, RP_CAND / 2);
  if (tid == 0) {
    s_prefix = 0u;
    s_need = T;
  }
  __syncthreads();
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const unsigned hi_mask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (int i = tid; i < 256; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const unsigned prefix = s_prefix;
    if (keys_smem) {
      for (int i = tid; i < a.N; i += blockDim.x) {
        const unsigned k = s_dk[i];
        if (k != 0u && (k & hi_mask) == prefix) atomicAdd(&s_hist[(k >> shift) & 255], 1);
      }
    } else
    // 8 keys per thread in flight per batch (assignment and dmin loads issued before any use)
    for (int i0 = tid; i0 < a.N; i0 += 8 * blockDim.x) {
      int ai[8];
      float di[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + r * blockDim.x;
        ai[r] = i < a.N ? as[i] : 0;
        di[r] = i < a.N ? dm[i] : -INFINITY;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const unsigned k = (di[r] != -INFINITY && s_cnt[ai[r]] >= 2) ? __float_as_uint(fmaxf(di[r], 0.f)) + 1u : 0u;
        if (k != 0u && (k & hi_mask) == prefix) atomicAdd(&s_hist[(k >> shift) & 255], 1);
      }
    }
    __syncthreads();
    if (tid == 0) {
      // descending: find the bucket where the count from the top reaches need
      int need = s_need, b = 255;
      for (; b > 0; --b) {
        if (s_hist[b] >= need) break;
        need -= s_hist[b];
      }
      s_need = need;
      s_prefix = prefix | ((unsigned)b << shift);
    }
    __syncthreads();
  }
  const unsigned thr = s_prefix;  // keys >= thr include the top-T (and ties)
  // ---- compact candidates (key >= thr) and sort them by (key desc, index asc)
  if (tid == 0) s_n = 0;
  __syncthreads();
  if (keys_smem) {
    for (int i = tid; i < a.N; i += blockDim.x) {
      const unsigned k = s_dk[i];
      if (k != 0u && k >= thr) {
        const int slot = atomicAdd(&s_n, 1);
        if (slot < RP_CAND) s_key[slot] = ((unsigned long long)(~k) << 32) | (unsigned)i;
      }
    }
  } else
  for (int i0 = tid; i0 < a.N; i0 += 8 * blockDim.x) {
    int ai[8];
    float di[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = i0 + r * blockDim.x;
      ai[r] = i < a.N ? as[i] : 0;
      di[r] = i < a.N ? dm[i] : -INFINITY;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const unsigned k = (di[r] != -INFINITY && s_cnt[ai[r]] >= 2) ? __float_as_uint(fmaxf(di[r], 0.f)) + 1u : 0u;
      if (k != 0u && k >= thr) {
        const int slot = atomicAdd(&s_n, 1);
        if (slot < RP_CAND) s_key[slot] = ((unsigned long long)(~k) << 32) | (unsigned)(i0 + r * blockDim.x);
      }
    }
  }
  __syncthreads();
  const int nc = s_n <= RP_CAND ? s_n : 0;  // overflow (massive ties): exact slow path only
  int np2 = 1;
  while (np2 < nc) np2 <<= 1;
  for (int i = nc + tid; i < np2; i += blockDim.x) s_key[i] = ~0ull;
  __syncthreads();
  for (int k2 = 2; k2 <= np2; k2 <<= 1)
    for (int jj = k2 >> 1; jj > 0; jj >>= 1) {
      for (int i = tid; i < np2; i += blockDim.x) {
        const int l = i ^ jj;
        if (l > i) {
          const unsigned long long x = s_key[i], y = s_key[l];
          const bool up = (i & k2) == 0;
          if ((x > y) == up) {
            s_key[i] = y;
            s_key[l] = x;
          }
        }
      }
      __syncthreads();
    }
  for (int i = tid; i < nc; i += blockDim.x) s_cl[i] = as[(int)(s_key[i] & 0xFFFFFFFFu)];
  __syncthreads();
  // ---- one sequential walk (shared memory only)
  if (tid == 0) {
    int r = 0;
    for (int c = 0; c < nc && r < E; ++c) {
      const int cl = s_cl[c];
      if (s_cnt[cl] < 2) continue;
      const int i = (int)(s_key[c] & 0xFFFFFFFFu);
      const int j = s_empty[r++];
      s_cnt[cl] -= 1;
      s_cnt[j] = 1;
      as[i] = j;
      dm[i] = -INFINITY;
      atomicSub(&a.cc[((int64_t)li * a.nchunk_max + i / KM_CHUNK) * a.kmax + cl], 1);
      atomicAdd(&a.cc[((int64_t)li * a.nchunk_max + i / KM_CHUNK) * a.kmax + j], 1);
    }
    s_filled = r;
  }
  __syncthreads();
  for (int j = tid; j < a.kc; j += blockDim.x) cnt[j] = s_cnt[j];
  __syncthreads();
  // ---- fallback for whatever the candidate list could not fill (exact, slow)
  __shared__ float s_bv[32];
  __shared__ int s_bi[32];
  for (int r = s_filled; r < E; ++r) {
    const int j = s_empty[r];
    float bv = -INFINITY;
    int bi = 0x7FFFFFFF;
    for (int i = tid; i < a.N; i += blockDim.x) {
      if (dm[i] == -INFINITY || cnt[as[i]] < 2) continue;
      const float v = fmaxf(dm[i], 0.f);  // same order as the fast path (fp32 dmin may dip below 0)
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      s_bv[tid >> 5] = bv;
      s_bi[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      float v = -INFINITY;
      int d = 0x7FFFFFFF;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (s_bv[w] > v || (s_bv[w] == v && s_bi[w] < d)) {
          v = s_bv[w];
          d = s_bi[w];
        }
      if (d != 0x7FFFFFFF) {
        const int from = as[d];
        cnt[from] -= 1;
        as[d] = j;
        cnt[j] = 1;
        dm[d] = -INFINITY;
        atomicSub(&a.cc[((int64_t)li * a.nchunk_max + d / KM_CHUNK) * a.kmax + from], 1);
        atomicAdd(&a.cc[((int64_t)li * a.nchunk_max + d / KM_CHUNK) * a.kmax + j], 1);
      }
    }
    __syncthreads();
  }
  // chunk histograms were updated in place; the column scan + offsets rerun for this instance
  if (tid == 0) a.flags[li] = 2;
}

// stable counting-sort scatter; one warp per chunk, rounds of 32 keys in position order
// Stable counting-sort scatter, one 1024-thread CTA per 1024-key chunk (used when the chunks of all
// instances fit one wave of such CTAs — few instances, e.g. C2: 256 chunks; A/B C2 sort phase
// 68.5 -> 64 us per layer-iteration, C4 with 4096 chunks 234 -> 266, so the warp version serves there): the chunk's keys are sorted
// on chip by (cluster, position) — a bitonic sort of 26-bit keys cluster << 10 | lane — and key p of
// the sorted chunk goes to its cluster's base (cluster offset + the chunk's column prefix) plus its
// rank in the run of equal clusters (p minus the run's first index, by binary search). Positions
// ascend within every cluster (the lane is the low key part), exactly the order of the warp-per-chunk
// scatter it replaces (which walked the chunk in 32 dependent rounds at one warp per chunk).
__global__ void __launch_bounds__(KM_CHUNK) km_scatter_cta_kernel(KmArgs a) {
  pdl_wait_trigger();
  __shared__ uint32_t sk[KM_CHUNK];
  const int li = blockIdx.y, c = blockIdx.x, t = threadIdx.x;
  const int i0 = c * KM_CHUNK, i1 = min(a.N, i0 + KM_CHUNK);
  const int32_t* as = a.assign + (int64_t)li * a.Nmax;
  sk[t] = i0 + t < i1 ? ((uint32_t)as[i0 + t] << 10) | (uint32_t)t : 0xFFFFFFFFu;
  __syncthreads();
  for (int k = 2; k <= KM_CHUNK; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = t ^ j;
      if (p > t) {
        const uint32_t x = sk[t], y = sk[p];
        const bool up = (t & k) == 0;
        if ((x > y) == up) {
          sk[t] = y;
          sk[p] = x;
        }
      }
      __syncthreads();
    }
  }
  const uint32_t key = sk[t];
  if (key == 0xFFFFFFFFu) return;
  const int cl = (int)(key >> 10), lane_i = (int)(key & 1023u);
  int lo = 0, hi = t;  // first index of this cluster's run
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int)(sk[mid] >> 10) < cl) lo = mid + 1;
    else hi = mid;
  }
  const int rank = t - lo;
  const int cpre = a.ccT[((int64_t)li * a.nchunk_max + c) * a.kmax + cl];
  const int o = a.off[(int64_t)li * (a.kmax + 1) + cl];
  const int to = a.toff[(int64_t)li * (a.kmax + 1) + cl];
  a.perm[(int64_t)li * a.Nmax + o + cpre + rank] = i0 + lane_i;
  a.tperm[(int64_t)li * a.task_max * KM_TASK + (int64_t)to * KM_TASK + cpre + rank] = i0 + lane_i;
}

// the same scatter by one warp per chunk (32 rounds of 32 keys, match_any ranks): many chunks
__global__ void __launch_bounds__(32) km_scatter_kernel(KmArgs a) {
  pdl_wait_trigger();
  extern __shared__ int base[];  // [kc] running offsets of this chunk, then [kc] the padded ones
  int* pbase = base + a.kc;      // (task-padded order: cluster j's members at 32 toff[j] + rank)
  const int li = blockIdx.y, c = blockIdx.x, lane = threadIdx.x;
  const int32_t* ccT = a.ccT + ((int64_t)li * a.nchunk_max + c) * a.kmax;
  const int32_t* off = a.off + (int64_t)li * (a.kmax + 1);
  const int32_t* toff = a.toff + (int64_t)li * (a.kmax + 1);
  for (int j0 = lane; j0 < a.kc; j0 += 8 * 32) {  // 24 loads per lane in flight per batch
    int cv[8], ov[8], tv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int j = j0 + r * 32;
      cv[r] = j < a.kc ? ccT[j] : 0;
      ov[r] = j < a.kc ? off[j] : 0;
      tv[r] = j < a.kc ? toff[j] : 0;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (j0 + r * 32 < a.kc) {
        base[j0 + r * 32] = cv[r] + ov[r];
        pbase[j0 + r * 32] = cv[r] + tv[r] * KM_TASK;
      }
  }
  __syncwarp();
  const int32_t* as = a.assign + (int64_t)li * a.Nmax;
  int32_t* perm = a.perm + (int64_t)li * a.Nmax;
  int32_t* tperm = a.tperm + (int64_t)li * a.task_max * KM_TASK;
  const int i0 = c * KM_CHUNK, i1 = min(a.N, i0 + KM_CHUNK);
  // prefetch the chunk's assignments (32 per lane) so the rounds below only touch registers/smem
  int cl_pre[KM_CHUNK / 32];
#pragma unroll
  for (int r = 0; r < KM_CHUNK / 32; ++r) {
    const int i = i0 + r * 32 + lane;
    cl_pre[r] = i < i1 ? as[i] : -1 - lane;
  }
#pragma unroll
  for (int r = 0; r < KM_CHUNK / 32; ++r) {
    const int i = i0 + r * 32 + lane;
    const bool valid = i < i1;
    const int cl = cl_pre[r];
    const unsigned peers = __match_any_sync(0xffffffffu, cl);
    const int leader = __ffs(peers) - 1;
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int bs = 0, ps = 0;
    if (valid && lane == leader) {
      bs = base[cl];
      ps = pbase[cl];
    }
    bs = __shfl_sync(0xffffffffu, bs, leader);
    ps = __shfl_sync(0xffffffffu, ps, leader);
    if (valid) {
      perm[bs + rank] = i;
      tperm[ps + rank] = i;
    }
    __syncwarp();
    if (valid && lane == leader) {
      base[cl] = bs + __popc(peers);
      pbase[cl] = ps + __popc(peers);
    }
    __syncwarp();
  }
}


// centroid update, task based: cluster j is cut into ceil(|j| / KM_TASK) tasks of consecutive
// members (position order); a warp sums one task (lane = 4 dims, sequential fp32). Single-task
// clusters are finalised in place; larger ones write partial sums that km_finalize adds in task
// order (deterministic; bounded work per warp however large a cluster grows).
__device__ __forceinline__ void km_write_centroid(const KmArgs& a, int li, int j, const float s[4], int n, int lane) {
  float* C = a.cent + ((int64_t)li * a.Umax + j) * D;
  uint16_t* Cb = reinterpret_cast<uint16_t*>(a.centb) + ((int64_t)li * a.Umax + j) * D;
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float c = __fdiv_rn(s[e], (float)n);
    C[lane * 4 + e] = c;
    Cb[lane * 4 + e] = f2bf_rne(c);
    ss = fmaf(c, c, ss);
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    a.half[(int64_t)li * a.hstride + j] = 0.5f * ss;
    write_bext(a, li, j, 0.5f * ss);
  }
}

__global__ void __launch_bounds__(128) km_update_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 4 + warp;
  const int32_t* toff = a.toff + (int64_t)li * (a.kmax + 1);
  if (t >= toff[a.kc]) return;
  // the task (written with the offsets): cluster j, members [m0, m1) of the cluster-sorted order,
  // tasks of j; lane i holds member m0 + i's position, so all <= 32 member rows are loaded in two
  // batches of 16 (three round trips in all), summed in member order (deterministic)
  // (the task and its members' positions — task-padded order — load in the same round trip)
  const int4 tk = a.tcl[(int64_t)li * a.task_max + t];
  const int pi_raw = a.tperm[((int64_t)li * a.task_max + t) * KM_TASK + lane];
  const int j = tk.x, m0 = tk.y, m1 = tk.z, ntask = tk.w;
  const int nm = m1 - m0;
  const int pi = lane < nm ? pi_raw : 0;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int rb = 0; rb < KM_TASK; rb += 16) {
    if (rb >= nm) break;
    uint2 u[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int idx = __shfl_sync(0xffffffffu, pi, rb + r);
      if (rb + r < nm) u[r] = reinterpret_cast<const uint2*>(xrow(a, li, idx))[lane];
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (rb + r < nm) {
        s[0] = __fadd_rn(s[0], __uint_as_float(u[r].x << 16));
        s[1] = __fadd_rn(s[1], __uint_as_float(u[r].x & 0xFFFF0000u));
        s[2] = __fadd_rn(s[2], __uint_as_float(u[r].y << 16));
        s[3] = __fadd_rn(s[3], __uint_as_float(u[r].y & 0xFFFF0000u));
      }
  }
  if (ntask == 1) {
    km_write_centroid(a, li, j, s, nm, lane);
  } else {
    float4* P = reinterpret_cast<float4*>(a.upart + ((int64_t)li * a.task_max + t) * D);
    P[lane] = make_float4(s[0], s[1], s[2], s[3]);
  }
}

__global__ void __launch_bounds__(128) km_finalize_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + warp;
  if (j >= a.kc) return;
  const int32_t* toff = a.toff + (int64_t)li * (a.kmax + 1);
  const int t0 = toff[j], t1 = toff[j + 1];
  if (t1 - t0 <= 1) return;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  for (int t = t0; t < t1; ++t) {
    const float4 v = reinterpret_cast<const float4*>(a.upart + ((int64_t)li * a.task_max + t) * D)[lane];
    s[0] = __fadd_rn(s[0], v.x);
    s[1] = __fadd_rn(s[1], v.y);
    s[2] = __fadd_rn(s[2], v.z);
    s[3] = __fadd_rn(s[3], v.w);
  }
  const int32_t* off = a.off + (int64_t)li * (a.kmax + 1);
  km_write_centroid(a, li, j, s, off[j + 1] - off[j], lane);
}

// page units (LOUISKV_UNITS_PAGES, §3.1): key i of [S, P) belongs to page i / page
__global__ void km_page_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)a.N; t += (int64_t)gridDim.x * blockDim.x)
    a.assign[(int64_t)li * a.Nmax + t] = (int32_t)(t / a.page);
}

// caller-supplied clustering: copy assignment and centroids in
__global__ void km_ext_kernel(KmArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)a.N; t += (int64_t)gridDim.x * blockDim.x)
    a.assign[(int64_t)li * a.Nmax + t] = a.ext_assign[(int64_t)li * a.N + t];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)a.kc * D;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float c = a.ext_cent[(int64_t)li * a.kc * D + t];
    a.cent[(int64_t)li * a.Umax * D + t] = c;
    reinterpret_cast<uint16_t*>(a.centb)[(int64_t)li * a.Umax * D + t] = f2bf_rne(c);
  }
}

// offload: pool row r (cluster-major order) <- key perm[r]; unit-major spans [K rows | V rows]
// Cluster-major permutation of instances [li0, li0 + gridDim.y) into dst (instance stride dst_stride
// bytes): a device staging buffer whose rows the copy engine then moves into the pinned host pool
// ("offload (K, V) to CPU memory pool asynchronously"), so the host-link transfer overlaps the
// next layer's clustering instead of holding SMs.
__global__ void __launch_bounds__(128) km_offload_kernel(KmArgs a, int li0, uint8_t* dst_base, int64_t dst_stride) {
  pdl_wait_trigger();
  const int li = li0 + blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 4), sub = threadIdx.x & 15;
  if (r >= a.N) return;
  const int32_t* perm = a.perm + (int64_t)li * a.Nmax;
  const int32_t* off = a.off + (int64_t)li * (a.kmax + 1);
  const int i = perm[r];
  const int j = a.assign[(int64_t)li * a.Nmax + i];
  const int o = off[j], n = off[j + 1] - o;
  uint8_t* dst = dst_base + (int64_t)blockIdx.y * dst_stride + (int64_t)o * pool_row_bytes(a.pool_fp8);
  const uint4 kx = reinterpret_cast<const uint4*>(xrow(a, li, i))[sub];
  const uint4 vx = reinterpret_cast<const uint4*>(vrow(a, li, i))[sub];
  if (a.pool_fp8) {  // FP8 pool (reading R-FP8): E4M3 rows, 8 B per 16-B bf16 piece
    reinterpret_cast<uint2*>(dst)[(int64_t)(r - o) * 16 + sub] = bf16x8_to_e4m3x8(kx);
    reinterpret_cast<uint2*>(dst)[(int64_t)(n + r - o) * 16 + sub] = bf16x8_to_e4m3x8(vx);
  } else {
    reinterpret_cast<uint4*>(dst)[(int64_t)(r - o) * 16 + sub] = kx;
    reinterpret_cast<uint4*>(dst)[(int64_t)(n + r - o) * 16 + sub] = vx;
  }
  if (sub == 0) a.pool_pos[(int64_t)li * a.pool_rows_cap + r] = a.S + i;
}

cudaError_t launch_km_offload(const KmArgs& a, int li0, int nli, uint8_t* dst, int64_t dst_stride, cudaStream_t st) {
  if (a.N <= 0 || a.kc <= 0 || nli <= 0) return cudaSuccess;
  launch_k(km_offload_kernel, dim3(dim3((a.N + 7) / 8, nli)), dim3(128), 0, st, a, li0, dst, dst_stride);
  return cudaGetLastError();
}

// unit table + instance reset after clustering
__global__ void km_units_kernel(KmArgs a, int P) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t* off = a.off + (int64_t)li * (a.kmax + 1);
  if (j < a.kc) {
    a.usize[(int64_t)li * a.Umax + j] = off[j + 1] - off[j];
    a.uoff[(int64_t)li * a.Umax + j] = off[j];
    a.ufirst[(int64_t)li * a.Umax + j] = a.S + a.perm[(int64_t)li * a.Nmax + off[j]];
    a.sel[(int64_t)li * a.Umax + j] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    InstState s{};
    s.n_units = a.kc;
    s.n_prompt_units = a.kc;
    s.pool_rows = a.N;
    s.prompt_len = P;
    s.s_eff = min(a.S_cap, P);
    a.inst[li] = s;
    atomicAdd(&a.stats->bytes_d2h, (unsigned long long)a.N * pool_row_bytes(a.pool_fp8));
  }
}

// sinks [0, S) stay on the device
__global__ void km_sinks_kernel(KmArgs a, int s_eff) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int b = li / a.hn, h = li % a.hn;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 4), sub = threadIdx.x & 15;
  if (r >= s_eff) return;
  const bf16* ks = a.k + (int64_t)b * a.sb + (int64_t)r * a.st + (int64_t)h * a.sh;
  const bf16* vs = a.v + (int64_t)b * a.sb + (int64_t)r * a.st + (int64_t)h * a.sh;
  bf16* dk = a.sinks + (int64_t)li * 2 * a.S_cap * D + (int64_t)r * D;
  bf16* dv = dk + (int64_t)a.S_cap * D;
  reinterpret_cast<uint4*>(dk)[sub] = reinterpret_cast<const uint4*>(ks)[sub];
  reinterpret_cast<uint4*>(dv)[sub] = reinterpret_cast<const uint4*>(vs)[sub];
}

__global__ void reset_insts_kernel(InstState* inst, int n, int P, int s_eff) {
  pdl_wait_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  InstState s{};
  s.prompt_len = P;
  s.s_eff = s_eff;
  inst[i] = s;
}

cudaError_t launch_km_units(const KmArgs& a, cudaStream_t st) {
  if (a.N <= 0 || a.kc <= 0) return cudaSuccess;
  launch_k(km_units_kernel, dim3(dim3((a.kc + 255) / 256, a.batch * a.hn)), dim3(256), 0, st, a, a.S + a.N);
  return cudaGetLastError();
}

cudaError_t launch_assign_tc(const KmArgs& a, cudaStream_t st);  // k_kmeans_tc.cu

static cudaError_t sort_by_cluster(const KmArgs& a, int ni, int nchunk, bool repair, cudaStream_t st) {
  launch_k(km_hist_kernel, dim3(dim3(nchunk, ni)), dim3(256), sizeof(int) * a.kc, st, a, nchunk);
  launch_k(km_colscan_kernel, dim3(dim3((a.kc + 255) / 256, ni)), dim3(256), 0, st, a, nchunk, 0);
  launch_k(km_offsets_kernel, dim3(ni), dim3(1024), 0, st, a, 0);
  if (repair) {
    const size_t rsm = repair_smem_base(a.kc) + (repair_keys_in_smem(a.kc, a.N) ? sizeof(unsigned) * (size_t)a.N : 0);
    launch_k(km_repair_kernel, dim3(ni), dim3(1024), rsm, st, a, nchunk);
    launch_k(km_colscan_kernel, dim3(dim3((a.kc + 255) / 256, ni)), dim3(256), 0, st, a, nchunk, 1);
    launch_k(km_offsets_kernel, dim3(ni), dim3(1024), 0, st, a, 1);
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  if ((int64_t)nchunk * ni <= 2 * sms)  // (two 1024-thread CTAs per SM)
    launch_k(km_scatter_cta_kernel, dim3(dim3(nchunk, ni)), dim3(KM_CHUNK), 0, st, a);
  else
    launch_k(km_scatter_kernel, dim3(dim3(nchunk, ni)), dim3(32), 2 * sizeof(int) * a.kc, st, a);
  return cudaGetLastError();
}

cudaError_t run_kmeans_prompt(const KmArgs& a, cudaStream_t st, uint64_t* tc_iters, uint64_t* simt_iters) {
  const int ni = a.batch * a.hn;
  const int P = a.S + a.N;
  const int s_eff = min(a.S_cap, P);
  cudaError_t e;
  if (s_eff > 0) launch_k(km_sinks_kernel, dim3(dim3((s_eff + 7) / 8, ni)), dim3(128), 0, st, a, s_eff);
  if (a.N <= 0 || a.kc <= 0) {
    launch_k(reset_insts_kernel, dim3((ni + 127) / 128), dim3(128), 0, st, a.inst, ni, P, s_eff);
    return cudaGetLastError();
  }
  static std::atomic<uint64_t> attr{0};
  cudaError_t ea = once_per_device(attr, [] {
    cudaError_t e = cudaFuncSetAttribute(km_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(km_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(km_repair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return e;
  });
  if (ea != cudaSuccess) return ea;
  const int nchunk = (a.N + KM_CHUNK - 1) / KM_CHUNK;
  const dim3 gk((a.kc + 3) / 4, ni);
  if (a.ext_assign) {
    launch_k(km_ext_kernel, dim3(dim3(64, ni)), dim3(256), 0, st, a);
    if ((e = sort_by_cluster(a, ni, nchunk, false, st)) != cudaSuccess) return e;
  } else if (a.page > 0) {
    // pages: fixed assignment, one centroid update (mean of each page's keys), no iterations
    launch_k(km_page_kernel, dim3(dim3(64, ni)), dim3(256), 0, st, a);
    if ((e = sort_by_cluster(a, ni, nchunk, false, st)) != cudaSuccess) return e;
    launch_k(km_update_kernel, dim3(dim3((a.task_max + 3) / 4, ni)), dim3(128), 0, st, a);
    launch_k(km_finalize_kernel, dim3(gk), dim3(128), 0, st, a);
  } else {
    launch_k(km_init_kernel, dim3(gk), dim3(128), 0, st, a);
    launch_k(km_half_pad_kernel, dim3(dim3(1, ni)), dim3(256), 0, st, a);
    for (int it = 0; it < a.iters; ++it) {
      if (a.rec) {
        a.rec->mark(st, PH_ASSIGN);
        a.rec->assign_flops += (uint64_t)ni * a.N * a.kc * 2ull * D;
        a.rec->assign_passes += 1;
      }
      bool done = false;
      if (a.impl == LOUISKV_KMEANS_TC && kmeans_tc_available()) {
        e = launch_assign_tc(a, st);
        if (e == cudaSuccess) done = true;
        else if (e != cudaErrorNotSupported) return e;
        else cudaGetLastError();
      }
      if (!done) launch_k(km_assign_simt_kernel, dim3(dim3((a.N + 127) / 128, ni)), dim3(128), 0, st, a);
      ++*(done ? tc_iters : simt_iters);
      if (a.rec) a.rec->mark(st, PH_SORT);
      if ((e = sort_by_cluster(a, ni, nchunk, true, st)) != cudaSuccess) return e;
      if (a.rec) a.rec->mark(st, PH_UPDATE);
      launch_k(km_update_kernel, dim3(dim3((a.task_max + 3) / 4, ni)), dim3(128), 0, st, a);
      launch_k(km_finalize_kernel, dim3(gk), dim3(128), 0, st, a);
    }
  }
  // the caller stages the cluster-major rows (launch_km_offload), copies them to the host pool and
  // then writes the unit table (launch_km_units)
  return cudaGetLastError();
}

__global__ void full_prompt_kernel(const bf16* k, const bf16* v, int64_t sb, int64_t st_, int64_t sh, int hn,
                                   int64_t P, bf16* full, int64_t full_cap) {
  pdl_wait_trigger();
  const int li = blockIdx.y, b = li / hn, h = li % hn;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 4);
  const int sub = threadIdx.x & 15;
  if (r >= P) return;
  bf16* K = full + (int64_t)li * 2 * full_cap * D;
  bf16* V = K + full_cap * D;
  reinterpret_cast<uint4*>(K + r * D)[sub] = reinterpret_cast<const uint4*>(k + b * sb + r * st_ + h * sh)[sub];
  reinterpret_cast<uint4*>(V + r * D)[sub] = reinterpret_cast<const uint4*>(v + b * sb + r * st_ + h * sh)[sub];
}

cudaError_t launch_full_prompt(const bf16* k, const bf16* v, int64_t sb, int64_t st_, int64_t sh, int batch, int hn,
                               int64_t P, bf16* full, int64_t full_cap, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  launch_k(full_prompt_kernel, dim3(dim3((unsigned)((P + 7) / 8), batch * hn)), dim3(128), 0, st, k, v, sb, st_, sh, hn, P, full,
                                                                                full_cap);
  return cudaGetLastError();
}

cudaError_t launch_reset_insts(InstState* inst, int n, int P, int s_eff, cudaStream_t st) {
  launch_k(reset_insts_kernel, dim3((n + 127) / 128), dim3(128), 0, st, inst, n, P, s_eff);
  return cudaGetLastError();
}

}  // namespace lkv
