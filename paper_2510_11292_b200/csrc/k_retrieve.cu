// kvm.Retrieve(q_t, B) — P:279-285 [Alg. 1], App. B P:243-247 [group-consistent scores],
// §4.3 P:126 [batched budgeted selection kernel, row-granular CPU->GPU transfer].
//
// score_select_kernel: one CTA per flagged (b, owned kv-head) instance.
//   1. logits l_{j,u} = fl32(fmaf-chain_e(q_j,e * c_u,e)) * fl32(1/sqrt(d))    (recipe R2)
//   2. m_j = max_u l_{j,u}; e_{j,u} = exp_R3(l - m_j); Z_j from the exact fixed-point sum
//      Σ_u floor(e * 2^40) (order independent, so the parallel reduction is bit-exact)
//   3. A_u = (Σ_j e_{j,u} / Z_j) / g ; key_u = (~bits(A_u) << 16) | u  (A desc, id asc)
//   4. budgeted selection = greedy skip-and-continue in key order, computed as rounds of a
//      size-weighted radix select: find the pivot (first unit whose inclusion would exceed
//      the remaining budget) with 6 passes of 8-bit digits; every candidate below it is taken;
//      the pivot is skipped; the next round only considers later units that still fit.
//      Proof of equivalence: units bigger than the remaining budget are skipped by the greedy
//      anyway and the remaining budget never grows.
//   5. new working-set layout (selected units in id order, prefix sums of sizes), diff with
//      the previous selection: kept units copy device->device, new units read from the pinned
//      host pool; one RowSrc per destination row for the gather kernel.
// gather_kernel: copies the rows (256 B K + 256 B V) with 16-B vector loads; host rows are
//   read zero-copy over the host link ("directly transfer specific rows").
#include "lkv_internal.cuh"

namespace lkv {

constexpr int SS_THREADS = 512;
constexpr int MAX_G = 16;

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

__global__ void __launch_bounds__(SS_THREADS) score_select_kernel(RetrieveArgs a) {
  const int li = blockIdx.x;  // local instance = b*hn + h
  const int b = li / a.hn, h = li % a.hn;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = SS_THREADS / 32;
  if (!a.flag[b]) {
    if (tid == 0) a.jobs[li].n_rows = 0;
    return;
  }
  InstState* S = a.inst + li;
  const int n = S->n_units;
  const int g = a.g;

  __shared__ float sq[MAX_G][D];
  __shared__ float s_coef[7];
  __shared__ float s_red[NW][MAX_G];
  __shared__ float s_m[MAX_G];
  __shared__ unsigned long long s_z[MAX_G];
  __shared__ float s_Z[MAX_G];
  __shared__ int s_hist[256];
  __shared__ long long s_red64[NW];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_need;
  __shared__ int s_scan[SS_THREADS];
  extern __shared__ uint32_t s_taken[];  // bitmap [ceil(Umax/32)]

  // recipe constants (identical IEEE double evaluation on both sides)
  if (tid == 0) {
    double p = 1.0, fact = 1.0;
    const double ln2 = 0.6931471805599453094;
    for (int i = 0; i <= 6; ++i) {
      if (i > 0) {
        p = __dmul_rn(p, ln2);
        fact = __dmul_rn(fact, (double)i);
      }
      s_coef[i] = __double2float_rn(__ddiv_rn(p, fact));
    }
  }
  const uint16_t* qb = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b + (int64_t)h * g * D;
  for (int i = tid; i < g * D; i += SS_THREADS) sq[i / D][i % D] = bf2f(qb[i]);
  for (int i = tid; i < (a.Umax + 31) / 32; i += SS_THREADS) s_taken[i] = 0u;
  if (tid < MAX_G) s_z[tid] = 0ull;
  __syncthreads();

  const float inv_sqrt_d = __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn((double)D)));
  float* E = a.scratch_e + (int64_t)li * g * a.Umax;
  unsigned long long* KEY = a.scratch_key + (int64_t)li * a.Umax;
  const uint4* C = reinterpret_cast<const uint4*>(a.centb + (int64_t)li * a.Umax * D);
  const int32_t* usize = a.usize + (int64_t)li * a.Umax;

  // ---- 1. logits + per-head max
  float mymax[MAX_G];
#pragma unroll
  for (int j = 0; j < MAX_G; ++j) mymax[j] = -INFINITY;
  for (int u = tid; u < n; u += SS_THREADS) {
    float acc[MAX_G];
#pragma unroll
    for (int j = 0; j < MAX_G; ++j) acc[j] = 0.0f;
    const uint4* row = C + (int64_t)u * (D / 8);
#pragma unroll 2
    for (int c8 = 0; c8 < D / 8; ++c8) {
      float cf[8];
      unpack8(__ldg(row + c8), cf);
#pragma unroll
      for (int j = 0; j < MAX_G; ++j) {
        if (j < g) {
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[j] = __fmaf_rn(sq[j][c8 * 8 + k], cf[k], acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < MAX_G; ++j) {
      if (j < g) {
        float l = __fmul_rn(acc[j], inv_sqrt_d);
        E[(int64_t)j * a.Umax + u] = l;
        mymax[j] = fmaxf(mymax[j], l);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAX_G; ++j) {
    if (j < g) {
      float m = mymax[j];
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) s_red[warp][j] = m;
    }
  }
  __syncthreads();
  if (tid < g) {
    float m = -INFINITY;
    for (int w = 0; w < NW; ++w) m = fmaxf(m, s_red[w][tid]);
    s_m[tid] = m;
  }
  __syncthreads();

  // ---- 2. exp + exact fixed-point normaliser
  unsigned long long zl[MAX_G];
#pragma unroll
  for (int j = 0; j < MAX_G; ++j) zl[j] = 0ull;
  for (int u = tid; u < n; u += SS_THREADS) {
#pragma unroll
    for (int j = 0; j < MAX_G; ++j) {
      if (j < g) {
        float e = exp_r3(__fsub_rn(E[(int64_t)j * a.Umax + u], s_m[j]), s_coef);
        E[(int64_t)j * a.Umax + u] = e;
        zl[j] += __float2ull_rz(__fmul_rn(e, 1099511627776.0f));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAX_G; ++j) {
    if (j < g) {
      unsigned long long z = zl[j];
      for (int o = 16; o; o >>= 1) z += shfl_xor_u64(z, o);
      if (lane == 0) atomicAdd(&s_z[j], z);
    }
  }
  __syncthreads();
  if (tid < g) s_Z[tid] = __fmul_rn(__ull2float_rn(s_z[tid]), __int_as_float((127 - 40) << 23));
  __syncthreads();

  // ---- 3. group score and sort key
  for (int u = tid; u < n; u += SS_THREADS) {
    float A = 0.0f;
    for (int j = 0; j < g; ++j) A = __fadd_rn(A, __fdiv_rn(E[(int64_t)j * a.Umax + u], s_Z[j]));
    A = __fdiv_rn(A, (float)g);
    unsigned long long key = ((unsigned long long)(~__float_as_uint(A)) << 16) | (unsigned)u;
    KEY[u] = key;
  }
  __syncthreads();

  // ---- 4. budgeted greedy selection via weighted radix-select rounds
  int rem = a.budget;
  bool lo_valid = false;
  unsigned long long lo = 0ull;
  while (rem > 0 && n > 0) {
    // total candidate weight
    long long tot = 0;
    for (int u = tid; u < n; u += SS_THREADS) {
      unsigned long long k = KEY[u];
      int sz = usize[u];
      if ((!lo_valid || k > lo) && sz <= rem) tot += sz;
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) s_red64[warp] = tot;
    __syncthreads();
    if (tid == 0) {
      long long t2 = 0;
      for (int w = 0; w < NW; ++w) t2 += s_red64[w];
      s_red64[0] = t2;
    }
    __syncthreads();
    tot = s_red64[0];
    __syncthreads();
    if (tot <= rem) {
      for (int u = tid; u < n; u += SS_THREADS) {
        unsigned long long k = KEY[u];
        if ((!lo_valid || k > lo) && usize[u] <= rem) atomicOr(&s_taken[u >> 5], 1u << (u & 31));
      }
      __syncthreads();
      break;
    }
    if (tid == 0) {
      s_prefix = 0ull;
      s_need = rem;
    }
    __syncthreads();
    for (int pass = 0; pass < 6; ++pass) {
      const int shift = 40 - 8 * pass;
      const unsigned long long hi_mask = (pass == 0) ? 0ull : (~0ull << (shift + 8)) & 0xFFFFFFFFFFFFull;
      for (int i = tid; i < 256; i += SS_THREADS) s_hist[i] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix;
      for (int u = tid; u < n; u += SS_THREADS) {
        unsigned long long k = KEY[u];
        int sz = usize[u];
        if ((!lo_valid || k > lo) && sz <= rem && (k & hi_mask) == prefix)
          atomicAdd(&s_hist[(k >> shift) & 255], sz);
      }
      __syncthreads();
      if (warp == 0) {
        // bucket with cumulative weight > need; lane handles 8 consecutive buckets
        int v[8], ls = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = s_hist[lane * 8 + i];
          ls += v[i];
        }
        int incl = ls;
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        int excl = incl - ls;
        const int need = s_need;
        unsigned hit = __ballot_sync(0xffffffffu, incl > need);
        int first = __ffs(hit) - 1;  // lane containing the bucket (always exists: tot > rem)
        if (lane == first) {
          int cum = excl, bk = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (cum + v[i] > need) {
              bk = i;
              break;
            }
            cum += v[i];
          }
          s_need = need - cum;
          s_prefix = prefix | ((unsigned long long)(lane * 8 + bk) << shift);
        }
      }
      __syncthreads();
    }
    const unsigned long long pivot = s_prefix;
    for (int u = tid; u < n; u += SS_THREADS) {
      unsigned long long k = KEY[u];
      if ((!lo_valid || k > lo) && usize[u] <= rem && k < pivot) atomicOr(&s_taken[u >> 5], 1u << (u & 31));
    }
    rem = s_need;
    lo = pivot;
    lo_valid = true;
    __syncthreads();
  }
  __syncthreads();

  // ---- 5. layout of the new working set (id order) + row sources
  const int per = (n + SS_THREADS - 1) / SS_THREADS;
  const int u0 = tid * per, u1 = min(n, u0 + per);
  int local = 0, local_cnt = 0;
  for (int u = u0; u < u1; ++u)
    if (s_taken[u >> 5] >> (u & 31) & 1u) {
      local += usize[u];
      ++local_cnt;
    }
  s_scan[tid] = local;
  __syncthreads();
  // Hillis-Steele inclusive scan
  for (int o = 1; o < SS_THREADS; o <<= 1) {
    int y = tid >= o ? s_scan[tid - o] : 0;
    __syncthreads();
    s_scan[tid] += y;
    __syncthreads();
  }
  const int total = s_scan[SS_THREADS - 1];
  int dst = s_scan[tid] - local;

  const int cur = S->ws_cur, nxt = cur ^ 1;
  const int64_t gi = a.inst_global_base + li;
  const bf16* curK = a.ws + cur * a.ws_buf_stride + gi * a.ws_inst_stride;
  const bf16* curV = curK + (int64_t)a.budget * D;
  bf16* nxtK = a.ws + nxt * a.ws_buf_stride + gi * a.ws_inst_stride;
  bf16* nxtV = nxtK + (int64_t)a.budget * D;
  const uint8_t* pool = a.pool + (int64_t)li * a.pool_inst_bytes;
  uint8_t* sel = a.sel + (int64_t)li * a.Umax;
  int32_t* seloff = a.seloff + (int64_t)li * a.Umax;
  const int64_t* uoff = a.uoff + (int64_t)li * a.Umax;
  RowSrc* rows = a.rows + (int64_t)li * a.budget;
  unsigned long long reused = 0, fetched = 0, hbytes = 0;
  for (int u = u0; u < u1; ++u) {
    const bool take = s_taken[u >> 5] >> (u & 31) & 1u;
    const bool had = sel[u] != 0;
    if (take) {
      const int sz = usize[u];
      if (had) {
        const int so = seloff[u];
        for (int i = 0; i < sz; ++i)
          rows[dst + i] = RowSrc{reinterpret_cast<const uint4*>(curK + (int64_t)(so + i) * D),
                                 reinterpret_cast<const uint4*>(curV + (int64_t)(so + i) * D)};
        ++reused;
      } else {
        const uint8_t* base = pool + uoff[u] * POOL_ROW_BYTES;
        for (int i = 0; i < sz; ++i)
          rows[dst + i] = RowSrc{reinterpret_cast<const uint4*>(base + (int64_t)i * ROW_BYTES),
                                 reinterpret_cast<const uint4*>(base + (int64_t)(sz + i) * ROW_BYTES)};
        ++fetched;
        hbytes += (unsigned long long)sz * POOL_ROW_BYTES;
      }
      sel[u] = 1;
      seloff[u] = dst;
      dst += sz;
    } else if (had) {
      sel[u] = 0;
    }
  }
  // stats (warp-aggregated)
  for (int o = 16; o; o >>= 1) {
    reused += __shfl_xor_sync(0xffffffffu, reused, o);
    fetched += __shfl_xor_sync(0xffffffffu, fetched, o);
    hbytes += __shfl_xor_sync(0xffffffffu, hbytes, o);
  }
  if (lane == 0 && (reused | fetched)) {
    atomicAdd(&a.stats->units_reused, reused);
    atomicAdd(&a.stats->units_fetched, fetched);
    atomicAdd(&a.stats->bytes_h2d, hbytes);
  }
  int cnt = local_cnt;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt) atomicAdd(&a.stats->units_selected, (unsigned long long)cnt);
  if (tid == 0) {
    atomicAdd(&a.stats->units_scored, (unsigned long long)n);
    if (h == 0) atomicAdd(&a.stats->retrievals, 1ull);
    a.jobs[li] = GatherJob{total, 0, nxtK, nxtV};
    S->ws_cur = nxt;
    S->ws_rows = total;
  }
}

constexpr int GA_THREADS = 256;
constexpr int GA_ROWS_PER_PASS = GA_THREADS / 16;

__global__ void __launch_bounds__(GA_THREADS) gather_kernel(const GatherJob* __restrict__ jobs,
                                                            const RowSrc* __restrict__ rows, int budget) {
  const int li = blockIdx.x;
  const GatherJob J = jobs[li];
  if (J.n_rows <= 0) return;
  const RowSrc* R = rows + (int64_t)li * budget;
  const int sub = threadIdx.x & 15;
  int r = blockIdx.y * GA_ROWS_PER_PASS + (threadIdx.x >> 4);
  const int stride = gridDim.y * GA_ROWS_PER_PASS;
  uint4* dK = reinterpret_cast<uint4*>(J.dstK);
  uint4* dV = reinterpret_cast<uint4*>(J.dstV);
  // two rows in flight per thread per iteration (4 x 16 B loads outstanding)
  for (; r < J.n_rows; r += 2 * stride) {
    const int r2 = r + stride;
    RowSrc s0 = R[r];
    uint4 k0 = s0.k[sub], v0 = s0.v[sub];
    uint4 k1, v1;
    if (r2 < J.n_rows) {
      RowSrc s1 = R[r2];
      k1 = s1.k[sub];
      v1 = s1.v[sub];
    }
    dK[(int64_t)r * (D / 8) + sub] = k0;
    dV[(int64_t)r * (D / 8) + sub] = v0;
    if (r2 < J.n_rows) {
      dK[(int64_t)r2 * (D / 8) + sub] = k1;
      dV[(int64_t)r2 * (D / 8) + sub] = v1;
    }
  }
}

cudaError_t launch_score_select(const RetrieveArgs& a, cudaStream_t st) {
  if (a.g > MAX_G) return cudaErrorInvalidValue;
  const size_t smem = sizeof(uint32_t) * ((a.Umax + 31) / 32);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(score_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_set = true;
  }
  score_select_kernel<<<a.batch * a.hn, SS_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gather(const GatherJob* jobs, const RowSrc* rows, int n_inst, int budget, cudaStream_t st) {
  const int gy = budget >= 64 ? budget / 64 : 1;
  gather_kernel<<<dim3(n_inst, gy), GA_THREADS, 0, st>>>(jobs, rows, budget);
  return cudaGetLastError();
}

}  // namespace lkv
