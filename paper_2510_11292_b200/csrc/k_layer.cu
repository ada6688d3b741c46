// One decode step of one retrieval layer in ONE clustered launch (Algorithm 1 P:301-312 in order:
// trigger -> [retrieve] -> store_cache -> attention), behind louiskv_decode_layer.
//
// One 8-CTA cluster per (b, owned kv-head) instance; every rank:
//   1. recomputes r_t of its sequence with recipe R1 (bit-identical on every rank, so the flag is
//      uniform across the cluster without an exchange); (rank 0, head 0) publishes flag / r / q_ref;
//   2. if flagged, scores and selects with the units split into 8 contiguous id ranges, one per rank:
//      logits (R2) -> cluster max -> exp (R3) + exact fixed-point Z (integer sums, so the cluster sum
//      is order independent) -> A_u and keys (A desc, id asc) -> the same size-weighted radix select
//      and per-take tail as the multi-kernel select, with the 256-bin histograms and the per-take
//      minima summed across ranks through distributed shared memory -> layout by a cluster prefix
//      over the ranks' row counts; the gather of the new working set is spread over the 8 ranks;
//   3. rank 0 appends (k_t, v_t) (seal / append / evict) and commits the instance's step;
//   4. split-K attention over sinks ∪ working set ∪ local buffer, one split per rank, DSMEM merge.
// Every decision is made in the arithmetic of the multi-kernel path (lkv_score_dev.cuh), so both
// paths match the oracle bit for bit on trigger decisions and selections. Every rank executes the
// same sequence of cluster barriers (all branches depend only on cluster-uniform values).
#include "lkv_append_dev.cuh"
#include "lkv_attn_dev.cuh"
#include "lkv_score_dev.cuh"

namespace lkv {

constexpr int LK_MCAP = LAYER_UNITS_MAX / AT_CL;  // units per rank held in shared memory
constexpr int LK_W = AT_THREADS / 32;

// block-wide exclusive scan (AT_THREADS threads)
__device__ __forceinline__ int lk_scan(int v, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < LK_W ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < LK_W) s_warp[lane] = wi - w;
    if (lane == LK_W - 1) s_warp[LK_W] = wi;
  }
  __syncthreads();
  const int r = s_warp[warp] + incl - v;
  total = s_warp[LK_W];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int clamp16(int sz) { return sz > 0xFFFF ? 0xFFFF : sz; }

// Distributed group-consistent scoring + budgeted greedy + working-set layout of instance li.
// Returns the row count of the new working set (identical on every rank); the row table of the
// gather is complete in global memory after the caller's next cluster barrier.
// SMB: this rank's logits / keys / sizes / taken bits live in the (idle) attention staging smem;
// else (more than LK_MCAP units per rank) in the instance's global scratch.
template <int G, bool SMB>
__device__ __forceinline__ int lk_select(const RetrieveArgs& a, const AppendArgs& app, const int li, const int rank,
                                         const int n, const int ws_cur, const float (*sq)[D], uint8_t* dsm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = (n + AT_CL - 1) / AT_CL;
  const int lo = min(n, rank * m), hi = min(n, lo + m), cnt = hi - lo;
  const int ES = SMB ? LK_MCAP : m;  // row stride of E
  float* E;                           // [G][ES]
  unsigned long long* KEYS;           // [ES]
  uint16_t* SZ;                       // [ES]
  uint32_t* TK;                       // [ceil(ES/32)]
  if constexpr (SMB) {
    E = reinterpret_cast<float*>(dsm);
    KEYS = reinterpret_cast<unsigned long long*>(E + G * LK_MCAP);
    SZ = reinterpret_cast<uint16_t*>(KEYS + LK_MCAP);
    TK = reinterpret_cast<uint32_t*>(SZ + LK_MCAP);
  } else {  // 8 ranks x m <= Umax + 7 rounded: within [G][Umax] floats and Umax * 26 bytes per instance
    E = a.scratch_e + (int64_t)li * G * a.Umax + (int64_t)rank * G * m;
    uint8_t* base = a.scratch_sort + (int64_t)li * a.Umax * 26;
    KEYS = reinterpret_cast<unsigned long long*>(base) + (int64_t)rank * m;
    SZ = reinterpret_cast<uint16_t*>(base + (int64_t)a.Umax * 8) + (int64_t)rank * m;
    TK = reinterpret_cast<uint32_t*>(base + (int64_t)a.Umax * 12) + (int64_t)rank * ((m + 31) / 32);
  }

  __shared__ float s_coef[7];
  __shared__ float x_max[G];               // exchanged through DSMEM
  __shared__ unsigned long long x_z[G];    // exchanged
  __shared__ int x_hist[2][256];           // exchanged (double-buffered by pass parity)
  __shared__ unsigned long long x_min[2];  // exchanged (double-buffered by take parity)
  __shared__ int x_tot;                    // exchanged
  __shared__ float s_red[LK_W][G];
  __shared__ unsigned long long s_kmin[LK_W];
  __shared__ float s_M[G], s_Z[G];
  __shared__ int s_gh[256];
  __shared__ unsigned long long s_prefix, s_kt;
  __shared__ int s_need, s_all, s_off, s_total;
  __shared__ int s_warp[LK_W + 1];

  if (tid == 0) r3_coefs(s_coef);
  for (int i = tid; i < (ES + 31) / 32; i += AT_THREADS) TK[i] = 0u;
  if (tid < G) x_z[tid] = 0ull;

  // ---- logits (R2) of this rank's units, local max per head
  const bf16* centb = a.centb + (int64_t)li * a.Umax * D;
  float mymax[G];
#pragma unroll
  for (int j = 0; j < G; ++j) mymax[j] = -INFINITY;
  for (int i = tid; i < cnt; i += AT_THREADS) {
    float l[G];
    logits_row<G>(sq, reinterpret_cast<const uint4*>(centb + (int64_t)(lo + i) * D), l);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      E[j * ES + i] = l[j];
      mymax[j] = fmaxf(mymax[j], l[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    float v = mymax[j];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_red[warp][j] = v;
  }
  __syncthreads();
  if (tid < G) {
    float v = -INFINITY;
    for (int w = 0; w < LK_W; ++w) v = fmaxf(v, s_red[w][tid]);
    x_max[tid] = v;
  }
  cl.sync();
  if (tid < G) {
    float v = -INFINITY;
    for (int r = 0; r < AT_CL; ++r) v = fmaxf(v, *cl.map_shared_rank(&x_max[tid], r));
    s_M[tid] = v;
  }
  __syncthreads();

  // ---- exp (R3) + exact fixed-point normaliser, summed over the cluster
  unsigned long long zl[G];
#pragma unroll
  for (int j = 0; j < G; ++j) zl[j] = 0ull;
  for (int i = tid; i < cnt; i += AT_THREADS) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float e = exp_r3(__fsub_rn(E[j * ES + i], s_M[j]), s_coef);
      E[j * ES + i] = e;
      zl[j] += __float2ull_rz(__fmul_rn(e, 1099511627776.0f));
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    unsigned long long z = zl[j];
    for (int o = 16; o; o >>= 1) z += shfl_xor_u64(z, o);
    if (lane == 0 && z) atomicAdd(&x_z[j], z);
  }
  cl.sync();
  if (tid < G) {
    unsigned long long z = 0ull;
    for (int r = 0; r < AT_CL; ++r) z += *cl.map_shared_rank(&x_z[tid], r);
    s_Z[tid] = __fmul_rn(__ull2float_rn(z), __int_as_float((127 - 40) << 23));
  }
  __syncthreads();

  // ---- A_u and keys (A desc, id asc); sizes clamped to 16 bits (B <= 65534: a clamped unit never fits)
  const int32_t* usize = a.usize + (int64_t)li * a.Umax;
  for (int i = tid; i < cnt; i += AT_THREADS) {
    float A = 0.0f;
#pragma unroll
    for (int j = 0; j < G; ++j) A = __fadd_rn(A, __fdiv_rn(E[j * ES + i], s_Z[j]));
    A = __fdiv_rn(A, (float)G);
    KEYS[i] = ((unsigned long long)(~__float_as_uint(A)) << 16) | (unsigned)(lo + i);
    SZ[i] = (uint16_t)clamp16(usize[lo + i]);
  }
  if (tid == 0) {
    s_prefix = 0ull;
    s_need = a.budget;
    s_all = 0;
  }

  // ---- first-skip pivot: size-weighted radix select over the cluster (6 passes of 8-bit digits)
  for (int pass = 0; pass < 6; ++pass) {
    const int shift = 40 - 8 * pass;
    const unsigned long long hi_mask = (pass == 0) ? 0ull : (~0ull << (shift + 8)) & 0xFFFFFFFFFFFFull;
    int* H = x_hist[pass & 1];
    H[tid] = 0;  // AT_THREADS == 256 bins
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    for (int i0 = warp * 32; i0 < cnt; i0 += AT_THREADS) {
      const int i = i0 + lane;
      int bk = -1, sz = 0;
      if (i < cnt) {
        const unsigned long long k = KEYS[i];
        if ((k & hi_mask) == prefix) {
          bk = (int)((k >> shift) & 255);
          sz = SZ[i];
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, bk);
      const unsigned sum = __reduce_add_sync(peers, (unsigned)sz);
      if (bk >= 0 && lane == __ffs(peers) - 1) atomicAdd(&H[bk], (int)sum);
    }
    cl.sync();
    {
      int gsum = 0;
#pragma unroll
      for (int r = 0; r < AT_CL; ++r) gsum += *cl.map_shared_rank(&H[tid], r);
      s_gh[tid] = gsum;
    }
    __syncthreads();
    if (warp == 0) {
      int v[8], ls = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = s_gh[lane * 8 + i];
        ls += v[i];
      }
      int incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int excl = incl - ls;
      const int need = s_need;
      const unsigned hit = __ballot_sync(0xffffffffu, incl > need);
      if (hit == 0u) {
        if (lane == 0) s_all = 1;  // (pass 0 sees everything) the whole set fits the budget
      } else {
        const int first = __ffs(hit) - 1;
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
    }
    __syncthreads();
    if (s_all) break;
  }
  const bool all = s_all != 0;
  const unsigned long long pivot = all ? ~0ull : s_prefix;
  const int per = (cnt + AT_THREADS - 1) / AT_THREADS;
  const int u0 = tid * per, u1 = min(cnt, u0 + per);
  for (int i = u0; i < u1; ++i)
    if (KEYS[i] < pivot) atomicOr(&TK[i >> 5], 1u << (i & 31));
  // ---- tail: the greedy's next take = the smallest key after the last take among units that still
  // fit; one cluster-wide min per take
  {
    int rem = all ? 0 : s_need;
    unsigned long long last = pivot;
    int it = 0;
    while (rem > 0) {
      unsigned long long best = ~0ull;
      for (int i = u0; i < u1; ++i) {
        const unsigned long long k = KEYS[i];
        if (k > last && k < best && SZ[i] <= rem) best = k;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long y = shfl_xor_u64(best, o);
        best = y < best ? y : best;
      }
      if (lane == 0) s_kmin[warp] = best;
      __syncthreads();
      if (tid == 0) {
        unsigned long long v = ~0ull;
        for (int w = 0; w < LK_W; ++w) v = s_kmin[w] < v ? s_kmin[w] : v;
        x_min[it & 1] = v;
      }
      cl.sync();
      if (tid == 0) {
        unsigned long long v = ~0ull;
        for (int r = 0; r < AT_CL; ++r) {
          const unsigned long long y = *cl.map_shared_rank(&x_min[it & 1], r);
          v = y < v ? y : v;
        }
        s_kt = v;
      }
      __syncthreads();
      const unsigned long long kt = s_kt;
      if (kt == ~0ull) break;  // nothing else fits
      const int ut = (int)(kt & 0xFFFFull);
      rem -= clamp16(usize[ut]);
      last = kt;
      if (tid == 0 && ut >= lo && ut < hi) atomicOr(&TK[(ut - lo) >> 5], 1u << ((ut - lo) & 31));
      ++it;
    }
  }
  __syncthreads();

  // ---- layout (selected units in id order): rank offset = rows of the lower ranks
  int local = 0, local_cnt = 0;
  for (int i = u0; i < u1; ++i)
    if (TK[i >> 5] >> (i & 31) & 1u) {
      local += SZ[i];
      ++local_cnt;
    }
  int rank_total;
  int dst = lk_scan(local, s_warp, rank_total);
  if (tid == 0) x_tot = rank_total;
  cl.sync();
  if (tid == 0) {
    int off = 0, tot = 0;
    for (int r = 0; r < AT_CL; ++r) {
      const int v = *cl.map_shared_rank(&x_tot, r);
      if (r < rank) off += v;
      tot += v;
    }
    s_off = off;
    s_total = tot;
  }
  __syncthreads();
  dst += s_off;
  const int total = s_total;

  const int nxt = ws_cur ^ 1;
  const int64_t gi = a.inst_global_base + li;
  const bf16* curK = a.ws + ws_cur * a.ws_buf_stride + gi * a.ws_inst_stride;
  const bf16* curV = curK + (int64_t)a.budget * D;
  const uint8_t* pool = a.pool + (int64_t)li * a.pool_inst_bytes;
  uint8_t* sel = a.sel + (int64_t)li * a.Umax;
  int32_t* seloff = a.seloff + (int64_t)li * a.Umax;
  const int64_t* uoff = a.uoff + (int64_t)li * a.Umax;
  RowSrc* rows = a.rows + (int64_t)li * app.budget;
  unsigned long long reused = 0, fetched = 0, hbytes = 0;
  for (int i = u0; i < u1; ++i) {
    const int u = lo + i;
    const bool take = TK[i >> 5] >> (i & 31) & 1u;
    const bool had = sel[u] != 0;
    if (take) {
      const int sz = SZ[i];
      if (had) {
        const int so = seloff[u];
        for (int k = 0; k < sz; ++k)
          rows[dst + k] = RowSrc{reinterpret_cast<const uint4*>(curK + (int64_t)(so + k) * D),
                                 reinterpret_cast<const uint4*>(curV + (int64_t)(so + k) * D)};
        ++reused;
      } else {
        const uint8_t* base = pool + uoff[u] * POOL_ROW_BYTES;
        for (int k = 0; k < sz; ++k)
          rows[dst + k] = RowSrc{reinterpret_cast<const uint4*>(base + (int64_t)k * ROW_BYTES),
                                 reinterpret_cast<const uint4*>(base + (int64_t)(sz + k) * ROW_BYTES)};
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
  for (int o = 16; o; o >>= 1) {
    reused += __shfl_xor_sync(0xffffffffu, reused, o);
    fetched += __shfl_xor_sync(0xffffffffu, fetched, o);
    hbytes += __shfl_xor_sync(0xffffffffu, hbytes, o);
    local_cnt += __shfl_xor_sync(0xffffffffu, local_cnt, o);
  }
  if (lane == 0 && (reused | fetched)) {
    atomicAdd(&a.stats->units_reused, reused);
    atomicAdd(&a.stats->units_fetched, fetched);
    atomicAdd(&a.stats->bytes_h2d, hbytes);
    atomicAdd(&a.stats->units_selected, (unsigned long long)local_cnt);
  }
  if (rank == 0 && tid == 0) {
    atomicAdd(&a.stats->units_scored, (unsigned long long)n);
    if (li % a.hn == 0) atomicAdd(&a.stats->retrievals, 1ull);
    InstState* S = a.inst + li;
    S->ws_cur = nxt;
    S->ws_rows = total;
  }
  return total;
}

#ifdef LKV_PROF
__device__ unsigned long long g_lkv_prof[64][2048][PROF_SLOTS];
#endif

template <int G>
__global__ void __launch_bounds__(AT_THREADS, G <= 4 ? 2 : 1) layer_kernel(LayerArgs A) {
  namespace cg = cooperative_groups;
#ifdef LKV_PROF
  unsigned long long* prof = (A.layer < 64 && blockIdx.x < 2048) ? g_lkv_prof[A.layer][blockIdx.x] : nullptr;
#else
  unsigned long long* prof = nullptr;
#endif
  prof_stamp(prof, 0);
  pdl_wait_trigger();
  prof_stamp(prof, 1);
  const RetrieveArgs& a = A.r;
  const AppendArgs& app = A.at.app;
  const int li = blockIdx.x / AT_CL, rank = blockIdx.x % AT_CL;
  const int b = li / a.hn, h = li % a.hn, tid = threadIdx.x;
  extern __shared__ __align__(128) uint8_t lk_smem[];
  __shared__ int s_t, s_n, s_cur, s_flag;
  __shared__ double s_r;
  __shared__ double s_cos[64];
  __shared__ float sq[G][D];
  if (tid == 0) {
    const InstState* S = a.inst + li;
    s_t = S->step + 1;  // read before the first cluster barrier; rank 0 commits t in append_one
    s_n = S->n_units;
    s_cur = S->ws_cur;
  }
  __syncthreads();
  // every rank's read of the instance state happens-before rank 0's append commits it: split cluster
  // barrier, arrived here and waited on after the trigger (the trigger hides its latency)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  prof_stamp(prof, 2);
  const int t = s_t, par = t & 1;
  const uint16_t* qc = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b;
  const uint16_t* qr_old = reinterpret_cast<const uint16_t*>(a.qref) + ((int64_t)(par ^ 1) * a.Bmax + b) * a.Hq * D;

  // ---- 1. trigger (R1), identical on every rank
  if (a.shared_copy) {
    if (tid == 0) {
      s_flag = a.flag_src[b];
      s_r = a.r_src[b];
    }
  } else {
    trigger_cosines<AT_THREADS>(qc, qr_old, a.Hq, s_cos);
    __syncthreads();
    if (tid == 0) {
      const double rr = trigger_mean(s_cos, a.Hq);
      s_r = rr;
      s_flag = (t == 1) || (rr < a.tau);
    }
  }
  __syncthreads();
  const int flag = s_flag;
  prof_stamp(prof, 3);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && h == 0) {
    if (tid == 0) {
      a.flag[b] = (uint8_t)flag;
      a.r[b] = s_r;
      if (a.flag_out) a.flag_out[b] = (uint8_t)flag;
      if (a.r_out) a.r_out[b] = s_r;
    }
    if (!a.shared_copy) {
      const uint4* src = reinterpret_cast<const uint4*>((a.trigger_ref == LOUISKV_TRIG_PREV_STEP || flag) ? qc : qr_old);
      uint4* dst = reinterpret_cast<uint4*>(a.qref + ((int64_t)par * a.Bmax + b) * a.Hq * D);
      for (int i = tid; i < a.Hq * D / 8; i += AT_THREADS) dst[i] = src[i];
    }
  }

  // ---- 2. retrieve: distributed score + select, then the gather spread over the ranks
  if (flag) {
    const uint16_t* qb = qc + (int64_t)(a.h0 + h) * G * D;
    for (int i = tid; i < G * D; i += AT_THREADS) sq[i / D][i % D] = bf2f(qb[i]);
    __syncthreads();
    const int total = s_n <= AT_CL * LK_MCAP ? lk_select<G, true>(a, app, li, rank, s_n, s_cur, sq, lk_smem)
                                             : lk_select<G, false>(a, app, li, rank, s_n, s_cur, sq, lk_smem);
    prof_stamp(prof, 4);
    cg::this_cluster().sync();  // row table complete (cluster-scope release/acquire)
    if (total > 0) {
      const int64_t gi = a.inst_global_base + li;
      bf16* nxtK = a.ws + (s_cur ^ 1) * a.ws_buf_stride + gi * a.ws_inst_stride;
      const GatherJob J{total, 0, nxtK, nxtK + (int64_t)a.budget * D};
      const int per = (total + AT_CL - 1) / AT_CL;
      const int r0 = rank * per, r1 = min(total, r0 + per);
      if (r0 < r1) gather_rows(app, li, J, r0, r1);
    }
  }

  // ---- 3. store_cache (rank 0), publish to the cluster (generic writes -> TMA reads: proxy fences)
  prof_stamp(prof, 5);
  if (rank == 0) append_one(app, li, flag);
  prof_stamp(prof, 6);
  asm volatile("fence.proxy.async.global;" ::: "memory");
  cg::this_cluster().sync();
  prof_stamp(prof, 7);
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // select used the staging smem

  // ---- 4. attention, one split per rank
  attn_body<G, true>(A.at, li, rank, AT_CL, prof);
  prof_stamp(prof, 14);
}

template <int G>
static cudaError_t launch_layer_g(const LayerArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(layer_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    attr = true;
  }
  static_assert(G * LK_MCAP * 4 + LK_MCAP * 10 + LK_MCAP / 8 <= AT_STAGES * AT_STAGE_BYTES, "select smem");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.r.batch * a.r.hn * AT_CL);
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = AT_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = AT_CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, layer_kernel<G>, a);
}

cudaError_t launch_layer(const LayerArgs& a, cudaStream_t st) {
  if (a.r.Hq > 64) return cudaErrorInvalidValue;
  switch (a.r.g) {
    case 1: return launch_layer_g<1>(a, st);
    case 2: return launch_layer_g<2>(a, st);
    case 4: return launch_layer_g<4>(a, st);
    case 8: return launch_layer_g<8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lkv

#ifdef LKV_PROF
extern "C" int louiskv_prof_read(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, lkv::g_lkv_prof, bytes);
}
#endif
