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
#include "lkv_score_dev.cuh"

namespace lkv {

constexpr int SS_THREADS = 1024;
constexpr int SS_WARPS = SS_THREADS / 32;
constexpr int SORT_CAP = 12288;  // units whose keys/sizes live in shared memory (else global scratch)

// ---- should_retrieve: semantic-boundary trigger (recipe R1) fused with the
// logits of the flagged instances (recipe R2 step 1). Grid (unit slices, b*hn). Every CTA recomputes
// r_t of its sequence with the same fixed-order recipe (bit-identical), so no grid-wide dependency
// is needed; the (slice 0, head 0) CTA publishes flag/r and writes the next q_ref buffer
// (double-buffered by step parity so concurrent CTAs keep reading the old one).
constexpr int TL_THREADS = 256;
template <int G>
__global__ void __launch_bounds__(TL_THREADS) trig_logits_kernel(RetrieveArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.y;
  const int b = li / a.hn, h = li % a.hn;
  const int tid = threadIdx.x;
  const int t = a.inst[li].step + 1;  // this instance's decode step (committed by its append)
  const int par = t & 1;
  __shared__ double s_cos[64];
  __shared__ int s_flag;
  __shared__ double s_r;
  const uint16_t* qc = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b;
  const uint16_t* qr_old = reinterpret_cast<const uint16_t*>(a.qref) + ((int64_t)(par ^ 1) * a.Bmax + b) * a.Hq * D;
  if (a.shared_copy) {
    if (tid == 0) {
      s_flag = a.flag_src[b];
      s_r = a.r_src[b];
    }
  } else {
    trigger_cosines<TL_THREADS>(qc, qr_old, a.Hq, s_cos);
    __syncthreads();
    if (tid == 0) {
      const double rr = trigger_mean(s_cos, a.Hq);
      s_r = rr;
      s_flag = a.stride > 0 ? ((t - 1) % a.stride == 0) : ((t == 1) || (rr < a.tau));
    }
  }
  __syncthreads();
  const int flag = s_flag;
  if (blockIdx.x == 0 && h == 0) {
    if (tid == 0) {
      a.flag[b] = (uint8_t)flag;
      a.r[b] = s_r;
      if (a.flag_out) a.flag_out[b] = (uint8_t)flag;
      if (a.r_out) a.r_out[b] = s_r;
    }
    if (!a.shared_copy) {
      // q_ref for step t+1: q_t (PREV_STEP, or a retrieval step) else the old reference
      const uint4* src = reinterpret_cast<const uint4*>((a.trigger_ref == LOUISKV_TRIG_PREV_STEP || flag) ? qc : qr_old);
      uint4* dst = reinterpret_cast<uint4*>(a.qref + ((int64_t)par * a.Bmax + b) * a.Hq * D);
      for (int i = tid; i < a.Hq * D / 8; i += TL_THREADS) dst[i] = src[i];
    }
  }
  if (!flag) return;
  // ---- logits of the owned KV head's g query heads against this slice of units
  const int n = a.inst[li].n_units;
  if ((int)blockIdx.x * TL_THREADS >= n) return;
  __shared__ float sq[G][D];
  const uint16_t* qb = qc + (int64_t)(a.h0 + h) * G * D;
  for (int i = tid; i < G * D; i += TL_THREADS) sq[i / D][i % D] = bf2f(qb[i]);
  __syncthreads();
  const int u = blockIdx.x * TL_THREADS + tid;
  if (u >= n) return;
  float l[G];
  logits_row<G>(sq, reinterpret_cast<const uint4*>(a.centb + ((int64_t)li * a.Umax + u) * D), a.inv_sqrt_d, l);
  float* E = a.scratch_e + (int64_t)li * G * a.Umax;
#pragma unroll
  for (int j = 0; j < G; ++j) E[(int64_t)j * a.Umax + u] = l[j];
}

// block-wide exclusive scan of one int per thread (512 threads); returns the exclusive prefix
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
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
    int w = lane < SS_WARPS ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < SS_WARPS) s_warp[lane] = wi - w;
    if (lane == SS_WARPS - 1) s_warp[SS_WARPS] = wi;
  }
  __syncthreads();
  const int r = s_warp[warp] + incl - v;
  total = s_warp[SS_WARPS];
  __syncthreads();
  return r;
}

// ---- group scores, sort, budgeted greedy, working-set layout: one CTA per flagged instance
// SMB: the sort buffers live in shared memory (explicit LDS/STS); else in this instance's global scratch
template <int G, bool SMB>
__device__ __forceinline__ void select_body(const RetrieveArgs& a, const int li, const int n) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  InstState* S = a.inst + li;

  __shared__ float s_coef[7];
  __shared__ float s_red[SS_WARPS][G];
  __shared__ float s_m[G];
  __shared__ unsigned long long s_z[G];
  __shared__ float s_Z[G];
  __shared__ int s_warp[SS_WARPS + 1];
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* s_taken = s_dyn;  // bitmap [ceil(Umax/32)]
  // sort keys (~bits(A) << 16 | id) padded to a power of two, and unit sizes (by id): shared memory
  // when they fit, else this instance's global scratch
  unsigned long long* KEYS;
  uint16_t* s_sz;
  if constexpr (SMB) {
    KEYS = reinterpret_cast<unsigned long long*>(s_dyn + (((a.Umax + 31) / 32 + 1) & ~1));
    s_sz = reinterpret_cast<uint16_t*>(KEYS + SORT_CAP);
  } else {
    KEYS = reinterpret_cast<unsigned long long*>(a.scratch_sort + (int64_t)li * a.Umax * 26);
    s_sz = reinterpret_cast<uint16_t*>(KEYS + 3 * a.Umax);
  }

  if (tid < 7) s_coef[tid] = a.r3c[tid];
  for (int i = tid; i < (a.Umax + 31) / 32; i += SS_THREADS) s_taken[i] = 0u;
  if (tid < G) s_z[tid] = 0ull;
  float* E = a.scratch_e + (int64_t)li * G * a.Umax;
  const int32_t* usize = a.usize + (int64_t)li * a.Umax;

  // ---- max of the logits per head (exact, order independent)
  float mymax[G];
#pragma unroll
  for (int j = 0; j < G; ++j) mymax[j] = -INFINITY;
  for (int u = tid; u < n; u += SS_THREADS)
#pragma unroll
    for (int j = 0; j < G; ++j) mymax[j] = fmaxf(mymax[j], E[(int64_t)j * a.Umax + u]);
#pragma unroll
  for (int j = 0; j < G; ++j) {
    float m = mymax[j];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_red[warp][j] = m;
  }
  __syncthreads();
  if (tid < G) {
    float m = -INFINITY;
    for (int w = 0; w < SS_WARPS; ++w) m = fmaxf(m, s_red[w][tid]);
    s_m[tid] = m;
  }
  __syncthreads();

  // ---- exp + exact fixed-point normaliser (recipe R2/R3)
  unsigned long long zl[G];
#pragma unroll
  for (int j = 0; j < G; ++j) zl[j] = 0ull;
  for (int u = tid; u < n; u += SS_THREADS) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float e = exp_r3(__fsub_rn(E[(int64_t)j * a.Umax + u], s_m[j]), s_coef);
      E[(int64_t)j * a.Umax + u] = e;
      zl[j] += __float2ull_rz(__fmul_rn(e, 1099511627776.0f));
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    unsigned long long z = zl[j];
    for (int o = 16; o; o >>= 1) z += shfl_xor_u64(z, o);
    if (lane == 0) atomicAdd(&s_z[j], z);
  }
  __syncthreads();
  if (tid < G) s_Z[tid] = __fmul_rn(__ull2float_rn(s_z[tid]), __int_as_float((127 - 40) << 23));
  __syncthreads();

  // ---- A_u and the sort key ~bits(A_u); values = unit ids in ascending order (stable sort ->
  // ties keep the lower id first); sizes clamped to 16 bits (B <= 65534: a clamped unit never fits)
  for (int u = tid; u < n; u += SS_THREADS) {
    float A = 0.0f;
#pragma unroll
    for (int j = 0; j < G; ++j) A = __fadd_rn(A, __fdiv_rn(E[(int64_t)j * a.Umax + u], s_Z[j]));
    A = __fdiv_rn(A, (float)G);
    KEYS[u] = ((unsigned long long)(~__float_as_uint(A)) << 16) | (unsigned)u;  // (A desc, id asc)
    const int sz = usize[u];
    s_sz[u] = (uint16_t)(sz > 0xFFFF ? 0xFFFF : sz);
  }
  __syncthreads();

  // ---- budgeted greedy skip-and-continue in (A desc, id asc) order, exact:
  // (1) size-weighted radix select of the first-skip pivot K* = the smallest key whose running size
  //     sum exceeds B (6 passes of 8-bit digits over the 48-bit keys; warp-aggregated histograms);
  //     every key < K* is taken, K* is skipped, rem1 = B - (sizes below K*);
  // (2) after K* only units with size <= rem1 can still be taken (the budget never grows): they are
  //     compacted, bitonic-sorted (a small set) and walked by one warp until the budget is spent.
  {
    __shared__ int s_hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ int s_need, s_all;
    if (tid == 0) {
      s_prefix = 0ull;
      s_need = a.budget;
      s_all = 0;
    }
    __syncthreads();
    for (int pass = 0; pass < 6; ++pass) {
      const int shift = 40 - 8 * pass;
      const unsigned long long hi_mask = (pass == 0) ? 0ull : (~0ull << (shift + 8)) & 0xFFFFFFFFFFFFull;
      for (int i = tid; i < 256; i += SS_THREADS) s_hist[i] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix;
      for (int u0 = warp * 32; u0 < n; u0 += SS_THREADS) {
        const int u = u0 + lane;
        int bk = -1, sz = 0;
        if (u < n) {
          const unsigned long long k = KEYS[u];
          if ((k & hi_mask) == prefix) {
            bk = (int)((k >> shift) & 255);
            sz = s_sz[u];
          }
        }
        const unsigned peers = __match_any_sync(0xffffffffu, bk);
        const unsigned sum = __reduce_add_sync(peers, (unsigned)sz);
        if (bk >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_hist[bk], (int)sum);
      }
      __syncthreads();
      if (warp == 0) {
        int v[8], ls = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[i] = s_hist[lane * 8 + i];
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
        __syncwarp();  // (every lane has read s_need before lane `first` rewrites it)
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
    const int rem1 = all ? 0 : s_need;
    // prefix run: every key below the pivot is taken
    const int per = (n + SS_THREADS - 1) / SS_THREADS;
    const int u0 = tid * per, u1 = min(n, u0 + per);
    for (int u = u0; u < u1; ++u)
      if (KEYS[u] < pivot) atomicOr(&s_taken[u >> 5], 1u << (u & 31));
    // tail: the greedy's next take is the smallest key after the last taken one among the units
    // that still fit; one block-wide min-reduction per take (few: each take lowers the budget,
    // which starts below the pivot's size)
    __shared__ unsigned long long s_kmin[SS_WARPS];
    __shared__ unsigned long long s_last;
    if (tid == 0) s_last = pivot;
    int rem = rem1;
    while (rem > 0) {
      __syncthreads();
      const unsigned long long last = s_last;
      unsigned long long best = ~0ull;
      for (int u = u0; u < u1; ++u) {
        const unsigned long long k = KEYS[u];
        if (k > last && k < best && s_sz[u] <= rem) best = k;
      }
#pragma unroll
      for (int o2 = 16; o2; o2 >>= 1) {
        const unsigned long long y = shfl_xor_u64(best, o2);
        best = y < best ? y : best;
      }
      if (lane == 0) s_kmin[warp] = best;
      __syncthreads();
      if (warp == 0) {
        unsigned long long v = s_kmin[lane];
#pragma unroll
        for (int o2 = 16; o2; o2 >>= 1) {
          const unsigned long long y = shfl_xor_u64(v, o2);
          v = y < v ? y : v;
        }
        if (lane == 0) s_last = v;
      }
      __syncthreads();
      const unsigned long long kt = s_last;
      if (kt == ~0ull) break;  // nothing else fits
      const int ut = (int)(kt & 0xFFFFull);
      rem -= s_sz[ut];
      if (tid == 0) atomicOr(&s_taken[ut >> 5], 1u << (ut & 31));
    }
  }
  __syncthreads();

  // ---- layout of the new working set (selected units in id order) + row sources; diff with the
  // previous selection: kept units are copied device->device, new ones read from the host pool
  const int per = (n + SS_THREADS - 1) / SS_THREADS;
  const int u0 = tid * per, u1 = min(n, u0 + per);
  int local = 0, local_cnt = 0;
  for (int u = u0; u < u1; ++u)
    if (s_taken[u >> 5] >> (u & 31) & 1u) {
      local += s_sz[u];
      ++local_cnt;
    }
  int total;
  int dst = block_excl_scan(local, s_warp, total);

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
  // BATCHED_DMA: two spans (K rows, V rows) per selected unit, in unit-id order
  DmaSpan* spans = a.dma_spans ? a.dma_spans + (int64_t)li * a.dma_cap : nullptr;
  int ord = 0;
  if (spans) {
    int n_sel;
    ord = block_excl_scan(local_cnt, s_warp, n_sel);
    if (tid == 0) a.dma_n[li] = 2 * n_sel;
  }
  unsigned long long reused = 0, fetched = 0, hbytes = 0;
  for (int u = u0; u < u1; ++u) {
    const bool take = s_taken[u >> 5] >> (u & 31) & 1u;
    const bool had = sel[u] != 0;
    if (take && spans) {
      const int sz = s_sz[u];
      const uint64_t nb = (uint64_t)sz * ROW_BYTES;  // (BATCHED_DMA implies a bf16 pool)
      DmaSpan* sp = spans + 2 * ord++;
      if (had) {
        const int so = seloff[u];
        sp[0] = DmaSpan{(uint64_t)(curK + (int64_t)so * D), (uint64_t)(nxtK + (int64_t)dst * D), nb};
        sp[1] = DmaSpan{(uint64_t)(curV + (int64_t)so * D), (uint64_t)(nxtV + (int64_t)dst * D), nb};
        ++reused;
      } else {
        const uint8_t* base = pool + uoff[u] * POOL_ROW_BYTES;  // unit-major [K rows | V rows]
        sp[0] = DmaSpan{(uint64_t)base, (uint64_t)(nxtK + (int64_t)dst * D), nb};
        sp[1] = DmaSpan{(uint64_t)(base + nb), (uint64_t)(nxtV + (int64_t)dst * D), nb};
        ++fetched;
        hbytes += 2 * nb;
      }
      sel[u] = 1;
      seloff[u] = dst;
      dst += sz;
    } else if (take) {
      const int sz = s_sz[u];
      if (had) {
        const int so = seloff[u];
        for (int i = 0; i < sz; ++i)
          rows[dst + i] = RowSrc{reinterpret_cast<const uint4*>(curK + (int64_t)(so + i) * D),
                                 reinterpret_cast<const uint4*>(curV + (int64_t)(so + i) * D)};
        ++reused;
      } else {
        // unit-major pool span [K rows | V rows]; E4M3 rows (FP8 pool) are tagged in bit 0
        const int prb = pool_row_bytes(a.pool_fp8), hrb = prb / 2;
        const uint8_t* base = pool + uoff[u] * prb;
        const uintptr_t tag = a.pool_fp8 ? 1u : 0u;
        for (int i = 0; i < sz; ++i)
          rows[dst + i] = RowSrc{reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(base + (int64_t)i * hrb) | tag),
                                 reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(base + (int64_t)(sz + i) * hrb) | tag)};
        ++fetched;
        hbytes += (unsigned long long)sz * prb;
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
  if (tid == 0) {
    atomicAdd(&a.stats->units_scored, (unsigned long long)n);
    if (li % a.hn == 0) atomicAdd(&a.stats->retrievals, 1ull);
    S->ws_cur = nxt;
    S->ws_rows = total;
  }
  // (BATCHED_DMA: the host issues the copies; the gather of append_output has nothing to do)
  if (tid == 0) a.jobs[li] = GatherJob{spans ? 0 : total, 0, nxtK, nxtV};
}

template <int G>
__global__ void __launch_bounds__(SS_THREADS) select_kernel(RetrieveArgs a) {
  pdl_wait_trigger();
  const int li = blockIdx.x;
  const int b = li / a.hn;
  if (!a.flag[b]) {  // (jobs of unflagged instances were cleared by their consumer)
    if (a.dma_n && threadIdx.x == 0) a.dma_n[li] = 0;
    return;
  }
  const int n = a.inst[li].n_units;
  const int cap = a.Umax < SORT_CAP ? a.Umax : SORT_CAP;
  if (n <= cap)
    select_body<G, true>(a, li, n);
  else
    select_body<G, false>(a, li, n);
}

template <int G>
static cudaError_t set_attrs_once() {
  static std::atomic<uint64_t> attr{0};
  return once_per_device(attr, [] {
    return cudaFuncSetAttribute(select_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
}

cudaError_t launch_trigger_logits(const RetrieveArgs& a, cudaStream_t st) {
  if (a.Hq > 64) return cudaErrorInvalidValue;
  const dim3 grid((a.Umax + TL_THREADS - 1) / TL_THREADS, a.batch * a.hn);
  switch (a.g) {
    case 1: launch_k(trig_logits_kernel<1>, dim3(grid), dim3(TL_THREADS), 0, st, a); break;
    case 2: launch_k(trig_logits_kernel<2>, dim3(grid), dim3(TL_THREADS), 0, st, a); break;
    case 4: launch_k(trig_logits_kernel<4>, dim3(grid), dim3(TL_THREADS), 0, st, a); break;
    case 8: launch_k(trig_logits_kernel<8>, dim3(grid), dim3(TL_THREADS), 0, st, a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_select_gather(const RetrieveArgs& a, cudaStream_t st) {
  const int cap = a.Umax < SORT_CAP ? a.Umax : SORT_CAP;
  const size_t smem =
      sizeof(uint32_t) * ((((a.Umax + 31) / 32) + 1) & ~1) + 8ull * SORT_CAP + 2ull * cap;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  switch (a.g) {
    case 1: if (cudaError_t ea = set_attrs_once<1>()) return ea; launch_k(select_kernel<1>, dim3(a.batch * a.hn), dim3(SS_THREADS), smem, st, a); break;
    case 2: if (cudaError_t ea = set_attrs_once<2>()) return ea; launch_k(select_kernel<2>, dim3(a.batch * a.hn), dim3(SS_THREADS), smem, st, a); break;
    case 4: if (cudaError_t ea = set_attrs_once<4>()) return ea; launch_k(select_kernel<4>, dim3(a.batch * a.hn), dim3(SS_THREADS), smem, st, a); break;
    case 8: if (cudaError_t ea = set_attrs_once<8>()) return ea; launch_k(select_kernel<8>, dim3(a.batch * a.hn), dim3(SS_THREADS), smem, st, a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lkv
