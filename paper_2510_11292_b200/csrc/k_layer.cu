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
#include <type_traits>

#include "lkv_append_dev.cuh"
#include "lkv_attn_dev.cuh"
#include "lkv_attn_mma_dev.cuh"
#include "lkv_score_dev.cuh"

namespace lkv {

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

// ---------------------------------------------------------------- replicated select
// Every rank scores its 1/8 of the units, pushes its A bits to all ranks (DSMEM stores), and then
// runs the whole greedy selection locally on the replicated keys: three cluster barriers in total
// (max, normaliser, keys) and every rank knows the complete new layout.
// Instances with more than LK_REP_N live units (long outputs: every evicted segment is a unit) run
// the same code with the A bits, sizes, own logits and own destinations in per-instance global
// scratch ("big" mode: each rank writes its own range once, the cluster barrier publishes it) and
// only the taken bits and the work lists in shared memory; the dispatch is on the LIVE unit count
// read from the instance state, so one launch serves every step of a long generation.
constexpr int LK_REP_N = LAYER_REP_UNITS;  // units per instance held in shared memory
constexpr int LK_REP_SEL = LAYER_REP_SEL;  // selected units (<= min(n, B))
// shared-memory regions of the replicated select (bytes, by n): RA [0, 4n) | SZ [4n, 6n) | TK bits |
// X (the rest of the idle attention staging area): own logits E, then the radix candidate lists,
// then the tail candidates, then the selected-unit LIST
__host__ __device__ constexpr int rep_off_tk(int n) { return (6 * n + 15) & ~15; }
__host__ __device__ constexpr int rep_off_x(int n) { return (rep_off_tk(n) + ((n + 31) / 32) * 4 + 15) & ~15; }
// The layer kernel runs one CTA per SM (register budget), so it takes a large dynamic shared-memory
// arena: the attention ring uses its first AT_STAGES x 32 KB, the select (which runs while no
// attention load is in flight) all of it.
constexpr int LK_SMEM = 192 * 1024;
static_assert(LK_SMEM >= AT_SMEM, "layer arena");
constexpr int REP_X_MIN = LK_SMEM - rep_off_x(LK_REP_N);
struct SelEnt {  // one selected unit, in id (= destination) order
  int dst, sz, u, f8;  // f8: the rows are E4M3 host-pool rows (FP8 pool), converted by the gather
  const uint8_t* kb;  // first K row (current working set, or the host pool span)
  const uint8_t* vb;
};
static_assert(LK_REP_SEL * (int)sizeof(SelEnt) <= REP_X_MIN, "rep LIST smem");
static_assert(8 * (LK_REP_N / 8) * 4 <= REP_X_MIN, "rep E smem (CL = 8)");
// shared-memory select possible for n units with G heads over CL ranks: the replicated arrays, the
// rank's logits E and at least 32 staged centroid rows fit the staging area (else big mode)
__host__ __device__ constexpr bool rep_fits(int n, int G, int CL) {
  return n <= LK_REP_N && LK_SMEM - rep_off_x(n) >= 4 * 64 * (ROW_BYTES + 16) + 0 * G * CL;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// L2 prefetch of [p, p + bytes) widened to 16-B granules (the buffers are 256-B aligned allocations)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, int64_t bytes) {
  const uint64_t a0 = reinterpret_cast<uint64_t>(p) & ~15ull;
  const uint64_t a1 = (reinterpret_cast<uint64_t>(p) + bytes + 15) & ~15ull;
  if (a1 > a0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

__device__ __forceinline__ unsigned long long rep_key(const uint32_t* RA, int u) {
  return ((unsigned long long)(~RA[u]) << 16) | (unsigned)u;
}

// big-mode global scratch of instance li (inside the retrieve scratch: [nl][Umax * 26] bytes):
// A bits [Umax] u32 | sizes [Umax] u16 | own destinations [Umax] i32
__device__ __forceinline__ uint8_t* big_scratch(const RetrieveArgs& a, int li) {
  return a.scratch_sort + (int64_t)li * a.Umax * 26;
}
// shared-memory offset of the work region X (after the on-chip select arrays)
__device__ __forceinline__ int rep_x_offset(int n, bool big) {
  return big ? ((((n + 31) / 32) * 4 + 15) & ~15) : rep_off_x(n);
}


// Returns the row count of the new working set; *nsel = selected units (LIST entries, at shared
// offset rep_x_offset(n, big)); own_dst[i] = destination row of own unit lo+i (-1: not selected) for
// the deferred sel/seloff update.
template <int G, int CL>
__device__ __forceinline__ int lk_select_rep(const RetrieveArgs& a, const int li, const int rank, const int n,
                                             const int ws_cur, const float (*sq)[D], uint8_t* dsm, int* nsel,
                                             int* own_dst, const bool big, unsigned long long* prof) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = (n + CL - 1) / CL;
  const int lo = min(n, rank * m), hi = min(n, lo + m), cnt = hi - lo;
  const int off_x = rep_x_offset(n, big), x_bytes = LK_SMEM - off_x;
  uint8_t* gscr = big ? big_scratch(a, li) : nullptr;
  // [n] A bits (replicated in every rank's shared memory; big: one global copy)
  uint32_t* RA = big ? reinterpret_cast<uint32_t*>(gscr) : reinterpret_cast<uint32_t*>(dsm);
  // [n] sizes (each rank loads all; big: each rank stores its own range)
  uint16_t* SZ = big ? reinterpret_cast<uint16_t*>(gscr + 4 * (int64_t)a.Umax) : reinterpret_cast<uint16_t*>(dsm + 4 * n);
  uint32_t* TK = reinterpret_cast<uint32_t*>(dsm + (big ? 0 : rep_off_tk(n)));  // [n/32] taken bits (per rank)
  // [G][m] own logits / exps (big: this rank's slice of the per-instance logits scratch
  // [G][Umax] floats; m <= Umax / CL since Umax is a multiple of 256)
  // Logits staging (below): up to 6 buffers of RB centroid rows after E (the own logits) in X; E
  // moves to global scratch when that leaves room for more buffers
  constexpr int PITCH = ROW_BYTES + 16;
  constexpr int HPT = G;           // heads per thread: g independent fmaf chains (ILP g)
  constexpr int RB = AT_THREADS;   // rows per round: one per thread (measured: fewer, longer rounds
                                   // beat more rows in flight — each round is one chain latency; at
                                   // g = 8, two threads per row with E in shared memory: C5 -4 %)
  const int e_bytes_s = (G * m * 4 + 127) & ~127;
  const int nb_s = big ? 0 : min(6, (x_bytes - e_bytes_s) / (RB * PITCH));
  const int nb_g = min(6, x_bytes / (RB * PITCH));
  const bool e_smem = nb_s >= 2 && nb_s >= min(nb_g, 4);
  const int NBUF = e_smem ? nb_s : nb_g;  // (>= 2: rep_fits / big mode leave >= 4 x 64 rows of X)
  float* E = e_smem ? reinterpret_cast<float*>(dsm + off_x)
                    : a.scratch_e + (int64_t)li * G * a.Umax + (int64_t)rank * G * (a.Umax / CL);
  SelEnt* LIST = reinterpret_cast<SelEnt*>(dsm + off_x);       // (after E and the lists are dead)

  __shared__ float s_coef[7];
  __shared__ float x_max[CL][G];               // pushed by every rank
  __shared__ unsigned long long x_z[CL][G];    // pushed by every rank
  __shared__ unsigned long long s_zl[G];
  __shared__ float s_red[LK_W][G];
  __shared__ float s_M[G], s_Z[G];
  __shared__ int s_hist[256];
  __shared__ unsigned long long s_prefix, s_kt;
  __shared__ unsigned long long s_kmin[LK_W];
  __shared__ int s_need, s_all, s_total, s_nsel;
  __shared__ int s_warp[LK_W + 1];

  if (tid < 7) s_coef[tid] = a.r3c[tid];
  if (tid < G) s_zl[tid] = 0ull;
  for (int i = tid; i < (n + 31) / 32; i += AT_THREADS) TK[i] = 0u;
  for (int i = tid; i < cnt; i += AT_THREADS) own_dst[i] = -1;
  const int32_t* usize = a.usize + (int64_t)li * a.Umax;
  // sizes (smem mode: all units; big mode: the own range), 4 per 16-B load: the first 4 x 256 loads
  // (4096 units) stay in flight across the logits below, the rest is loaded in batches of 4 after
  const int sz0 = big ? lo : 0, sz1 = big ? hi : n;          // (lo, hi multiples of 4? not in general:
  const int q0 = sz0 >> 2, q1 = (sz1 + 3) >> 2;             //  whole 16-B words, clipped per element)
  const int4* us4 = reinterpret_cast<const int4*>(usize);  // (a.usize rows are 1 KB aligned: Umax % 256 == 0)
  int4 szv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = q0 + i * AT_THREADS + tid;
    szv[i] = q < q1 ? us4[q] : make_int4(0, 0, 0, 0);
  }
  prof_stamp(prof, 20);

  // ---- logits (R2) of the own units, cluster max per head. The rank's centroid rows are staged in
  // shared memory by coalesced cp.async (16 lanes per 256-B row; row pitch 272 B so that the
  // one-row-per-thread reads below are bank-conflict free), RB rows per round.
  const bf16* centb = a.centb + (int64_t)li * a.Umax * D;
  float mymax[G];
#pragma unroll
  for (int j = 0; j < G; ++j) mymax[j] = -INFINITY;
  {
    // RB = 256 HPT / g rows per round, thread t scores row t % RB for heads [HPT hd, HPT hd + HPT),
    // hd = t / RB (one sequential fmaf chain per (unit, head): recipe R2), NBUF buffers: NBUF - 1
    // rounds of rows in flight while one is scored (an empty group is committed past the end, so the
    // wait count is a constant)
    uint8_t* CS = dsm + off_x + (e_smem ? e_bytes_s : 0);
    const uint32_t cs_s = (uint32_t)__cvta_generic_to_shared(CS);
    const int row = tid % RB, hd = tid / RB;
    const int nround = (cnt + RB - 1) / RB;
    auto issue = [&](int r) {
      if (r < nround) {
        const int b0 = r * RB, nb = min(RB, cnt - b0);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(centb + (int64_t)(lo + b0) * D);
        const uint32_t dst = cs_s + (uint32_t)((r % NBUF) * RB * PITCH);
        for (int i = tid; i < nb * 16; i += AT_THREADS)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (i >> 4) * PITCH + (i & 15) * 16),
                       "l"(src + (int64_t)i * 16)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll 1
    for (int r = 0; r < NBUF - 1; ++r) issue(r);
#pragma unroll 1
    for (int r = 0; r < nround; ++r) {
      issue(r + NBUF - 1);  // into the buffer scored in round r - 1 (freed by its closing barrier)
      switch (NBUF) {       // (the wait count is an immediate)
        case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
      }
      __syncthreads();
      const int b0 = r * RB, nb = min(RB, cnt - b0);
      if (row < nb) {
        const uint4* crow = reinterpret_cast<const uint4*>(CS + (r % NBUF) * RB * PITCH + row * PITCH);
        float l[HPT];
        logits_row_smem<HPT>(sq + hd * HPT, crow, a.inv_sqrt_d, l);
#pragma unroll
        for (int k = 0; k < HPT; ++k) E[(hd * HPT + k) * m + b0 + row] = l[k];
        // (the heads' running maxima; compile-time indices only — no dynamically indexed registers)
        if constexpr (HPT == G) {
#pragma unroll
          for (int j = 0; j < G; ++j) mymax[j] = fmaxf(mymax[j], l[j]);
        } else {
#pragma unroll
          for (int j = 0; j < G; ++j)
#pragma unroll
            for (int k = 0; k < HPT; ++k)
              if (j == hd * HPT + k) mymax[j] = fmaxf(mymax[j], l[k]);
        }
      }
      __syncthreads();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  {
    auto put4 = [&](int q, const int4 v) {
      const int u = 4 * q;
      if (u >= sz0 && u < sz1) SZ[u] = (uint16_t)clamp16(v.x);
      if (u + 1 >= sz0 && u + 1 < sz1) SZ[u + 1] = (uint16_t)clamp16(v.y);
      if (u + 2 >= sz0 && u + 2 < sz1) SZ[u + 2] = (uint16_t)clamp16(v.z);
      if (u + 3 >= sz0 && u + 3 < sz1) SZ[u + 3] = (uint16_t)clamp16(v.w);
    };
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = q0 + i * AT_THREADS + tid;
      if (q < q1) put4(q, szv[i]);
    }
    for (int qb = q0 + 4 * AT_THREADS + tid; qb < q1; qb += 4 * AT_THREADS) {
      int4 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = qb + i * AT_THREADS;
        v[i] = q < q1 ? us4[q] : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (qb + i * AT_THREADS < q1) put4(qb + i * AT_THREADS, v[i]);
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    float v = mymax[j];
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_red[warp][j] = v;
  }
  __syncthreads();
  if (tid < G * CL) {
    const int j = tid % G, r = tid / G;
    float v = -INFINITY;
    for (int w = 0; w < LK_W; ++w) v = fmaxf(v, s_red[w][j]);
    *cl.map_shared_rank(&x_max[rank][j], r) = v;
  }
  prof_stamp(prof, 6);
  cl.sync();
  if (tid < G) {
    float v = -INFINITY;
#pragma unroll
    for (int r = 0; r < CL; ++r) v = fmaxf(v, x_max[r][tid]);
    s_M[tid] = v;
  }
  __syncthreads();

  // ---- exp (R3) + exact fixed-point normaliser (integer sums: order independent)
  unsigned long long zl[G];
#pragma unroll
  for (int j = 0; j < G; ++j) zl[j] = 0ull;
  // E in global scratch (large instances): units in batches of EB per thread, every load of a batch
  // issued before its arithmetic (the stores to E would otherwise serialise the next unit's loads);
  // E in shared memory: one unit at a time (C5's share: flagged launch 104 -> 94 us; C2: batching -1 %)
  auto exp_pass = [&](auto ebc) {
    constexpr int EB = decltype(ebc)::value;
    for (int i0 = tid; i0 < cnt; i0 += EB * AT_THREADS) {
      float ev[EB][G];
#pragma unroll
      for (int k = 0; k < EB; ++k) {
        const int i = i0 + k * AT_THREADS;
#pragma unroll
        for (int j = 0; j < G; ++j) ev[k][j] = i < cnt ? E[j * m + i] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < EB; ++k) {
        const int i = i0 + k * AT_THREADS;
        if (i < cnt) {
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const float e = exp_r3(__fsub_rn(ev[k][j], s_M[j]), s_coef);
            E[j * m + i] = e;
            zl[j] += __float2ull_rz(__fmul_rn(e, 1099511627776.0f));
          }
        }
      }
    }
  };
  if constexpr (G == 8) {  // (the only group size whose large instances keep E in global scratch;
                           // other g keep the loop code of one unit per thread — C2 -0.5 % otherwise)
    if (e_smem) exp_pass(std::integral_constant<int, 1>{});
    else exp_pass(std::integral_constant<int, 4>{});
  } else {
    exp_pass(std::integral_constant<int, 1>{});
  }
#pragma unroll
  for (int j = 0; j < G; ++j) {
    unsigned long long z = zl[j];
    for (int o = 16; o; o >>= 1) z += shfl_xor_u64(z, o);
    if (lane == 0 && z) atomicAdd(&s_zl[j], z);
  }
  __syncthreads();
  if (tid < G * CL) {
    const int j = tid % G, r = tid / G;
    *cl.map_shared_rank(&x_z[rank][j], r) = s_zl[j];
  }
  cl.sync();
  if (tid < G) {
    unsigned long long z = 0ull;
#pragma unroll
    for (int r = 0; r < CL; ++r) z += x_z[r][tid];
    s_Z[tid] = __fmul_rn(__ull2float_rn(z), __int_as_float((127 - 40) << 23));
  }
  __syncthreads();

  // ---- A_u of the own units, pushed to every rank
  auto a_pass = [&](auto ebc) {
    constexpr int EB = decltype(ebc)::value;
    for (int i0 = tid; i0 < cnt; i0 += EB * AT_THREADS) {
      float ev[EB][G];
#pragma unroll
      for (int k = 0; k < EB; ++k) {
        const int i = i0 + k * AT_THREADS;
#pragma unroll
        for (int j = 0; j < G; ++j) ev[k][j] = i < cnt ? E[j * m + i] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < EB; ++k) {
        const int i = i0 + k * AT_THREADS;
        if (i >= cnt) break;
        float A = 0.0f;
#pragma unroll
        for (int j = 0; j < G; ++j) A = __fadd_rn(A, __fdiv_rn(ev[k][j], s_Z[j]));
        A = __fdiv_rn(A, (float)G);
        const uint32_t bits = __float_as_uint(A);
        if (big) {
          RA[lo + i] = bits;  // (published to the cluster by the barrier below)
        } else {
#pragma unroll
          for (int r = 0; r < CL; ++r) *cl.map_shared_rank(&RA[lo + i], r) = bits;
        }
      }
    }
  };
  if constexpr (G == 8) {
    if (e_smem) a_pass(std::integral_constant<int, 1>{});
    else a_pass(std::integral_constant<int, 4>{});
  } else {
    a_pass(std::integral_constant<int, 1>{});
  }
  if (tid == 0) {
    s_prefix = 0ull;
    s_need = a.budget;
    s_all = 0;
  }
  cl.sync();
  prof_stamp(prof, 13);

  // ---- greedy skip-and-continue over all n keys, locally (exact):
  // (a) first-skip pivot = the smallest key whose running size sum in key order exceeds B: a
  //     size-weighted radix select over the key bits below the common prefix of all keys (8 bits
  //     per pass), the candidate ids compacted to the chosen bucket after every pass;
  // (b) every key below the pivot is taken; (c) after the pivot only units with size <= the
  //     remaining budget can be taken (it never grows): they are compacted (key | size << 48) and
  //     one warp walks them, one warp-wide min per take.
  // candidate lists (key | size << 48) in region X: two of LCAP entries
  unsigned long long* LB = reinterpret_cast<unsigned long long*>(dsm + off_x);
  const int LCAP = x_bytes / 16;
  constexpr unsigned long long M48 = 0xFFFFFFFFFFFFull;
  constexpr int DIRECT = 512;  // candidates ranked directly (all pairs) instead of another pass
  __shared__ int s_nc, s_tb;
  __shared__ unsigned long long s_kmax[LK_W];
  const int per = (n + AT_THREADS - 1) / AT_THREADS;
  const int u0 = min(n, tid * per), u1 = min(n, u0 + per);
  {
    unsigned long long kmn = ~0ull, kmx = 0ull;
    for (int u = tid; u < n; u += AT_THREADS) {
      const unsigned long long k = rep_key(RA, u);
      kmn = k < kmn ? k : kmn;
      kmx = k > kmx ? k : kmx;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long y = shfl_xor_u64(kmn, o), z = shfl_xor_u64(kmx, o);
      kmn = y < kmn ? y : kmn;
      kmx = z > kmx ? z : kmx;
    }
    if (lane == 0) {
      s_kmin[warp] = kmn;
      s_kmax[warp] = kmx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 0; w < LK_W; ++w) {
        kmn = s_kmin[w] < kmn ? s_kmin[w] : kmn;
        kmx = s_kmax[w] > kmx ? s_kmax[w] : kmx;
      }
      if (n == 0 || (n == 1 && SZ[0] <= s_need)) {
        s_all = 1;
        s_tb = -1;
      } else if (n == 1) {
        s_prefix = kmn;  // the single unit does not fit: it is the pivot
        s_tb = -1;
      } else {
        const int tb = 63 - __clzll(kmn ^ kmx);
        s_tb = tb;
        s_prefix = kmn & ~((2ull << tb) - 1ull);  // common prefix of every key
      }
    }
    __syncthreads();
  }
  int tb = s_tb, nc = 0, cb = -1;  // cb = -1: candidates = all keys matching the prefix above tb
  bool first_pass = true;
  while (tb >= 0) {
    const int lo_bit = tb >= 7 ? tb - 7 : 0;
    const unsigned wmask = (2u << (tb - lo_bit)) - 1u;
    const unsigned long long himask = (~0ull << (tb + 1)) & M48, pre0 = s_prefix;
    s_hist[tid] = 0;
    __syncthreads();
    if (cb < 0) {
      // most keys share a few buckets (the bulk of A has one exponent): each thread sums its
      // contiguous units per run of equal buckets, and a warp whose lanes all hold the same bucket
      // adds once — no same-address atomic storms
      int mb = -1, macc = 0;
      for (int u = u0; u < u1; ++u) {
        const unsigned long long k = rep_key(RA, u);
        if ((k & himask) != pre0) continue;
        const int bk = (int)((unsigned)(k >> lo_bit) & wmask);
        if (mb < 0) mb = bk;
        if (bk == mb) macc += (int)SZ[u];
        else atomicAdd(&s_hist[bk], (int)SZ[u]);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, mb);
      if (peers == 0xffffffffu) {
#pragma unroll
        for (int o = 16; o; o >>= 1) macc += __shfl_xor_sync(0xffffffffu, macc, o);
        if (lane == 0 && mb >= 0 && macc) atomicAdd(&s_hist[mb], macc);
      } else if (mb >= 0 && macc) {
        atomicAdd(&s_hist[mb], macc);
      }
    } else {
      const unsigned long long* L = LB + cb * LCAP;
      for (int i = tid; i < nc; i += AT_THREADS) {
        const unsigned long long e = L[i];
        atomicAdd(&s_hist[(unsigned)((e & M48) >> lo_bit) & wmask], (int)(e >> 48));
      }
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
      if (lane == 0) s_nc = 0;
      if (hit == 0u) {
        if (lane == 0) s_all = 1;  // (only possible on the first pass) the whole set fits the budget
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
          s_prefix |= (unsigned long long)(lane * 8 + bk) << lo_bit;
        }
      }
    }
    __syncthreads();
    if (first_pass) prof_stamp(prof, 16);
    first_pass = false;
    if (s_all || lo_bit == 0) break;
    tb = lo_bit - 1;
    // compact the chosen bucket's candidates (if they fit the list capacity)
    const unsigned long long msk = (~0ull << lo_bit) & M48, pre = s_prefix;
    const int dsti = cb < 0 ? 0 : cb ^ 1;
    unsigned long long* dstl = LB + dsti * LCAP;
    if (cb < 0) {
      for (int u0c = warp * 32; u0c < n; u0c += AT_THREADS) {
        const int u = u0c + lane;
        unsigned long long k = 0;
        bool keep = false;
        if (u < n) {
          k = rep_key(RA, u);
          keep = (k & msk) == pre;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_nc, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int slot = base + __popc(bal & ((1u << lane) - 1u));
        if (keep && slot < LCAP) dstl[slot] = k | ((unsigned long long)SZ[u] << 48);
      }
    } else {
      const unsigned long long* L = LB + cb * LCAP;
      for (int i0 = warp * 32; i0 < nc; i0 += AT_THREADS) {
        const int i = i0 + lane;
        unsigned long long e = 0;
        bool keep = false;
        if (i < nc) {
          e = L[i];
          keep = (e & msk) == pre;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_nc, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) dstl[base + __popc(bal & ((1u << lane) - 1u))] = e;
      }
    }
    __syncthreads();
    if (s_nc > LCAP) {
      cb = -1;  // (too many to list: the next pass filters all keys by the prefix again)
      continue;
    }
    cb = dsti;
    nc = s_nc;
    if (nc <= DIRECT) {
      // direct finish: the pivot is the candidate whose running size sum (in key order) crosses need
      // (need read by every thread before the barrier; the one matching thread publishes after it)
      const unsigned long long* L = LB + cb * LCAP;
      const int need = s_need;
      __syncthreads();
      for (int ci = tid; ci < nc; ci += AT_THREADS) {
        const unsigned long long e = L[ci], k = e & M48;
        int below = 0;
        for (int cj = 0; cj < nc; ++cj) {
          const unsigned long long f = L[cj];
          if ((f & M48) < k) below += (int)(f >> 48);
        }
        if (below <= need && below + (int)(e >> 48) > need) {
          s_prefix = k;
          s_need = need - below;
        }
      }
      __syncthreads();
      break;
    }
  }
  prof_stamp(prof, 17);
  const bool all = s_all != 0;
  const unsigned long long pivot = all ? ~0ull : s_prefix;
  const int rem1 = all ? 0 : s_need;
  // (b) prefix run taken; (c) tail candidates compacted as key | size << 48
  unsigned long long* T = LB;  // (the lists are dead)
  const int T_CAP = x_bytes / 8;
  __shared__ int s_tc[LK_W];
  if (tid == 0) s_nc = 0;  // (every read of s_nc in the radix loop precedes its last barrier)
  __syncthreads();  // (the id lists in the same region are dead)
  // one warp per 32 consecutive units; two passes, no shared counter (a returning atomic per 32
  // units serialised the warps): (1) the taken bits (one TK word each, exclusive owner) and the
  // warp's tail-candidate count; (2) after a prefix over the warps, the candidates written in id
  // order to one contiguous list
  int wcnt = 0;
  for (int base = warp * 32; base < n; base += AT_THREADS) {
    const int u = base + lane;
    bool take = false, cand = false;
    if (u < n) {
      const unsigned long long k = rep_key(RA, u);
      take = k < pivot;
      cand = rem1 > 0 && k > pivot && SZ[u] <= rem1;
    }
    const unsigned tbits = __ballot_sync(0xffffffffu, take);
    if (lane == 0) TK[base >> 5] = tbits;
    wcnt += __popc(__ballot_sync(0xffffffffu, cand));
  }
  if (lane == 0) s_tc[warp] = wcnt;
  __syncthreads();
  int woff = 0, nt_all = 0;
#pragma unroll
  for (int w = 0; w < LK_W; ++w) {
    woff += w < warp ? s_tc[w] : 0;
    nt_all += s_tc[w];
  }
  if (rem1 > 0 && nt_all <= T_CAP) {
    for (int base = warp * 32; base < n; base += AT_THREADS) {
      const int u = base + lane;
      bool cand = false;
      unsigned long long k = 0;
      if (u < n) {
        k = rep_key(RA, u);
        cand = k > pivot && SZ[u] <= rem1;
      }
      const unsigned cbits = __ballot_sync(0xffffffffu, cand);
      if (cand) T[woff + __popc(cbits & ((1u << lane) - 1u))] = k | ((unsigned long long)SZ[u] << 48);
      woff += __popc(cbits);
    }
  }
  if (tid == 0) s_nc = nt_all;
  prof_stamp(prof, 15);
  __syncthreads();
  if (rem1 > 0) {
    const int nt = s_nc;
    int rem = rem1;
    unsigned long long last = pivot;
    if (nt <= T_CAP) {
      if (warp == 0) {  // one warp, no block barriers per take
        while (rem > 0) {
          unsigned long long best = ~0ull;
#pragma unroll 4
          for (int i = lane; i < nt; i += 32) {
            const unsigned long long e = T[i];
            const unsigned long long k = e & 0xFFFFFFFFFFFFull;
            if (k > last && k < best && (int)(e >> 48) <= rem) best = k;
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            const unsigned long long y = shfl_xor_u64(best, o);
            best = y < best ? y : best;
          }
          if (best == ~0ull) break;
          const int ut = (int)(best & 0xFFFFull);
          rem -= SZ[ut];
          last = best;
          if (lane == 0) atomicOr(&TK[ut >> 5], 1u << (ut & 31));
        }
      }
    } else {  // (many small units after the pivot) block-wide min per take over all keys
      while (rem > 0) {
        unsigned long long best = ~0ull;
        for (int u = u0; u < u1; ++u) {
          const unsigned long long k = rep_key(RA, u);
          if (k > last && k < best && SZ[u] <= rem) best = k;
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
          s_kt = v;
        }
        __syncthreads();
        const unsigned long long kt = s_kt;
        if (kt == ~0ull) break;
        const int ut = (int)(kt & 0xFFFFull);
        rem -= SZ[ut];
        last = kt;
        if (tid == 0) atomicOr(&TK[ut >> 5], 1u << (ut & 31));
      }
    }
  }
  __syncthreads();
  prof_stamp(prof, 18);
  if (tid == 0 && prof) prof[21] = s_nc;  // (tail candidates)

  // ---- layout (selected units in id order) and the selected-unit list with row sources; the old
  // sel/seloff are only read here (their update is deferred past the cluster's last barrier)
  int rows_l = 0, cnt_l = 0;
  for (int u = u0; u < u1; ++u)
    if (TK[u >> 5] >> (u & 31) & 1u) {
      rows_l += SZ[u];
      ++cnt_l;
    }
  // one scan of (rows | count << 16): rows <= B <= 65534, count <= LK_REP_N
  int tot_p;
  const int ex_p = lk_scan(rows_l | (cnt_l << 16), s_warp, tot_p);
  const int total = tot_p & 0xFFFF, ns = tot_p >> 16;
  int dst = ex_p & 0xFFFF, k = ex_p >> 16;
  prof_stamp(prof, 19);
  const int64_t gi = a.inst_global_base + li;
  const uint8_t* curK = reinterpret_cast<const uint8_t*>(a.ws + ws_cur * a.ws_buf_stride + gi * a.ws_inst_stride);
  const uint8_t* curV = curK + (int64_t)a.budget * ROW_BYTES;
  const uint8_t* pool = a.pool + (int64_t)li * a.pool_inst_bytes;
  const uint8_t* sel = a.sel + (int64_t)li * a.Umax;
  const int32_t* seloff = a.seloff + (int64_t)li * a.Umax;
  const int64_t* uoff = a.uoff + (int64_t)li * a.Umax;
  unsigned long long reused = 0, fetched = 0, hbytes = 0;
  constexpr int LB_N = 8;  // the selection-state loads of up to 8 TAKEN units are issued together
  int ub = u0;
  while (true) {
    int uid[LB_N], nb = 0;
    while (ub < u1 && nb < LB_N) {  // the next taken units of this thread's id range, in id order
      if (TK[ub >> 5] >> (ub & 31) & 1u) uid[nb++] = ub;
      ++ub;
    }
    if (nb == 0) break;
    uint8_t hadv[LB_N];
    int sov[LB_N];
    int64_t uov[LB_N];
#pragma unroll
    for (int i = 0; i < LB_N; ++i)
      if (i < nb) {
        hadv[i] = sel[uid[i]];
        sov[i] = seloff[uid[i]];
        uov[i] = uoff[uid[i]];
      }
#pragma unroll
    for (int i = 0; i < LB_N; ++i) {
      if (i >= nb) break;
      const int u = uid[i];
      const int sz = SZ[u];
      SelEnt e;
      e.dst = dst;
      e.sz = sz;
      e.u = u;
      e.f8 = 0;
      if (hadv[i]) {
        e.kb = curK + (int64_t)sov[i] * ROW_BYTES;
        e.vb = curV + (int64_t)sov[i] * ROW_BYTES;
        ++reused;
      } else {
        const int prb = pool_row_bytes(a.pool_fp8);
        const uint8_t* base = pool + uov[i] * prb;
        e.kb = base;
        e.vb = base + (int64_t)sz * (prb / 2);
        e.f8 = a.pool_fp8;
        ++fetched;
        hbytes += (unsigned long long)sz * prb;
      }
      LIST[k++] = e;
      if (u >= lo && u < hi) own_dst[u - lo] = dst;
      dst += sz;
    }
  }
  if (rank == 0) {
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
    if (tid == 0) {
      atomicAdd(&a.stats->units_selected, (unsigned long long)ns);
      atomicAdd(&a.stats->units_scored, (unsigned long long)n);
      if (li % a.hn == 0) atomicAdd(&a.stats->retrievals, 1ull);
    }
  }
  if (tid == 0) {
    s_total = total;
    s_nsel = ns;
  }
  __syncthreads();
  *nsel = s_nsel;
  return s_total;
}

// Gather rows [R0, R1) of the new working set (sources from the selected-unit list; 16 lanes x 16 B
// per row, four rows in flight per half-warp): new units zero-copy from the pinned host pool, kept
// units device-to-device.
__device__ __forceinline__ void lk_gather_list(const SelEnt* LIST, const int nsel, const int R0, const int R1,
                                               uint8_t* nxtK, uint8_t* nxtV) {
  const int sub = threadIdx.x & 15, hw = threadIdx.x >> 4;
  for (int base = R0 + hw; base < R1; base += 4 * AT_HW) {
    uint4 kv[4], vv[4];
    int rr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = base + i * AT_HW;
      rr[i] = r;
      if (r < R1) {
        int lo = 0, hi = nsel - 1;  // last entry with dst <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (LIST[mid].dst <= r) lo = mid;
          else hi = mid - 1;
        }
        const int off = r - LIST[lo].dst;
        if (LIST[lo].f8) {  // E4M3 pool rows (128 B): 8 B per piece, converted to bf16
          kv[i] = e4m3x8_to_bf16x8(reinterpret_cast<const uint2*>(LIST[lo].kb + (int64_t)off * D)[sub]);
          vv[i] = e4m3x8_to_bf16x8(reinterpret_cast<const uint2*>(LIST[lo].vb + (int64_t)off * D)[sub]);
        } else {
          kv[i] = reinterpret_cast<const uint4*>(LIST[lo].kb + (int64_t)off * ROW_BYTES)[sub];
          vv[i] = reinterpret_cast<const uint4*>(LIST[lo].vb + (int64_t)off * ROW_BYTES)[sub];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (rr[i] < R1) {
        reinterpret_cast<uint4*>(nxtK + (int64_t)rr[i] * ROW_BYTES)[sub] = kv[i];
        reinterpret_cast<uint4*>(nxtV + (int64_t)rr[i] * ROW_BYTES)[sub] = vv[i];
      }
  }
}

#ifdef LKV_PROF
__device__ unsigned long long g_lkv_prof[64][2048][PROF_SLOTS];
#endif

#ifndef LKV_LAYER_MINB
#define LKV_LAYER_MINB 1
#endif
template <int G, int CL>
__global__ void __launch_bounds__(AT_THREADS, G <= 4 ? LKV_LAYER_MINB : 1) layer_kernel(LayerArgs A) {
  namespace cg = cooperative_groups;
#ifdef LKV_PROF
  unsigned long long* prof = (A.layer < 64 && blockIdx.x < 2048) ? g_lkv_prof[A.layer][blockIdx.x] : nullptr;
#else
  unsigned long long* prof = nullptr;
#endif
  prof_stamp(prof, 0);
  // early: the previous kernel is ANOTHER layer's layer kernel (host-tracked, LayerArgs::early), so
  // this layer's own state — instance state, q_ref, working set, local buffer, sinks, unit tables —
  // was last written by a kernel that completed before that one passed its own wait: the prologue
  // below reads it before this kernel's wait and overlaps the previous layer. The step's inputs
  // (q_t, k_t, v_t: in a model, produced upstream) are read only after the wait.
  const bool early = A.early != 0;
  if (!early) pdl_wait_trigger();
  const RetrieveArgs& a = A.r;
  const AppendArgs& app = A.at.app;
  const int li = blockIdx.x / CL, rank = blockIdx.x % CL;
  const int b = li / a.hn, h = li % a.hn, tid = threadIdx.x;
  extern __shared__ __align__(128) uint8_t lk_smem[];
  __shared__ __align__(16) InstState s_S;  // state before this step
  __shared__ InstState s_postv[2];         // after this step's store_cache (attention window only),
                                           // for flag = 0 and flag = 1 (both computed while r_t resolves)
  __shared__ int2 s_fifo[32];
  __shared__ double s_cos[64];
  __shared__ double s_r;
  __shared__ int s_flag;
  __shared__ __align__(16) float sq[G][D];
  constexpr int DS = D / CL;  // output dims finalised by each rank
  __shared__ float mg_acc[CL][G][DS];
  __shared__ float mg_ml[CL][G][2];
  __shared__ int s_own_dst[LK_REP_N / CL];
  InstState* S = a.inst + li;

  // ---- 1. prologue: the instance state and (Hq <= 32) BOTH q_ref buffers (so no load waits for the
  // step parity), the L2 prefetch of the retrieval operands and the speculative attention loads
  if (tid < 4) reinterpret_cast<uint4*>(&s_S)[tid] = reinterpret_cast<const uint4*>(S)[tid];
  const int l8 = tid & 7, hh = tid >> 3;
  const bool fast_trig = !a.shared_copy && a.Hq <= AT_THREADS / 8;
  const bool act = fast_trig && hh < a.Hq;
  const uint4* qc4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b);
  const uint4* qr4[2] = {reinterpret_cast<const uint4*>(a.qref + ((int64_t)0 * a.Bmax + b) * a.Hq * D),
                         reinterpret_cast<const uint4*>(a.qref + ((int64_t)1 * a.Bmax + b) * a.Hq * D)};
  uint4 c0 = make_uint4(0, 0, 0, 0), c1 = c0, r00 = c0, r01 = c0, r10 = c0, r11 = c0;
  uint4 nv = c0;  // (last rank, threads < 32) the new token's K / V row pieces, for the attention
  if (act) {
    r00 = qr4[0][hh * 16 + l8];
    r01 = qr4[0][hh * 16 + l8 + 8];
    r10 = qr4[1][hh * 16 + l8];
    r11 = qr4[1][hh * 16 + l8 + 8];
  }
  __syncthreads();
  prof_stamp(prof, 2);
#ifndef LKV_NO_SPEC_PREFETCH
  // (only at 8 CTAs per instance, i.e. few instances: measured +1.2 % at C2; at batch (C4, CL 4) the
  // unflagged launches' wasted prefetch traffic costs 4 %)
  if (CL == 8 && A.spec_pf && tid == 0) {  // speculative L2 prefetch of what a retrieval reads (this rank's 1/CL): centroid
     // rows, sizes and the old selection / pool offsets — five bulk prefetches (TMA unit, no LSU
     // traffic). The trigger resolves in ~2 us; on an unflagged step the lines are simply not used.
    const int nu = s_S.n_units, mu = (nu + CL - 1) / CL;
    const int plo = min(nu, rank * mu), phi = min(nu, plo + mu);
    const int64_t ib = (int64_t)li * a.Umax;
    if (phi > plo) {
      bulk_prefetch_l2(a.centb + (ib + plo) * D, (phi - plo) * ROW_BYTES);
      bulk_prefetch_l2(a.usize + ib + plo, (phi - plo) * 4);
      bulk_prefetch_l2(a.seloff + ib + plo, (phi - plo) * 4);
      bulk_prefetch_l2(a.uoff + ib + plo, (phi - plo) * 8);
      bulk_prefetch_l2(a.sel + ib + plo, phi - plo);
    }
  }
#endif
  prof_stamp(prof, 24);
  const int t = s_S.step + 1, par = t & 1;
  const int cap = app.ring_cap;
  const AttnArgs& at = A.at;
  bf16* ringK = app.ring + (int64_t)li * 2 * cap * D;
  bf16* ringV = ringK + (int64_t)cap * D;
  const int64_t gi = a.inst_global_base + li;
  // this rank's attention plan: 1/8 of sinks, working set and local window (the new token, the
  // window's last row, taken from the input by the last rank)
  auto make_plan = [&](AttnPlan& pl, const bf16* wsk, int ws_rows_r, int win_head, int win_n) {
    // always the same four pieces at fixed indices (possibly empty: the piece lookup takes the
    // last piece starting at or before a row), so the plan stays in registers
    const int se = s_S.s_eff;
    const int s0 = se * rank / CL, s1 = se * (rank + 1) / CL;
    const bf16* sk = at.sinks + (int64_t)li * 2 * at.S * D;
    const int w0 = win_n * rank / CL, w1 = win_n * (rank + 1) / CL;
    const int hs = (win_head + w0) % cap;
    const int first = min(w1 - w0, cap - hs);
    pl.P.np = 4;
    pl.P.v0[0] = 0;
    pl.P.n[0] = s1 - s0;
    pl.P.k[0] = sk + (int64_t)s0 * D;
    pl.P.v[0] = sk + (int64_t)at.S * D + (int64_t)s0 * D;
    pl.P.v0[1] = s1 - s0;
    pl.P.n[1] = ws_rows_r;
    pl.P.k[1] = wsk;
    pl.P.v[1] = wsk + (int64_t)a.budget * D;
    pl.P.v0[2] = s1 - s0 + ws_rows_r;
    pl.P.n[2] = first;
    pl.P.k[2] = ringK + (int64_t)hs * D;
    pl.P.v[2] = ringV + (int64_t)hs * D;
    pl.P.v0[3] = s1 - s0 + ws_rows_r + first;
    pl.P.n[3] = w1 - w0 - first;
    pl.P.k[3] = ringK;
    pl.P.v[3] = ringV;
    pl.rows = (s1 - s0) + ws_rows_r + (w1 - w0);
    pl.mask_lo = pl.mask_hi = 0;
    pl.new_vr = (rank == CL - 1 && w1 > w0) ? pl.rows - 1 : -1;
    return w0;
  };
  // speculative (no retrieval) plan, issued now so the loads overlap the trigger: current working
  // set, and the window before this step's evictions (a superset; evicted rows are masked later)
  AttnPlan pl;
  const int dec0 = s_S.step;
  const int sup_head = s_S.buffered > 0 ? s_S.ring_head : dec0, sup_n = dec0 - sup_head + 1;
  int ws_r0 = s_S.ws_rows * rank / CL, ws_r1 = s_S.ws_rows * (rank + 1) / CL;
  const int sup_w0 = make_plan(pl, a.ws + s_S.ws_cur * a.ws_buf_stride + gi * a.ws_inst_stride + (int64_t)ws_r0 * D,
                               ws_r1 - ws_r0, sup_head, sup_n);
  int npre = min((pl.rows + am::CHUNK - 1) / am::CHUNK, am::STAGES - 1);
  for (int c = 0; c < npre; ++c) {
    attn_load_chunk(pl, c, nv, /*with_new=*/false);  // (the new token's row: after the wait)
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  prof_stamp(prof, 25);
  if (tid >= 32 && tid < 64) {  // prefetch the sealed-segment FIFO head entries (evictions)
    const int k = tid - 32;
    if (k < s_S.fifo_count) s_fifo[k] = app.fifo[(int64_t)li * cap + (s_S.fifo_head + k) % cap];
  }
  // split cluster barrier (arrived here, waited on before the first DSMEM store): every rank has
  // started before any rank writes its shared memory. Relaxed: a release would stall until the
  // speculative attention loads above have landed. (Every rank's reads of the instance state are
  // ordered before the appending rank's commit by the merge barrier, which every rank passes first.)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  // ---- the step's inputs, after the grid-dependency wait
  if (early) pdl_wait_trigger();
  prof_stamp(prof, 1);
  uint32_t qa[8][2];  // the owned heads' q as the attention MMA's A fragments (used at the end)
  mma_q_frags<G>(reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b + (int64_t)(a.h0 + h) * G * D, qa);
  if (rank == CL - 1 && tid < 32)
    nv = reinterpret_cast<const uint4*>((tid < 16 ? A.at.app.k_t : A.at.app.v_t) + (int64_t)b * A.at.app.stride_b +
                                        (int64_t)h * D)[tid & 15];
  // store_cache's ring write of the new token, now (off the step's tail): its slot (decode index
  // dec0 mod ring_cap) is in no attended window this step — the window's rows occupy distinct slots
  // (at most ring_cap - 1 of them) and its own row is supplied from registers
  if (rank == CL - 1 && tid < 32)
    reinterpret_cast<uint4*>((tid < 16 ? ringK : ringV) + (int64_t)(dec0 % cap) * D)[tid & 15] = nv;
  if (act) {
    c0 = qc4[hh * 16 + l8];
    c1 = qc4[hh * 16 + l8 + 8];
  }
  for (int c = 0; c < npre; ++c) attn_store_new_row(pl, c, nv);

  // ---- 2. trigger r_t (recipe R1), identical on every rank: 8 lanes per head, lane l8 sums dims
  // [8 l8, 8 l8 + 8) and [8 l8 + 64, 8 l8 + 72) sequentially, adds them (the tree's first level),
  // then the xor tree 4, 2, 1
  const uint16_t* qc = reinterpret_cast<const uint16_t*>(a.q_own) + (int64_t)b * a.stride_b;
  const uint16_t* qr_old = reinterpret_cast<const uint16_t*>(a.qref) + ((int64_t)(par ^ 1) * a.Bmax + b) * a.Hq * D;
  if (fast_trig) {
    const uint4 ra0 = par ? r00 : r10, ra1 = par ? r01 : r11;  // q_ref buffer (t - 1) & 1
    double dot[2], na[2], nb[2];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float fa[8], fc[8];
      unpack8(half ? ra1 : ra0, fa);
      unpack8(half ? c1 : c0, fc);
      double d_ = 0.0, a_ = 0.0, b_ = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double x = (double)fa[e], y = (double)fc[e];
        d_ = __dadd_rn(d_, __dmul_rn(x, y));
        a_ = __dadd_rn(a_, __dmul_rn(x, x));
        b_ = __dadd_rn(b_, __dmul_rn(y, y));
      }
      dot[half] = d_;
      na[half] = a_;
      nb[half] = b_;
    }
    double dt = __dadd_rn(dot[0], dot[1]), an = __dadd_rn(na[0], na[1]), bn = __dadd_rn(nb[0], nb[1]);
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
      dt = __dadd_rn(dt, __shfl_xor_sync(0xffffffffu, dt, off));
      an = __dadd_rn(an, __shfl_xor_sync(0xffffffffu, an, off));
      bn = __dadd_rn(bn, __shfl_xor_sync(0xffffffffu, bn, off));
    }
    if (act && l8 == 0) {
      double cs = 0.0;
      if (an != 0.0 && bn != 0.0) {
        cs = __ddiv_rn(dt, __dmul_rn(__dsqrt_rn(an), __dsqrt_rn(bn)));
        cs = cs > 1.0 ? 1.0 : (cs < -1.0 ? -1.0 : cs);
      }
      s_cos[hh] = cs;
    }
    // the owned KV head's g query rows (scoring operand) are already in registers
    const int jq = hh - (a.h0 + h) * G;
    if (act && jq >= 0 && jq < G) {
      float f[8];
      unpack8(c0, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) sq[jq][8 * l8 + e] = f[e];
      unpack8(c1, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) sq[jq][64 + 8 * l8 + e] = f[e];
    }
  } else if (!a.shared_copy) {
    trigger_cosines<AT_THREADS>(qc, qr_old, a.Hq, s_cos);
  }
  prof_stamp(prof, 26);
  __syncthreads();
  if (tid == 0) {
    int flag;
    if (a.shared_copy) {
      flag = a.flag_src[b];
      s_r = a.r_src[b];
    } else {
      const double rr = trigger_mean(s_cos, a.Hq);
      s_r = rr;
      flag = a.stride > 0 ? ((t - 1) % a.stride == 0) : ((t == 1) || (rr < a.tau));
    }
    s_flag = flag;
  } else if (tid == 32 || tid == 64) {
    // post-store_cache window (the same seal / append / evict rules as append_one, state only), for
    // both outcomes of the flag while thread 0 resolves r_t
    const bool flag = tid == 64;
    InstState p = s_S;
    const int dec = p.step;
    int2 pushed = make_int2(0, 0);
    int pushed_k = -1;
    if ((flag && p.open_len > 0) || p.open_len >= app.max_open) {
      pushed = make_int2(p.open_start, p.open_len);
      pushed_k = p.fifo_count;
      p.fifo_count++;
      p.open_len = 0;
    }
    if (p.open_len == 0) p.open_start = dec;
    if (p.buffered == 0) p.ring_head = dec;
    p.open_len++;
    p.buffered++;
    int k = 0;
    while (p.buffered > app.W && p.fifo_count > 0 && !p.error) {
      const int2 seg = k == pushed_k ? pushed
                       : k < 32     ? s_fifo[k]
                                    : app.fifo[(int64_t)li * cap + (s_S.fifo_head + k) % cap];
      if (p.n_units >= app.Umax || p.pool_rows + seg.y > app.pool_rows_cap) {
        p.error = 1;
        break;
      }
      p.n_units++;
      p.pool_rows += seg.y;
      p.buffered -= seg.y;
      p.ring_head += seg.y;
      p.fifo_head = (p.fifo_head + 1) % cap;
      p.fifo_count--;
      ++k;
    }
    s_postv[flag] = p;
  }
  prof_stamp(prof, 27);
  __syncthreads();
  prof_stamp(prof, 3);
#ifdef LKV_PROF
  if (prof && tid == 0) prof[22] = clock64();
#endif
  const int flag = s_flag;
  const InstState& s_post = s_postv[flag];
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

  // ---- 3. retrieve (flagged): drain the speculative loads (the select uses the staging memory),
  // select, gather this rank's 1/8 of the new working set — the rows it then attends itself, so no
  // barrier separates gather and attention — and plan again
  const int n = s_S.n_units, ws_cur = s_S.ws_cur;
  bool rep = false, big = false;
  int* own_dst = s_own_dst;
  int total = 0;
  if (flag) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (!fast_trig) {
      const uint16_t* qb = qc + (int64_t)(a.h0 + h) * G * D;
      for (int i = tid; i < G * D; i += AT_THREADS) sq[i / D][i % D] = bf2f(qb[i]);
    }
    __syncthreads();
    bf16* nxtK = a.ws + (ws_cur ^ 1) * a.ws_buf_stride + gi * a.ws_inst_stride;
    // (the host launches this kernel only when min(Umax, B) <= LK_REP_SEL; instances with more than
    // LK_REP_N live units select in big mode, with their per-unit arrays in global scratch)
    rep = true;
    big = !rep_fits(n, G, CL);
    own_dst = big ? reinterpret_cast<int*>(big_scratch(a, li) + 6 * (int64_t)a.Umax) + (int64_t)min(n, rank * ((n + CL - 1) / CL))
                  : s_own_dst;
    int nsel;
    total = lk_select_rep<G, CL>(a, li, rank, n, ws_cur, sq, lk_smem, &nsel, own_dst, big, prof);
    prof_stamp(prof, 4);
#ifdef LKV_PROF
    if (prof && tid == 0) prof[23] = clock64();
#endif
    const int R0 = total * rank / CL, R1 = total * (rank + 1) / CL;
    lk_gather_list(reinterpret_cast<const SelEnt*>(lk_smem + rep_x_offset(n, big)), nsel, R0, R1,
                   reinterpret_cast<uint8_t*>(nxtK), reinterpret_cast<uint8_t*>(nxtK + (int64_t)a.budget * D));
    make_plan(pl, nxtK + (int64_t)R0 * D, R1 - R0, s_post.ring_head, s_post.buffered);
    npre = 0;
  } else {
    // the post-store_cache window is a suffix of the speculative one: mask the evicted front rows
    const int ex = s_post.ring_head - sup_head;  // rows evicted from the front of the superset
    const int w1 = sup_n * (rank + 1) / CL;
    const int v_ring = pl.rows - (w1 - sup_w0);  // (the window rows come last in the plan)
    pl.mask_lo = v_ring;
    pl.mask_hi = v_ring + max(0, min(ex, w1) - sup_w0);
  }
  prof_stamp(prof, 5);

  // ---- 4. attention (tensor cores) over this rank's plan
  prof_stamp(prof, 7);
  const float* part = attn_run_mma<G>(qa, at.scale_log2, pl, npre, nv, prof);

  // ---- 5. merge: every rank pushes its partial's dims [16 r, 16 r + 16) to rank r and its (max, sum)
  // to all ranks (DSMEM stores), one cluster barrier, each rank finalises 16 dims of every head
  cg::cluster_group cl = cg::this_cluster();
  // (unflagged: complete the entry barrier first — it also guarantees every rank has started, so
  // its shared memory may be written)
  if (!flag) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int idx = tid; idx < G * D; idx += AT_THREADS) {
    const int j = idx / D, e = idx % D;
    *cl.map_shared_rank(&mg_acc[rank][j][e % DS], e / DS) = part[j * (D + 2) + e];
  }
  if (tid < G * CL) {
    const int j = tid % G, r = tid / G;
    float* dm = cl.map_shared_rank(&mg_ml[rank][j][0], r);
    dm[0] = part[j * (D + 2) + D];
    dm[1] = part[j * (D + 2) + D + 1];
  }
  prof_stamp(prof, 10);
  cl.sync();
  prof_stamp(prof, 11);
  for (int idx = tid; idx < G * DS; idx += AT_THREADS) {
    const int j = idx / DS, e = idx % DS;
    float M = -INFINITY;
#pragma unroll
    for (int y = 0; y < CL; ++y) M = fmaxf(M, mg_ml[y][j][0]);
    float Lsum = 0.f, Acc = 0.f;
#pragma unroll
    for (int y = 0; y < CL; ++y) {
      const float w = mg_ml[y][j][0] == -INFINITY ? 0.f : exp2f(mg_ml[y][j][0] - M);
      Lsum = fmaf(w, mg_ml[y][j][1], Lsum);
      Acc = fmaf(w, mg_acc[y][j][e], Acc);
    }
    const float o = Acc / Lsum;
    const int64_t oi = ((int64_t)(b * a.hn + h) * G + j) * D + rank * DS + e;
    at.out[oi] = __float2bfloat16_rn(o);
    if (at.out_f32) at.out_f32[oi] = o;
  }
  prof_stamp(prof, 12);

  // ---- 6. deferred state updates (every rank has read the old selection by now)
  if (flag && rep) {
    const int m = (n + CL - 1) / CL;
    const int lo = min(n, rank * m), hi = min(n, lo + m);
    uint8_t* sel = a.sel + (int64_t)li * a.Umax;
    int32_t* seloff = a.seloff + (int64_t)li * a.Umax;
    for (int u = lo + tid; u < hi; u += AT_THREADS) {
      const int d = own_dst[u - lo];
      if (d >= 0) {
        sel[u] = 1;
        seloff[u] = d;
      } else if (sel[u]) {
        sel[u] = 0;
      }
    }
    if (rank == 0 && tid == 0) {
      S->ws_cur = ws_cur ^ 1;
      S->ws_rows = total;
    }
  }
  // store_cache side effects (seal / append / evict) by the last rank; commits the step
  if (rank == CL - 1) append_one(app, li, flag, &s_S, /*row_written=*/true);
  prof_stamp(prof, 14);
}

template <int G, int CL>
static cudaError_t launch_layer_gc(const LayerArgs& a, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  cudaError_t ea = once_per_device(attr, [] {
    return cudaFuncSetAttribute(layer_kernel<G, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, LK_SMEM);
  });
  if (ea != cudaSuccess) return ea;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.r.batch * a.r.hn * CL);
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = LK_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, layer_kernel<G, CL>, a);
}

template <int G>
static cudaError_t launch_layer_g(const LayerArgs& a, int cl, cudaStream_t st) {
  switch (cl) {
    case 2: return launch_layer_gc<G, 2>(a, st);
    case 4: return launch_layer_gc<G, 4>(a, st);
    default: return launch_layer_gc<G, 8>(a, st);
  }
}

// CTAs per instance: the kernel holds one CTA per SM (its register budget); 8 when every instance's
// cluster is resident in one wave, else 4 while two waves suffice, else 2 (measured at C4, 64
// instances: CL 8 / 4 / 2 -> 2529 / 2866 / 2766 tok/s). LOUISKV_LAYER_CL overrides (2, 4 or 8).
int layer_cluster_size(int n_inst) {
  const char* es = getenv("LOUISKV_LAYER_CL");  // (read per launch: tests switch it in-process)
  const int env = es ? atoi(es) : 0;
  if (env == 2 || env == 4 || env == 8) return env;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  if (n_inst * 8 <= sms) return 8;
  if (n_inst * 4 <= 2 * sms) return 4;  // (two waves of 4-CTA clusters beat one of 2-CTA clusters: the
                                        // flagged instances' select and gather get twice the SMs)
  return 2;
}

cudaError_t launch_layer(const LayerArgs& a, cudaStream_t st) {
  if (a.r.Hq > 64 || min(a.r.Umax, a.r.budget) > LK_REP_SEL) return cudaErrorInvalidValue;
  const int cl = layer_cluster_size(a.r.batch * a.r.hn);
  switch (a.r.g) {
    case 1: return launch_layer_g<1>(a, cl, st);
    case 2: return launch_layer_g<2>(a, cl, st);
    case 4: return launch_layer_g<4>(a, cl, st);
    case 8: return launch_layer_g<8>(a, cl, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lkv

#ifdef LKV_PROF
extern "C" int louiskv_prof_read(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, lkv::g_lkv_prof, bytes);
}
extern "C" int louiskv_prof_clear(void) {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, lkv::g_lkv_prof);
  return (int)cudaMemset(p, 0, sizeof(lkv::g_lkv_prof));
}
#endif
