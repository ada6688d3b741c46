// Internal declarations of the LouisKV B200 library (not part of the ABI).
// Kernels live in k_*.cu; the C ABI and all state management in api.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "louiskv.h"

namespace lkv {

constexpr int D = 128;               // head_dim (the paper's models all use 128)
constexpr int ROW_BYTES = D * 2;     // one bf16 K (or V) row
constexpr int POOL_ROW_BYTES = 2 * ROW_BYTES;  // K+V of one token in the host pool (bf16 pool)
// FP8 pool (config pool_dtype = LOUISKV_POOL_FP8_E4M3, reading R-FP8): E4M3 rows, half the bytes
__host__ __device__ constexpr int pool_row_bytes(int fp8) { return fp8 ? 2 * D : POOL_ROW_BYTES; }

typedef __nv_bfloat16 bf16;

// Per (retrieval layer, b, owned kv-head) decode state, device resident.
struct InstState {
  int32_t n_units;        // prompt clusters + evicted segments (scorable units)
  int32_t n_prompt_units; // k
  int64_t pool_rows;      // rows used in this instance's host-pool region
  int32_t ws_cur;         // which working-set buffer is current (0/1)
  int32_t ws_rows;        // rows in the current working set
  int32_t open_len;       // tokens in the open segment
  int32_t open_start;     // decode index (0-based) of the first open token
  int32_t buffered;       // tokens in the local buffer (sealed + open)
  int32_t ring_head;      // decode index of the oldest buffered token
  int32_t fifo_head;      // sealed-segment FIFO (ring of ring_cap int2 entries)
  int32_t fifo_count;
  int32_t error;          // capacity overflow (sticky)
  int32_t prompt_len;     // P
  int32_t s_eff;          // min(S, P)
  int32_t step;           // decode steps completed (read by the trigger, committed by the append)
};

// Gather job of one instance: written by select (retrieve), consumed by the gather of append_output
// or by the clustered append+attention kernel, which clear it.
struct GatherJob {
  int32_t n_rows;
  int32_t pad;
  bf16* dstK;
  bf16* dstV;
};
struct RowSrc {
  const uint4* k;
  const uint4* v;
};
// One copy of the BATCHED_DMA fetch (louiskv.h LOUISKV_FETCH_BATCHED_DMA): a contiguous span of K or
// V rows of one selected unit, from the host pool (new unit) or the current working set (kept unit)
// into the next working set. Written by select_kernel into mapped pinned host memory, read by the
// host, which issues the copies (contiguous spans merged) on the copy engines.
struct DmaSpan {
  uint64_t src, dst, bytes;
};

struct StatsDev {
  unsigned long long retrievals, units_scored, units_selected, units_reused, units_fetched, bytes_h2d,
      bytes_d2h, segments_evicted;
};

// ---------------------------------------------------------------- kernel launchers
// retrieve (k_retrieve.cu)
struct RetrieveArgs {
  const bf16* q_own;         // (select) owned heads; (trigger+logits) = q_all
  int64_t stride_b;
  int batch, hn, g, Umax, budget;
  // trigger (fused into the logits kernel launched by should_retrieve)
  int Hq, h0, Bmax, trigger_ref, shared_copy;
  double tau;
  int stride;  // trigger_stride: 0 = semantic boundary (r_t < tau), k >= 1 = every k steps
  bf16* qref;                // layer base [2][Bmax][Hq][D], read buffer (t-1)&1, write t&1
  const uint8_t* flag_src;   // SHARED mode: designated layer's flags / r
  const double* r_src;
  double* r;                 // [batch] of this layer
  uint8_t* flag_out;         // optional caller outputs
  double* r_out;
  uint8_t* flag;             // [batch] of this layer
  GatherJob* jobs;           // [batch*hn] per-layer gather jobs
  InstState* inst;           // layer base, [batch*hn]
  const bf16* centb;         // layer base [batch*hn][Umax][D]
  const int32_t* usize;      // [batch*hn][Umax]
  const int64_t* uoff;       // [batch*hn][Umax]
  uint8_t* sel;              // [batch*hn][Umax]
  int32_t* seloff;           // [batch*hn][Umax]
  const uint8_t* pool;       // host pool (device-mapped pointer), layer base
  int64_t pool_inst_bytes;   // bytes per instance region
  bf16* ws;                  // working sets: [2][n_inst_total][2][B][D]
  int64_t ws_buf_stride;     // elements between buffer 0 and 1
  int64_t ws_inst_stride;    // elements per instance (2*B*D)
  int64_t inst_global_base;  // global instance index of this layer's first instance
  float* scratch_e;          // [batch*hn][g][Umax]
  uint8_t* scratch_sort;     // [batch*hn][Umax * 14] sort buffers when n exceeds the smem capacity
  RowSrc* rows;              // [batch*hn][B]
  DmaSpan* dma_spans;        // BATCHED_DMA: [batch*hn][dma_cap] spans (device-mapped host), else null
  int32_t* dma_n;            // BATCHED_DMA: [batch*hn] span counts (device-mapped host)
  int dma_cap;               // spans per instance (2 per selected unit, <= 2*B)
  int pool_fp8;              // host-pool rows are E4M3 (converted to bf16 by the gather)
  StatsDev* stats;
  float r3c[7];              // recipe R3 Taylor coefficients fl32(ln2^i / i!) (r3_coefs)
  float inv_sqrt_d;          // recipe R2 scale fl32(1 / fl64(sqrt(d)))
};
// should_retrieve on a retrieval layer: r_t / flag (recipe R1) + logits of flagged instances
cudaError_t launch_trigger_logits(const RetrieveArgs& a, cudaStream_t st);
// retrieve: select (sort + greedy) + working-set layout -> gather job
cudaError_t launch_select_gather(const RetrieveArgs& a, cudaStream_t st);

// append (k_append.cu)
struct AppendArgs {
  GatherJob* jobs;      // [batch*hn] pending gathers of this layer (consumed here)
  const RowSrc* rows;   // [batch*hn][budget]
  int budget;
  const bf16* k_t;
  const bf16* v_t;
  int64_t stride_b;
  int batch, hn, W, max_open, ring_cap, Umax;
  const uint8_t* flag;  // [batch]
  InstState* inst;
  bf16* ring;           // layer base [batch*hn][2][ring_cap][D]
  int2* fifo;           // [batch*hn][ring_cap]
  float* cent;          // [batch*hn][Umax][D]
  bf16* centb;
  int32_t* usize;
  int64_t* uoff;
  int32_t* ufirst;
  uint8_t* sel;
  int32_t* pool_pos;    // [batch*hn][pool_rows_cap]
  int64_t pool_rows_cap;
  uint8_t* pool;        // host pool (device-mapped), layer base
  int64_t pool_inst_bytes;
  int pool_fp8;         // evicted rows are written to the pool as E4M3; E4M3 gather sources
  StatsDev* stats;
};
cudaError_t launch_append(const AppendArgs& a, cudaStream_t st);  // gather kernel + append kernel
// full-cache layer step: append (k_t, v_t) at P + t - 1 and commit the step counter (one CTA)
cudaError_t launch_full_step(const bf16* k_t, const bf16* v_t, int64_t stride_b, int batch, int hn, bf16* full,
                             int64_t full_cap, int64_t P, int* step, int* error, cudaStream_t st);

// attention (k_attn.cu)
struct AttnArgs {
  const bf16* q_own;
  int64_t stride_b;
  int batch, hn, g;
  float scale_log2;  // log2(e)/sqrt(d)
  // sparse layers
  const InstState* inst;  // may be null for full layers
  const bf16* sinks;      // [batch*hn][2][S][D]
  int S;
  const bf16* ws;         // global working-set base
  int64_t ws_buf_stride, ws_inst_stride, inst_global_base;
  int B;
  const bf16* ring;       // [batch*hn][2][ring_cap][D]
  int ring_cap;
  // full layers
  const bf16* full;       // [batch*hn][2][full_cap][D]
  int64_t full_cap;
  int64_t full_P;         // rows = full_P + *step (capped at full_cap)
  const int* step;
  // outputs
  bf16* out;
  float* out_f32;
  // scratch
  float* part;            // [batch*hn][splits][g][D+2]
  int* counters;          // [batch*hn]
  int splits;
  // fused append + attention (clustered launch, sparse layers)
  int fused;
  AppendArgs app;
};
cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st);
// full-cache layers on tensor cores (k_attn_tc.cu); cudaErrorNotSupported -> use launch_attn
// store_cache fused into the full-cache attention (one launch per full-cache layer step)
struct FullStepArgs {
  const bf16* k_t;
  const bf16* v_t;
  int64_t stride_kv;
  int* error;
  uint8_t* flag_out;
  double* r_out;
  int batch;
};
cudaError_t launch_attn_full_tc(const AttnArgs& a, int n_inst_layer, cudaStream_t st,
                                const FullStepArgs* fs = nullptr);

// one decode step of one retrieval layer in ONE clustered launch (k_layer.cu): trigger (R1),
// distributed score + select (R2/R3, greedy), gather, append, attention. r.q_own = q_all.
struct LayerArgs {
  RetrieveArgs r;
  AttnArgs at;  // fused = 1, at.app = the append arguments
  int layer;    // (LKV_PROF builds: timestamp rows of this layer)
  int early;    // 1: the previous kernel in the stream is another layer's layer kernel, so this layer's own
                // state (written only by kernels that completed before that one passed its wait) may be
                // read before griddepcontrol.wait — the prologue overlaps the previous layer
  int spec_pf;  // speculative L2 prefetch of the retrieval operands (small unit tables only: the
                // prefetch runs on every launch, flagged or not; C2 +1.2 %, C5's 33 MB per launch -1.4 %)
};
constexpr int PROF_SLOTS = 32;  // LKV_PROF: [64 layers][2048 CTAs][PROF_SLOTS] globaltimer stamps
// the single launch selects on-chip for instances with at most LAYER_REP_UNITS live units (more: the
// per-unit select arrays move to global scratch, same launch) and handles at most LAYER_REP_SEL
// selectable units (min(Umax, B)); larger budgets run the multi-kernel sequence
constexpr int LAYER_REP_UNITS = 8192;
constexpr int LAYER_REP_SEL = 1024;
cudaError_t launch_layer(const LayerArgs& a, cudaStream_t st);

// Prefill phase timer (louiskv_set_prefill_timing): stream-ordered CUDA events between the phases of
// cluster_prompt; the time from one mark to the next is charged to the earlier mark's phase.
enum { PH_INIT = 0, PH_ASSIGN, PH_SORT, PH_UPDATE, PH_STAGE, PH_END, PH_N };
struct PhaseRec {
  bool on = false;
  std::vector<std::pair<int, cudaEvent_t>> marks;       // main (caller) stream
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> d2h;  // copy-engine offload on the library's stream
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  uint64_t assign_flops = 0, keys = 0, d2h_bytes = 0, assign_passes = 0;
  int calls = 0;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[used++];
  }
  void mark(cudaStream_t st, int ph) {
    if (!on) return;
    cudaEvent_t e = ev();
    if (e && cudaEventRecord(e, st) == cudaSuccess) marks.push_back({ph, e});
  }
};

// k-means / prompt (k_kmeans.cu)
struct KmArgs {
  const bf16* k;
  const bf16* v;
  int64_t sb, st, sh;
  int batch, hn, S, N, kc, iters, impl;
  int pool_fp8;      // the prompt offload writes E4M3 rows
  // outputs / state (layer bases)
  float* cent;       // [ni][Umax][D]
  bf16* centb;
  int Umax;
  int32_t* usize;
  int64_t* uoff;
  int32_t* ufirst;
  uint8_t* sel;
  int32_t* pool_pos;
  int64_t pool_rows_cap;
  uint8_t* pool;
  int64_t pool_inst_bytes;
  bf16* sinks;       // [ni][2][S][D]
  int S_cap;
  InstState* inst;
  // scratch
  float* half;       // [ni][hstride], entries [kc, hstride) = +inf (masked centroid columns)
  int hstride;       // multiple of 256
  uint16_t* bext;    // [ni][Umax][8] bf16: (-h_hi, -h_mid, -h_lo, 0...) — the 9th GEMM K-step
  int32_t* assign;   // [ni][Nmax]
  float* dmin;       // [ni][Nmax]
  int32_t* cc;       // [ni][kmax][nchunk_max] (transposed chunk histograms)
  int32_t* ccT;      // [ni][nchunk_max][kmax] chunk-major exclusive prefixes (scatter bases)
  int32_t* toff;     // [ni][kmax+1] update-task offsets
  int4* tcl;         // [ni][task_max] update tasks: (cluster, first member, end member, tasks of the cluster)
  float* upart;      // [ni][task_max][D] partial sums of multi-task clusters
  int task_max;      // kmax + ceil(Nmax / 32)
  int32_t* off;      // [ni][kmax+1]
  int32_t* cnt;      // [ni][kmax]
  int32_t* perm;     // [ni][Nmax]
  int32_t* tperm;    // [ni][task_max][32] members in task-padded order (update task t: slots 32 t ..)
  int32_t* flags;    // [ni]
  int64_t Nmax;
  int kmax;
  int nchunk_max;
  StatsDev* stats;
  const int32_t* ext_assign;   // device copy of caller-provided assignment (set_prompt_units)
  const float* ext_cent;       // device copy of caller-provided centroids
  int page;                    // > 0: page units of `page` tokens (LOUISKV_UNITS_PAGES), no k-means
  PhaseRec* rec;               // optional phase timer (null: no events)
};
// tc_iters / simt_iters: host counters of which assignment kernel ran
cudaError_t run_kmeans_prompt(const KmArgs& a, cudaStream_t st, uint64_t* tc_iters, uint64_t* simt_iters);
// cluster-major rows of instances [li0, li0+nli) -> dst (+ pool positions); then the unit table
cudaError_t launch_km_offload(const KmArgs& a, int li0, int nli, uint8_t* dst, int64_t dst_stride, cudaStream_t st);
cudaError_t launch_km_units(const KmArgs& a, cudaStream_t st);
cudaError_t launch_full_prompt(const bf16* k, const bf16* v, int64_t sb, int64_t st_, int64_t sh, int batch, int hn,
                               int64_t P, bf16* full, int64_t full_cap, cudaStream_t st);
cudaError_t launch_reset_insts(InstState* inst, int n, int P, int s_eff, cudaStream_t st);

bool kmeans_tc_available();

// Recipe R3's 7 Taylor coefficients fl32(ln2^i / i!): IEEE double products and quotient (round to
// nearest), then one rounding to float; computed on the host once per call.
inline void r3_coefs(float* c) {
  double p = 1.0, fact = 1.0;
  const double ln2 = 0.6931471805599453094;
  for (int i = 0; i <= 6; ++i) {
    if (i > 0) {
      p = p * ln2;
      fact = fact * (double)i;
    }
    c[i] = (float)(p / fact);
  }
}

// Kernel attributes (the >48 KB dynamic shared-memory opt-in) are per device context: set them once
// per device (bit `dev` of `mask`), checking the result; idempotent, so a race between two threads
// only sets them twice.
template <typename F>
inline cudaError_t once_per_device(std::atomic<uint64_t>& mask, F&& set_attrs) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = set_attrs();
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Launch with the programmatic-stream-serialization attribute (PDL); captured into CUDA graphs as
// programmatic edges.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace lkv

// ---------------------------------------------------------------- device helpers
#ifdef __CUDACC__
namespace lkv {
__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

// ---- FP8 pool conversions (reading R-FP8): 8 bf16 <-> 8 E4M3, element order kept (lower byte first)
// bf16 -> fp32 is exact; fp32 -> E4M3 rounds to nearest even and saturates at +-448 (satfinite)
__device__ __forceinline__ uint2 bf16x8_to_e4m3x8(const uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
    unsigned short p;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(p) : "f"(hi), "f"(lo));  // (a -> upper byte)
    o[i] = p;
  }
  return make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
}
// E4M3 -> fp16 is exact, fp16 -> fp32 exact, and every E4M3 value has a 3-bit mantissa and an
// exponent in [-9, 8], so its fp32 bits truncated to bf16 are exact
__device__ __forceinline__ uint4 e4m3x8_to_bf16x8(const uint2 v) {
  const uint32_t in[2] = {v.x, v.y};
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned short p = (unsigned short)(in[i >> 1] >> (16 * (i & 1)));
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(p));
    float f0, f1;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f0) : "h"((unsigned short)(h2 & 0xFFFFu)));
    asm("cvt.f32.f16 %0, %1;" : "=f"(f1) : "h"((unsigned short)(h2 >> 16)));
    o[i] = (__float_as_uint(f0) >> 16) | (__float_as_uint(f1) & 0xFFFF0000u);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}
// 16-B piece `sub` of a working-set row source: bf16 rows are read as is; a source pointer tagged in
// bit 0 is an E4M3 pool row (8 B per piece), converted
__device__ __forceinline__ uint4 load_row_piece(const uint4* p, int sub) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(p);
  if (u & 1u) return e4m3x8_to_bf16x8(reinterpret_cast<const uint2*>(u & ~(uintptr_t)1)[sub]);
  return p[sub];
}
__device__ __forceinline__ void unpack8(const uint4 u, float* f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xFFFF0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xFFFF0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xFFFF0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xFFFF0000u);
}
// ---- programmatic dependent launch: every kernel waits for its predecessor grid (memory visible)
// before touching shared state, then lets its dependent grid launch early (the launch latency of the
// next kernel overlaps this one; the dependent still waits at its own griddepcontrol.wait)
// (default on: measured -1..3 % on the C2 decode step; -DLKV_PDL_LATE_TRIGGER restores the implicit
// trigger at grid completion)
__device__ __forceinline__ void pdl_wait_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifndef LKV_PDL_LATE_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ---- optional phase timestamps (-DLKV_PROF builds only): thread 0 writes %globaltimer into slot
__device__ __forceinline__ void prof_stamp(unsigned long long* p, int slot) {
#ifdef LKV_PROF
  if (p && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p[slot] = g;
  }
#endif
}

// ---- mbarrier / bulk-copy (TMA engine) helpers
__device__ __forceinline__ uint32_t ptx_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ptx_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ptx_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void ptx_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ptx_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ptx_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(ptx_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy on the TMA engine; completes `bytes` of transaction on `bar`
__device__ __forceinline__ void ptx_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx_smem_u32(bar))
               : "memory");
}
// fp32 -> bf16 bits, round to nearest even (NaN-free inputs)
__device__ __forceinline__ uint16_t f2bf_rne(float x) {
  uint32_t u = __float_as_uint(x);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
}  // namespace lkv
#endif
