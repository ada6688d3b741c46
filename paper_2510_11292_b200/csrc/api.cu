// C ABI of the LouisKV B200 library: context, capacities, state machine, kernel sequencing.
// See include/louiskv.h for the contract of every entry point (paper citations there).
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lkv_internal.cuh"

using namespace lkv;

struct louiskv_ctx {
  louiskv_config cfg{};
  int L = 0, Hq = 0, Hkv = 0, h0 = 0, hn = 0, g = 0, Bmax = 0, S = 0, W = 0, Bud = 0, c = 0, iters = 0;
  int max_open = 0, ring_cap = 0, kmax = 0, Umax = 0, nchunk_max = 0;
  int64_t Pmax = 0, Mmax = 0, Nmax = 0, pool_rows_cap = 0, full_cap = 0;
  int n_r = 0, n_f = 0;
  std::vector<int> ridx, fidx;
  int batch = 0;
  std::vector<int64_t> P;
  std::vector<int> t, stage;
  int64_t n_inst = 0;  // n_r * Bmax * hn
  int inst_per_layer = 0;
  // device state
  InstState* d_inst = nullptr;
  bf16* d_sinks = nullptr;
  bf16* d_ws = nullptr;
  int64_t ws_buf_stride = 0, ws_inst_stride = 0;
  bf16* d_ring = nullptr;
  int2* d_fifo = nullptr;
  float* d_cent = nullptr;   // unit index (centroids); index_offload: device-mapped host memory
  bf16* d_centb = nullptr;
  float* h_cent = nullptr;   // index_offload: the pinned host arrays behind d_cent / d_centb
  bf16* h_centb = nullptr;
  float* d_km_cent = nullptr;  // index_offload: one layer's device k-means centroids, copied out after
  bf16* d_km_centb = nullptr;
  uint64_t index_host_bytes = 0;
  int32_t* d_usize = nullptr;
  int64_t* d_uoff = nullptr;
  int32_t* d_ufirst = nullptr;
  uint8_t* d_sel = nullptr;
  int32_t* d_seloff = nullptr;
  int32_t* d_pool_pos = nullptr;
  uint8_t* d_flag = nullptr;
  double* d_r = nullptr;
  bf16* d_qref = nullptr;
  bf16* d_full = nullptr;
  uint8_t* h_pool = nullptr;
  bool pool_registered = false;  // mmap + mbind + cudaHostRegister (NUMA-local) instead of cudaHostAlloc
  int pool_numa_node = -1;
  uint8_t* d_pool = nullptr;
  int64_t pool_inst_bytes = 0;
  // scratch
  float* d_se = nullptr;
  uint8_t* d_ssort = nullptr;
  RowSrc* d_rows = nullptr;
  GatherJob* d_jobs = nullptr;  // [L][Bmax*hn]
  // BATCHED_DMA fetch: span lists written by select into mapped pinned memory
  DmaSpan* h_spans = nullptr;
  int32_t* h_span_n = nullptr;
  DmaSpan* d_spans = nullptr;
  int32_t* d_span_n = nullptr;
  int dma_cap = 0;
  uint64_t dma_copies = 0;  // copies issued (louiskv_stats.dma_copies)
  int prb = POOL_ROW_BYTES;  // host-pool bytes per token (K + V): 512 bf16, 256 E4M3
  int sms = 148;             // SMs of the context's device (split-K grid sizing)
  float* d_part = nullptr;
  int* d_counters = nullptr;
  int max_splits = 64;
  float* d_km_half = nullptr;
  int32_t* d_km_assign = nullptr;
  float* d_km_dmin = nullptr;
  int32_t* d_km_cc = nullptr;
  int32_t* d_km_off = nullptr;
  int32_t* d_km_cnt = nullptr;
  int32_t* d_km_perm = nullptr;
  int32_t* d_km_tperm = nullptr;
  int32_t* d_km_flags = nullptr;
  int32_t* d_km_toff = nullptr;
  int4* d_km_tcl = nullptr;
  int32_t* d_km_ccT = nullptr;
  uint16_t* d_km_bext = nullptr;
  float* d_km_upart = nullptr;
  int km_task_max = 0;
  StatsDev* d_stats = nullptr;
  int* d_step = nullptr;   // [L] device decode-step counters (graph-replay safe)
  int* d_error = nullptr;  // device capacity-overflow flag
  uint64_t km_tc_iters = 0, km_simt_iters = 0;
  // prompt offload: cluster-major rows are staged on the device (double buffer) and moved into the
  // pinned pool by the copy engine on off_stream, overlapping the next layer's clustering
  uint8_t* d_stage[2] = {nullptr, nullptr};
  int64_t stage_bytes = 0;
  int stage_next = 0;
  bool stage_used[2] = {false, false};
  cudaStream_t off_stream = nullptr;
  cudaEvent_t ev_free[2] = {nullptr, nullptr}, ev_staged = nullptr;
  std::vector<cudaEvent_t> ev_done;  // [L] offload of layer l complete
  std::vector<char> off_pending;     // [L] a decode-path stream has not yet waited on ev_done[l]
  std::vector<void*> allocs;
  int last_layer = -1;  // layer of the last launch when it was a one-launch layer step, else -1
  void* last_stream = nullptr;  // ... and the stream it went to
  uint64_t dev_bytes = 0, host_bytes = 0;  // louiskv_get_memory
  PhaseRec prec;                            // louiskv_set_prefill_timing
  // decode-state checkpoint (louiskv_state_save / _restore): device copies of every buffer the decode
  // path writes that is not dead beyond the saved counters
  struct SnapBuf {
    void* src;
    size_t bytes;
    void* dst;
  };
  std::vector<SnapBuf> snap;
  bool snap_valid = false;
  std::vector<int> snap_t, snap_stage;
  std::string err;
  bool sticky = false;
};

namespace {

// NUMA node of the GPU's PCI device (sysfs), -1 if unknown; number of NUMA nodes of the host
int device_numa_node(int dev) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, (int)sizeof(bus), dev) != cudaSuccess) return -1;
  for (char* p = bus; *p; ++p) *p = (char)tolower(*p);
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = fopen(path.c_str(), "r");
  if (!f) return -1;
  int node = -1;
  if (fscanf(f, "%d", &node) != 1) node = -1;
  fclose(f);
  return node;
}
int numa_node_count() {
  int n = 0;
  for (int i = 0; i < 64; ++i) {
    std::string p = "/sys/devices/system/node/node" + std::to_string(i);
    if (access(p.c_str(), F_OK) == 0) ++n;
  }
  return n;
}
// The pinned pool on the GPU's NUMA node (multi-socket hosts: every GPU's host-link traffic stays on
// its own socket): anonymous mmap, MPOL_BIND to the node (raw mbind syscall, no libnuma), then pinned
// and mapped with cudaHostRegister. Returns nullptr (caller falls back to cudaHostAlloc) on any failure.
void* alloc_pool_numa(size_t bytes, int node) {
  if (node < 0 || node >= 64) return nullptr;
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  unsigned long mask = 1ul << node;
  const long MPOL_BIND_ = 2;
  if (syscall(SYS_mbind, p, bytes, MPOL_BIND_, &mask, (unsigned long)(sizeof(mask) * 8), 0) != 0) {
    munmap(p, bytes);
    return nullptr;
  }
  if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, bytes);
    return nullptr;
  }
  return p;
}

louiskv_status fail(louiskv_ctx* c, louiskv_status s, const std::string& m) {
  if (c) {
    c->err = m;
    if (s == LOUISKV_ERR_CUDA || s == LOUISKV_ERR_CAPACITY) c->sticky = true;
  }
  return s;
}

louiskv_status cuda_fail(louiskv_ctx* c, cudaError_t e, const char* where) {
  return fail(c, LOUISKV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

template <typename T>
bool dalloc(louiskv_ctx* c, T** p, size_t n) {
  if (n == 0) n = 1;
  void* v = nullptr;
  if (cudaMalloc(&v, n * sizeof(T)) != cudaSuccess) return false;
  cudaMemset(v, 0, n * sizeof(T));
  c->allocs.push_back(v);
  c->dev_bytes += n * sizeof(T);
  *p = reinterpret_cast<T*>(v);
  return true;
}

#define LKV_CHECK_CTX(c)                                                        \
  do {                                                                          \
    if (!(c)) return LOUISKV_ERR_INVALID_ARG;                                   \
    if ((c)->sticky) return fail((c), LOUISKV_ERR_CUDA, (c)->err);               \
    if (cudaSetDevice((c)->cfg.device) != cudaSuccess)                           \
      return fail((c), LOUISKV_ERR_CUDA, "cudaSetDevice failed");                \
  } while (0)

#define LKV_LAUNCH(c, expr, where)                            \
  do {                                                        \
    (c)->last_layer = -1;                                     \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return cuda_fail((c), _e, where);  \
  } while (0)

bool is_full(const louiskv_ctx* c, int layer) { return (c->cfg.full_cache_layers >> layer) & 1ull; }

int64_t inst_base(const louiskv_ctx* c, int layer) { return (int64_t)c->ridx[layer] * c->inst_per_layer; }

RetrieveArgs retrieve_args(louiskv_ctx* c, int layer, const void* q, int64_t stride_b) {
  const int64_t ib = inst_base(c, layer);
  RetrieveArgs a{};
  a.q_own = reinterpret_cast<const bf16*>(q);
  a.stride_b = stride_b;
  a.batch = c->batch;
  a.hn = c->hn;
  a.g = c->g;
  a.Umax = c->Umax;
  a.budget = c->Bud;
  a.Hq = c->Hq;
  a.h0 = c->h0;
  a.Bmax = c->Bmax;
  a.trigger_ref = c->cfg.trigger_ref;
  a.tau = c->cfg.tau;
  a.stride = c->cfg.trigger_stride;
  a.qref = c->d_qref + (size_t)layer * 2 * c->Bmax * c->Hq * D;
  a.r = c->d_r + (size_t)layer * c->Bmax;
  a.flag = c->d_flag + (size_t)layer * c->Bmax;
  a.inst = c->d_inst + ib;
  a.centb = c->d_centb + ib * c->Umax * D;
  a.usize = c->d_usize + ib * c->Umax;
  a.uoff = c->d_uoff + ib * c->Umax;
  a.sel = c->d_sel + ib * c->Umax;
  a.seloff = c->d_seloff + ib * c->Umax;
  a.pool = c->d_pool + ib * c->pool_inst_bytes;
  a.pool_inst_bytes = c->pool_inst_bytes;
  a.pool_fp8 = c->cfg.pool_dtype == LOUISKV_POOL_FP8_E4M3;
  a.ws = c->d_ws;
  a.ws_buf_stride = c->ws_buf_stride;
  a.ws_inst_stride = c->ws_inst_stride;
  a.inst_global_base = ib;
  a.scratch_e = c->d_se;
  a.scratch_sort = c->d_ssort;
  a.rows = c->d_rows;
  a.jobs = c->d_jobs + (size_t)layer * c->inst_per_layer;
  a.stats = c->d_stats;
  r3_coefs(a.r3c);
  a.inv_sqrt_d = (float)(1.0 / std::sqrt((double)D));
  return a;
}

AppendArgs append_args(louiskv_ctx* c, int layer, const void* k_t, const void* v_t, int64_t stride_b) {
  const int64_t ib = inst_base(c, layer);
  AppendArgs a{};
  a.k_t = reinterpret_cast<const bf16*>(k_t);
  a.v_t = reinterpret_cast<const bf16*>(v_t);
  a.stride_b = stride_b;
  a.batch = c->batch;
  a.hn = c->hn;
  a.W = c->W;
  a.max_open = c->max_open;
  a.ring_cap = c->ring_cap;
  a.Umax = c->Umax;
  a.flag = c->d_flag + (size_t)layer * c->Bmax;
  a.inst = c->d_inst + ib;
  a.ring = c->d_ring + ib * 2 * c->ring_cap * D;
  a.fifo = c->d_fifo + ib * c->ring_cap;
  a.cent = c->d_cent + ib * c->Umax * D;
  a.centb = c->d_centb + ib * c->Umax * D;
  a.usize = c->d_usize + ib * c->Umax;
  a.uoff = c->d_uoff + ib * c->Umax;
  a.ufirst = c->d_ufirst + ib * c->Umax;
  a.sel = c->d_sel + ib * c->Umax;
  a.pool_pos = c->d_pool_pos + ib * c->pool_rows_cap;
  a.pool_rows_cap = c->pool_rows_cap;
  a.pool = c->d_pool + ib * c->pool_inst_bytes;
  a.pool_inst_bytes = c->pool_inst_bytes;
  a.pool_fp8 = c->cfg.pool_dtype == LOUISKV_POOL_FP8_E4M3;
  a.stats = c->d_stats;
  a.jobs = c->d_jobs + (size_t)layer * c->inst_per_layer;
  a.rows = c->d_rows;
  a.budget = std::max(c->Bud, 1);
  return a;
}

AttnArgs attn_args(louiskv_ctx* c, int layer, const void* q_own, int64_t stride_b, void* out, float* out_f32) {
  AttnArgs a{};
  a.q_own = reinterpret_cast<const bf16*>(q_own);
  a.stride_b = stride_b;
  a.batch = c->batch;
  a.hn = c->hn;
  a.g = c->g;
  a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  a.out = reinterpret_cast<bf16*>(out);
  a.out_f32 = out_f32;
  a.part = c->d_part;
  a.counters = c->d_counters;
  const int n_ctas = c->batch * c->hn;
  int64_t max_rows;
  if (is_full(c, layer)) {
    a.full = c->d_full + (size_t)c->fidx[layer] * c->inst_per_layer * 2 * c->full_cap * D;
    a.full_cap = c->full_cap;
    a.full_P = c->P[layer];
    a.step = c->d_step + layer;
    max_rows = c->P[layer] + c->t[layer];
  } else {
    const int64_t ib = inst_base(c, layer);
    a.inst = c->d_inst + ib;
    a.sinks = c->d_sinks + ib * 2 * std::max(c->S, 1) * D;
    a.S = std::max(c->S, 1);
    a.ws = c->d_ws;
    a.ws_buf_stride = c->ws_buf_stride;
    a.ws_inst_stride = c->ws_inst_stride;
    a.inst_global_base = ib;
    a.B = std::max(c->Bud, 1);
    a.ring = c->d_ring + ib * 2 * c->ring_cap * D;
    a.ring_cap = c->ring_cap;
    max_rows = std::min<int64_t>(c->S, c->P[layer]) + c->Bud + c->ring_cap;
  }
  // split-K grid: splits per instance = floor(slots / instances), so the grid never spills into a
  // partial second wave (the ceiling of 296 / instances had left C4 a 24-CTA second wave: 413 us per
  // full-cache layer); slots = one CTA per SM for few instances (at most SMs / 4: fewer split partials
  // to merge — C2 33.5 -> 29.7 us, C5's share 167.6 -> 163.6 us), two per SM otherwise (C4: 318 us vs
  // 326 at one per SM). A split never ends with a tiny tail chunk (rows per split rounded to whole
  // 64-row pipeline chunks).
#ifdef FA_SPLIT_CTAS
  const int64_t slots = FA_SPLIT_CTAS;  // (experiments)
#else
  const int64_t slots = (int64_t)n_ctas * 4 <= c->sms ? c->sms : 2 * (int64_t)c->sms;
#endif
  const int64_t want = std::max<int64_t>(1, slots / n_ctas);
  const int64_t chunks = (max_rows + 63) / 64;
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(want, chunks));
  if (chunks > splits) splits = (int)((chunks + (chunks + splits - 1) / splits - 1) / ((chunks + splits - 1) / splits));
  a.splits = std::min(splits, c->max_splits);
  return a;
}

// BATCHED_DMA fetch (§4.3: selected rows moved by the DMA engines, the analogue of the paper's
// DGL row transfer): wait for select's span lists (mapped pinned memory), merge spans that are
// contiguous in both source and destination (runs of kept units; a new unit's K and V spans are
// adjacent in the pool but not in the working set), then one stream-ordered cudaMemcpyAsync per merged
// span — new units host pool -> next working set over the host link, kept units current -> next
// working set on the device. The copies are mutually independent (disjoint destinations).
cudaError_t batched_dma_fetch(louiskv_ctx* c, cudaStream_t st) {
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  const uint64_t dp = reinterpret_cast<uint64_t>(c->d_pool), hp = reinterpret_cast<uint64_t>(c->h_pool);
  uint64_t src0 = 0, dst0 = 0, len = 0;
  auto flush = [&]() -> cudaError_t {
    if (!len) return cudaSuccess;
    const cudaError_t r = cudaMemcpyAsync(reinterpret_cast<void*>(dst0), reinterpret_cast<const void*>(src0),
                                          (size_t)len, cudaMemcpyDefault, st);
    len = 0;
    return r;
  };
  const int ni = c->batch * c->hn;
  for (int li = 0; li < ni; ++li) {
    const int n = c->h_span_n[li];
    if (n < 0 || n > c->dma_cap) return cudaErrorIllegalState;
    const DmaSpan* sp = c->h_spans + (size_t)li * c->dma_cap;
    for (int i = 0; i < n; ++i) {
      uint64_t src = sp[i].src;
      // host-pool sources: device-mapped address -> the pool's host address
      if (c->d_pool && src >= dp && src < dp + c->host_bytes) src = hp + (src - dp);
      if (len && src == src0 + len && sp[i].dst == dst0 + len) {
        len += sp[i].bytes;
        continue;
      }
      if ((e = flush()) != cudaSuccess) return e;
      ++c->dma_copies;
      src0 = src;
      dst0 = sp[i].dst;
      len = sp[i].bytes;
    }
  }
  return flush();
}

}  // namespace

extern "C" {

const char* louiskv_version(void) { return "louiskv-b200 0.1 (sm_100a, tcgen05/TMEM k-means, zero-copy gather)"; }

const char* louiskv_last_error(const louiskv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void louiskv_destroy(louiskv_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  for (cudaEvent_t e : ctx->ev_done)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {ctx->ev_free[0], ctx->ev_free[1], ctx->ev_staged})
    if (e) cudaEventDestroy(e);
  if (ctx->off_stream) cudaStreamDestroy(ctx->off_stream);
  if (ctx->h_spans) cudaFreeHost(ctx->h_spans);
  if (ctx->h_cent) cudaFreeHost(ctx->h_cent);
  if (ctx->h_centb) cudaFreeHost(ctx->h_centb);
  if (ctx->h_span_n) cudaFreeHost(ctx->h_span_n);
  for (cudaEvent_t e : ctx->prec.pool)
    if (e) cudaEventDestroy(e);
  for (auto& sb : ctx->snap)
    if (sb.dst) cudaFree(sb.dst);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->h_pool) {
    if (ctx->pool_registered) {
      cudaHostUnregister(ctx->h_pool);
      munmap(ctx->h_pool, (size_t)ctx->host_bytes);
    } else {
      cudaFreeHost(ctx->h_pool);
    }
  }
  delete ctx;
}

louiskv_status louiskv_create(const louiskv_config* cfg, louiskv_ctx** out) {
  if (!cfg || !out) return LOUISKV_ERR_INVALID_ARG;
  *out = nullptr;
  const louiskv_config& k = *cfg;
  if (k.head_dim != D || k.num_layers <= 0 || k.num_layers > 64 || k.num_q_heads <= 0 || k.num_q_heads > 64 ||
      k.num_kv_heads <= 0 ||
      k.num_q_heads % k.num_kv_heads != 0 || k.kv_head_begin < 0 || k.kv_head_count <= 0 ||
      k.kv_head_begin + k.kv_head_count > k.num_kv_heads || k.max_batch <= 0 || k.max_prompt_len <= 0 ||
      k.max_output_len <= 0 || k.budget_tokens < 0 || k.sink_tokens < 0 || k.window_tokens < 1 ||
      k.avg_cluster_size < 1 || k.kmeans_iters < 0 || !(std::isfinite(k.tau)) || k.trigger_stride < 0 ||
      (k.prompt_units != LOUISKV_UNITS_KMEANS && k.prompt_units != LOUISKV_UNITS_PAGES) ||
      (k.fetch_mode != LOUISKV_FETCH_ZERO_COPY && k.fetch_mode != LOUISKV_FETCH_BATCHED_DMA) ||
      (k.index_offload != 0 && k.index_offload != 1) ||
      (k.pool_dtype != LOUISKV_POOL_BF16 && k.pool_dtype != LOUISKV_POOL_FP8_E4M3) ||
      (k.pool_dtype == LOUISKV_POOL_FP8_E4M3 && k.fetch_mode == LOUISKV_FETCH_BATCHED_DMA) ||
      (k.boundary_mode == LOUISKV_BOUNDARY_SHARED && (k.shared_layer < 0 || k.shared_layer >= k.num_layers)))
    return LOUISKV_ERR_INVALID_ARG;
  const int g = k.num_q_heads / k.num_kv_heads;
  if (g != 1 && g != 2 && g != 4 && g != 8) return LOUISKV_ERR_INVALID_ARG;
  if (k.max_prompt_len > (1ll << 30) || k.max_output_len > (1ll << 30)) return LOUISKV_ERR_INVALID_ARG;
  if (cudaSetDevice(k.device) != cudaSuccess) return LOUISKV_ERR_CUDA;

  louiskv_ctx* c = new louiskv_ctx();
  c->cfg = k;
  if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, k.device) != cudaSuccess || c->sms <= 0)
    c->sms = 148;
  c->L = k.num_layers;
  c->Hq = k.num_q_heads;
  c->Hkv = k.num_kv_heads;
  c->h0 = k.kv_head_begin;
  c->hn = k.kv_head_count;
  c->g = g;
  c->Bmax = k.max_batch;
  c->S = k.sink_tokens;
  c->W = k.window_tokens;
  c->Bud = k.budget_tokens;
  c->c = k.avg_cluster_size;
  c->iters = k.kmeans_iters;
  c->max_open = k.max_open_segment > 0 ? k.max_open_segment : k.window_tokens;
  c->ring_cap = std::max(c->W, c->max_open) + 2;
  c->Pmax = k.max_prompt_len;
  c->Mmax = k.max_output_len;
  c->Nmax = std::max<int64_t>(0, c->Pmax - c->S);
  c->kmax = (int)((c->Nmax + c->c - 1) / c->c);
  // unit-table rows padded to whole 256-row centroid tiles (the tcgen05 k-means TMA box)
  c->Umax = (int)((((int64_t)c->kmax + c->Mmax) + 255) / 256 * 256);
  if (c->Umax > (1 << 16) || k.budget_tokens > 65534) {  // 16-bit unit ids / sizes in the selection
    delete c;
    return LOUISKV_ERR_INVALID_ARG;
  }
  c->nchunk_max = (int)((c->Nmax + 1023) / 1024);
  c->pool_rows_cap = c->Nmax + c->Mmax;
  c->full_cap = c->Pmax + c->Mmax;
  c->ridx.assign(c->L, -1);
  c->fidx.assign(c->L, -1);
  for (int l = 0; l < c->L; ++l) {
    if (is_full(c, l))
      c->fidx[l] = c->n_f++;
    else
      c->ridx[l] = c->n_r++;
  }
  c->P.assign(c->L, -1);
  c->t.assign(c->L, 0);
  c->stage.assign(c->L, 0);
  c->inst_per_layer = c->Bmax * c->hn;
  c->n_inst = (int64_t)c->n_r * c->inst_per_layer;
  const int64_t ni = c->n_inst, nl = c->inst_per_layer;

  bool ok = true;
  ok = ok && dalloc(c, &c->d_inst, ni);
  ok = ok && dalloc(c, &c->d_sinks, (size_t)ni * 2 * std::max(c->S, 1) * D);
  c->ws_inst_stride = (int64_t)2 * std::max(c->Bud, 1) * D;
  c->ws_buf_stride = ni * c->ws_inst_stride;
  ok = ok && dalloc(c, &c->d_ws, (size_t)2 * c->ws_buf_stride);
  ok = ok && dalloc(c, &c->d_ring, (size_t)ni * 2 * c->ring_cap * D);
  ok = ok && dalloc(c, &c->d_fifo, (size_t)ni * c->ring_cap);
  if (k.index_offload) {
    // the unit index in pinned, device-mapped host memory (the paper's future work): scoring
    // reads the centroid rows over the host link; k-means runs on one layer's device scratch
    const size_t ne = std::max<size_t>((size_t)ni * c->Umax * D, 1);
    void *hc = nullptr, *hb = nullptr, *dc = nullptr, *db = nullptr;
    ok = ok && cudaHostAlloc(&hc, ne * sizeof(float), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess &&
         cudaHostAlloc(&hb, ne * sizeof(bf16), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess;
    c->h_cent = reinterpret_cast<float*>(hc);
    c->h_centb = reinterpret_cast<bf16*>(hb);
    if (ok) {
      memset(hc, 0, ne * sizeof(float));
      memset(hb, 0, ne * sizeof(bf16));
      c->index_host_bytes = ne * (sizeof(float) + sizeof(bf16));
    }
    ok = ok && cudaHostGetDevicePointer(&dc, hc, 0) == cudaSuccess && cudaHostGetDevicePointer(&db, hb, 0) == cudaSuccess;
    c->d_cent = reinterpret_cast<float*>(dc);
    c->d_centb = reinterpret_cast<bf16*>(db);
    if (!ok) cudaGetLastError();
    ok = ok && dalloc(c, &c->d_km_cent, (size_t)nl * c->Umax * D);
    ok = ok && dalloc(c, &c->d_km_centb, (size_t)nl * c->Umax * D);
  } else {
    ok = ok && dalloc(c, &c->d_cent, (size_t)ni * c->Umax * D);
    ok = ok && dalloc(c, &c->d_centb, (size_t)ni * c->Umax * D);
  }
  ok = ok && dalloc(c, &c->d_usize, (size_t)ni * c->Umax);
  ok = ok && dalloc(c, &c->d_uoff, (size_t)ni * c->Umax);
  ok = ok && dalloc(c, &c->d_ufirst, (size_t)ni * c->Umax);
  ok = ok && dalloc(c, &c->d_sel, (size_t)ni * c->Umax);
  ok = ok && dalloc(c, &c->d_seloff, (size_t)ni * c->Umax);
  ok = ok && dalloc(c, &c->d_pool_pos, (size_t)ni * c->pool_rows_cap);
  ok = ok && dalloc(c, &c->d_flag, (size_t)c->L * c->Bmax);
  ok = ok && dalloc(c, &c->d_r, (size_t)c->L * c->Bmax);
  ok = ok && dalloc(c, &c->d_qref, (size_t)c->L * 2 * c->Bmax * c->Hq * D);
  ok = ok && dalloc(c, &c->d_full, (size_t)c->n_f * nl * 2 * c->full_cap * D);
  ok = ok && dalloc(c, &c->d_se, (size_t)nl * g * c->Umax);
  ok = ok && dalloc(c, &c->d_ssort, (size_t)nl * c->Umax * 26);
  ok = ok && dalloc(c, &c->d_rows, (size_t)nl * std::max(c->Bud, 1));
  ok = ok && dalloc(c, &c->d_jobs, (size_t)c->L * nl);
  ok = ok && dalloc(c, &c->d_part, (size_t)nl * c->max_splits * g * (D + 4));  // (>= every kernel's partial stride)
  ok = ok && dalloc(c, &c->d_counters, (size_t)nl + 1);  // + the fused full-cache step's layer ticket
  ok = ok && dalloc(c, &c->d_km_half, (size_t)nl * (((std::max(c->kmax, 1) + 255) / 256) * 256));
  ok = ok && dalloc(c, &c->d_km_assign, (size_t)nl * std::max<int64_t>(c->Nmax, 1));
  ok = ok && dalloc(c, &c->d_km_dmin, (size_t)nl * std::max<int64_t>(c->Nmax, 1));
  ok = ok && dalloc(c, &c->d_km_cc, (size_t)nl * std::max(c->nchunk_max, 1) * std::max(c->kmax, 1));
  ok = ok && dalloc(c, &c->d_km_off, (size_t)nl * (c->kmax + 1));
  ok = ok && dalloc(c, &c->d_km_cnt, (size_t)nl * std::max(c->kmax, 1));
  ok = ok && dalloc(c, &c->d_km_perm, (size_t)nl * std::max<int64_t>(c->Nmax, 1));
  ok = ok && dalloc(c, &c->d_km_flags, (size_t)nl);
  c->km_task_max = std::max(c->kmax, 1) + (int)((c->Nmax + 31) / 32);
  ok = ok && dalloc(c, &c->d_km_toff, (size_t)nl * (c->kmax + 1));
  ok = ok && dalloc(c, &c->d_km_tcl, (size_t)nl * c->km_task_max);
  ok = ok && dalloc(c, &c->d_km_tperm, (size_t)nl * c->km_task_max * 32);
  ok = ok && dalloc(c, &c->d_km_bext, (size_t)nl * c->Umax * 8);
  ok = ok && dalloc(c, &c->d_km_ccT, (size_t)nl * std::max(c->nchunk_max, 1) * std::max(c->kmax, 1));
  ok = ok && dalloc(c, &c->d_km_upart, (size_t)nl * c->km_task_max * D);
  ok = ok && dalloc(c, &c->d_stats, 1);
  ok = ok && dalloc(c, &c->d_step, (size_t)c->L);
  ok = ok && dalloc(c, &c->d_error, 1);
  {
    // staging for the prompt offload: whole layers up to 256 MiB per buffer, else instance chunks
    const int64_t inst_b = std::max<int64_t>(c->Nmax, 1) * POOL_ROW_BYTES;
    c->stage_bytes = std::max<int64_t>(inst_b, std::min<int64_t>(inst_b * nl, 256ll << 20));
    if (c->n_r > 0 && c->Nmax > 0) {
      ok = ok && dalloc(c, &c->d_stage[0], (size_t)c->stage_bytes);
      ok = ok && dalloc(c, &c->d_stage[1], (size_t)c->stage_bytes);
    }
    ok = ok && cudaStreamCreateWithFlags(&c->off_stream, cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_free[0], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_free[1], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming) == cudaSuccess;
    c->ev_done.assign(c->L, nullptr);
    c->off_pending.assign(c->L, 0);
    for (int l = 0; l < c->L && ok; ++l)
      ok = cudaEventCreateWithFlags(&c->ev_done[l], cudaEventDisableTiming) == cudaSuccess;
  }
  if (ok && k.fetch_mode == LOUISKV_FETCH_BATCHED_DMA) {
    c->dma_cap = 2 * std::max(c->Bud, 1);
    void *hs = nullptr, *hn_ = nullptr, *ds = nullptr, *dn = nullptr;
    ok = cudaHostAlloc(&hs, sizeof(DmaSpan) * nl * c->dma_cap, cudaHostAllocMapped) == cudaSuccess &&
         cudaHostAlloc(&hn_, sizeof(int32_t) * nl, cudaHostAllocMapped) == cudaSuccess;
    c->h_spans = reinterpret_cast<DmaSpan*>(hs);
    c->h_span_n = reinterpret_cast<int32_t*>(hn_);
    ok = ok && cudaHostGetDevicePointer(&ds, hs, 0) == cudaSuccess &&
         cudaHostGetDevicePointer(&dn, hn_, 0) == cudaSuccess;
    c->d_spans = reinterpret_cast<DmaSpan*>(ds);
    c->d_span_n = reinterpret_cast<int32_t*>(dn);
    if (!ok) cudaGetLastError();
  }
  if (!ok) {
    louiskv_destroy(c);
    return LOUISKV_ERR_OOM_DEVICE;
  }
  c->prb = pool_row_bytes(k.pool_dtype == LOUISKV_POOL_FP8_E4M3);
  c->pool_inst_bytes = c->pool_rows_cap * c->prb;
  const size_t pool_bytes = (size_t)std::max<int64_t>(ni, 1) * c->pool_inst_bytes;
  if (pool_bytes > 0) {
    void* hp = nullptr;
    // NUMA-local pool on multi-node hosts (LOUISKV_POOL_NUMA=0 disables, =1 forces it on one node)
    const char* ne = getenv("LOUISKV_POOL_NUMA");
    const int numa_mode = ne ? atoi(ne) : -1;
    int node = device_numa_node(k.device);
    if (numa_mode == 1 && node < 0) node = 0;  // (forced on a host whose sysfs reports no node)
    if (numa_mode != 0 && node >= 0 && (numa_mode == 1 || numa_node_count() > 1)) {
      hp = alloc_pool_numa(pool_bytes, node);
      if (hp) {
        c->pool_registered = true;
        c->pool_numa_node = node;
      }
    }
    if (!hp && cudaHostAlloc(&hp, pool_bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      louiskv_destroy(c);
      return LOUISKV_ERR_OOM_HOST;
    }
    c->h_pool = reinterpret_cast<uint8_t*>(hp);
    c->host_bytes = pool_bytes;
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, hp, 0) != cudaSuccess) {
      louiskv_destroy(c);
      return LOUISKV_ERR_CUDA;
    }
    c->d_pool = reinterpret_cast<uint8_t*>(dp);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    louiskv_destroy(c);
    return LOUISKV_ERR_CUDA;
  }
  *out = c;
  return LOUISKV_OK;
}

// Prompt offload: stage the cluster-major K/V rows of a chunk of instances on the
// device, then one strided copy-engine transfer into the pinned pool on off_stream. Two staging
// buffers alternate, so the D2H of layer l overlaps the clustering of layer l+1; the decode-path
// calls of layer l wait on ev_done[l] (offload_wait).
static cudaError_t offload_prompt(louiskv_ctx* c, int layer, const KmArgs& a, cudaStream_t st) {
  cudaError_t e;
  const int ni = a.batch * a.hn;
  c->prec.mark(st, PH_STAGE);
  if (a.N > 0 && a.kc > 0) {
    const int64_t inst_b = (int64_t)a.N * c->prb;
    const int per = (int)std::max<int64_t>(1, std::min<int64_t>(ni, c->stage_bytes / inst_b));
    const int64_t ib = inst_base(c, layer);
    for (int li0 = 0; li0 < ni; li0 += per) {
      const int nli = std::min(per, ni - li0);
      const int buf = c->stage_next;
      c->stage_next ^= 1;
      if (c->stage_used[buf] && (e = cudaStreamWaitEvent(st, c->ev_free[buf], 0)) != cudaSuccess) return e;
      if ((e = launch_km_offload(a, li0, nli, c->d_stage[buf], inst_b, st)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(c->ev_staged, st)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(c->off_stream, c->ev_staged, 0)) != cudaSuccess) return e;
      cudaEvent_t d0 = nullptr, d1 = nullptr;
      if (c->prec.on && (d0 = c->prec.ev()) && (d1 = c->prec.ev())) cudaEventRecord(d0, c->off_stream);
      if ((e = cudaMemcpy2DAsync(c->h_pool + (ib + li0) * c->pool_inst_bytes, (size_t)c->pool_inst_bytes,
                                 c->d_stage[buf], (size_t)inst_b, (size_t)inst_b, (size_t)nli,
                                 cudaMemcpyDeviceToHost, c->off_stream)) != cudaSuccess)
        return e;
      if (d0 && d1) {
        cudaEventRecord(d1, c->off_stream);
        c->prec.d2h.push_back({d0, d1});
        c->prec.d2h_bytes += (uint64_t)inst_b * nli;
      }
      if ((e = cudaEventRecord(c->ev_free[buf], c->off_stream)) != cudaSuccess) return e;
      c->stage_used[buf] = true;
    }
    if ((e = launch_km_units(a, st)) != cudaSuccess) return e;
  }
  c->prec.mark(st, PH_END);
  if ((e = cudaEventRecord(c->ev_done[layer], c->off_stream)) != cudaSuccess) return e;
  c->off_pending[layer] = 1;
  return cudaSuccess;
}

// Make `st` wait for the prompt offload of `layer` (once; inside a graph capture the wait becomes an
// external event-wait node, which is free once the offload has completed).
static cudaError_t offload_wait(louiskv_ctx* c, int layer, cudaStream_t st) {
  if (!c->off_pending[layer]) return cudaSuccess;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  if (cs == cudaStreamCaptureStatusActive) return cudaStreamWaitEvent(st, c->ev_done[layer], cudaEventWaitExternal);
  e = cudaStreamWaitEvent(st, c->ev_done[layer], 0);
  if (e == cudaSuccess) c->off_pending[layer] = 0;
  return e;
}

static louiskv_status prompt_common(louiskv_ctx* c, int32_t layer, const void* k, const void* v, int64_t sb,
                                    int64_t st_, int64_t sh, int32_t batch, int64_t P, int32_t n_clusters,
                                    const int32_t* h_assign, const float* h_cent, void* stream) {
  LKV_CHECK_CTX(c);
  c->last_layer = -1;  // (prefill kernels follow: no early prologue for the next decode launch)
  if (layer < 0 || layer >= c->L || !k || !v || batch <= 0 || batch > c->Bmax || P < 0 || P > c->Pmax)
    return fail(c, LOUISKV_ERR_INVALID_ARG, "cluster_prompt: bad layer/pointer/batch/prompt_len");
  if (c->batch != 0 && batch != c->batch)
    return fail(c, LOUISKV_ERR_INVALID_ARG, "cluster_prompt: batch differs from an earlier layer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  c->batch = batch;
  c->P[layer] = P;
  c->t[layer] = 0;
  c->stage[layer] = 0;
  LKV_LAUNCH(c, cudaMemsetAsync(c->d_qref + (size_t)layer * 2 * c->Bmax * c->Hq * D, 0,
                                 sizeof(bf16) * 2 * c->Bmax * c->Hq * D, st),
             "memset q_ref");
  LKV_LAUNCH(c, cudaMemsetAsync(c->d_flag + (size_t)layer * c->Bmax, 0, c->Bmax, st), "memset flag");
  LKV_LAUNCH(c, cudaMemsetAsync(c->d_step + layer, 0, sizeof(int), st), "memset step");
  LKV_LAUNCH(c, cudaMemsetAsync(c->d_jobs + (size_t)layer * c->inst_per_layer, 0, sizeof(GatherJob) * c->inst_per_layer, st),
             "memset jobs");
  if (is_full(c, layer)) {
    if (h_assign) return fail(c, LOUISKV_ERR_INVALID_ARG, "set_prompt_units on a full-cache layer");
    LKV_LAUNCH(c,
               launch_full_prompt(reinterpret_cast<const bf16*>(k), reinterpret_cast<const bf16*>(v), sb, st_, sh, batch,
                                  c->hn, P, c->d_full + (size_t)c->fidx[layer] * c->inst_per_layer * 2 * c->full_cap * D,
                                  c->full_cap, st),
               "full prompt");
    return LOUISKV_OK;
  }
  const int64_t N = std::max<int64_t>(0, P - c->S);
  const int kc = N > 0 ? (int)((N + c->c - 1) / c->c) : 0;
  const int64_t ib = inst_base(c, layer);
  KmArgs a{};
  a.k = reinterpret_cast<const bf16*>(k);
  a.v = reinterpret_cast<const bf16*>(v);
  a.sb = sb;
  a.st = st_;
  a.sh = sh;
  a.batch = batch;
  a.hn = c->hn;
  a.S = (int)std::min<int64_t>(c->S, P);
  a.N = (int)N;
  a.kc = kc;
  a.iters = c->iters;
  a.impl = c->cfg.kmeans_impl;
  a.page = c->cfg.prompt_units == LOUISKV_UNITS_PAGES ? c->cfg.avg_cluster_size : 0;
  const bool idx_off = c->cfg.index_offload != 0;
  a.cent = idx_off ? c->d_km_cent : c->d_cent + ib * c->Umax * D;
  a.centb = idx_off ? c->d_km_centb : c->d_centb + ib * c->Umax * D;
  a.Umax = c->Umax;
  a.usize = c->d_usize + ib * c->Umax;
  a.uoff = c->d_uoff + ib * c->Umax;
  a.ufirst = c->d_ufirst + ib * c->Umax;
  a.sel = c->d_sel + ib * c->Umax;
  a.pool_pos = c->d_pool_pos + ib * c->pool_rows_cap;
  a.pool_rows_cap = c->pool_rows_cap;
  a.pool = c->d_pool + ib * c->pool_inst_bytes;
  a.pool_inst_bytes = c->pool_inst_bytes;
  a.pool_fp8 = c->cfg.pool_dtype == LOUISKV_POOL_FP8_E4M3;
  a.sinks = c->d_sinks + ib * 2 * std::max(c->S, 1) * D;
  a.S_cap = c->S;
  a.inst = c->d_inst + ib;
  a.half = c->d_km_half;
  a.hstride = ((std::max(c->kmax, 1) + 255) / 256) * 256;
  a.assign = c->d_km_assign;
  a.dmin = c->d_km_dmin;
  a.cc = c->d_km_cc;
  a.off = c->d_km_off;
  a.cnt = c->d_km_cnt;
  a.perm = c->d_km_perm;
  a.tperm = c->d_km_tperm;
  a.flags = c->d_km_flags;
  a.toff = c->d_km_toff;
  a.tcl = c->d_km_tcl;
  a.ccT = c->d_km_ccT;
  a.bext = c->d_km_bext;
  a.upart = c->d_km_upart;
  a.task_max = c->km_task_max;
  a.Nmax = std::max<int64_t>(c->Nmax, 1);
  a.kmax = std::max(c->kmax, 1);
  a.nchunk_max = std::max(c->nchunk_max, 1);
  a.stats = c->d_stats;
  int32_t* d_ea = nullptr;
  float* d_ec = nullptr;
  if (h_assign) {
    if (n_clusters != kc) return fail(c, LOUISKV_ERR_INVALID_ARG, "set_prompt_units: n_clusters != ceil((P-S)/c)");
    const size_t na = (size_t)batch * c->hn * N, nc = (size_t)batch * c->hn * kc * D;
    for (size_t i = 0; i < na; ++i)
      if (h_assign[i] < 0 || h_assign[i] >= kc) return fail(c, LOUISKV_ERR_INVALID_ARG, "set_prompt_units: id out of range");
    if (cudaMalloc(&d_ea, std::max<size_t>(na, 1) * 4) != cudaSuccess ||
        cudaMalloc(&d_ec, std::max<size_t>(nc, 1) * 4) != cudaSuccess)
      return fail(c, LOUISKV_ERR_OOM_DEVICE, "set_prompt_units scratch");
    cudaMemcpy(d_ea, h_assign, na * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ec, h_cent, nc * 4, cudaMemcpyHostToDevice);
    a.ext_assign = d_ea;
    a.ext_cent = d_ec;
  }
  if (c->prec.on) {
    a.rec = &c->prec;
    c->prec.mark(st, PH_INIT);
    c->prec.keys += (uint64_t)batch * c->hn * N;
    c->prec.calls += 1;
  }
  cudaError_t e = run_kmeans_prompt(a, st, &c->km_tc_iters, &c->km_simt_iters);
  if (e == cudaSuccess && idx_off) {
    // the layer's centroids (fp32 master + bf16 scoring copy) out to the host-resident index
    const size_t ne = (size_t)batch * c->hn * c->Umax * D;
    e = cudaMemcpyAsync(c->h_cent + ib * c->Umax * D, c->d_km_cent, ne * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(c->h_centb + ib * c->Umax * D, c->d_km_centb, ne * sizeof(bf16), cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = offload_prompt(c, layer, a, st);
  if (h_assign) {
    cudaStreamSynchronize(st);
    cudaFree(d_ea);
    cudaFree(d_ec);
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "cluster_prompt");
  return LOUISKV_OK;
}

louiskv_status louiskv_cluster_prompt(louiskv_ctx* ctx, int32_t layer, const void* k, const void* v, int64_t stride_b,
                                      int64_t stride_t, int64_t stride_h, int32_t batch, int64_t prompt_len,
                                      void* stream) {
  return prompt_common(ctx, layer, k, v, stride_b, stride_t, stride_h, batch, prompt_len, 0, nullptr, nullptr, stream);
}

louiskv_status louiskv_set_prompt_units(louiskv_ctx* ctx, int32_t layer, const void* k, const void* v, int64_t stride_b,
                                        int64_t stride_t, int64_t stride_h, int32_t batch, int64_t prompt_len,
                                        int32_t n_clusters, const int32_t* h_assign, const float* h_centroids,
                                        void* stream) {
  if (!h_assign || !h_centroids) return fail(ctx, LOUISKV_ERR_INVALID_ARG, "set_prompt_units: null host arrays");
  return prompt_common(ctx, layer, k, v, stride_b, stride_t, stride_h, batch, prompt_len, n_clusters, h_assign,
                       h_centroids, stream);
}

louiskv_status louiskv_should_retrieve(louiskv_ctx* c, int32_t layer, const void* q_all, int64_t stride_b,
                                       uint8_t* d_flag_out, double* d_r_out, void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !q_all) return fail(c, LOUISKV_ERR_INVALID_ARG, "should_retrieve: bad args");
  if (c->P[layer] < 0) return fail(c, LOUISKV_ERR_STATE, "should_retrieve before cluster_prompt");
  if (c->stage[layer] != 0 && c->stage[layer] != 3)
    return fail(c, LOUISKV_ERR_STATE, "should_retrieve: previous step incomplete");
  if (c->t[layer] >= c->Mmax) return fail(c, LOUISKV_ERR_STATE, "should_retrieve: max_output_len reached");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
  const int t = c->t[layer] + 1;
  if (is_full(c, layer)) {
    // full-cache layers never retrieve; the step counter advances in append_output
    if (d_flag_out) LKV_LAUNCH(c, cudaMemsetAsync(d_flag_out, 0, c->batch, st), "flags");
    if (d_r_out) LKV_LAUNCH(c, cudaMemsetAsync(d_r_out, 0, sizeof(double) * c->batch, st), "r");
  } else {
    RetrieveArgs a = retrieve_args(c, layer, q_all, stride_b);
    a.flag_out = d_flag_out;
    a.r_out = d_r_out;
    if (c->cfg.boundary_mode == LOUISKV_BOUNDARY_SHARED && layer != c->cfg.shared_layer) {
      const int sl = c->cfg.shared_layer;
      if (c->t[sl] < t) return fail(c, LOUISKV_ERR_STATE, "SHARED: designated layer not yet called this step");
      a.shared_copy = 1;
      a.flag_src = c->d_flag + (size_t)sl * c->Bmax;
      a.r_src = c->d_r + (size_t)sl * c->Bmax;
    }
    LKV_LAUNCH(c, launch_trigger_logits(a, st), "trigger+logits");
  }
  c->t[layer] = t;
  c->stage[layer] = 1;
  return LOUISKV_OK;
}

louiskv_status louiskv_retrieve(louiskv_ctx* c, int32_t layer, const void* q_own, int64_t stride_b, void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !q_own) return fail(c, LOUISKV_ERR_INVALID_ARG, "retrieve: bad args");
  if (c->stage[layer] != 1) return fail(c, LOUISKV_ERR_STATE, "retrieve must follow should_retrieve");
  c->stage[layer] = 2;
  if (is_full(c, layer)) return LOUISKV_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
  RetrieveArgs a = retrieve_args(c, layer, q_own, stride_b);
  a.budget = std::max(c->Bud, 0);
  if (c->cfg.fetch_mode == LOUISKV_FETCH_BATCHED_DMA) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LKV_LAUNCH(c, cudaStreamIsCapturing(st, &cs), "retrieve: capture status");
    if (cs != cudaStreamCaptureStatusNone)
      return fail(c, LOUISKV_ERR_STATE, "retrieve: BATCHED_DMA synchronises the host and cannot be graph-captured");
    a.dma_spans = c->d_spans;
    a.dma_n = c->d_span_n;
    a.dma_cap = c->dma_cap;
    LKV_LAUNCH(c, launch_select_gather(a, st), "select (span list)");
    LKV_LAUNCH(c, batched_dma_fetch(c, st), "batched DMA fetch");
    return LOUISKV_OK;
  }
  LKV_LAUNCH(c, launch_select_gather(a, st), "select+gather");
  return LOUISKV_OK;
}

louiskv_status louiskv_append_output(louiskv_ctx* c, int32_t layer, const void* k_t, const void* v_t, int64_t stride_b,
                                     void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !k_t || !v_t) return fail(c, LOUISKV_ERR_INVALID_ARG, "append_output: bad args");
  if (c->stage[layer] != 1 && c->stage[layer] != 2)
    return fail(c, LOUISKV_ERR_STATE, "append_output must follow should_retrieve/retrieve");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");

  if (is_full(c, layer)) {
    LKV_LAUNCH(c,
               launch_full_step(reinterpret_cast<const bf16*>(k_t), reinterpret_cast<const bf16*>(v_t), stride_b,
                                c->batch, c->hn,
                                c->d_full + (size_t)c->fidx[layer] * c->inst_per_layer * 2 * c->full_cap * D,
                                c->full_cap, c->P[layer], c->d_step + layer, c->d_error, st),
               "full step");
  } else {
    AppendArgs a = append_args(c, layer, k_t, v_t, stride_b);
    LKV_LAUNCH(c, launch_append(a, st), "append");
  }
  c->stage[layer] = 3;
  return LOUISKV_OK;
}

louiskv_status louiskv_sparse_attn(louiskv_ctx* c, int32_t layer, const void* q_own, int64_t stride_b, void* out,
                                   float* out_f32, void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !q_own || !out) return fail(c, LOUISKV_ERR_INVALID_ARG, "sparse_attn: bad args");
  if (c->stage[layer] != 3) return fail(c, LOUISKV_ERR_STATE, "sparse_attn must follow append_output");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
  AttnArgs a = attn_args(c, layer, q_own, stride_b, out, out_f32);
  if (is_full(c, layer) && c->cfg.attn_impl != LOUISKV_ATTN_SIMT) {
    const cudaError_t e = launch_attn_full_tc(a, c->inst_per_layer, st);
    if (e == cudaSuccess) return LOUISKV_OK;
    if (e != cudaErrorNotSupported) return cuda_fail(c, e, "attn (tensor cores)");
  }
  LKV_LAUNCH(c, launch_attn(a, st), "attn");
  return LOUISKV_OK;
}

louiskv_status louiskv_append_attn(louiskv_ctx* c, int32_t layer, const void* k_t, const void* v_t,
                                  int64_t stride_kv, const void* q_own, int64_t stride_q, void* out, float* out_f32,
                                  void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !k_t || !v_t || !q_own || !out)
    return fail(c, LOUISKV_ERR_INVALID_ARG, "append_attn: bad args");
  if (is_full(c, layer)) {
    louiskv_status s = louiskv_append_output(c, layer, k_t, v_t, stride_kv, stream);
    if (s != LOUISKV_OK) return s;
    return louiskv_sparse_attn(c, layer, q_own, stride_q, out, out_f32, stream);
  }
  if (c->stage[layer] != 1 && c->stage[layer] != 2)
    return fail(c, LOUISKV_ERR_STATE, "append_attn must follow should_retrieve/retrieve");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
  AttnArgs a = attn_args(c, layer, q_own, stride_q, out, out_f32);
  a.fused = 1;
  a.app = append_args(c, layer, k_t, v_t, stride_kv);
  LKV_LAUNCH(c, launch_attn(a, st), "append+attn");
  c->stage[layer] = 3;
  return LOUISKV_OK;
}

louiskv_status louiskv_decode_layer(louiskv_ctx* c, int32_t layer, const void* q_all, int64_t stride_q,
                                    const void* k_t, const void* v_t, int64_t stride_kv, void* out, float* out_f32,
                                    uint8_t* d_flag_out, double* d_r_out, void* stream) {
  LKV_CHECK_CTX(c);
  if (layer < 0 || layer >= c->L || !q_all || !k_t || !v_t || !out)
    return fail(c, LOUISKV_ERR_INVALID_ARG, "decode_layer: bad args");
  const void* q_own = reinterpret_cast<const bf16*>(q_all) + (int64_t)c->h0 * c->g * D;
  // the previous launch on this context was another layer's one-launch step: PDL-early prologue allowed
  // (same stream only: PDL orders a kernel after its predecessor in its own stream)
  const int early = (c->last_layer >= 0 && c->last_layer != layer && c->last_stream == stream) ? 1 : 0;
  if (is_full(c, layer) && c->cfg.attn_impl != LOUISKV_ATTN_SIMT) {
    // full-cache layer: ONE launch — flags 0, store_cache of (k_t, v_t), dense attention, step commit
    if (c->P[layer] < 0) return fail(c, LOUISKV_ERR_STATE, "decode_layer before cluster_prompt");
    if (c->stage[layer] != 0 && c->stage[layer] != 3)
      return fail(c, LOUISKV_ERR_STATE, "decode_layer: previous step incomplete");
    if (c->t[layer] >= c->Mmax) return fail(c, LOUISKV_ERR_STATE, "decode_layer: max_output_len reached");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
    AttnArgs a = attn_args(c, layer, q_own, stride_q, out, out_f32);
    FullStepArgs fs{reinterpret_cast<const bf16*>(k_t), reinterpret_cast<const bf16*>(v_t), stride_kv, c->d_error,
                    d_flag_out, d_r_out, c->batch};
    const cudaError_t e = launch_attn_full_tc(a, c->inst_per_layer, st, &fs);
    if (e == cudaSuccess) {
      c->last_layer = layer;
      c->last_stream = stream;
      c->t[layer] += 1;
      c->stage[layer] = 3;
      return LOUISKV_OK;
    }
    if (e != cudaErrorNotSupported) return cuda_fail(c, e, "full-cache step (tensor cores)");
  }
  if (is_full(c, layer) || std::min(c->Umax, c->Bud) > LAYER_REP_SEL || c->Hq > 64 ||
      c->cfg.fetch_mode == LOUISKV_FETCH_BATCHED_DMA) {
    // full-cache layer (SIMT attention), a budget / head count beyond the single launch, or the
    // host-issued batched DMA fetch (the selection must reach the host between select and attention)
    louiskv_status s = louiskv_should_retrieve(c, layer, q_all, stride_q, d_flag_out, d_r_out, stream);
    if (s == LOUISKV_OK) s = louiskv_retrieve(c, layer, q_own, stride_q, stream);
    if (s == LOUISKV_OK) s = louiskv_append_attn(c, layer, k_t, v_t, stride_kv, q_own, stride_q, out, out_f32, stream);
    return s;
  }
  if (c->P[layer] < 0) return fail(c, LOUISKV_ERR_STATE, "decode_layer before cluster_prompt");
  if (c->stage[layer] != 0 && c->stage[layer] != 3)
    return fail(c, LOUISKV_ERR_STATE, "decode_layer: previous step incomplete");
  if (c->t[layer] >= c->Mmax) return fail(c, LOUISKV_ERR_STATE, "decode_layer: max_output_len reached");
  const int t = c->t[layer] + 1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LKV_LAUNCH(c, offload_wait(c, layer, st), "prompt offload wait");
  LayerArgs la{};
  la.r = retrieve_args(c, layer, q_all, stride_q);
  la.r.budget = std::max(c->Bud, 0);
  la.r.flag_out = d_flag_out;
  la.r.r_out = d_r_out;
  if (c->cfg.boundary_mode == LOUISKV_BOUNDARY_SHARED && layer != c->cfg.shared_layer) {
    const int sl = c->cfg.shared_layer;
    if (c->t[sl] < t) return fail(c, LOUISKV_ERR_STATE, "SHARED: designated layer not yet called this step");
    la.r.shared_copy = 1;
    la.r.flag_src = c->d_flag + (size_t)sl * c->Bmax;
    la.r.r_src = c->d_r + (size_t)sl * c->Bmax;
  }
  la.at = attn_args(c, layer, q_own, stride_q, out, out_f32);
  la.at.fused = 1;
  la.at.app = append_args(c, layer, k_t, v_t, stride_kv);
  la.layer = layer;
  la.early = early;
  // the speculative prefetch of the centroid rows etc. pays only while a launch's unit index is small
  la.spec_pf = (int64_t)c->batch * c->hn * std::max(c->kmax, 1) * ROW_BYTES <= (8ll << 20) ? 1 : 0;
  LKV_LAUNCH(c, launch_layer(la, st), "decode_layer");
  c->last_layer = layer;
  c->last_stream = stream;
  c->t[layer] = t;
  c->stage[layer] = 3;
  return LOUISKV_OK;
}

// ---------------------------------------------------------------- introspection
louiskv_status louiskv_prompt_fence(louiskv_ctx* c, void* stream) {
  LKV_CHECK_CTX(c);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int l = 0; l < c->L; ++l) LKV_LAUNCH(c, offload_wait(c, l, st), "prompt fence");
  return LOUISKV_OK;
}

static louiskv_status inst_lookup(louiskv_ctx* c, int layer, int b, int h, int64_t* gi) {
  if (c->off_stream && cudaStreamSynchronize(c->off_stream) != cudaSuccess)
    return fail(c, LOUISKV_ERR_CUDA, "prompt offload failed");
  if (layer < 0 || layer >= c->L || b < 0 || b >= c->Bmax || h < 0 || h >= c->hn)
    return fail(c, LOUISKV_ERR_INVALID_ARG, "bad (layer, b, h)");
  if (is_full(c, layer)) return fail(c, LOUISKV_ERR_INVALID_ARG, "full-cache layer has no units");
  *gi = inst_base(c, layer) + (int64_t)b * c->hn + h;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_selection(louiskv_ctx* c, int32_t layer, int32_t b, int32_t h, int32_t* ids, int32_t cap,
                                     int32_t* n) {
  LKV_CHECK_CTX(c);
  int64_t gi;
  louiskv_status s = inst_lookup(c, layer, b, h, &gi);
  if (s) return s;
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_selection");
  InstState is;
  cudaMemcpy(&is, c->d_inst + gi, sizeof(is), cudaMemcpyDeviceToHost);
  std::vector<uint8_t> sel(std::max(is.n_units, 1));
  cudaMemcpy(sel.data(), c->d_sel + gi * c->Umax, is.n_units, cudaMemcpyDeviceToHost);
  int cnt = 0;
  for (int u = 0; u < is.n_units; ++u)
    if (sel[u]) {
      if (ids && cnt < cap) ids[cnt] = u;
      ++cnt;
    }
  if (n) *n = cnt;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_units(louiskv_ctx* c, int32_t layer, int32_t b, int32_t h, int32_t cap, float* cf,
                                 int32_t* sizes, int32_t* first_pos, int32_t* n_units) {
  LKV_CHECK_CTX(c);
  int64_t gi;
  louiskv_status s = inst_lookup(c, layer, b, h, &gi);
  if (s) return s;
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_units");
  InstState is;
  cudaMemcpy(&is, c->d_inst + gi, sizeof(is), cudaMemcpyDeviceToHost);
  const int n = std::min(is.n_units, std::max(cap, 0));
  if (cf && n) cudaMemcpy(cf, c->d_cent + gi * c->Umax * D, sizeof(float) * n * D, cudaMemcpyDefault);
  if (sizes && n) cudaMemcpy(sizes, c->d_usize + gi * c->Umax, sizeof(int32_t) * n, cudaMemcpyDeviceToHost);
  if (first_pos && n) cudaMemcpy(first_pos, c->d_ufirst + gi * c->Umax, sizeof(int32_t) * n, cudaMemcpyDeviceToHost);
  if (n_units) *n_units = is.n_units;
  if (is.error) return fail(c, LOUISKV_ERR_CAPACITY, "unit table / host pool capacity exceeded");
  return LOUISKV_OK;
}

louiskv_status louiskv_get_unit_positions(louiskv_ctx* c, int32_t layer, int32_t b, int32_t h, int32_t* positions,
                                          int64_t cap, int64_t* n) {
  LKV_CHECK_CTX(c);
  int64_t gi;
  louiskv_status s = inst_lookup(c, layer, b, h, &gi);
  if (s) return s;
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_unit_positions");
  InstState is;
  cudaMemcpy(&is, c->d_inst + gi, sizeof(is), cudaMemcpyDeviceToHost);
  const int64_t m = std::min<int64_t>(is.pool_rows, std::max<int64_t>(cap, 0));
  if (positions && m)
    cudaMemcpy(positions, c->d_pool_pos + gi * c->pool_rows_cap, sizeof(int32_t) * m, cudaMemcpyDeviceToHost);
  if (n) *n = is.pool_rows;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_working_set(louiskv_ctx* c, int32_t layer, int32_t b, int32_t h, uint16_t* k_rows,
                                       uint16_t* v_rows, int32_t cap, int32_t* n_rows) {
  LKV_CHECK_CTX(c);
  int64_t gi;
  louiskv_status s = inst_lookup(c, layer, b, h, &gi);
  if (s) return s;
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_working_set");
  InstState is;
  cudaMemcpy(&is, c->d_inst + gi, sizeof(is), cudaMemcpyDeviceToHost);
  const int m = std::min(is.ws_rows, std::max(cap, 0));
  const bf16* K = c->d_ws + is.ws_cur * c->ws_buf_stride + gi * c->ws_inst_stride;
  const bf16* V = K + (int64_t)std::max(c->Bud, 1) * D;
  if (k_rows && m) cudaMemcpy(k_rows, K, sizeof(bf16) * m * D, cudaMemcpyDeviceToHost);
  if (v_rows && m) cudaMemcpy(v_rows, V, sizeof(bf16) * m * D, cudaMemcpyDeviceToHost);
  if (n_rows) *n_rows = is.ws_rows;
  return LOUISKV_OK;
}

louiskv_status louiskv_set_prefill_timing(louiskv_ctx* c, int32_t enable) {
  LKV_CHECK_CTX(c);
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "set_prefill_timing");
  PhaseRec& r = c->prec;
  r.on = enable != 0;
  r.marks.clear();
  r.d2h.clear();
  r.used = 0;
  r.assign_flops = r.keys = r.d2h_bytes = r.assign_passes = 0;
  r.calls = 0;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_prefill_times(louiskv_ctx* c, louiskv_prefill_times* out) {
  LKV_CHECK_CTX(c);
  if (!out) return fail(c, LOUISKV_ERR_INVALID_ARG, "get_prefill_times: null");
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_prefill_times");
  const PhaseRec& r = c->prec;
  double acc[PH_N] = {0};
  for (size_t i = 0; i + 1 < r.marks.size(); ++i) {
    if (r.marks[i].first == PH_END) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.marks[i].second, r.marks[i + 1].second) != cudaSuccess)
      return cuda_fail(c, cudaGetLastError(), "get_prefill_times: events");
    acc[r.marks[i].first] += ms;
  }
  double d2h = 0.0;
  for (const auto& pr : r.d2h) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) d2h += ms;
  }
  *out = louiskv_prefill_times{};
  out->init_ms = acc[PH_INIT];
  out->assign_ms = acc[PH_ASSIGN];
  out->sort_ms = acc[PH_SORT];
  out->update_ms = acc[PH_UPDATE];
  out->stage_ms = acc[PH_STAGE];
  out->d2h_ms = d2h;
  out->assign_flops = r.assign_flops;
  out->keys = r.keys;
  out->d2h_bytes = r.d2h_bytes;
  out->assign_passes = r.assign_passes;
  out->calls = r.calls;
  return LOUISKV_OK;
}

// decode-state checkpoint: everything the decode path writes whose validity is not bounded by the
// saved instance counters (rows appended beyond n_units / pool_rows / the full-cache step are dead
// after a restore and are rewritten by the next steps)
static void snap_list(louiskv_ctx* c, std::vector<std::pair<void*, size_t>>& v) {
  const int64_t ni = c->n_inst, nl = c->inst_per_layer;
  v.push_back({c->d_inst, sizeof(InstState) * (size_t)std::max<int64_t>(ni, 1)});
  v.push_back({c->d_sel, (size_t)std::max<int64_t>(ni, 1) * c->Umax});
  v.push_back({c->d_seloff, sizeof(int32_t) * (size_t)std::max<int64_t>(ni, 1) * c->Umax});
  v.push_back({c->d_ws, sizeof(bf16) * (size_t)2 * c->ws_buf_stride});
  v.push_back({c->d_ring, sizeof(bf16) * (size_t)std::max<int64_t>(ni, 1) * 2 * c->ring_cap * D});
  v.push_back({c->d_fifo, sizeof(int2) * (size_t)std::max<int64_t>(ni, 1) * c->ring_cap});
  v.push_back({c->d_flag, (size_t)c->L * c->Bmax});
  v.push_back({c->d_r, sizeof(double) * (size_t)c->L * c->Bmax});
  v.push_back({c->d_qref, sizeof(bf16) * (size_t)c->L * 2 * c->Bmax * c->Hq * D});
  v.push_back({c->d_step, sizeof(int) * (size_t)c->L});
  v.push_back({c->d_jobs, sizeof(GatherJob) * (size_t)c->L * nl});
  v.push_back({c->d_stats, sizeof(StatsDev)});
  v.push_back({c->d_error, sizeof(int)});
}

louiskv_status louiskv_state_save(louiskv_ctx* c, void* stream) {
  LKV_CHECK_CTX(c);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int l = 0; l < c->L; ++l) {
    if (c->P[l] < 0) return fail(c, LOUISKV_ERR_STATE, "state_save before cluster_prompt on every layer");
    if (c->stage[l] != 0 && c->stage[l] != 3) return fail(c, LOUISKV_ERR_STATE, "state_save inside a step");
    LKV_LAUNCH(c, offload_wait(c, l, st), "state_save: prompt offload wait");
  }
  std::vector<std::pair<void*, size_t>> v;
  snap_list(c, v);
  if (c->snap.empty()) {
    for (auto& pr : v) {
      void* d = nullptr;
      if (cudaMalloc(&d, pr.second) != cudaSuccess) {
        cudaGetLastError();
        for (auto& sb : c->snap) cudaFree(sb.dst);
        c->snap.clear();
        return fail(c, LOUISKV_ERR_OOM_DEVICE, "state_save: checkpoint buffers");
      }
      c->snap.push_back({pr.first, pr.second, d});
    }
  }
  for (auto& sb : c->snap)
    LKV_LAUNCH(c, cudaMemcpyAsync(sb.dst, sb.src, sb.bytes, cudaMemcpyDeviceToDevice, st), "state_save copy");
  c->snap_t = c->t;
  c->snap_stage = c->stage;
  c->snap_valid = true;
  return LOUISKV_OK;
}

louiskv_status louiskv_state_restore(louiskv_ctx* c, void* stream) {
  LKV_CHECK_CTX(c);
  if (!c->snap_valid) return fail(c, LOUISKV_ERR_STATE, "state_restore without state_save");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (auto& sb : c->snap)
    LKV_LAUNCH(c, cudaMemcpyAsync(sb.src, sb.dst, sb.bytes, cudaMemcpyDeviceToDevice, st), "state_restore copy");
  c->t = c->snap_t;
  c->stage = c->snap_stage;
  c->last_layer = -1;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_pool_numa_node(const louiskv_ctx* c, int32_t* node) {
  if (!c || !node) return LOUISKV_ERR_INVALID_ARG;
  *node = c->pool_registered ? c->pool_numa_node : -1;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_memory(const louiskv_ctx* c, uint64_t* device_bytes, uint64_t* host_pool_bytes) {
  if (!c) return LOUISKV_ERR_INVALID_ARG;
  if (device_bytes) *device_bytes = c->dev_bytes;
  if (host_pool_bytes) *host_pool_bytes = c->host_bytes + c->index_host_bytes;
  return LOUISKV_OK;
}

louiskv_status louiskv_get_stats(louiskv_ctx* c, louiskv_stats* out) {
  LKV_CHECK_CTX(c);
  if (!out) return fail(c, LOUISKV_ERR_INVALID_ARG, "get_stats: null");
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_fail(c, cudaGetLastError(), "get_stats");
  StatsDev sd;
  cudaMemcpy(&sd, c->d_stats, sizeof(sd), cudaMemcpyDeviceToHost);
  int derr = 0;
  cudaMemcpy(&derr, c->d_error, sizeof(int), cudaMemcpyDeviceToHost);
  std::vector<InstState> is(std::max<int64_t>(c->n_inst, 1));
  if (c->n_inst) cudaMemcpy(is.data(), c->d_inst, sizeof(InstState) * c->n_inst, cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < c->n_inst; ++i) derr |= is[i].error;
  out->retrievals = sd.retrievals;
  out->units_scored = sd.units_scored;
  out->units_selected = sd.units_selected;
  out->units_reused = sd.units_reused;
  out->units_fetched = sd.units_fetched;
  out->bytes_h2d = sd.bytes_h2d;
  out->bytes_d2h = sd.bytes_d2h;
  out->segments_evicted = sd.segments_evicted;
  out->kmeans_tc_iters = c->km_tc_iters;
  out->kmeans_simt_iters = c->km_simt_iters;
  out->dma_copies = c->dma_copies;
  if (derr) return fail(c, LOUISKV_ERR_CAPACITY, "device capacity exceeded (host pool, unit table or full cache)");
  return LOUISKV_OK;
}

}  // extern "C"
