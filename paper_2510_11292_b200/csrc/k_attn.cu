// Sparse decode attention — o = softmax(q K_I^T / sqrt(d)) V_I  (P:63-65 [§3.1]),
// I = sinks ∪ KV_critical ∪ KV_local (P:143, P:307 [Alg. 1 KV_attn]); the full-cache layers
// attend to all P+t rows.
//
// Split-K flash-decode, GQA-packed: one CTA per (instance, split); the g query heads of a KV
// head share every K/V row read (one HBM read serves g heads). Inside a CTA, each half-warp
// (16 lanes x 8 dims) walks rows with an online softmax in the log2 domain; half-warps merge
// through shared memory; splits merge in a fixed order by the last CTA to finish (atomic
// ticket), so the result is deterministic. HBM-bound: 512 B of K+V per row.
#include <cooperative_groups.h>

#include "lkv_append_dev.cuh"
#include "lkv_attn_dev.cuh"

namespace cg = cooperative_groups;

namespace lkv {

template <int G, bool FUSED>
__global__ void __launch_bounds__(AT_THREADS, G <= 4 ? 2 : 1) attn_kernel(AttnArgs a) {
  pdl_wait_trigger();
  int li, split, nsplit;
  if constexpr (FUSED) {
    // one 8-CTA cluster per instance: rank 0 runs kvm.store_cache(k_t, v_t) (seal / append / evict),
    // the cluster barrier publishes the new local-buffer state to the other ranks
    li = blockIdx.x / AT_CL;
    split = blockIdx.x % AT_CL;
    nsplit = AT_CL;
    {  // every rank copies 1/AT_CL of the pending gather job (selected rows -> working set)
      const GatherJob J = a.app.jobs[li];
      if (J.n_rows > 0) {
        const int per = (J.n_rows + AT_CL - 1) / AT_CL;
        const int r0 = split * per, r1 = min(J.n_rows, r0 + per);
        if (r0 < r1) gather_rows(a.app, li, J, r0, r1);
      }
    }
    if (split == 0) append_one(a.app, li, a.app.flag ? a.app.flag[li / a.hn] : 0);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    cg::this_cluster().sync();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (split == 0 && threadIdx.x == 0) a.app.jobs[li].n_rows = 0;
  } else {
    li = blockIdx.x;
    split = blockIdx.y;
    nsplit = gridDim.y;
  }
  attn_body<G, FUSED>(a, li, split, nsplit);
}

template <int G>
static cudaError_t launch_attn_g(const AttnArgs& a, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  cudaError_t ea = once_per_device(attr, [] {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    return e != cudaSuccess ? e : cudaFuncSetAttribute(attn_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
  });
  if (ea != cudaSuccess) return ea;
  if (!a.fused) return launch_k(attn_kernel<G, false>, dim3(a.batch * a.hn, a.splits), dim3(AT_THREADS), AT_SMEM, st, a);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.batch * a.hn * AT_CL);
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
  return cudaLaunchKernelEx(&cfg, attn_kernel<G, true>, a);
}

cudaError_t launch_attn(const AttnArgs& a, cudaStream_t st) {
  switch (a.g) {
    case 1: return launch_attn_g<1>(a, st);
    case 2: return launch_attn_g<2>(a, st);
    case 4: return launch_attn_g<4>(a, st);
    case 8: return launch_attn_g<8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lkv
