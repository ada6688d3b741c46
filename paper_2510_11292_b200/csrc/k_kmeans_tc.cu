// k-means assignment on the 5th-gen tensor cores (P:120 k-means, P:126 clustering kernel).
//
//   a_i = argmax_j ( x_i · bf16(C_j) - ½||C_j||² ),  ties -> lower j;   dmin_i = ||x_i||² - 2 max
//
// The cross term is a dense GEMM X[N×128] · C[k×128]^T (bf16 in, fp32 accumulate), so it runs as
// tcgen05.mma kind::f16 with the accumulator in TMEM and a fused row-argmax epilogue; nothing of
// the N×k score matrix ever reaches memory.
//
// Persistent kernel, one CTA per SM (512 TMEM columns, ~193 KB smem), warp roles:
//   warp 0  TMA producer: A tile (128 keys × 128 dims, two 64-dim SWIZZLE_128B boxes, straight
//           from the caller's strided K tensor through a 4-D tensor map) once per work item,
//           B tiles (256 centroids × 128 dims, bf16) through a 2-stage ring;
//   warp 1  MMA issuer (one thread): 8 × tcgen05.mma M=128 N=256 K=16 per B tile into one of two
//           TMEM accumulator buffers, tcgen05.commit -> mbarriers;
//   warp 2  TMEM allocator;
//   warps 4-7 epilogue: tcgen05.ld 32x32b.x32 (thread = key row = TMEM lane), subtract the
//           half-norms, chunk max + rare index search, running (best, index) per row in registers.
// Work item = (instance, 128-key block); the n loop over all centroid tiles stays inside the item.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "lkv_internal.cuh"

namespace lkv {

namespace tc {

constexpr int BM = 128;            // keys per tile (UMMA M)
constexpr int BN = 256;            // centroids per tile (UMMA N)
constexpr int KH = 64;             // bf16 elements per 128-B swizzle row
constexpr int A_BYTES = BM * D * 2;       // 32 KB
constexpr int B_BYTES = BN * D * 2;       // 64 KB
constexpr int B_STAGES = 2;
constexpr int THREADS = 384;  // 4 non-epilogue warps + 8 epilogue warps
constexpr int BX_BYTES = BN * 16;        // B extension block: 256 centroids x 8 bf16 (4 KB)
constexpr int AX_BYTES = BM * 16;        // A extension block: 128 keys x 8 bf16 (1,1,1,0...) (2 KB)
constexpr int ZERO_BYTES = BN * 16;      // the second (all-zero) core-matrix column of the 9th K-step
constexpr int SMEM_BYTES = 2 * A_BYTES + B_STAGES * (B_BYTES + BX_BYTES) + AX_BYTES + ZERO_BYTES + 1024 /*align*/ +
                           256 /*barriers*/ + 2 * BM * 4 + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
#ifndef LKV_KM_X_NOHINT
  // the key tiles with an L2 evict_last policy: the layer's keys (C2: 67 MB) stay in L2 for the
  // centroid update that follows (it gathers member rows) and the next iteration's assignment
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
#endif
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart (SBO), version 1
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // version (sm100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// UMMA descriptor for the 9th K-step: K-major, SWIZZLE_NONE, core matrices (8 rows x 16 B) packed
// at 128 B (SBO); the second 8-element K half sits LBO bytes further (the shared zero block)
__device__ __forceinline__ uint64_t umma_desc_none(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // layout type 0 = SWIZZLE_NONE
}
// instruction descriptor kind::f16: D=F32, A=B=BF16, K-major both, N=256, M=128
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define TMEM_LD32(taddr, r)                                                                                       \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),           \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(taddr))

struct TcParams {
  int ni, N, kc, n_mblk, n_ntile;
  const float* half;   // [ni][hstride]
  int hstride;
  int32_t* assign;     // [ni][Nmax]
  float* dmin;
  int64_t Nmax;
  int hn;
};

__global__ void __launch_bounds__(THREADS, 1)
    kmeans_assign_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ CUtensorMap tmBx, TcParams p) {
  pdl_wait_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                              // [2][A_BYTES]
  uint8_t* sB = smem + 2 * A_BYTES;                // [B_STAGES][B_BYTES]
  uint8_t* sBx = sB + B_STAGES * B_BYTES;          // [B_STAGES][BX_BYTES]
  uint8_t* sAx = sBx + B_STAGES * BX_BYTES;        // [AX_BYTES] constant (1,1,1,0,...) rows
  uint8_t* sZero = sAx + AX_BYTES;                 // [ZERO_BYTES] zeros
  uint64_t* bars = reinterpret_cast<uint64_t*>(sZero + ZERO_BYTES);
  uint64_t* a_full = bars;           // [2]
  uint64_t* a_empty = bars + 2;      // [2]
  uint64_t* b_full = bars + 4;       // [B_STAGES]
  uint64_t* b_empty = bars + 6;      // [B_STAGES]
  uint64_t* acc_full = bars + 8;     // [2]
  uint64_t* acc_empty = bars + 10;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = p.ni * p.n_mblk;
  // constant operand blocks of the 9th K-step (generic-proxy stores, fenced for the async proxy)
  for (int i = threadIdx.x; i < BM; i += blockDim.x)
    reinterpret_cast<uint4*>(sAx)[i] = make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u);
  for (int i = threadIdx.x; i < ZERO_BYTES / 16; i += blockDim.x) reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1 + 8);  // MMA commit + the 8 epilogue warps (half of them read ||x||^2 from sA)
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);
    }
    for (int i = 0; i < B_STAGES; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0, bstage = 0;
      uint32_t bphase = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int inst = item / p.n_mblk, mb = item % p.n_mblk;
        const int b = inst / p.hn, h = inst % p.hn;
        const int ab = it & 1;
        if (it >= 2) mbar_wait(&a_empty[ab], ((it >> 1) - 1) & 1);
        mbar_expect_tx(&a_full[ab], A_BYTES);
        tma_load_4d(sA + ab * A_BYTES, &tmA, &a_full[ab], 0, h, mb * BM, b);
        tma_load_4d(sA + ab * A_BYTES + A_BYTES / 2, &tmA, &a_full[ab], KH, h, mb * BM, b);
        for (int nt = 0; nt < p.n_ntile; ++nt) {
          mbar_wait(&b_empty[bstage], bphase ^ 1);
          mbar_expect_tx(&b_full[bstage], B_BYTES + BX_BYTES);
          tma_load_3d(sB + bstage * B_BYTES, &tmB, &b_full[bstage], 0, nt * BN, inst);
          tma_load_3d(sB + bstage * B_BYTES + B_BYTES / 2, &tmB, &b_full[bstage], KH, nt * BN, inst);
          tma_load_3d(sBx + bstage * BX_BYTES, &tmBx, &b_full[bstage], 0, nt * BN, inst);
          if (++bstage == B_STAGES) {
            bstage = 0;
            bphase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int it = 0, bstage = 0, acc = 0;
      uint32_t bphase = 0, accphase = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int ab = it & 1;
        mbar_wait(&a_full[ab], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + ab * A_BYTES);
        for (int nt = 0; nt < p.n_ntile; ++nt) {
          mbar_wait(&acc_empty[acc], accphase ^ 1);
          mbar_wait(&b_full[bstage], bphase);
          tc_fence_after();
          const uint32_t b_base = smem_u32(sB + bstage * B_BYTES);
          const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t koff = (uint32_t)((k >> 2) * (BM * 128) + (k & 3) * 32);
            const uint32_t kofb = (uint32_t)((k >> 2) * (BN * 128) + (k & 3) * 32);
            mma_bf16(tmem_d, umma_desc(a_base + koff), umma_desc(b_base + kofb), k > 0 ? 1u : 0u);
          }
          {  // 9th K-step: + (1,1,1) . (-h_hi, -h_mid, -h_lo)  ==  - ½||c||²
            const uint32_t ax = smem_u32(sAx), bx = smem_u32(sBx + bstage * BX_BYTES), z = smem_u32(sZero);
            mma_bf16(tmem_d, umma_desc_none(ax, z - ax), umma_desc_none(bx, z - bx), 1u);
          }
          mma_commit(&b_empty[bstage]);
          mma_commit(&acc_full[acc]);
          if (nt == p.n_ntile - 1) mma_commit(&a_empty[ab]);
          if (++bstage == B_STAGES) {
            bstage = 0;
            bphase ^= 1;
          }
          if (++acc == 2) {
            acc = 0;
            accphase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: 8 warps; thread = key row = TMEM lane (warp % 4 selects the lane
    // quarter), column half = (warp - 4) / 4; the two halves of a row merge through smem per item
    const int e = warp - 4;
    const int q = warp & 3;
    const int chalf = e >> 2;
    const int row = q * 32 + lane;
    int it = 0, acc = 0;
    uint32_t accphase = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int inst = item / p.n_mblk, mb = item % p.n_mblk;
      float best = -INFINITY;
      int bidx = 0x7FFFFFFF;
      const int ab = it & 1;
      float xn = 0.f;
      mbar_wait(&a_full[ab], (it >> 1) & 1);
      if (chalf == 0) {
        // ||x||^2 from the swizzled A tile (row = TMEM lane)
        const uint8_t* arow = sA + ab * A_BYTES;
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int pc = c ^ (row & 7);
            const uint4 u = *reinterpret_cast<const uint4*>(arow + kh * (A_BYTES / 2) + row * 128 + pc * 16);
            float f[8];
            unpack8(u, f);
#pragma unroll
            for (int x = 0; x < 8; ++x) xn = fmaf(f[x], f[x], xn);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_empty[ab]);
      for (int nt = 0; nt < p.n_ntile; ++nt) {
        mbar_wait(&acc_full[acc], accphase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + chalf * (BN / 2));
        const int colbase = nt * BN + chalf * (BN / 2);
        uint32_t r[2][32];
        TMEM_LD32(taddr, r[0]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int ch = 0; ch < BN / 64; ++ch) {
          // software pipeline: the next 32 columns are in flight while this chunk is reduced
          if (ch + 1 < BN / 64) TMEM_LD32(taddr + (ch + 1) * 32, r[(ch + 1) & 1]);
          const uint32_t* rc = r[ch & 1];
          const int col0 = colbase + ch * 32;
          float v[32];  // the accumulator already holds x.c - ½||c||² (9th K-step)
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(rc[c]);
          float m01[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) m01[i] = fmaxf(v[2 * i], v[2 * i + 1]);
#pragma unroll
          for (int i = 0; i < 8; ++i) m01[i] = fmaxf(m01[2 * i], m01[2 * i + 1]);
#pragma unroll
          for (int i = 0; i < 4; ++i) m01[i] = fmaxf(m01[2 * i], m01[2 * i + 1]);
          const float m = fmaxf(fmaxf(m01[0], m01[1]), fmaxf(m01[2], m01[3]));
          if (m > best) {
            int idx = 0;
#pragma unroll
            for (int c = 31; c >= 0; --c)
              if (v[c] == m) idx = c;
            best = m;
            bidx = col0 + idx;
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
        if (++acc == 2) {
          acc = 0;
          accphase ^= 1;
        }
      }
      // merge the two column halves of each row (strictly greater wins; ties -> lower index)
      float* s_best = reinterpret_cast<float*>(tmem_slot + 4);
      int* s_idx = reinterpret_cast<int*>(s_best + BM);
      if (chalf == 1) {
        s_best[row] = best;
        s_idx[row] = bidx;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (chalf == 0) {
        const float ob = s_best[row];
        const int oi = s_idx[row];
        if (ob > best || (ob == best && oi < bidx)) {
          best = ob;
          bidx = oi;
        }
        const int grow = mb * BM + row;
        if (grow < p.N) {
          p.assign[(int64_t)inst * p.Nmax + grow] = bidx;
          p.dmin[(int64_t)inst * p.Nmax + grow] = fmaf(-2.f, best, xn);
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

}  // namespace tc

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return get_encode(); }

bool kmeans_tc_available() {
  static int avail = -1;
  if (avail < 0) {
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    avail = (major == 10 && minor == 0 && get_encode() != nullptr) ? 1 : 0;
  }
  return avail == 1;
}

static void tc_debug(const char* what, int rc) {
  if (getenv("LOUISKV_DEBUG")) fprintf(stderr, "[louiskv] tcgen05 k-means unavailable: %s (rc=%d)\n", what, rc);
}

cudaError_t launch_assign_tc(const KmArgs& a, cudaStream_t st) {
  auto enc = get_encode();
  if (!enc) {
    tc_debug("cuTensorMapEncodeTiled entry point", 0);
    return cudaErrorNotSupported;
  }
  // TMA needs 16-B aligned base and strides; element strides must be monotone for this map
  const uintptr_t base = reinterpret_cast<uintptr_t>(a.k + (int64_t)a.S * a.st);
  // strides of size-1 dimensions are irrelevant (torch reports arbitrary values for them)
  const bool bad_h = a.hn > 1 && ((a.sh * 2) % 16 || a.sh <= 0 || a.st < a.sh * a.hn);
  const bool bad_b = a.batch > 1 && ((a.sb * 2) % 16 || a.sb < a.st * (int64_t)(a.S + a.N));
  if ((base & 15) || (a.st * 2) % 16 || bad_h || bad_b) {
    if (getenv("LOUISKV_DEBUG"))
      fprintf(stderr, "[louiskv] K base=%p sb=%lld st=%lld sh=%lld hn=%d batch=%d S=%d N=%d\n", (void*)base,
              (long long)a.sb, (long long)a.st, (long long)a.sh, a.hn, a.batch, a.S, a.N);
    tc_debug("K strides/alignment not TMA-compatible", 0);
    return cudaErrorNotSupported;
  }
  CUtensorMap tmA, tmB;
  {
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)a.hn, (cuuint64_t)a.N, (cuuint64_t)a.batch};
    // a single owned head: give the (always 0) head coordinate a stride past the key rows
    const int64_t hstride = a.hn > 1 ? a.sh * 2 : (int64_t)a.st * 2 * (a.S + a.N);
    const int64_t bstride = a.batch > 1 ? a.sb * 2 : hstride * a.hn + (int64_t)a.st * 2 * (a.S + a.N);
    cuuint64_t strides[3] = {(cuuint64_t)hstride, (cuuint64_t)a.st * 2, (cuuint64_t)bstride};
    cuuint32_t box[4] = {tc::KH, 1, tc::BM, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, reinterpret_cast<void*>(base), dims, strides,
                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      tc_debug("tensor map of K", (int)r);
      return cudaErrorNotSupported;
    }
  }
  const int ni = a.batch * a.hn;
  {
    cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)a.Umax, (cuuint64_t)ni};
    cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)a.Umax * D * 2};
    cuuint32_t box[3] = {tc::KH, tc::BN, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)a.centb, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      tc_debug("tensor map of centroids", (int)r);
      return cudaErrorNotSupported;
    }
  }
  CUtensorMap tmBx;
  {
    cuuint64_t dims[3] = {8, (cuuint64_t)a.Umax, (cuuint64_t)ni};
    cuuint64_t strides[2] = {16, (cuuint64_t)a.Umax * 16};
    cuuint32_t box[3] = {8, tc::BN, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = enc(&tmBx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)a.bext, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      tc_debug("tensor map of the half-norm extension", (int)r);
      return cudaErrorNotSupported;
    }
  }
  tc::TcParams p;
  p.ni = ni;
  p.N = a.N;
  p.kc = a.kc;
  p.n_mblk = (a.N + tc::BM - 1) / tc::BM;
  p.n_ntile = (a.kc + tc::BN - 1) / tc::BN;
  p.half = a.half;
  p.hstride = a.hstride;
  p.assign = a.assign;
  p.dmin = a.dmin;
  p.Nmax = a.Nmax;
  p.hn = a.hn;
  static std::atomic<uint64_t> attr{0};
  cudaError_t ea = once_per_device(attr, [] {
    return cudaFuncSetAttribute(tc::kmeans_assign_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES);
  });
  if (ea != cudaSuccess) return ea;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int items = ni * p.n_mblk;
  const int grid = items < sms ? items : sms;
  launch_k(tc::kmeans_assign_tc_kernel, dim3(grid), dim3(tc::THREADS), tc::SMEM_BYTES, st, tmA, tmB, tmBx, p);
  return cudaGetLastError();
}

}  // namespace lkv
