// gemm_tc.cu — tcgen05 (5th-generation tensor core) GEMM for sm_100a: the two chained products of
// Algorithm 1 line 3, U = A' X^T and Y[0:n,0:n'] = A U^T + lambda K, in 3xTF32 (fp32-
// accurate: a = big + small, big = rna_tf32(a), small = rna_tf32(a - big); C += Ps Qb + Pb Qs +
// Pb Qb, the small*small term (2^-22 relative) dropped) or plain 1xTF32.
//
// C[M x N] = P[M x K] Q[N x K]^T, both operands K-major (row-major, K contiguous), fp32 in HBM.
//  * TMA (cp.async.bulk.tensor, SWIZZLE_128B) loads 128-row x 32-float (128 B) boxes of the big
//    and small parts into a 3-stage shared-memory ring guarded by mbarriers (full/empty).
//  * One elected thread issues tcgen05.mma.kind::tf32 with the accumulator in TMEM; with
//    CG = 2 (cta_group::2) a CTA pair computes a 256 x 256 tile: each CTA stages 128 rows of P and
//    128 rows of Q (its half of B), the leader CTA issues the MMA for both.
//  * Two TMEM accumulator buffers let the epilogue of tile i overlap the MMAs of tile i+1.
//  * Epilogue warps read TMEM with tcgen05.ld.32x32b and apply the fused epilogue: the TF32 split
//    of U for the next GEMM (kEpiSplit) or + lambda K into the Y block (kEpiAxpy).
//  * Persistent: grid = min(#tiles, #SMs / CG) clusters, grouped tile raster for L2 reuse.
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4-7 epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fpfp {

namespace {

using namespace tc;

constexpr int kBK = 32;                 // fp32 per 128-byte swizzle row
constexpr int kRowsPerCta = 128;        // rows of P and of Q staged per CTA per stage
constexpr int kStages = 3;
constexpr int kBoxBytes = kRowsPerCta * kBK * 4;  // 16 KB
constexpr int kThreads = 256;

template <int CG>
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  }
}

struct TcParams {
  int M, N, K;
  int q3d, qk;      // Q is [K/qk][N][qk] blocks (3-D tensor map) when q3d != 0
  int epi;
  float* C; float* C2; float* C3; int64_t ldC;
  const float* D; int64_t ldD; float lam;
  const float* D2; int64_t ldD2; float scale;
  const int* done;
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mt, int& nt) {
  constexpr int kGroup = 8;
  const int per_group = kGroup * num_n;
  const int g = t / per_group;
  const int first_m = g * kGroup;
  const int gsz = min(num_m - first_m, kGroup);
  const int r = t - g * per_group;
  mt = first_m + r % gsz;
  nt = r / gsz;
}

template <int CG, int PASSES>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap mPb, const __grid_constant__ CUtensorMap mPs,
               const __grid_constant__ CUtensorMap mQb, const __grid_constant__ CUtensorMap mQs,
               TcParams p) {
  if (p.done && *p.done) return;  // uniform across the grid

  constexpr int kTileM = 128 * CG, kTileN = 128 * CG;
  constexpr int kAccCols = kTileN;                     // fp32 accumulator columns per buffer
  constexpr uint32_t kTmemCols = 2 * kAccCols;         // 256 (CG=1) or 512 (CG=2)
  constexpr int kBoxesPerStage = PASSES == 1 ? 2 : 4;  // Pb, Qb (+ Ps, Qs)
  constexpr uint32_t kStageBytes = kBoxesPerStage * kBoxBytes;
  constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTileN >> 3) << 17) |
                              ((uint32_t)(kTileM >> 4) << 24);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_sm;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 1 ? 0 : cta_rank();
  const bool leader = rank == 0;
  const int num_m = (int)ceil_div(p.M, kTileM), num_n = (int)ceil_div(p.N, kTileN);
  const int num_tiles = num_m * num_n;
  const int num_kb = (int)ceil_div(p.K, kBK);
  const int cid = CG == 1 ? (int)blockIdx.x : (int)cluster_id_x();
  const int ncl = CG == 1 ? (int)gridDim.x : (int)num_clusters_x();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull_bar[a], 1); mbar_init(&tempty_bar[a], 4 * CG); }
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sm)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sm)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sm;

  if (warp == 0) {
    // ===================== TMA producer (one elected lane per CTA) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        int mt, nt;
        tile_coords(t, num_m, num_n, mt, nt);
        const int prow = mt * kTileM + (int)rank * kRowsPerCta;
        const int qrow = nt * kTileN + (int)rank * kRowsPerCta;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint32_t bar = smem_u32(&full_bar[stage]);
          if (CG == 2) bar = mapa(bar, 0);        // the leader CTA's full barrier
          if (leader) mbar_expect_tx(&full_bar[stage], kStageBytes * CG);
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          const int kc = kb * kBK;
          tma_load<CG>(&mPb, base + 0 * kBoxBytes, bar, kc, prow);
          if (p.q3d) {
            const int blk = kc / p.qk, kin = kc - blk * p.qk;
            tma_load3<CG>(&mQb, base + 1 * kBoxBytes, bar, kin, qrow, blk);
          } else {
            tma_load<CG>(&mQb, base + 1 * kBoxBytes, bar, kc, qrow);
          }
          if (PASSES == 3) {
            tma_load<CG>(&mPs, base + 2 * kBoxBytes, bar, kc, prow);
            if (p.q3d) {
              const int blk = kc / p.qk, kin = kc - blk * p.qk;
              tma_load3<CG>(&mQs, base + 3 * kBoxBytes, bar, kin, qrow, blk);
            } else {
              tma_load<CG>(&mQs, base + 3 * kBoxBytes, bar, kc, qrow);
            }
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA; warp-uniform loop, one elected lane issues) =====
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);   // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kAccCols);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kStageBytes);
          if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {            // K = 8 tf32 (32 bytes) per MMA
            const uint32_t off = (uint32_t)k * 32u;
            const uint64_t pb = smem_desc(base + 0 * kBoxBytes + off);
            const uint64_t qb = smem_desc(base + 1 * kBoxBytes + off);
            const uint32_t first = (kb == 0 && k == 0) ? 0u : 1u;
            if constexpr (PASSES == 3) {
              const uint64_t ps = smem_desc(base + 2 * kBoxBytes + off);
              const uint64_t qs = smem_desc(base + 3 * kBoxBytes + off);
              mma_tf32<CG>(d_tmem, ps, qb, kIdesc, first);   // small terms first
              mma_tf32<CG>(d_tmem, pb, qs, kIdesc, 1u);
              mma_tf32<CG>(d_tmem, pb, qb, kIdesc, 1u);
            } else {
              mma_tf32<CG>(d_tmem, pb, qb, kIdesc, first);
            }
          }
          umma_commit<CG>(&empty_bar[stage]);            // frees the smem slot in both CTAs
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit<CG>(&tfull_bar[acc]);   // accumulator ready (both CTAs)
        __syncwarp();
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> registers -> global =====================
    const int ew = warp & 3;                 // TMEM lane quarter of this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader = CG == 2 ? mapa(smem_u32(&tempty_bar[0]), 0) : 0;
    for (int t = cid; t < num_tiles; t += ncl) {
      int mt, nt;
      tile_coords(t, num_m, num_n, mt, nt);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mt * kTileM + (int)rank * kRowsPerCta + ew * 32 + lane;
      const bool row_ok = row < p.M;
      const uint32_t tbase = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * kAccCols);
#pragma unroll 1
      for (int cc = 0; cc < kTileN / 32; ++cc) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32(tbase + (uint32_t)(cc * 32), v);
        const int col0 = nt * kTileN + cc * 32;
        if (!row_ok || col0 >= p.N) continue;
        const bool full = col0 + 32 <= p.N;
        float* c = p.C + (int64_t)row * p.ldC + col0;
        if (p.epi == kEpiSplit) {
          float* c2 = p.C2 + (int64_t)row * p.ldC + col0;
          float* c3 = p.C3 ? p.C3 + (int64_t)row * p.ldC + col0 : nullptr;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 hb, sm, pl;
            float* h = reinterpret_cast<float*>(&hb);
            float* s = reinterpret_cast<float*>(&sm);
            float* q = reinterpret_cast<float*>(&pl);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = __uint_as_float(v[j + e]);
              q[e] = a;
              h[e] = tf32_rna(a);
              s[e] = tf32_rna(a - h[e]);
            }
            if (full) {
              *reinterpret_cast<float4*>(c + j) = hb;
              *reinterpret_cast<float4*>(c2 + j) = sm;
              if (c3) *reinterpret_cast<float4*>(c3 + j) = pl;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (col0 + j + e < p.N) { c[j + e] = h[e]; c2[j + e] = s[e]; if (c3) c3[j + e] = q[e]; }
            }
          }
        } else {
          const float* dd = ((p.epi == kEpiAxpy || p.epi == kEpiPG) && p.D) ? p.D + (int64_t)row * p.ldD + col0 : nullptr;
          const float* d2 = p.epi == kEpiPG ? p.D2 + (int64_t)row * p.ldD2 + col0 : nullptr;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o;
            float* oe = reinterpret_cast<float*>(&o);
            if (dd && full) {
              const float4 dv = *reinterpret_cast<const float4*>(dd + j);
              const float* de = reinterpret_cast<const float*>(&dv);
#pragma unroll
              for (int e = 0; e < 4; ++e) oe[e] = __uint_as_float(v[j + e]) + p.lam * de[e];
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float a = __uint_as_float(v[j + e]);
                if (dd && col0 + j + e < p.N) a += p.lam * dd[j + e];
                oe[e] = a;
              }
            }
            if (d2) {   // Projected Gradient: X + alpha (A X A' + lambda K)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (full || col0 + j + e < p.N) oe[e] = p.scale * oe[e] + d2[j + e];
            }
            if (full) {
              *reinterpret_cast<float4*>(c + j) = o;
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (col0 + j + e < p.N) c[j + e] = oe[e];
            }
          }
        }
      }
      // release the accumulator to the MMA issuer (leader CTA's barrier)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * sizeof(uint64_t)));
        else mbar_arrive_local(&tempty_bar[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  // teardown
  __syncwarp();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// rows x K fp32 row-major matrix with row stride ld (floats); box = 128 rows x 32 floats, SW128
bool make_map(CUtensorMap* m, const float* base, int rows, int K, int64_t ld) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * sizeof(float))};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kRowsPerCta};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// [blocks][rows][qk] blocks of row stride ld and block stride bstride (floats); box 128 x 32 x 1
bool make_map3(CUtensorMap* m, const float* base, int rows, int qk, int blocks, int64_t ld,
               int64_t bstride) {
  cuuint64_t dims[3] = {(cuuint64_t)qk, (cuuint64_t)rows, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * sizeof(float)), (cuuint64_t)(bstride * sizeof(float))};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)kRowsPerCta, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int CG, int PASSES>
cudaError_t launch_impl(const GemmArgs& g, cudaStream_t s, int device) {
  CUtensorMap mPb, mPs, mQb, mQs;
  const float* ps = PASSES == 3 ? g.Ps : g.Pb;
  const float* qs = PASSES == 3 ? g.Qs : g.Qb;
  const bool q3d = g.q_blocks > 1;
  bool ok = make_map(&mPb, g.Pb, g.M, g.K, g.ldP) && make_map(&mPs, ps, g.M, g.K, g.ldP);
  if (q3d)
    ok = ok && make_map3(&mQb, g.Qb, g.N, g.q_block_k, g.q_blocks, g.ldQ, g.q_block_stride) &&
         make_map3(&mQs, qs, g.N, g.q_block_k, g.q_blocks, g.ldQ, g.q_block_stride);
  else
    ok = ok && make_map(&mQb, g.Qb, g.N, g.K, g.ldQ) && make_map(&mQs, qs, g.N, g.K, g.ldQ);
  if (!ok) return cudaErrorInvalidValue;
  TcParams p{g.M, g.N, g.K, q3d ? 1 : 0, q3d ? g.q_block_k : 0, g.epi, g.C, g.C2, g.C3, g.ldC,
             g.D, g.ldD, g.lam, g.D2, g.ldD2, g.scale, g.done};
  constexpr int kBoxes = PASSES == 1 ? 2 : 4;
  const size_t smem = (size_t)kStages * kBoxes * kBoxBytes + 1024;
  auto kern = gemm_tc_kernel<CG, PASSES>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t tiles = ceil_div(g.M, 128 * CG) * ceil_div(g.N, 128 * CG);
  const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, sms / CG));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, mPb, mPs, mQb, mQs, p);
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
  if (!get_encode()) return false;
  if (!g.Pb || !g.Qb || g.M < 1 || g.N < 1 || g.K < 1) return false;
  // TMA: 16-byte aligned bases and row strides
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
  if (g.q_blocks > 1 && (g.q_block_k % kBK != 0 || (int64_t)g.q_block_k * g.q_blocks != g.K))
    return false;
  return al(g.Pb) && al(g.Ps) && al(g.Qb) && al(g.Qs) && (g.ldP % 4 == 0) && (g.ldQ % 4 == 0) &&
         (g.ldC % 4 == 0);
}

cudaError_t launch_gemm_tc(const GemmArgs& g, int passes, cudaStream_t s, int device) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.cta_group == 1)
    return passes == 1 ? launch_impl<1, 1>(g, s, device) : launch_impl<1, 3>(g, s, device);
  return passes == 1 ? launch_impl<2, 1>(g, s, device) : launch_impl<2, 3>(g, s, device);
}

}  // namespace fpfp
