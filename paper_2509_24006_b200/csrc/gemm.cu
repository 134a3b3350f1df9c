// gemm.cu -- batched bf16 tcgen05 GEMM, the workhorse of the linear (marginal) branch:
//   H   = M0 . h        (aggregation.cpp:40-56 as a GEMM; M0 is the 0/1 marginal indicator)
//   h_j = phi(K_j)^T V_j (summaries.cpp:17-42, batched over key blocks)
//   dH_agg = M0^T . dH  (backward.cpp:170-178)
// C[b] = A[b] . B[b] with A either K-major ([M][K] rows) or M-major ([K][M] rows) and
// B either N-major ([K][N] rows) or K-major ([N][K] rows); fp32 accumulate in TMEM.
//
// Warp roles (224 threads): warp 0 = TMA producer of A, warp 6 = TMA producer of B (one issuing
// warp's TMA stream saturates at ~40 B/cycle, two reach ~70 B/cycle per SM -- csrc/diag.cu
// sla_b200_diag_tma_bw -- so each stage is filled by both), warp 1 = MMA issuer (one elected thread), warps 2-5 = epilogue
// (TMEM -> registers -> global).  4-stage smem ring with full/empty mbarriers; the
// accumulator lives in TMEM (BN columns).
#include <algorithm>
#include <cstdio>

#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

namespace {

constexpr int kStages = 4;
#ifndef SLAB_GEMM_P2_STAGES
#define SLAB_GEMM_P2_STAGES 6  // a P2 stage is 32 KB (A 16 KB + half of B 16 KB)
#endif
constexpr int kBK = 64;  // K elements per stage (one 128-byte swizzle row of bf16)

template <int BM, int BN, int ST = kStages>
struct GemmSmem {
  static constexpr int kStagesN = ST;
  static constexpr int kA = BM * kBK * 2;
  static constexpr int kB = BN * kBK * 2;
  static constexpr int kStage = kA + kB;
  static constexpr int kOut = BM * 64 * 2;  // one [BM][64] bf16 output box (TMA-store staging)
  static constexpr int oOut = ST * kStage;
  static constexpr int kBytes = oOut + 2 * kOut + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(kBytes <= 232448, "smem");
};

// Persistent: each CTA walks tiles blockIdx.x, +gridDim.x, ...; the smem ring runs across tile
// boundaries and the TMEM accumulator is double-buffered (2 x BN columns) so the epilogue of
// tile t overlaps the main loop of tile t+1.
// MC: 2-CTA clusters whose CTAs take the two M-halves of a 2*BM x BN tile pair; each CTA
// loads half of the pair's B k-block and multicasts it to both, so B crosses L2 -> SM once per
// pair (the aggregation GEMMs are L2-bandwidth-bound).  A stage is refilled only after BOTH
// CTAs' MMAs released it (every MMA commit arrives on the empty barrier of both CTAs).
// P2: a cta_group::2 pair -- the leader issues M = 2*BM MMAs over both CTAs' smem; each CTA
// holds its own BM rows of A and half (BN/2 columns) of B.  Every TMA load completes on the
// leader's full barrier; the leader's commits arrive on both CTAs' empty / tfull barriers; both
// epilogues arrive on the leader's tempty.
template <int BM, int BN, bool A_MN, bool B_MN, typename OutT, bool MC = false, bool P2 = false>
__global__ void __launch_bounds__(224, 1)
    k_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap tc_out,
           OutT* __restrict__ C, int M, int N, int K, int batch, long long c_batch, int ldc,
           RowLayout arl, RowLayout brl, int a_rpu, int b_rpu) {
  pdl_entry();  // launched by launch_pdl
  static_assert(!(MC && P2), "one pairing mode");
  using L = GemmSmem<BM, P2 ? BN / 2 : BN, P2 ? SLAB_GEMM_P2_STAGES : kStages>;  // P2: a stage holds half of B
  constexpr int kStages = L::kStagesN;
  constexpr bool PAIRED = MC || P2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::oOut + 2 * L::kOut);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + kBK - 1) / kBK;
  const int tiles_n = N / BN, tiles_m = (M + BM - 1) / BM;
  // work units: tiles, or (MC) pairs of M-adjacent tiles, one per CTA of the cluster
  const int rank = PAIRED ? int(tc::cluster_rank()) : 0;
  const long long unit0 = PAIRED ? blockIdx.x / 2 : blockIdx.x;
  const long long ustep = PAIRED ? gridDim.x / 2 : gridDim.x;
  const int units_m = PAIRED ? tiles_m / 2 : tiles_m;
  const long long total = (long long)tiles_n * units_m * batch;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&ta);
      tc::tma_prefetch(&tb);
      for (int s = 0; s < kStages; ++s) {
        tc::mbar_init(&full[s], P2 ? 4 : 2);     // one arrive.expect_tx per producer (P2: of both CTAs)
        tc::mbar_init(&empty[s], MC ? 2 : 1);    // (MC) both CTAs' MMA commits
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(&tfull[s], 1);
        tc::mbar_init(&tempty[s], P2 ? 8 : 4);  // (P2) both CTAs' epilogue warps
      }
      tc::fence_barrier_init();
    }
    __syncwarp();
    if constexpr (P2)
      tc::tmem_alloc_pair<2 * BN>(tmem_slot);
    else
      tc::tmem_alloc<2 * BN>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (PAIRED) tc::cluster_sync();  // the peer's barriers are initialised before any multicast / remote arrive
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto coords = [&](long long t, int& n0, int& m0, int& b) {
    n0 = int(t % tiles_n) * BN;
    m0 = (PAIRED ? 2 * int((t / tiles_n) % units_m) + rank : int((t / tiles_n) % units_m)) * BM;
    b = int(t / ((long long)tiles_n * units_m));
  };

  if (warp == 0 || warp == 6) {
    if (lane == 0) {
      const bool loads_a = warp == 0;
      int kc = 0;  // k-blocks issued by this CTA (ring position)
      for (long long t = unit0; t < total; t += ustep) {
        int n0, m0, b;
        coords(t, n0, m0, b);
        for (int kb = 0; kb < nk; ++kb, ++kc) {
          const int s = kc % kStages;
          tc::mbar_wait(&empty[s], ((kc / kStages) & 1) ^ 1);
          uint8_t* sa = smem + s * L::kStage;
          uint8_t* sb = sa + L::kA;
          const int k0 = kb * kBK;
          if constexpr (P2) {  // own half, completing on the leader's full barrier
            const uint32_t lf = tc::mapa_shared(tc::smem_u32(&full[s]), 0);
            if (loads_a) {
              tc::mbar_expect_tx_cluster_relaxed(lf, L::kA);
              if (A_MN) {
#pragma unroll
                for (int c = 0; c < BM / 64; ++c) tc::tma_load_3d_pair(sa + c * 8192, &ta, lf, m0 + 64 * c, k0, b);
              } else {
                tc::tma_load_3d_pair(sa, &ta, lf, k0, m0, b);
              }
            } else {
              static_assert(!P2 || (B_MN && BN % 128 == 0), "P2: N-major B, 64-column chunks per half");
              tc::mbar_expect_tx_cluster_relaxed(lf, L::kB);
#pragma unroll
              for (int c = 0; c < BN / 128; ++c)
                tc::tma_load_3d_pair(sb + c * 8192, &tb, lf, n0 + rank * (BN / 2) + 64 * c, k0, b);
            }
            continue;
          }
          if (loads_a) {
            tc::mbar_expect_tx(&full[s], L::kA);
            if (A_MN && arl.mode) {  // a caller tensor in place: chunk b % a_rpu of unit b / a_rpu
#pragma unroll
              for (int c = 0; c < BM / 64; ++c)
                tc::tma_load_rows(sa + c * 8192, &ta, &full[s], m0 + 64 * c, (b % a_rpu) * K + k0, row_tma(arl, b / a_rpu, 0));
            } else if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c) tc::tma_load_3d(sa + c * 8192, &ta, &full[s], m0 + 64 * c, k0, b);
            } else {
              tc::tma_load_3d(sa, &ta, &full[s], k0, m0, b);
            }
          } else {
            tc::mbar_expect_tx(&full[s], L::kB);
            if (MC) {  // my half of the pair's B chunks, to both CTAs
              static_assert(!MC || (B_MN && BN % 128 == 0), "MC: N-major B, even chunk count");
#pragma unroll
              for (int c = rank * (BN / 128); c < (rank + 1) * (BN / 128); ++c)
                tc::tma_load_3d_mc(sb + c * 8192, &tb, &full[s], n0 + 64 * c, k0, b, uint16_t(3));
            } else if (B_MN && brl.mode) {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c)
                tc::tma_load_rows(sb + c * 8192, &tb, &full[s], n0 + 64 * c, (b % b_rpu) * K + k0, row_tma(brl, b / b_rpu, 0));
            } else if (B_MN) {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c) tc::tma_load_3d(sb + c * 8192, &tb, &full[s], n0 + 64 * c, k0, b);
            } else {
              tc::tma_load_3d(sb, &tb, &full[s], k0, n0, b);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (P2 && rank != 0) {
      // the pair's MMAs are issued by the leader
    } else {
    constexpr uint32_t idesc = tc::idesc_bf16(P2 ? 2 * BM : BM, BN, A_MN, B_MN);
    int kc = 0, lt = 0;
    for (long long t = unit0; t < total; t += ustep, ++lt) {
      const int ab = lt & 1;
      tc::mbar_wait(&tempty[ab], ((lt >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t acc = tmem + ab * BN;
      for (int kb = 0; kb < nk; ++kb, ++kc) {
        const int s = kc % kStages;
        tc::mbar_wait(&full[s], (kc / kStages) & 1);
        tc::tc_fence_after();
        {  // whole warp, one elected lane issues (warp-uniform descriptors, see tc::mma_bf16_w)
          const uint32_t sa = tc::smem_u32(smem + s * L::kStage);
          const uint32_t sb = sa + L::kA;
          const uint64_t a0 = A_MN ? tc::desc_mnmajor(sa, 8192) : tc::desc_kmajor(sa);
          const uint64_t b0 = B_MN ? tc::desc_mnmajor(sb, 8192) : tc::desc_kmajor(sb);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t da = tc::desc_add(a0, A_MN ? kk * 2048 : kk * 32);
            const uint64_t db = tc::desc_add(b0, B_MN ? kk * 2048 : kk * 32);
            if constexpr (P2)
              tc::mma_bf16_pair_w(acc, da, db, idesc, (kb | kk) != 0);
            else
              tc::mma_bf16_w(acc, da, db, idesc, (kb | kk) != 0);
          }
          if (P2)
            tc::mma_commit_pair_mc_w(&empty[s], uint16_t(3));
          else if (MC)
            tc::mma_commit_mc_w(&empty[s], uint16_t(3));
          else
            tc::mma_commit_w(&empty[s]);
          if (kb == nk - 1) {
            if (P2)
              tc::mma_commit_pair_mc_w(&tfull[ab], uint16_t(3));
            else
              tc::mma_commit_w(&tfull[ab]);
          }
        }
      }
    }
    }
  } else if (warp <= 5) {
    // epilogue warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3;
    int lt = 0;
    // output chunks staged so far by this CTA: the staging-buffer parity runs across tiles (with
    // BN = 64 a tile is one chunk, and restarting the parity per tile would overwrite the buffer
    // the previous tile's TMA store may still be reading)
    int oc = 0;
    for (long long t = unit0; t < total; t += ustep, ++lt) {
      int n0, m0, b;
      coords(t, n0, m0, b);
      const int ab = lt & 1;
      tc::mbar_wait(&tfull[ab], (lt >> 1) & 1);
      tc::tc_fence_after();
      const int row = BM == 128 ? 32 * q + lane : 16 * q + lane;
      const bool live = (BM == 128 || lane < 16) && (m0 + row) < M;
      if constexpr (sizeof(OutT) == 2) {
        // bf16: each 64-column chunk goes TMEM -> registers -> SW128 smem box -> one TMA store
        // (coalesced; row-per-thread global stores were as slow as the MMAs of the tile)
        const uint32_t ob = tc::smem_u32(smem + L::oOut);
#pragma unroll 1
        for (int c = 0; c < BN / 64; ++c, ++oc) {
          uint32_t r0[32], r1[32];
          const uint32_t ta0 = tmem + ab * BN + (uint32_t(32 * q) << 16) + 64 * c;
          tc::tmem_ld32(ta0, r0);
          tc::tmem_ld32(ta0 + 32, r1);
          tc::tmem_ld_wait();
          // staging buffer (oc & 1) is free once the store issued two chunks ago has read it
          if (threadIdx.x == 64) tc::bulk_wait_read<1>();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const uint32_t buf = ob + (oc & 1) * L::kOut;
          if (BM == 128 || lane < 16) {
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint32_t* src = ch < 4 ? r0 + 8 * ch : r1 + 8 * (ch - 4);
              uint4 v;
              v.x = tc::pack_bf16(__uint_as_float(src[0]), __uint_as_float(src[1]));
              v.y = tc::pack_bf16(__uint_as_float(src[2]), __uint_as_float(src[3]));
              v.z = tc::pack_bf16(__uint_as_float(src[4]), __uint_as_float(src[5]));
              v.w = tc::pack_bf16(__uint_as_float(src[6]), __uint_as_float(src[7]));
              tc::sts_u4(buf + tc::sw128_off(row, ch), v);
            }
          }
          tc::fence_proxy_async();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 64) {
            tc::tma_store_3d(&tc_out, smem + L::oOut + (oc & 1) * L::kOut, n0 + 64 * c, m0, b);
            tc::bulk_commit();
          }
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (P2)
            tc::mbar_arrive_cluster_relaxed(tc::mapa_shared(tc::smem_u32(&tempty[ab]), 0));  // TMEM reads waited (wait::ld)
          else
            tc::mbar_arrive(&tempty[ab]);
        }
        continue;
      }
      OutT* crow = C + (long long)b * c_batch + (long long)(m0 + row) * ldc + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + ab * BN + (uint32_t(32 * q) << 16) + c0, r);
        tc::tmem_ld_wait();
        if (live) {
          if constexpr (sizeof(OutT) == 4) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(crow + c0 + e) =
                  make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                              __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
          } else {
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 v;
              v.x = tc::pack_bf16(__uint_as_float(r[e]), __uint_as_float(r[e + 1]));
              v.y = tc::pack_bf16(__uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
              v.z = tc::pack_bf16(__uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]));
              v.w = tc::pack_bf16(__uint_as_float(r[e + 6]), __uint_as_float(r[e + 7]));
              *reinterpret_cast<uint4*>(crow + c0 + e) = v;
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (P2)
          tc::mbar_arrive_cluster_relaxed(tc::mapa_shared(tc::smem_u32(&tempty[ab]), 0));  // TMEM reads waited (wait::ld)
        else
          tc::mbar_arrive(&tempty[ab]);
      }
    }
  }
  if (threadIdx.x == 64) tc::bulk_wait_read<0>();
  tc::tc_fence_before();
  __syncthreads();
  if (PAIRED) tc::cluster_sync();  // no remote arrive may target a CTA that has exited
  if (warp == 0) {
    if constexpr (P2)
      tc::tmem_dealloc_pair<2 * BN>(tmem);
    else
      tc::tmem_dealloc<2 * BN>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SLAB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

template <int BM, int BN, bool A_MN, bool B_MN, typename OutT, bool MC = false, bool P2 = false>
void launch_gemm_t(const GemmArgs& g, cudaStream_t st) {
  CUtensorMap ta, tb;
  // A: K-major -> tensor [batch][M][K], box [BM][64]; M-major -> [batch][K][M], box [64][64]
  if (g.a_rl.mode && !A_MN) throw InvalidArgument("sla_b200 gemm: in-place A must be M-major");
  if (g.b_rl.mode && !B_MN) throw InvalidArgument("sla_b200 gemm: in-place B must be N-major");
  if (g.a_rl.mode)
    make_tmap_rows(&ta, g.A, g.M, g.units, 0, g.a_rl, 64);
  else if (A_MN)
    make_tmap_bf16(&ta, g.A, g.M, g.K, g.batch, g.lda, g.a_batch, 64);
  else
    make_tmap_bf16(&ta, g.A, g.K, g.M, g.batch, g.lda, g.a_batch, BM);
  if (g.b_rl.mode)
    make_tmap_rows(&tb, g.B, g.N, g.units, 0, g.b_rl, 64);
  else if (B_MN)
    make_tmap_bf16(&tb, g.B, g.N, g.K, g.batch, g.ldb, g.b_batch, 64);
  else
    make_tmap_bf16(&tb, g.B, g.K, g.N, g.batch, g.ldb, g.b_batch, BN);
  CUtensorMap tcm{};
  if (sizeof(OutT) == 2)  // output boxes [BM rows][64 cols] of C [batch][M][ldc]
    make_tmap_bf16(&tcm, g.C, g.N, g.M, g.batch, g.ldc, g.c_batch, BM);
  auto kern = k_gemm<BM, BN, A_MN, B_MN, OutT, MC, P2>;
  constexpr int smem = GemmSmem<BM, P2 ? BN / 2 : BN, P2 ? SLAB_GEMM_P2_STAGES : kStages>::kBytes;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const long long tiles = (long long)(g.N / BN) * ((g.M + BM - 1) / BM) * g.batch;
  static int sms = 0;
  if (!sms) SLAB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  if (MC || P2) {  // 2-CTA clusters, one tile pair per cluster at a time
    const int grid = int(std::min<long long>(tiles, sms)) & ~1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(224);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = SLAB_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, static_cast<OutT*>(g.C), g.M, g.N, g.K, g.batch, g.c_batch, g.ldc,
                       g.a_rl, g.b_rl, g.a_rpu, g.b_rpu);
  } else {
    const int grid = int(std::min<long long>(tiles, sms));
    launch_pdl(kern, grid, 224, smem, st, ta, tb, tcm, static_cast<OutT*>(g.C), g.M, g.N, g.K, g.batch, g.c_batch, g.ldc,
               g.a_rl, g.b_rl, g.a_rpu, g.b_rpu);
  }
  check_launch(g.name ? g.name : "k_gemm", st);
}

#ifndef SLAB_GEMM_2SM
#define SLAB_GEMM_2SM 1  // cta_group::2 pairs for the aggregation GEMMs (takes precedence over MC)
#endif
#ifndef SLAB_GEMM_MC
#define SLAB_GEMM_MC 1  // measured: gemm_aggregate_t 0.098 -> 0.093 ms, gemm_aggregate 0.098 -> 0.097
#endif
template <int BM, int BN, typename OutT>
void dispatch_major(const GemmArgs& g, cudaStream_t st) {
  // B multicast across 2-CTA clusters where the tile grid pairs up (the aggregation GEMMs)
  if constexpr (BM == 128 && BN == 256 && sizeof(OutT) == 2) {
    const int tiles_m = (g.M + BM - 1) / BM;
    if (SLAB_GEMM_2SM && g.b_mn && tiles_m % 2 == 0 && g.M % BM == 0 && !g.a_rl.mode && !g.b_rl.mode) {
      if (g.a_mn) launch_gemm_t<BM, BN, true, true, OutT, false, true>(g, st);
      else launch_gemm_t<BM, BN, false, true, OutT, false, true>(g, st);
      return;
    }
    if (SLAB_GEMM_MC && g.b_mn && tiles_m % 2 == 0 && g.M % BM == 0) {
      if (g.a_mn) launch_gemm_t<BM, BN, true, true, OutT, true>(g, st);
      else launch_gemm_t<BM, BN, false, true, OutT, true>(g, st);
      return;
    }
  }
  if (g.a_mn && g.b_mn) launch_gemm_t<BM, BN, true, true, OutT>(g, st);
  else if (g.a_mn) launch_gemm_t<BM, BN, true, false, OutT>(g, st);
  else if (g.b_mn) launch_gemm_t<BM, BN, false, true, OutT>(g, st);
  else launch_gemm_t<BM, BN, false, false, OutT>(g, st);
}

template <typename OutT>
void dispatch_tile(const GemmArgs& g, cudaStream_t st) {
  const int BM = (g.M % 128 == 0 || g.M > 192) ? 128 : 64;
  const int BN = g.N % 256 == 0 ? 256 : (g.N % 128 == 0 ? 128 : 64);
  if (BM == 128) {
    if (BN == 256) dispatch_major<128, 256, OutT>(g, st);
    else if (BN == 128) dispatch_major<128, 128, OutT>(g, st);
    else dispatch_major<128, 64, OutT>(g, st);
  } else {
    if (BN == 256) dispatch_major<64, 256, OutT>(g, st);
    else if (BN == 128) dispatch_major<64, 128, OutT>(g, st);
    else dispatch_major<64, 64, OutT>(g, st);
  }
}

}  // namespace

bool make_tmap_rows(CUtensorMap* map, const void* base, uint64_t d, long long U, long long N,
                    const RowLayout& rl, uint32_t box_rows) {
  // always 4-D {d, h, rows, z} so the kernels address every layout as (c, t.h, t.y0 + r, t.z)
  // (row_tma) without branching: mode 0 [U*N][d], mode 1 [U][nv][d], mode 2 [B][nv][H][d]
  uint64_t dims_h = 1, rows, outer;
  uint64_t s_h = d * 2, s_row, s_outer;
  if (rl.mode == 0) {
    rows = uint64_t(U) * uint64_t(N);
    outer = 1;
    s_row = d * 2;
    s_outer = rows * d * 2;
  } else if (rl.mode == 1) {
    rows = uint64_t(rl.nv);
    outer = uint64_t(U);
    s_row = d * 2;
    s_outer = rows * d * 2;
  } else {
    dims_h = uint64_t(rl.H);
    rows = uint64_t(rl.nv);
    outer = uint64_t(U) / dims_h;
    s_h = d * 2;
    s_row = dims_h * d * 2;
    s_outer = rows * dims_h * d * 2;
  }
  cuuint64_t dims[4] = {d, dims_h, rows, outer};
  cuuint64_t strides[3] = {s_h, s_row, s_outer};
  cuuint32_t box[4] = {64, 1, box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled (4-D rows) failed (" + std::to_string(int(r)) + ")");
  return true;
}

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t outer,
                    uint64_t row_stride_elems, uint64_t outer_stride_elems, uint32_t box_rows) {
  cuuint64_t dims[3] = {cols, rows, outer};
  cuuint64_t strides[2] = {row_stride_elems * 2, outer_stride_elems * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return true;
}

void launch_gemm(const GemmArgs& g, cudaStream_t st) {
  // N must tile exactly; M and K tails are handled by TMA zero fill + masked stores
  if (g.N % 64 || g.M <= 0 || g.N <= 0 || g.K <= 0)
    throw InvalidArgument("sla_b200 gemm: N must be a positive multiple of 64");
  if (g.out_f32)
    dispatch_tile<float>(g, st);
  else
    dispatch_tile<__nv_bfloat16>(g, st);
}

}  // namespace slab
