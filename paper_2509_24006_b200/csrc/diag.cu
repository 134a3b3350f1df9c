#include <type_traits>
// diag.cu -- diagnostics used by tests/test_gpu_tmem.py to pin TMEM data-path layouts that the
// kernels rely on: (1) the thread <-> (lane, column) map of tcgen05.ld.16x32bx2, and (2) that
// an M=64 MMA whose D address carries lane offset 16 fills lanes 16-31 of each quarter.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {
namespace {

__device__ __forceinline__ void tmem_ld_16x32bx2_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16], 16;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// out[(w*32 + t)*16 + k]: value thread t of warp w read with 16x32bx2.x16 (offset 16) after
// every (lane, col) was set to lane*1000 + col by 32x32b stores.
__global__ void k_diag_tmem_x2(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc<64>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t t = slot + (uint32_t(32 * warp) << 16);
  uint32_t v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = uint32_t((32 * warp + lane) * 1000 + c);
  tc::tmem_st32(t, v);
  tc::tmem_st_wait();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  uint32_t r[16];
  tmem_ld_16x32bx2_x16(t, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int k = 0; k < 16; ++k) out[(warp * 32 + lane) * 16 + k] = r[k];
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<64>(slot);
}

// A = ones(64 x 16) (K-major SW128 in smem), B = identity-ish (16 x 64): D = A B written by an
// M=64 MMA at lane offset `loff`; out[(w*32+t)*2 + {0,1}] = (col 0, col 1) of TMEM lane 32w+t.
__global__ void k_diag_m64_lane(uint32_t loff, float* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: 64 rows x 64 (K) bf16, row m = (m+1) in column 0, zeros elsewhere; B: N=64 rows x 64 (K),
  // row n = 1 in column 0 -> D[m][n] = m + 1
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int rr = e / 64, c = e % 64;
    const uint32_t off = tc::sw128_off(rr, c / 8) + (c % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sm + off) = __float2bfloat16(c == 0 ? float(rr + 1) : 0.f);
    *reinterpret_cast<__nv_bfloat16*>(sm + 8192 + off) = __float2bfloat16(c == 0 ? 1.f : 0.f);
  }
  tc::fence_proxy_async();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<64>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // zero TMEM first
  {
    uint32_t z[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) z[c] = 0u;
    tc::tmem_st32(slot + (uint32_t(32 * warp) << 16), z);
    tc::tmem_st32(slot + (uint32_t(32 * warp) << 16) + 32, z);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(sm);
    tc::mma_bf16(slot + (loff << 16), tc::desc_kmajor(a), tc::desc_kmajor(a + 8192), tc::idesc_bf16(64, 64, false, false), 0);
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  uint32_t r[32];
  tc::tmem_ld32(slot + (uint32_t(32 * warp) << 16), r);
  tc::tmem_ld_wait();
  out[(warp * 32 + lane) * 2 + 0] = __uint_as_float(r[0]);
  out[(warp * 32 + lane) * 2 + 1] = __uint_as_float(r[1]);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<64>(slot);
}

}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_tmem(void* out_x2, void* out_m64_lo, void* out_m64_hi, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  slab::k_diag_tmem_x2<<<1, 128, 0, st>>>(static_cast<uint32_t*>(out_x2));
  cudaFuncSetAttribute(slab::k_diag_m64_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  slab::k_diag_m64_lane<<<1, 128, 20480, st>>>(0u, static_cast<float*>(out_m64_lo));
  slab::k_diag_m64_lane<<<1, 128, 20480, st>>>(16u, static_cast<float*>(out_m64_hi));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

namespace slab {
namespace {
// L2 read bandwidth probe: every CTA streams 16-byte loads over an L2-resident buffer.
__global__ void k_diag_l2bw(const uint4* __restrict__ buf, long long n16, int iters, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it)
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n16;
         e += (long long)gridDim.x * blockDim.x) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + e));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678u) sink[0] = acc;
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_l2bw(const void* buf, long long bytes, int iters, void* sink, int blocks, int threads) {
  slab::k_diag_l2bw<<<blocks, threads>>>(static_cast<const uint4*>(buf), bytes / 16, iters, static_cast<uint4*>(sink));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// (3) tcgen05.mma issue-to-completion cost per shape: one CTA, one thread issues `reps`
// back-to-back M x N x 16 bf16 MMAs (SS operands, K-major or MN-major SW128) into one TMEM
// accumulator; cycles between the first issue and the commit's mbarrier completing.
namespace slab {
namespace {
__global__ void k_diag_mma_rate(int m, int n, int a_mn, int b_mn, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < (128 + 256) * 64 / 8; e += blockDim.x)
    reinterpret_cast<uint4*>(sm)[e] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  tc::fence_proxy_async();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(sm), b = a + 128 * 128;
    const uint32_t id = tc::idesc_bf16(m, n, a_mn == 1, b_mn != 0 && a_mn < 3);
    const long long t0 = clock64();
    if (a_mn == 2) {  // A from TMEM (ts form): M lanes x 16 bf16 (8 columns) at column 256 + 8 kk
      for (int r = 0; r < reps; ++r) {
        const int kk = r & 3;
        const uint64_t db = b_mn ? tc::desc_mnmajor(b + kk * 2048, 8192) : tc::desc_kmajor(b + kk * 32);
        tc::mma_bf16_ts(slot, slot + 256 + 8 * kk, db, id, r > 0);
      }
    } else if (a_mn >= 3) {  // SS, K-major, round-robin over (a_mn - 2) accumulators 128 columns apart
      uint64_t da[4], db[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        da[kk] = tc::desc_kmajor(a + kk * 32);
        db[kk] = tc::desc_kmajor(b + kk * 32);
      }
      auto run = [&](auto nacc_c) {
        constexpr int NA = decltype(nacc_c)::value;
        for (int r = 0; r < reps; r += 4 * NA) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
#pragma unroll
            for (int q = 0; q < NA; ++q) tc::mma_bf16(slot + 128 * q, da[kk], db[kk], id, (r | kk) != 0);
        }
      };
      if (a_mn == 3) run(std::integral_constant<int, 1>{});
      else if (a_mn == 4) run(std::integral_constant<int, 2>{});
      else run(std::integral_constant<int, 4>{});
    } else {
      for (int r = 0; r < reps; ++r) {
        const int kk = r & 3;
        const uint64_t db = b_mn ? tc::desc_mnmajor(b + kk * 2048, 8192) : tc::desc_kmajor(b + kk * 32);
        const uint64_t da = a_mn ? tc::desc_mnmajor(a + kk * 2048, 8192) : tc::desc_kmajor(a + kk * 32);
        tc::mma_bf16(slot, da, db, id, r > 0);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(slot);
}
}  // namespace
}  // namespace slab

// (3b) the same for a cta_group::2 pair (cluster of 2): the leader issues `reps` M = 256 x N x 16
// MMAs over both CTAs' smem (each holds 128 rows of A and N/2 columns of B, K-major)
namespace slab {
namespace {
__global__ void k_diag_mma_pair_rate(int n, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = tc::cluster_rank();
  for (int e = threadIdx.x; e < (128 + 128) * 64 / 8; e += blockDim.x)
    reinterpret_cast<uint4*>(sm)[e] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  tc::fence_proxy_async();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::cluster_sync();
  if (warp == 0) tc::tmem_alloc_pair<256>(&slot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    if (rank == 0) {
      const uint32_t a = tc::smem_u32(sm), b = a + 128 * 128;
      const uint32_t id = tc::idesc_bf16(256, n, false, false);
      for (int r = 0; r < reps; ++r) {
        const int kk = r & 3;
        tc::mma_bf16_pair(slot, tc::desc_kmajor(a + kk * 32), tc::desc_kmajor(b + kk * 32), id, r > 0);
      }
      tc::mma_commit_pair_mc(&bar, uint16_t(3));
    }
    tc::mbar_wait(&bar, 0);
    if (rank == 0) out[0] = clock64() - t0;
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc_pair<256>(slot);
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_mma_pair_rate(int n, int reps, long long* host_cycles) {
  long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(long long)) != cudaSuccess) return 1;
  const int bytes = (128 + 128) * 128 + 1024;
  cudaFuncSetAttribute(slab::k_diag_mma_pair_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, slab::k_diag_mma_pair_rate, n, reps, d) != cudaSuccess) return 1;
  int rc = cudaMemcpy(host_cycles, d, sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
  cudaFree(d);
  return rc;
}

extern "C" int sla_b200_diag_mma_rate(int m, int n, int a_mn, int b_mn, int reps, long long* host_cycles) {
  long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(long long)) != cudaSuccess) return 1;
  const int bytes = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(slab::k_diag_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  slab::k_diag_mma_rate<<<1, 128, bytes>>>(m, n, a_mn, b_mn, reps, d);
  int rc = cudaMemcpy(host_cycles, d, sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
  cudaFree(d);
  return rc;
}

// (4) TMA throughput per SM vs bytes in flight: each CTA streams `iters` random 64x128 bf16
// tiles (16 KB, two SW128 boxes) from an L2-resident buffer through a ring of `slots` tiles.
namespace slab {
namespace {
__global__ void k_diag_tma_bw(const __grid_constant__ CUtensorMap tm, int rows, int slots, int iters,
                              int producers, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) tc::mbar_init(bars + s, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  // producer p (lane 0 of warp p) runs its own ring of slots/producers tiles
  const int pw = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && pw < producers) {
    const int ps = slots / producers, s0 = pw * ps, my_iters = iters / producers;
    uint32_t x = 12345u + 7919u * blockIdx.x + 104729u * pw;
    const int tiles = rows / 64;
    const long long t0 = clock64();
    for (int it = 0; it < my_iters + ps; ++it) {
      const int s = s0 + it % ps;
      if (it >= ps) tc::mbar_wait(bars + s, ((it / ps) - 1) & 1);
      if (it < my_iters) {
        x = x * 1664525u + 1013904223u;
        const int row = int((x >> 8) % uint32_t(tiles)) * 64;
        tc::mbar_expect_tx(bars + s, 16384);
        tc::tma_load_3d(sm + s * 16384, &tm, bars + s, 0, row, 0);
        tc::tma_load_3d(sm + s * 16384 + 8192, &tm, bars + s, 64, row, 0);
      }
    }
    const long long dt = clock64() - t0;
    if (pw == 0) out[blockIdx.x] = dt;
  }
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_tma_bw(const void* buf, int rows, int ctas, int slots, int iters,
                                    int producers, long long* host_cycles) {
  try {
    CUtensorMap tm;
    slab::make_tmap_bf16(&tm, buf, 128, uint64_t(rows), 1, 128, 0, 64);
    long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(long long) * ctas) != cudaSuccess) return 1;
    const int bytes = slots * 16384 + 1024;
    cudaFuncSetAttribute(slab::k_diag_tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    slab::k_diag_tma_bw<<<ctas, 32 * producers, bytes>>>(tm, rows, slots, iters, producers, d);
    int rc = cudaMemcpy(host_cycles, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
    cudaFree(d);
    return rc;
  } catch (...) {
    return 1;
  }
}

// (5) contention: the MMA stream of (3) while warp 1 streams TMA tile loads (16 KB each, ring
// of 4) into a separate smem region of the same CTA (tma_on = 0: MMAs alone).
namespace slab {
namespace {
__global__ void k_diag_mma_tma(const __grid_constant__ CUtensorMap tm, int rows, int m, int n, int reps,
                               int tma_on, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = sm + (128 + 256) * 128;
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, rb[4];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < (128 + 256) * 64 / 8; e += blockDim.x)
    reinterpret_cast<uint4*>(sm)[e] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  tc::fence_proxy_async();
  if (threadIdx.x == 0) {
    stop = 0;
    tc::mbar_init(&bar, 1);
    for (int s = 0; s < 4; ++s) tc::mbar_init(rb + s, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(sm), b = a + 128 * 128;
    const uint32_t id = tc::idesc_bf16(m, n, false, false);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int kk = r & 3;
      tc::mma_bf16(slot, tc::desc_kmajor(a + kk * 32), tc::desc_kmajor(b + kk * 32), id, r > 0);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[2 * blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (threadIdx.x == 32 && tma_on) {
    uint32_t x = 777u + blockIdx.x;
    const int tiles = rows / 64;
    long long loads = 0;
    for (int it = 0;; ++it) {
      const int s = it & 3;
      if (it >= 4) tc::mbar_wait(rb + s, ((it >> 2) - 1) & 1);
      if (stop) {
        for (int k = it + 1; k < it + 4; ++k)
          if (k >= 4 && k - 4 < it) tc::mbar_wait(rb + (k & 3), ((k >> 2) - 1) & 1);
        break;
      }
      x = x * 1664525u + 1013904223u;
      const int row = int((x >> 8) % uint32_t(tiles)) * 64;
      tc::mbar_expect_tx(rb + s, 16384);
      tc::tma_load_3d(ring + s * 16384, &tm, rb + s, 0, row, 0);
      tc::tma_load_3d(ring + s * 16384 + 8192, &tm, rb + s, 64, row, 0);
      ++loads;
    }
    out[2 * blockIdx.x + 1] = loads;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(slot);
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_mma_tma(const void* buf, int rows, int ctas, int m, int n, int reps, int tma_on,
                                     long long* host2) {
  try {
    CUtensorMap tm;
    slab::make_tmap_bf16(&tm, buf, 128, uint64_t(rows), 1, 128, 0, 64);
    long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(long long) * 2 * ctas) != cudaSuccess) return 1;
    cudaMemset(d, 0, sizeof(long long) * 2 * ctas);
    const int bytes = (128 + 256) * 128 + 4 * 16384 + 1024;
    cudaFuncSetAttribute(slab::k_diag_mma_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    slab::k_diag_mma_tma<<<ctas, 64, bytes>>>(tm, rows, m, n, reps, tma_on, d);
    int rc = cudaMemcpy(host2, d, sizeof(long long) * 2 * ctas, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
    cudaFree(d);
    return rc;
  } catch (...) {
    return 1;
  }
}

// (6) TMA load latency: each producer warp (lane 0) loads one item of `boxes` 8 KB SW128 boxes
// (random 64-row blocks, both 64-column halves) and waits for it before issuing the next, so
// cycles / item is the issue-to-complete latency of a ring slot of that size.
namespace slab {
namespace {
__global__ void k_diag_tma_lat(const __grid_constant__ CUtensorMap tm, int rows, int boxes, int iters,
                               int producers, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) tc::mbar_init(bars + s, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  const int pw = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && pw < producers) {
    uint8_t* dst = sm + pw * boxes * 8192;
    uint32_t x = 12345u + 7919u * blockIdx.x + 104729u * pw;
    const int tiles = rows / 64;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      tc::mbar_expect_tx(bars + pw, boxes * 8192);
      for (int b = 0; b < boxes; b += 2) {
        x = x * 1664525u + 1013904223u;
        const int row = int((x >> 8) % uint32_t(tiles)) * 64;
        tc::tma_load_3d(dst + b * 8192, &tm, bars + pw, 0, row, 0);
        tc::tma_load_3d(dst + (b + 1) * 8192, &tm, bars + pw, 64, row, 0);
      }
      tc::mbar_wait(bars + pw, it & 1);
    }
    out[blockIdx.x * 8 + pw] = clock64() - t0;
  }
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_tma_lat(const void* buf, int rows, int ctas, int boxes, int iters,
                                     int producers, long long* host_cycles) {
  try {
    CUtensorMap tm;
    slab::make_tmap_bf16(&tm, buf, 128, uint64_t(rows), 1, 128, 0, 64);
    long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(long long) * 8 * ctas) != cudaSuccess) return 1;
    const int bytes = producers * boxes * 8192 + 1024;
    cudaFuncSetAttribute(slab::k_diag_tma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    slab::k_diag_tma_lat<<<ctas, 32 * producers, bytes>>>(tm, rows, boxes, iters, producers, d);
    int rc = cudaMemcpy(host_cycles, d, sizeof(long long) * 8 * ctas, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
    cudaFree(d);
    return rc;
  } catch (...) {
    return 1;
  }
}

// (7) what slows TMA inside the backward kernels: two producer warps each load 32 KB items
// (one in flight, so cycles / item = latency) while, per `mode` bit, (1) one thread streams
// M=128 N=64 SS MMAs over distinct smem tiles, (2) 8 warps loop tcgen05.ld + exp + st.shared +
// fence.proxy.async (the softmax-gradient phase), (4) those warps skip the proxy fence.
namespace slab {
namespace {
__global__ void __launch_bounds__(352, 1)
    k_diag_contention(const __grid_constant__ CUtensorMap tm, int rows, int iters, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ld = sm;                 // 2 x 32 KB TMA destinations
  uint8_t* ops = sm + 65536;        // 96 KB MMA operand tiles
  uint8_t* pd = sm + 65536 + 98304; // 32 KB generic-proxy stores
  __shared__ uint64_t bars[2], mbar, mb2[2];
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    stop = 0;
    tc::mbar_init(bars, 1);
    tc::mbar_init(bars + 1, 1);
    tc::mbar_init(&mbar, 1);
    tc::mbar_init(mb2, 1);
    tc::mbar_init(mb2 + 1, 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp < 2) {
    if (lane == 0) {
      uint32_t x = 12345u + 7919u * blockIdx.x + 104729u * warp;
      const int tiles = rows / 64;
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        tc::mbar_expect_tx(bars + warp, 32768);
        for (int b = 0; b < 4; b += 2) {
          x = x * 1664525u + 1013904223u;
          const int row = int((x >> 8) % uint32_t(tiles)) * 64;
          tc::tma_load_3d(ld + warp * 32768 + b * 8192, &tm, bars + warp, 0, row, 0);
          tc::tma_load_3d(ld + warp * 32768 + (b + 1) * 8192, &tm, bars + warp, 64, row, 0);
        }
        tc::mbar_wait(bars + warp, it & 1);
      }
      out[blockIdx.x * 2 + warp] = clock64() - t0;
    }
    __syncwarp();
  } else if (warp == 2) {
    if (lane == 0 && (mode & 1)) {
      const uint32_t a = tc::smem_u32(ops);
      constexpr uint32_t id = tc::idesc_bf16(128, 64, false, false);
      constexpr uint32_t id_mn = tc::idesc_bf16(128, 64, true, true);
      int r = 0;
      while (!stop) {
        if (mode & 16) {  // dQ^T-like: both operands MN-major
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            tc::mma_bf16(slot + 128 * (kk & 1), tc::desc_mnmajor(a + (r % 3) * 32768 + kk * 2048, 16384),
                         tc::desc_mnmajor(a + ((r + 1) % 3) * 32768 + kk * 2048, 16384), id_mn, kk > 1);
        } else {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t base = a + ((r + kk) % 3) * 32768;
            tc::mma_bf16(slot + 128 * (kk & 1), tc::desc_kmajor(base + (kk >> 2) * 16384 + (kk & 3) * 32),
                         tc::desc_kmajor(base + 24576 + (kk & 3) * 32), id, kk > 1);
          }
        }
        if (mode & 8) {  // keep the pipe full: wait for the group before the previous one
          tc::mma_commit(mb2 + (r & 1));
          if (r >= 1) tc::mbar_wait(mb2 + ((r - 1) & 1), ((r - 1) >> 1) & 1);
        } else {
          tc::mma_commit(&mbar);
          tc::mbar_wait(&mbar, r & 1);
        }
        ++r;
      }
      if (mode & 8) tc::mbar_wait(mb2 + ((r - 1) & 1), ((r - 1) >> 1) & 1);
    }
  } else if (mode & 2) {
    const int q4 = warp & 3, grp = (warp - 3) >> 2;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const int rq = 32 * q4 + lane;
    while (!stop) {
      uint32_t sv[32], pp[16];
      tc::tmem_ld32(slot + 256 + lane_base + 32 * (grp & 1), sv);
      tc::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float p0, p1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(__uint_as_float(sv[e]) * 0.01f - 1.f));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(__uint_as_float(sv[e + 1]) * 0.01f - 1.f));
        pp[e >> 1] = tc::pack_bf16(p0, p1);
      }
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        *reinterpret_cast<uint4*>(pd + (grp & 1) * 16384 + tc::sw128_off(rq, 4 * (grp >> 1) + ch)) =
            make_uint4(pp[4 * ch], pp[4 * ch + 1], pp[4 * ch + 2], pp[4 * ch + 3]);
      if (!(mode & 4)) tc::fence_proxy_async();
      __syncwarp();
    }
  }
  if (threadIdx.x == 0) {
    // producers finished (thread 0 is producer 0); wait for producer 1 via its output slot
    while (out[blockIdx.x * 2 + 1] == 0) {
    }
    stop = 1;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc<512>(slot);
}
}  // namespace
}  // namespace slab

extern "C" int sla_b200_diag_contention(const void* buf, int rows, int ctas, int iters, int mode,
                                        long long* host2) {
  try {
    CUtensorMap tm;
    slab::make_tmap_bf16(&tm, buf, 128, uint64_t(rows), 1, 128, 0, 64);
    long long* d = nullptr;
    if (cudaMalloc(&d, sizeof(long long) * 2 * ctas) != cudaSuccess) return 1;
    cudaMemset(d, 0, sizeof(long long) * 2 * ctas);
    const int bytes = 65536 + 98304 + 32768 + 1024;
    cudaFuncSetAttribute(slab::k_diag_contention, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    slab::k_diag_contention<<<ctas, 352, bytes>>>(tm, rows, iters, mode, d);
    int rc = cudaMemcpy(host2, d, sizeof(long long) * 2 * ctas, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
    cudaFree(d);
    return rc;
  } catch (...) {
    return 1;
  }
}

// tcgen05 GEMM of gemm.cu on plain row-major operands (tests/test_gpu_gemm.py)
extern "C" int sla_b200_diag_gemm(const void* A, const void* B, void* C, int batch, int M, int N,
                                  int K, int a_mn, int b_mn, int out_f32, void* stream) {
  try {
    slab::GemmArgs g{};
    g.A = A;
    g.B = B;
    g.C = C;
    g.batch = batch;
    g.M = M;
    g.N = N;
    g.K = K;
    g.a_mn = a_mn;
    g.b_mn = b_mn;
    g.out_f32 = out_f32;
    g.lda = a_mn ? M : K;
    g.ldb = b_mn ? N : K;
    g.ldc = N;
    g.a_batch = (long long)M * K;
    g.b_batch = (long long)K * N;
    g.c_batch = (long long)M * N;
    slab::launch_gemm(g, static_cast<cudaStream_t>(stream));
    return 0;
  } catch (const slab::InvalidArgument& e) {
    std::fprintf(stderr, "%s\n", e.msg.c_str());
    return 2;
  } catch (const slab::CudaError& e) {
    std::fprintf(stderr, "%s\n", e.msg.c_str());
    return 1;
  }
}

// rows of k_classify_rank that fall back to the exact P_c ranking are counted into *dev_counter
// (a device int; null stops counting) -- tests/test_gpu_classify.py checks the fallback is rare
extern "C" int sla_b200_diag_classify_exact(int* dev_counter) {
  slab::set_classify_exact_counter(dev_counter);
  return 0;
}
