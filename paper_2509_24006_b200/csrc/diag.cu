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
    const uint32_t id = tc::idesc_bf16(m, n, a_mn != 0, b_mn != 0);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int kk = r & 3;
      const uint64_t da = a_mn ? tc::desc_mnmajor(a + kk * 2048, 8192) : tc::desc_kmajor(a + kk * 32);
      const uint64_t db = b_mn ? tc::desc_mnmajor(b + kk * 2048, 8192) : tc::desc_kmajor(b + kk * 32);
      tc::mma_bf16(slot, da, db, id, r > 0);
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
