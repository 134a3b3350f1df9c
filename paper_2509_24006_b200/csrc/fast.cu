// fast.cu -- the tcgen05 fast path (b_q = b_kv = 64, d in {64, 128}, bf16):
//   K3  phi(K) (bf16) and z_j = colsum phi(K_j)                 k_phi_kz
//       h_j = phi(K_j)^T V_j for every key block                tcgen05 batched GEMM
//   K4  H = M0 . h (M0 = marginal indicator, bf16 0/1)          tcgen05 GEMM
//       Z = sum over marginal z_j (ascending, f32)              k_aggregate_z
//   K5  fused sparse + linear + projection forward              attn_fwd.cu
// References: summaries.cpp:17-42, aggregation.cpp:40-56, forward.cpp:81-195.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

namespace {

// phi(K) rows -> bf16, and z_j = sum over the block's rows of phi(K) (f32).  grid (Tn, U),
// 8 warps, each warp 8 rows; lane owns D/32 consecutive columns.
template <int D>
__global__ void __launch_bounds__(256) k_phi_kz(const __nv_bfloat16* __restrict__ k,
                                                __nv_bfloat16* __restrict__ kfb,
                                                float* __restrict__ z, long long N, int Tn, int phi) {
  constexpr int C = D / 32;
  __shared__ float zpart[8][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  float zacc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) zacc[c] = 0.f;
  for (int rr = 0; rr < 8; ++rr) {
    const long long row = u * N + (long long)j * 64 + warp * 8 + rr;
    const __nv_bfloat16* src = k + row * D + lane * C;
    float x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = __bfloat162float(src[c]);
    if (phi == 2) {
      float m = -INFINITY;
#pragma unroll
      for (int c = 0; c < C; ++c) m = fmaxf(m, x[c]);
      m = warp_max(m);
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x[c] = __expf(x[c] - m);
        s += x[c];
      }
      s = warp_sum(s);
      const float inv = 1.f / s;
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] *= inv;
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = phi_elem(phi, x[c]);
    }
    __nv_bfloat16* dst = kfb + row * D + lane * C;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      dst[c] = __float2bfloat16_rn(x[c]);
      zacc[c] += x[c];
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) zpart[warp][lane * C + c] = zacc[c];
  __syncthreads();
  for (int a = threadIdx.x; a < D; a += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += zpart[w][a];
    z[(u * Tn + j) * D + a] = s;
  }
}

// Z_i = sum_{j marginal, ascending} z_j (aggregation.cpp:40-56); grid (Tm, U), D threads.
__global__ void k_aggregate_z(const int8_t* __restrict__ labels, const float* __restrict__ z,
                              int d, int Tm, int Tn, float* __restrict__ Z) {
  extern __shared__ int slist[];
  __shared__ int s_cnt;
  const long long u = blockIdx.y;
  const int i = blockIdx.x;
  if (threadIdx.x < 32) {
    const int8_t* lrow = labels + (u * Tm + i) * (long long)Tn;
    int base = 0;
    for (int j0 = 0; j0 < Tn; j0 += 32) {
      const int j = j0 + threadIdx.x;
      const bool m = j < Tn && lrow[j] == 0;
      const unsigned b = __ballot_sync(0xffffffffu, m);
      if (m) slist[base + __popc(b & ((1u << threadIdx.x) - 1u))] = j;
      base += __popc(b);
    }
    if (threadIdx.x == 0) s_cnt = base;
  }
  __syncthreads();
  const int cnt = s_cnt;
  const float* zu = z + u * (long long)Tn * d;
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < cnt; ++p) acc += zu[(long long)slist[p] * d + a];
    Z[(u * Tm + i) * d + a] = acc;
  }
}

}  // namespace

bool fast_supported(const Dims& D, int dtype) {
  return dtype == 0 && D.bq == 64 && D.bkv == 64 && (D.d == 64 || D.d == 128);
}

void fast_prepare_linear(const Dims& Dm, const void* k, const void* v, const StateBufs& s,
                         const WorkBufs& wb, cudaStream_t st) {
  const int d = Dm.d;
  if (d == 128)
    k_phi_kz<128><<<dim3(Dm.Tn, unsigned(Dm.U)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z, Dm.N, Dm.Tn, Dm.phi);
  else
    k_phi_kz<64><<<dim3(Dm.Tn, unsigned(Dm.U)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z, Dm.N, Dm.Tn, Dm.phi);
  check_launch("k_phi_kz", st);
  // h_j = phi(K_j)^T V_j: batch = every key block, M = N = d, K = 64 tokens
  GemmArgs g{};
  g.A = wb.kfb;
  g.B = v;
  g.C = wb.hb;
  g.batch = int(Dm.U * Dm.Tn);
  g.M = d;
  g.N = d;
  g.K = 64;
  g.a_mn = true;
  g.b_mn = true;
  g.out_f32 = false;
  g.lda = d;
  g.ldb = d;
  g.ldc = d;
  g.a_batch = 64LL * d;
  g.b_batch = 64LL * d;
  g.c_batch = (long long)d * d;
  g.name = "gemm_summaries";
  launch_gemm(g, st);
  // H = M0 . h per unit: M = Tm, N = d*d, K = Tn
  launch_build_m0(Dm, s, st);
  GemmArgs a{};
  a.A = s.M0;
  a.B = wb.hb;
  a.C = s.Hb;
  a.batch = int(Dm.U);
  a.M = Dm.Tm;
  a.N = d * d;
  a.K = Dm.Tn;
  a.a_mn = false;
  a.b_mn = true;
  a.out_f32 = false;
  a.lda = m0_stride(Dm);
  a.ldb = (long long)d * d;
  a.ldc = (long long)d * d;
  a.a_batch = (long long)Dm.Tm * m0_stride(Dm);
  a.b_batch = (long long)Dm.Tn * d * d;
  a.c_batch = (long long)Dm.Tm * d * d;
  a.name = "gemm_aggregate";
  launch_gemm(a, st);
  k_aggregate_z<<<dim3(Dm.Tm, unsigned(Dm.U)), d, size_t(Dm.Tn) * 4, st>>>(s.labels, wb.z, d, Dm.Tm,
                                                                            Dm.Tn, s.Z);
  check_launch("k_aggregate_z", st);
}

void fast_forward(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                  void* o, void* o_s, void* o_l, float* lse, const StateBufs& s,
                  const WorkBufs& wb, cudaStream_t st) {
  fast_prepare_linear(Dm, k, v, s, wb, st);
  launch_attn_fwd(Dm, q, k, v, w, o, o_s, o_l, lse, s, st);
}

void fast_backward(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                   const void* o_s, const void* o_l, const float* lse, const void* d_out,
                   void* dq, void* dk, void* dv, float* dw, const StateBufs& s,
                   const WorkBufs& wb, cudaStream_t st) {
  // first fast-path revision: the SIMT backward over the fast path's bf16 H state
  generic_backward(Dm, 0, q, k, v, w, o_s, o_l, lse, d_out, dq, dk, dv, dw, s, wb, st);
}

}  // namespace slab
