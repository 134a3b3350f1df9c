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

// Marginal aggregation of the per-block vectors as a tiled fp32 GEMM with the 0/1 marginal
// indicator: Z = M0 z (forward, aggregation.cpp:40-56) or dZ_agg = M0^T dZ (backward,
// backward.cpp:170-178).  grid (ceil(T_out/64), U); 256 threads, 64 output rows x d columns
// per CTA, K (= block index) staged 32 at a time.
template <bool kTrans>
__global__ void __launch_bounds__(256) k_aggregate_vec(const int8_t* __restrict__ labels,
                                                       const float* __restrict__ x, int d, int Tm,
                                                       int Tn, float* __restrict__ out) {
  constexpr int BM = 16, BK = 32;
  __shared__ float sa[BK][BM + 1];   // indicator tile, [k][m]
  __shared__ float sx[BK][128];      // x tile, [k][a]
  const long long u = blockIdx.y;
  const int m0 = blockIdx.x * BM;
  const int Mo = kTrans ? Tn : Tm, Kd = kTrans ? Tm : Tn;
  const int8_t* lu = labels + u * (long long)Tm * Tn;
  const float* xu = x + u * (long long)Kd * d;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 8 row groups x 32 column lanes
  constexpr int RPT = BM / 8;  // rows per thread group
  float acc[RPT][4];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
  for (int k0 = 0; k0 < Kd; k0 += BK) {
    __syncthreads();
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      const int kk = e / BM, m = e % BM;
      const int gm = m0 + m, gk = k0 + kk;
      float v = 0.f;
      if (gm < Mo && gk < Kd) {
        const int8_t l = kTrans ? lu[(long long)gk * Tn + gm] : lu[(long long)gm * Tn + gk];
        v = l == 0 ? 1.f : 0.f;
      }
      sa[kk][m] = v;
    }
    for (int e = threadIdx.x; e < BK * d; e += 256) {
      const int kk = e / d, a = e % d;
      sx[kk][a] = (k0 + kk < Kd) ? xu[(long long)(k0 + kk) * d + a] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      float xv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) xv[c] = (tx + 32 * c < d) ? sx[kk][tx + 32 * c] : 0.f;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const float w = sa[kk][ty * RPT + i];
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = fmaf(w, xv[c], acc[i][c]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int gm = m0 + ty * RPT + i;
    if (gm >= Mo) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (tx + 32 * c < d) out[(u * Mo + gm) * d + tx + 32 * c] = acc[i][c];
  }
}

// dW[h] = sum over the batch and the split-K chunks of O^l^T dO (backward.cpp:46).
__global__ void k_reduce_dw(const float* __restrict__ part, int chunks_per_unit, long long B,
                            long long H, int dd, float* __restrict__ dw) {
  const int h = blockIdx.y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < dd; e += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (long long b = 0; b < B; ++b) {
      const long long u = b * H + h;
      for (int c = 0; c < chunks_per_unit; ++c) acc += part[(u * chunks_per_unit + c) * (long long)dd + e];
    }
    dw[(long long)h * dd + e] = acc;
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
  k_aggregate_vec<false><<<dim3((Dm.Tm + 15) / 16, unsigned(Dm.U)), 256, 0, st>>>(s.labels, wb.z, d, Dm.Tm,
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
  const int d = Dm.d;
  launch_build_csc(Dm, s, st);
  // row phase: the linear branch (dH_i reusing the forward's h scratch, dZ_i, D^s, dQ^phi),
  // then the sparse dQ over critical pairs with dq_total = J_phi^T dQ^phi + dQ
  launch_bwd_lin(Dm, q, w, o_s, o_l, d_out, s, wb.hb, wb.gZ, wb.Ds, wb.dqphi, st);
  launch_bwd_rows(Dm, q, k, v, lse, d_out, dq, s, wb.Ds, wb.dqphi, st);
  // dH_agg = M0^T dH (A = M0 read M-major), dZ_agg
  GemmArgs a{};
  a.A = s.M0;
  a.B = wb.hb;
  a.C = wb.hab;
  a.batch = int(Dm.U);
  a.M = Dm.Tn;
  a.N = d * d;
  a.K = Dm.Tm;
  a.a_mn = true;
  a.b_mn = true;
  a.out_f32 = false;
  a.lda = m0_stride(Dm);
  a.ldb = (long long)d * d;
  a.ldc = (long long)d * d;
  a.a_batch = (long long)Dm.Tm * m0_stride(Dm);
  a.b_batch = (long long)Dm.Tm * d * d;
  a.c_batch = (long long)Dm.Tn * d * d;
  a.name = "gemm_aggregate_t";
  launch_gemm(a, st);
  k_aggregate_vec<true><<<dim3((Dm.Tn + 15) / 16, unsigned(Dm.U)), 256, 0, st>>>(s.labels, wb.gZ, d, Dm.Tm,
                                                                               Dm.Tn, wb.gZa);
  check_launch("k_aggregate_dz", st);
  // columns pass: dk_total, dv
  launch_bwd_cols(Dm, q, k, v, lse, d_out, dk, dv, s, wb.hab, wb.gZa, wb.Ds, st);
  // dW = O^l^T dO per head, split-K over row chunks of each unit, then reduced over chunks + batch
  const long long KC = 64LL * dw_chunk_tiles(Dm);
  const int chunks = int(dw_chunks(Dm));
  GemmArgs g{};
  g.A = o_l;
  g.B = d_out;
  g.C = wb.dwp;
  g.batch = int(Dm.U * chunks);
  g.M = d;
  g.N = d;
  g.K = int(KC);
  g.a_mn = true;
  g.b_mn = true;
  g.out_f32 = true;
  g.lda = d;
  g.ldb = d;
  g.ldc = d;
  g.a_batch = KC * d;
  g.b_batch = KC * d;
  g.c_batch = (long long)d * d;
  g.name = "gemm_dw";
  launch_gemm(g, st);
  k_reduce_dw<<<dim3((d * d + 255) / 256, unsigned(Dm.H)), 256, 0, st>>>(wb.dwp, chunks, Dm.B, Dm.H, d * d, dw);
  check_launch("k_reduce_dw", st);
}

}  // namespace slab
