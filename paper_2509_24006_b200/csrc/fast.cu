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
                                                float* __restrict__ z, long long N, int Tn, int phi,
                                                long long n_valid) {
  constexpr int C = D / 32;
  __shared__ float zpart[8][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  float zacc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) zacc[c] = 0.f;
  for (int rr = 0; rr < 8; ++rr) {
    const long long rin = (long long)j * 64 + warp * 8 + rr;  // row within the unit
    const long long row = u * N + rin;
    const __nv_bfloat16* src = k + row * D + lane * C;
    float x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = __bfloat162float(src[c]);
    if (rin >= n_valid) {  // ragged N: padded keys have no feature map (no summary weight)
      __nv_bfloat16* dst = kfb + row * D + lane * C;
#pragma unroll
      for (int c = 0; c < C; ++c) dst[c] = __float2bfloat16_rn(0.f);
      continue;
    }
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
// indicator M0 (bf16, the A operand of the H GEMM): Z = M0 z (forward, aggregation.cpp:40-56)
// or dZ_agg = M0^T dZ (backward, backward.cpp:170-178).  grid (ceil(T_out/32), U); 256
// threads, 32 output rows x d (<= 128) columns per CTA, 2 rows x 8 columns per thread; K (the
// block index) staged 64 at a time with coalesced 16-byte loads of M0 and x.
template <bool kTrans>
__global__ void __launch_bounds__(256) k_aggregate_vec(const __nv_bfloat16* __restrict__ m0, int ld,
                                                       const float* __restrict__ x, int d, int Tm,
                                                       int Tn, float* __restrict__ out) {
  constexpr int BM = 32, BK = 64;
  __shared__ __align__(16) float sa[BK][BM];   // indicator tile, [k][m]
  __shared__ __align__(16) float sx[BK][128];  // x tile, [k][a]
  const long long u = blockIdx.y;
  const int m0r = blockIdx.x * BM;
  const int Mo = kTrans ? Tn : Tm, Kd = kTrans ? Tm : Tn;
  const __nv_bfloat16* mu = m0 + u * (long long)Tm * ld;
  const float* xu = x + u * (long long)Kd * d;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;  // rows 2*ty, 2*ty+1; columns 4*tx.. and 64+4*tx..
  float acc[2][8];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
  // chunk k0 is staged from registers loaded during chunk k0 - BK (software pipelining)
  uint4 ra;
  float4 rx[8];
  auto load = [&](int k0) {
    ra = make_uint4(0, 0, 0, 0);
    if (!kTrans) {  // A[m][k] = M0[m][k]: row m = tid/8, k chunk 8*(tid%8)
      const int gm = m0r + (tid >> 3), gk = k0 + 8 * (tid & 7);
      if (gm < Mo && gk < ld) ra = *reinterpret_cast<const uint4*>(mu + (long long)gm * ld + gk);
    } else {  // A[m][k] = M0[k][m]: row k = tid/4, m chunk 8*(tid%4)
      const int gk = k0 + (tid >> 2), gm = m0r + 8 * (tid & 3);
      if (gk < Kd && gm < ld) ra = *reinterpret_cast<const uint4*>(mu + (long long)gk * ld + gm);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // x: 64 rows x 128 columns as float4, 8 per thread
      const int e = tid + 256 * r;
      const int kk = e >> 5, a4 = 4 * (e & 31);
      rx[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k0 + kk < Kd && a4 < d) rx[r] = *reinterpret_cast<const float4*>(xu + (long long)(k0 + kk) * d + a4);
    }
  };
  load(0);
  for (int k0 = 0; k0 < Kd; k0 += BK) {
    __syncthreads();
    {
      float v[8];
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&ra);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h2[e]);
        v[2 * e] = f.x;
        v[2 * e + 1] = f.y;
      }
      if (!kTrans) {
        const int m = tid >> 3, kc = 8 * (tid & 7);
#pragma unroll
        for (int e = 0; e < 8; ++e) sa[kc + e][m] = k0 + kc + e < Kd ? v[e] : 0.f;
      } else {
        const int kk = tid >> 2, mc = 8 * (tid & 3);
#pragma unroll
        for (int e = 0; e < 8; ++e) sa[kk][mc + e] = m0r + mc + e < Mo ? v[e] : 0.f;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int e = tid + 256 * r;
        *reinterpret_cast<float4*>(&sx[e >> 5][4 * (e & 31)]) = rx[r];
      }
    }
    __syncthreads();
    if (k0 + BK < Kd) load(k0 + BK);
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      const float2 w = *reinterpret_cast<const float2*>(&sa[kk][2 * ty]);
      const float4 x0 = *reinterpret_cast<const float4*>(&sx[kk][4 * tx]);
      const float4 x1 = *reinterpret_cast<const float4*>(&sx[kk][64 + 4 * tx]);
      const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc[0][c] = fmaf(w.x, xv[c], acc[0][c]);
        acc[1][c] = fmaf(w.y, xv[c], acc[1][c]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int gm = m0r + 2 * ty + i;
    if (gm >= Mo) continue;
    float* orow = out + (u * Mo + gm) * d;
    if (4 * tx < d) *reinterpret_cast<float4*>(orow + 4 * tx) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    if (64 + 4 * tx < d)
      *reinterpret_cast<float4*>(orow + 64 + 4 * tx) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
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

// Z = M0 z (and dZ_agg = M0^T dZ) on the tensor core without losing f32: z = hi + mid + lo in
// three bf16 parts (8 + 8 + 8 significant bits cover f32's 24), M0 is an exact 0/1 bf16
// matrix, so the GEMM's products are exact and its f32 accumulation matches an f32 sum.
__global__ void k_split3(const float* __restrict__ x, long long rows, int d, __nv_bfloat16* __restrict__ out) {
  const long long total = rows * d;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / d;
    const int a = int(e % d);
    const float v = x[e];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    __nv_bfloat16* o = out + r * 3 * d + a;
    o[0] = hi;
    o[d] = mid;
    o[2 * d] = lo;
  }
}
__global__ void k_sum3(const float* __restrict__ x3, long long rows, int d, float* __restrict__ out) {
  const long long total = rows * d;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / d;
    const int a = int(e % d);
    const float* x = x3 + r * 3 * d + a;
    out[e] = (x[0] + x[d]) + x[2 * d];
  }
}

// out[u] = A[u] x[u] with A = M0 (trans = false, [Tm x Tn]) or M0^T; x, out f32 [rows][d]
void aggregate_vec_tc(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, bool trans, const float* x,
                      float* out, const char* name, cudaStream_t st) {
  const int d = Dm.d;
  const int Mo = trans ? Dm.Tn : Dm.Tm, Kd = trans ? Dm.Tm : Dm.Tn;
  const long long xrows = Dm.U * (long long)Kd, orows = Dm.U * (long long)Mo;
  const int grid = 148 * 4;
  k_split3<<<grid, 256, 0, st>>>(x, xrows, d, wb.z3b);
  check_launch("k_split3", st);
  GemmArgs a{};
  a.A = s.M0;
  a.B = wb.z3b;
  a.C = wb.z3f;
  a.batch = int(Dm.U);
  a.M = Mo;
  a.N = 3 * d;
  a.K = Kd;
  a.a_mn = trans;
  a.b_mn = true;
  a.out_f32 = true;
  a.lda = m0_stride(Dm);
  a.ldb = 3LL * d;
  a.ldc = 3LL * d;
  a.a_batch = (long long)Dm.Tm * m0_stride(Dm);
  a.b_batch = (long long)Kd * 3 * d;
  a.c_batch = (long long)Mo * 3 * d;
  a.name = name;
  launch_gemm(a, st);
  k_sum3<<<grid, 256, 0, st>>>(wb.z3f, orows, d, out);
  check_launch("k_sum3", st);
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
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z, Dm.N, Dm.Tn, Dm.phi, Dm.N_valid);
  else
    k_phi_kz<64><<<dim3(Dm.Tn, unsigned(Dm.U)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z, Dm.N, Dm.Tn, Dm.phi, Dm.N_valid);
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
#ifdef SLAB_SIMT_AGG
  k_aggregate_vec<false><<<dim3((Dm.Tm + 31) / 32, unsigned(Dm.U)), 256, 0, st>>>(s.M0, int(m0_stride(Dm)), wb.z, d,
                                                                                Dm.Tm, Dm.Tn, s.Z);
  check_launch("k_aggregate_z", st);
#else
  aggregate_vec_tc(Dm, s, wb, false, wb.z, s.Z, "gemm_aggregate_z", st);
#endif
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
#ifdef SLAB_SIMT_AGG
  k_aggregate_vec<true><<<dim3((Dm.Tn + 31) / 32, unsigned(Dm.U)), 256, 0, st>>>(s.M0, int(m0_stride(Dm)), wb.gZ, d,
                                                                               Dm.Tm, Dm.Tn, wb.gZa);
  check_launch("k_aggregate_dz", st);
#else
  aggregate_vec_tc(Dm, s, wb, true, wb.gZ, wb.gZa, "gemm_aggregate_dz", st);
#endif
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
