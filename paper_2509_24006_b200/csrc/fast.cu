// fast.cu -- the tcgen05 fast path (b_q = b_kv = 64, d in {64, 128}, bf16):
//   K3  phi(K) (bf16) and z_j = colsum phi(K_j)                 k_phi_kz
//       h_j = phi(K_j)^T V_j for every key block                tcgen05 batched GEMM
//   K4  H = M0 . h (M0 = marginal indicator, bf16 0/1)          tcgen05 GEMM
//       Z = sum over marginal z_j (ascending, f32)              k_aggregate_z
//   K5  fused sparse + linear + projection forward              attn_fwd.cu
// References: summaries.cpp:17-42, aggregation.cpp:40-56, forward.cpp:81-195.
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

namespace {

// phi(K) rows -> bf16, and z_j = sum over the block's rows of phi(K) (f32).  grid (Tn, U),
// 8 warps, each warp 8 rows; lane owns D/32 consecutive columns.
template <int D>
__global__ void __launch_bounds__(256) k_phi_kz(const __nv_bfloat16* __restrict__ k,
                                                __nv_bfloat16* __restrict__ kfb,
                                                __nv_bfloat16* __restrict__ z3b, long long N, int Tn, int phi,
                                                long long n_valid, RowLayout rl) {
  pdl_entry();  // launched by launch_pdl
  constexpr int C = D / 32;
  __shared__ float zpart[8][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  float zacc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) zacc[c] = 0.f;
  // all 8 rows' loads in flight before any reduction (C bf16 = 2C bytes per lane and row)
  using V = typename std::conditional<C == 4, uint2, uint32_t>::type;
  static_assert(C == 2 || C == 4, "d in {64, 128}");
  const long long rin0 = (long long)j * 64 + warp * 8;
  V raw[8];
  const RowMap rm = row_map(rl, u, N);  // the caller's K in place (rows past a ragged N do not exist)
  const V* src = reinterpret_cast<const V*>(k + (rm.base + rin0 * rm.stride) * D) + lane;
  const long long rs = rm.stride * (D / C);
  if (rin0 + 8 <= n_valid && rm.stride == 1) {  // unit-major rows: constant strides
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) raw[rr] = src[rr * (D / C)];
  } else if (rin0 + 8 <= n_valid) {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) raw[rr] = src[rr * rs];
  } else {
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) raw[rr] = rin0 + rr < n_valid ? src[rr * rs] : V{};
  }
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const long long rin = rin0 + rr;  // row within the unit
    V* dst = reinterpret_cast<V*>(kfb + (u * N + rin) * D) + lane;
    if (rin >= n_valid) {  // ragged N: padded keys have no feature map (no summary weight)
      *dst = V{};
      continue;
    }
    float x[C];
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[rr]);
#pragma unroll
    for (int c = 0; c < C; c += 2) {
      const float2 f = __bfloat1622float2(h2[c / 2]);
      x[c] = f.x;
      x[c + 1] = f.y;
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
    V out;
    uint32_t* o32 = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
    for (int c = 0; c < C; c += 2) {
      o32[c / 2] = tc::pack_bf16(x[c], x[c + 1]);
      zacc[c] += x[c];
      zacc[c + 1] += x[c + 1];
    }
    *dst = out;
  }
#pragma unroll
  for (int c = 0; c < C; ++c) zpart[warp][lane * C + c] = zacc[c];
  __syncthreads();
  for (int a = threadIdx.x; a < D; a += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += zpart[w][a];
    tc::store_split3(z3b + (u * Tn + j) * 3 * D + a, D, s);  // z_j in 3 bf16 parts
  }
}

// dW[h] = sum over the batch and the split-K chunks of O^l^T dO (backward.cpp:46).
__global__ void k_reduce_dw(const float* __restrict__ part, int chunks_per_unit, long long B,
                            long long H, int dd, float* __restrict__ dw) {
  pdl_entry();  // launched by launch_pdl
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

// identity [H, d, d] bf16: W of the linear-branch MMA when dO^l is given (dO^l I = dO^l exactly)
__global__ void k_fill_identity(__nv_bfloat16* __restrict__ w, long long total, int d) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long m = e % ((long long)d * d);
    w[e] = __float2bfloat16_rn(m / d == m % d ? 1.f : 0.f);
  }
}

// out[r] = <a_r, b_r> over d columns, one warp per row (bf16 in, f32 sum)
__global__ void k_rowdot(const __nv_bfloat162* __restrict__ a, const __nv_bfloat162* __restrict__ b,
                         float* __restrict__ out, long long rows, int d2, long long N, RowLayout rl) {
  const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;  // [U, N] kernel row
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const long long cr = caller_row(rl, r / N, r % N, N);  // the caller's a, b in place
  float acc = 0.f;
  for (int j = lane; cr >= 0 && j < d2; j += 32) {
    const float2 x = __bfloat1622float2(a[cr * d2 + j]), y = __bfloat1622float2(b[cr * d2 + j]);
    acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
  }
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

// out = (add ? add : 0) + x M, M = W[u % H] or its transpose; 64 rows per CTA, W staged as f32
template <typename In>
__global__ void __launch_bounds__(256) k_rowmat(const In* __restrict__ x, const In* __restrict__ w,
                                                int transpose_w, const In* __restrict__ add,
                                                In* __restrict__ out, long long N, long long H, int d) {
  extern __shared__ float sm[];
  const int dp = d + 1;
  float* sW = sm;              // sW[b * dp + a] = M[b][a]
  float* sX = sm + d * dp;     // [8 warps][d]
  const long long u = blockIdx.y;
  const In* wh = w + (u % H) * (long long)d * d;
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    const int r = e / d, c = e % d;  // W[r][c]
    const float v = to_f(wh[e]);
    if (transpose_w) sW[c * dp + r] = v;
    else sW[r * dp + c] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xr = sX + warp * d;
  for (int rr = warp; rr < 64; rr += 8) {
    const long long row = (long long)blockIdx.x * 64 + rr;
    if (row >= N) break;
    const long long g = (u * N + row) * d;
    for (int c = lane; c < d; c += 32) xr[c] = to_f(x[g + c]);
    __syncwarp();
    for (int a = lane; a < d; a += 32) {
      float acc = 0.f;
      for (int b = 0; b < d; ++b) acc = fmaf(xr[b], sW[b * dp + a], acc);
      if (add) acc += to_f(add[g + a]);
      out[g + a] = from_f<In>(acc);
    }
    __syncwarp();
  }
}

// Z3 = M0 [z_hi | z_mid | z_lo] (trans: M0^T [dZ parts]) on the tensor core: the z parts are
// written by their producers (k_phi_kz, k_bwd_lin) with tc::store_split3, M0 is an exact 0/1
// bf16 matrix, so products are exact and the f32 accumulation matches an f32 sum; consumers
// add the three output columns back (tc::load_sum3).
void aggregate_vec_tc(const Dims& Dm, const StateBufs& s, const __nv_bfloat16* z3, bool trans, float* out3,
                      const char* name, cudaStream_t st) {
  const int d = Dm.d;
  const int Mo = trans ? Dm.Tn : Dm.Tm, Kd = trans ? Dm.Tm : Dm.Tn;
  GemmArgs a{};
  a.A = s.M0;
  a.B = z3;
  a.C = out3;
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
}

}  // namespace

#ifndef SLAB_AGG_Z_SIDE
#define SLAB_AGG_Z_SIDE 0  // Z / dZ aggregation on the side stream beside H / dH_agg: measured no gain (2.764-2.797 vs 2.773-2.776 ms)
#endif

bool fast_supported(const Dims& D, int dtype) {
  return dtype == 0 && D.bq == 64 && D.bkv == 64 && (D.d == 64 || D.d == 128);
}

void launch_rowmat(const Dims& D, int dtype, const void* x, const void* w, bool transpose_w,
                   const void* add, void* out, cudaStream_t st) {
  const size_t smem = (size_t(D.d) * (D.d + 1) + 8 * size_t(D.d)) * 4;
  const dim3 grid(unsigned((D.N + 63) / 64), unsigned(D.U));
  if (dtype == 0) {
    using T = __nv_bfloat16;
    SLAB_CUDA(cudaFuncSetAttribute(k_rowmat<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_rowmat<T><<<grid, 256, smem, st>>>((const T*)x, (const T*)w, transpose_w, (const T*)add, (T*)out, D.N,
                                         D.H, D.d);
  } else {
    SLAB_CUDA(cudaFuncSetAttribute(k_rowmat<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_rowmat<float><<<grid, 256, smem, st>>>((const float*)x, (const float*)w, transpose_w, (const float*)add,
                                             (float*)out, D.N, D.H, D.d);
  }
  check_launch("k_rowmat", st);
}

void launch_rowdot(const Dims& D, const void* a, const void* b, float* out, cudaStream_t st) {
  const long long rows = D.U * D.N;
  k_rowdot<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(static_cast<const __nv_bfloat162*>(a),
                                                             static_cast<const __nv_bfloat162*>(b), out, rows,
                                                             D.d / 2, D.N, D.rl);
  check_launch("k_rowdot", st);
}

// dW = O^l^T dO per head (backward.cpp:46): split-K over row chunks of each unit on the tensor
// core, then reduced over the chunks and the batch
void launch_dw_fast(const Dims& Dm, const void* o_l, const void* d_out, float* dw, const WorkBufs& wb,
                    cudaStream_t ds) {
  const int d = Dm.d;
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
  g.a_rl = Dm.rl;  // O^l and dO in place: chunk c of unit u
  g.b_rl = Dm.rl;
  g.a_rpu = g.b_rpu = chunks;
  g.units = Dm.U;
  launch_gemm(g, ds);
  launch_pdl(k_reduce_dw, dim3((d * d + 255) / 256, unsigned(Dm.H)), 256, 0, ds, (const float*)wb.dwp, chunks,
             (long long)Dm.B, (long long)Dm.H, d * d, dw);
  check_launch("k_reduce_dw", ds);
}

// phi(K), z_j and h_j = phi(K_j)^T V_j: independent of the mask, so the C-ABI forward runs them
// on a side stream while the classification kernels (latency / FP64 bound) run
void fast_summaries(const Dims& Dm, const void* k, const void* v, const WorkBufs& wb, cudaStream_t st) {
  const int d = Dm.d;
  if (d == 128)
    launch_pdl(k_phi_kz<128>, dim3(Dm.Tn, unsigned(Dm.U)), 256, 0, st,
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z3b, Dm.Nk, Dm.Tn, Dm.phi, Dm.Nk_valid, Dm.rl);
  else
    launch_pdl(k_phi_kz<64>, dim3(Dm.Tn, unsigned(Dm.U)), 256, 0, st,
        static_cast<const __nv_bfloat16*>(k), wb.kfb, wb.z3b, Dm.Nk, Dm.Tn, Dm.phi, Dm.Nk_valid, Dm.rl);
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
  g.b_rl = Dm.rl;  // V in place: key block j of unit u is chunk j of u's rows
  g.b_rpu = Dm.Tn;
  g.units = Dm.U;
  launch_gemm(g, st);
}

// H = M0 . h per unit: M = Tm, N = d*d, K = Tn
void fast_aggregate_h(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, cudaStream_t st) {
  const int d = Dm.d;
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
}

// H = M0 h, Z = M0 z (needs the mask); M0 itself unless the classifier wrote it
void fast_aggregate(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, bool m0_ready, cudaStream_t st) {
  if (!m0_ready) launch_build_m0(Dm, s, st);  // the classifier writes M0 itself
  fast_aggregate_h(Dm, s, wb, st);
  aggregate_vec_tc(Dm, s, wb.z3b, false, s.Z, "gemm_aggregate_z", st);  // s.Z: [U, Tm, 3d]
}

void fast_forward(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                  void* o, void* o_s, void* o_l, float* lse, const StateBufs& s,
                  const WorkBufs& wb, bool m0_ready, const SideFork& side, cudaStream_t st) {
  if (!side.s) {
    fast_summaries(Dm, k, v, wb, st);
    fast_aggregate(Dm, s, wb, m0_ready, st);
  } else if (!SLAB_AGG_Z_SIDE) {
    SLAB_CUDA(cudaStreamWaitEvent(st, side.join, 0));
    fast_aggregate(Dm, s, wb, m0_ready, st);
  } else {  // Z = M0 z (a thin GEMM, N = 3d) on the side stream beside H = M0 h
    if (!m0_ready) launch_build_m0(Dm, s, st);
    SLAB_CUDA(cudaEventRecord(side.mid, st));
    SLAB_CUDA(cudaStreamWaitEvent(side.s, side.mid, 0));  // M0 (the side has the z parts)
    aggregate_vec_tc(Dm, s, wb.z3b, false, s.Z, "gemm_aggregate_z", side.s);
    SLAB_CUDA(cudaEventRecord(side.join3, side.s));
    SLAB_CUDA(cudaStreamWaitEvent(st, side.join, 0));  // h (summaries)
    fast_aggregate_h(Dm, s, wb, st);
    SLAB_CUDA(cudaStreamWaitEvent(st, side.join3, 0));
  }
  launch_attn_fwd(Dm, q, k, v, w, o, o_s, o_l, lse, s, st);
}

// dH_agg = M0^T dH and dZ_agg = M0^T dZ (A = M0 read M-major) from the row phase's dH_i / dZ_i
static void launch_agg_t(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, const __nv_bfloat16* gH,
                         const __nv_bfloat16* z3, cudaStream_t as) {
  const int d = Dm.d;
  GemmArgs a{};
  a.A = s.M0;
  a.B = gH;
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
  launch_gemm(a, as);
  if (z3) aggregate_vec_tc(Dm, s, z3, true, wb.gZa, "gemm_aggregate_dz", as);  // gZa: [U, Tn, 3d]
}

// row phase (backward.cpp:46-120): the linear branch (dH_i, dZ_i, D^s, dQ^phi) and the sparse dQ
// with dq_total.  dH_i -> gH [U, Tm, d, d], dZ_i parts -> z3 [U, Tm, 3d], D^s -> Ds [U, N].
// Independent cotangents: the linear kernel multiplies the given dO^l by an identity W (exact)
// and D^s = <dO^s, O^s> comes from its own row-dot kernel.
// rows_st: the stream of the sparse dQ pass (k_bwd_rows), ordered after k_bwd_lin on st through
// `after_lin` (null: st)
static void backward_rows_phase(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                                const void* o_s, const void* o_l, const float* lse, const void* d_out,
                                const void* d_out_l, void* dq, const GradParts& parts, const StateBufs& s,
                                const WorkBufs& wb, __nv_bfloat16* gH, __nv_bfloat16* z3, float* Ds,
                                cudaStream_t st, cudaStream_t rows_st = nullptr, cudaEvent_t after_lin = nullptr) {
  const int d = Dm.d;
  const bool split = d_out_l != nullptr;
  const void* lin_w = w;
  const void* lin_do = d_out;
  if (split) {
    const long long total = Dm.H * (long long)d * d;
    k_fill_identity<<<unsigned((total + 255) / 256), 256, 0, st>>>(wb.wid, total, d);
    check_launch("k_fill_identity", st);
    launch_rowdot(Dm, d_out, o_s, Ds, st);
    lin_w = wb.wid;
    lin_do = d_out_l;
  }
  launch_bwd_lin(Dm, q, lin_w, o_s, o_l, lin_do, s, gH, z3, Ds, wb.dqphi, split, st);
  if (rows_st) {
    SLAB_CUDA(cudaEventRecord(after_lin, st));
    SLAB_CUDA(cudaStreamWaitEvent(rows_st, after_lin, 0));
  }
  launch_bwd_rows(Dm, q, k, v, lse, d_out, dq, s, Ds, wb.dqphi, parts.dq, parts.dq_feat, rows_st ? rows_st : st);
}

// SLA_B200_ROWS_SIDE=1 (A/B switch): the sparse dQ pass runs on the side stream, beside the dH
// aggregation and the columns pass (neither reads its output)
static bool rows_on_side() {
  static const bool on = [] {
    const char* e = getenv("SLA_B200_ROWS_SIDE");
    return e && e[0] == '1';
  }();
  return on;
}

void fast_backward(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                   const void* o_s, const void* o_l, const float* lse, const void* d_out,
                   const void* d_out_l, void* dq, void* dk, void* dv, float* dw,
                   const GradParts& parts, const StateBufs& s, const WorkBufs& wb, cudaStream_t st,
                   const SideFork& side) {
  // the column lists (labels only) build on the side stream while k_bwd_lin, a latency-bound
  // kernel with registers and threads to spare on every SM, runs; joined before the columns pass.
  // dW needs only O^l and dO: it fills SMs beside the row / column passes.
  SideJoin guard(side, st);
  if (side.s) {
    SLAB_CUDA(cudaEventRecord(side.fork, st));
    SLAB_CUDA(cudaStreamWaitEvent(side.s, side.fork, 0));
    guard.arm(side.join2);
    launch_build_csc(Dm, s, side.s);
    SLAB_CUDA(cudaEventRecord(side.join, side.s));
    if (dw) launch_dw_fast(Dm, o_l, d_out, dw, wb, side.s);
    SLAB_CUDA(cudaEventRecord(side.join2, side.s));
  } else {
    launch_build_csc(Dm, s, st);
  }
  const bool rside = side.s && rows_on_side();
  backward_rows_phase(Dm, q, k, v, w, o_s, o_l, lse, d_out, d_out_l, dq, parts, s, wb, wb.hb, wb.z3b, wb.Ds, st,
                      rside ? side.s : nullptr, rside ? side.mid : nullptr);
  // dH_agg and dZ_agg need only k_bwd_lin's dH / dZ (measured: dH_agg on a side stream beside the
  // rows pass 2.81 ms per step against 2.73-2.78 here -- rows loses SMs, cols waits); the thin
  // dZ_agg GEMM runs on the side stream beside dH_agg
  if (side.s && SLAB_AGG_Z_SIDE && !rside) {
    SLAB_CUDA(cudaEventRecord(side.mid, st));
    SLAB_CUDA(cudaStreamWaitEvent(side.s, side.mid, 0));
    aggregate_vec_tc(Dm, s, wb.z3b, true, wb.gZa, "gemm_aggregate_dz", side.s);
    SLAB_CUDA(cudaEventRecord(side.join3, side.s));
    launch_agg_t(Dm, s, wb, wb.hb, nullptr, st);
    SLAB_CUDA(cudaStreamWaitEvent(st, side.join3, 0));
  } else {
    launch_agg_t(Dm, s, wb, wb.hb, wb.z3b, st);
  }
  // columns pass: dk_total, dv
  if (side.s) SLAB_CUDA(cudaStreamWaitEvent(st, side.join, 0));
  launch_bwd_cols(Dm, q, k, v, lse, d_out, dk, dv, s, wb.hab, wb.gZa, wb.Ds, parts.dk, parts.dk_feat, wb.work_ctr, st);
  if (!side.s && dw) launch_dw_fast(Dm, o_l, d_out, dw, wb, st);
  if (rside) SLAB_CUDA(cudaEventRecord(side.join2, side.s));  // after the rows pass
  guard.release();
  if (side.s) SLAB_CUDA(cudaStreamWaitEvent(st, side.join2, 0));
}

void fast_backward_rows(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                        const void* o_s, const void* o_l, const float* lse, const void* d_out,
                        const void* d_out_l, void* dq, float* dw, const StateBufs& s, const WorkBufs& wb,
                        __nv_bfloat16* gH, __nv_bfloat16* z3, float* Ds, cudaStream_t st) {
  backward_rows_phase(Dm, q, k, v, w, o_s, o_l, lse, d_out, d_out_l, dq, GradParts{}, s, wb, gH, z3, Ds, st);
  if (dw) launch_dw_fast(Dm, o_l, d_out, dw, wb, st);
}

void fast_backward_cols(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                        const void* d_out, const float* Ds, const __nv_bfloat16* gH, const __nv_bfloat16* z3,
                        void* dk, void* dv, const StateBufs& s, const WorkBufs& wb, cudaStream_t st) {
  launch_build_m0(Dm, s, st);
  launch_build_csc(Dm, s, st);
  launch_agg_t(Dm, s, wb, gH, z3, st);
  launch_bwd_cols(Dm, q, k, v, lse, d_out, dk, dv, s, wb.hab, wb.gZa, Ds, nullptr, nullptr, wb.work_ctr, st);
}

}  // namespace slab
