// generic.cu -- shape-generic SIMT kernels (fp32 arithmetic) for any b_q, b_kv, d that fit
// shared memory.  They serve the reference's own test shapes (b in {4, 8, 16}, d in
// {4, 8, 16}), f32 inputs, and every shape the tcgen05 fast path does not cover.  Loop
// orders follow the reference so f32 results track its f32 path closely.
//
// Reference: feature_map.cpp:24-73, summaries.cpp:17-42, aggregation.cpp:40-56,
// forward.cpp:29-195, backward.cpp:12-216 (paths relative to /root/reference/proj/core).
#include <algorithm>

#include "buffers.hpp"
#include "kernels.hpp"

namespace slab {

namespace {

constexpr int kThreads = 256;

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    SLAB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(bytes)));
}

// ---------------------------------------------------------------------------------------
// phi(X) -> f32 (feature_map.cpp:24-40); one warp per row.
// ---------------------------------------------------------------------------------------
template <typename In>
__global__ void k_phi(const In* __restrict__ x, float* __restrict__ out, long long rows, int d,
                      int phi) {
  const long long r = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const In* xr = x + r * d;
  float* orow = out + r * d;
  if (phi != 2) {
    for (int c = lane; c < d; c += 32) orow[c] = phi_elem(phi, to_f(xr[c]));
    return;
  }
  float m = -INFINITY;
  for (int c = lane; c < d; c += 32) m = fmaxf(m, to_f(xr[c]));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += expf(to_f(xr[c]) - m);
  s = warp_sum(s);
  for (int c = lane; c < d; c += 32) orow[c] = expf(to_f(xr[c]) - m) / s;
}

// ---------------------------------------------------------------------------------------
// KV summaries h_j = phi(K_j)^T V_j, z_j (summaries.cpp:17-42); grid (Tn, U).
// ---------------------------------------------------------------------------------------
template <typename In>
__global__ void k_summaries(const float* __restrict__ kf, const In* __restrict__ v, long long N,
                            int d, int bkv, int Tn, float* __restrict__ h,
                            float* __restrict__ z) {
  extern __shared__ float sm[];
  float* skf = sm;               // [bkv][d]
  float* sv = sm + bkv * d;      // [bkv][d]
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  const long long base = (u * N + (long long)j * bkv) * d;
  for (int e = threadIdx.x; e < bkv * d; e += blockDim.x) {
    skf[e] = kf[base + e];
    sv[e] = to_f(v[base + e]);
  }
  __syncthreads();
  float* hj = h + (u * Tn + j) * (long long)d * d;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int a = idx / d, b = idx % d;
    float acc = 0.f;
    for (int t = 0; t < bkv; ++t) acc = add_rn(acc, mul_rn(skf[t * d + a], sv[t * d + b]));
    hj[idx] = acc;
  }
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    float acc = 0.f;
    for (int t = 0; t < bkv; ++t) acc = add_rn(acc, skf[t * d + a]);
    z[(u * Tn + j) * d + a] = acc;
  }
}

// ---------------------------------------------------------------------------------------
// Row aggregation H_i = sum_{j marginal} h_j, ascending, first term copied
// (aggregation.cpp:40-56); grid (Tm, U).
// ---------------------------------------------------------------------------------------
__global__ void k_aggregate_rows(const int8_t* __restrict__ labels, const float* __restrict__ h,
                                 const float* __restrict__ z, int d, int Tm, int Tn,
                                 float* __restrict__ H, float* __restrict__ Z) {
  extern __shared__ int slist[];  // [Tn]
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
  const float* hu = h + u * (long long)Tn * d * d;
  float* Hi = H + (u * Tm + i) * (long long)d * d;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < cnt; ++p) {
      const float x = hu[(long long)slist[p] * d * d + idx];
      acc = p == 0 ? x : add_rn(acc, x);
    }
    Hi[idx] = acc;
  }
  const float* zu = z + u * (long long)Tn * d;
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < cnt; ++p) {
      const float x = zu[(long long)slist[p] * d + a];
      acc = p == 0 ? x : add_rn(acc, x);
    }
    Z[(u * Tm + i) * d + a] = acc;
  }
}

// ---------------------------------------------------------------------------------------
// Fused forward of one block row: sparse online softmax (forward.cpp:29-79), linear branch
// (forward.cpp:126-149) and the projection combine (forward.cpp:187-195).  grid (Tm, U).
// ---------------------------------------------------------------------------------------
struct FwdSmem {
  int q, r1, s, acc, misc;
  size_t bytes;
};
inline FwdSmem fwd_smem(const Dims& D) {
  FwdSmem L;
  const int d = D.d, bq = D.bq, bkv = D.bkv;
  L.q = 0;
  L.r1 = L.q + bq * d;
  const int r1 = std::max(bkv * (d + 1) + bkv * d, d * d);
  L.s = L.r1 + r1;
  L.acc = L.s + bq * bkv;
  L.misc = L.acc + bq * d;
  L.bytes = size_t(L.misc + 4 * bq + d) * 4;
  return L;
}

template <typename In>
__global__ void k_fwd_generic(Dims D, FwdSmem L, const In* __restrict__ q,
                              const In* __restrict__ k, const In* __restrict__ v,
                              const In* __restrict__ w, const float* __restrict__ qf,
                              const int* __restrict__ crit_cnt, const int* __restrict__ crit_idx,
                              const int* __restrict__ marg_cnt, const float* __restrict__ H,
                              const float* __restrict__ Z, In* __restrict__ o,
                              In* __restrict__ o_s, In* __restrict__ o_l,
                              float* __restrict__ lse) {
  extern __shared__ float sm[];
  const int d = D.d, bq = D.bq, bkv = D.bkv, dp = d + 1;
  float* sQ = sm + L.q;
  float* sK = sm + L.r1;
  float* sV = sK + bkv * dp;
  float* sS = sm + L.s;
  float* sAcc = sm + L.acc;
  float* sM = sm + L.misc;
  float* sL = sM + bq;
  float* sAl = sL + bq;
  float* sDen = sAl + bq;
  float* sZ = sDen + bq;
  const long long u = blockIdx.y;
  const int i = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31;
  const long long row0 = u * D.N + (long long)i * bq;

  for (int e = tid; e < bq * d; e += nt) {
    sQ[e] = to_f(q[row0 * d + e]);
    sAcc[e] = 0.f;
  }
  for (int r = tid; r < bq; r += nt) {
    sM[r] = -INFINITY;
    sL[r] = 0.f;
  }
  const int cnt = crit_cnt[u * D.Tm + i];
  const int* list = crit_idx + (u * D.Tm + i) * (long long)D.Tn;
  for (int t = 0; t < cnt; ++t) {
    const long long kv0 = (u * D.N + (long long)list[t] * bkv) * d;
    __syncthreads();
    for (int e = tid; e < bkv * d; e += nt) {
      const int c = e / d, x = e % d;
      sK[c * dp + x] = to_f(k[kv0 + e]);
      sV[c * d + x] = to_f(v[kv0 + e]);
    }
    __syncthreads();
    for (int idx = tid; idx < bq * bkv; idx += nt) {
      const int r = idx / bkv, c = idx % bkv;
      float acc = 0.f;
      for (int e = 0; e < d; ++e) acc = add_rn(acc, mul_rn(sQ[r * d + e], sK[c * dp + e]));
      sS[idx] = mul_rn(acc, D.scale_f);
    }
    __syncthreads();
    for (int r = warp; r < bq; r += nt / 32) {
      float rmax = -INFINITY;
      for (int c = lane; c < bkv; c += 32) rmax = fmaxf(rmax, sS[r * bkv + c]);
      rmax = warp_max(rmax);
      const float m_old = sM[r];
      const float m_new = fmaxf(m_old, rmax);
      const float alpha = expf(m_old - m_new);
      float ps = 0.f;
      for (int c = lane; c < bkv; c += 32) {
        const float p = expf(sS[r * bkv + c] - m_new);
        sS[r * bkv + c] = p;
        ps += p;
      }
      ps = warp_sum(ps);
      __syncwarp();
      if (lane == 0) {
        sL[r] = alpha * sL[r] + ps;
        sM[r] = m_new;
        sAl[r] = alpha;
      }
    }
    __syncthreads();
    for (int idx = tid; idx < bq * d; idx += nt) {
      const int r = idx / d, e = idx % d;
      float a = mul_rn(sAcc[idx], sAl[r]);
      for (int c = 0; c < bkv; ++c) a = add_rn(a, mul_rn(sS[r * bkv + c], sV[c * d + e]));
      sAcc[idx] = a;
    }
  }
  __syncthreads();
  // finalize the sparse branch (forward.cpp:68-78)
  for (int idx = tid; idx < bq * d; idx += nt) {
    const int r = idx / d;
    const float l = sL[r];
    const float val = l == 0.f ? 0.f : div_rn(sAcc[idx], l);
    sAcc[idx] = val;
    if (o_s) o_s[row0 * d + idx] = from_f<In>(val);
  }
  for (int r = tid; r < bq; r += nt) {
    const float l = sL[r];
    lse[row0 + r] = l == 0.f ? kLseSentinel : sM[r] + logf(l);
  }
  // linear branch: O^l rows = phi(q) H_i / (phi(q) . Z_i), zero without marginal blocks
  const int mc = marg_cnt[u * D.Tm + i];
  float* sOl = sQ;  // Q no longer needed
  float* sH = sm + L.r1;
  __syncthreads();
  if (mc > 0) {
    const float* Hi = H + (u * D.Tm + i) * (long long)d * d;
    for (int e = tid; e < d * d; e += nt) sH[e] = Hi[e];
    for (int a = tid; a < d; a += nt) sZ[a] = Z[(u * D.Tm + i) * d + a];
    __syncthreads();
    for (int r = tid; r < bq; r += nt) {
      const float* qr = qf + (row0 + r) * d;
      float den = 0.f;
      for (int a = 0; a < d; ++a) den = add_rn(den, mul_rn(qr[a], sZ[a]));
      sDen[r] = den;
    }
    __syncthreads();
    for (int idx = tid; idx < bq * d; idx += nt) {
      const int r = idx / d, b = idx % d;
      const float den = sDen[r];
      float acc = 0.f;
      if (den != 0.f) {
        const float* qr = qf + (row0 + r) * d;
        for (int a = 0; a < d; ++a) {
          const float qa = qr[a];
          if (qa == 0.f) continue;
          acc = add_rn(acc, mul_rn(qa, sH[a * d + b]));
        }
        acc = div_rn(acc, den);
      }
      sOl[idx] = acc;
    }
  } else {
    for (int idx = tid; idx < bq * d; idx += nt) sOl[idx] = 0.f;
  }
  __syncthreads();
  for (int idx = tid; idx < bq * d; idx += nt)
    if (o_l) o_l[row0 * d + idx] = from_f<In>(sOl[idx]);
  if (!w || !o) return;
  // combine O = O^l W + O^s with matmul's skip-zero ascending order
  float* sW = sH;
  const In* wh = w + (u % D.H) * (long long)d * d;
  for (int e = tid; e < d * d; e += nt) sW[e] = to_f(wh[e]);
  __syncthreads();
  for (int idx = tid; idx < bq * d; idx += nt) {
    const int r = idx / d, b = idx % d;
    float acc = 0.f;
    for (int a = 0; a < d; ++a) {
      const float x = sOl[r * d + a];
      if (x == 0.f) continue;
      acc = add_rn(acc, mul_rn(x, sW[a * d + b]));
    }
    o[row0 * d + idx] = from_f<In>(add_rn(acc, sAcc[idx]));
  }
}

// ---------------------------------------------------------------------------------------
// Backward prologue: dO^l = dO W^T, D^s, D^l (backward.cpp:12-22, 48-58).
// grid (ceil(N / 64), U); warp per row.
// ---------------------------------------------------------------------------------------
template <typename In>
__global__ void k_bwd_prep(Dims D, const In* __restrict__ w, const In* __restrict__ d_out,
                           const In* __restrict__ d_out_l, const In* __restrict__ o_s,
                           const In* __restrict__ o_l, float* __restrict__ dOl,
                           float* __restrict__ Ds, float* __restrict__ Dl) {
  // d_out_l != null: independent cotangents (sla_backward's dO^l, backward.hpp:25-38) -- dO^l is
  // taken as given; else dO^l = dO W^T (proj_backward, backward.cpp:12-22)
  extern __shared__ float sm[];
  const int d = D.d, dp = d + 1;
  float* sW = sm;                         // [d][d+1]
  float* sRow = sm + d * dp;              // [warps][d]
  const long long u = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (!d_out_l) {
    const In* wh = w + (u % D.H) * (long long)d * d;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) sW[(e / d) * dp + e % d] = to_f(wh[e]);
  }
  __syncthreads();
  float* myrow = sRow + warp * d;
  for (int rr = warp; rr < 64; rr += nw) {
    const long long r = (long long)blockIdx.x * 64 + rr;
    if (r >= D.N) break;
    const long long g = (u * D.N + r) * d;
    for (int c = lane; c < d; c += 32) myrow[c] = to_f(d_out[g + c]);
    __syncwarp();
    float ds = 0.f, dl = 0.f;
    for (int c = lane; c < d; c += 32) ds += myrow[c] * to_f(o_s[g + c]);
    for (int a = lane; a < d; a += 32) {
      float acc = 0.f;
      if (d_out_l)
        acc = to_f(d_out_l[g + a]);
      else
        for (int b = 0; b < d; ++b) acc = add_rn(acc, mul_rn(myrow[b], sW[a * dp + b]));
      dOl[g + a] = acc;
      dl += acc * to_f(o_l[g + a]);
    }
    ds = warp_sum(ds);
    dl = warp_sum(dl);
    if (lane == 0) {
      Ds[u * D.N + r] = ds;
      Dl[u * D.N + r] = dl;
    }
    __syncwarp();
  }
}

// dW[h] += O^l^T dO over 32-row chunks (backward.cpp:46, summed over the batch per head)
template <typename In>
__global__ void k_dw(Dims D, const In* __restrict__ o_l, const In* __restrict__ d_out,
                     float* __restrict__ dw) {
  extern __shared__ float sm[];
  const int d = D.d;
  constexpr int R = 32;
  float* sOl = sm;
  float* sdO = sm + R * d;
  const long long u = blockIdx.y;
  const long long r0 = (long long)blockIdx.x * R;
  const int rows = int(std::min<long long>(R, D.N - r0));
  for (int e = threadIdx.x; e < rows * d; e += blockDim.x) {
    sOl[e] = to_f(o_l[(u * D.N + r0) * d + e]);
    sdO[e] = to_f(d_out[(u * D.N + r0) * d + e]);
  }
  __syncthreads();
  float* dwh = dw + (u % D.H) * (long long)d * d;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int a = idx / d, b = idx % d;
    float acc = 0.f;
    for (int r = 0; r < rows; ++r) acc += sOl[r * d + a] * sdO[r * d + b];
    atomicAdd(dwh + idx, acc);
  }
}

// Row phase, linear branch (backward.cpp:70-95): dH_i, dZ_i, dQ^phi.  grid (Tm, U).
template <typename HT>
__global__ void k_bwd_rows_lin(Dims D, const int* __restrict__ marg_cnt,
                               const float* __restrict__ qf, const float* __restrict__ dOl,
                               const float* __restrict__ Dl, const HT* __restrict__ H,
                               const float* __restrict__ Z, float* __restrict__ gH,
                               float* __restrict__ gZ, float* __restrict__ dqf) {
  extern __shared__ float sm[];
  const int d = D.d, bq = D.bq, dp = d + 1;
  float* sQF = sm;                 // [bq][d]
  float* sDO = sQF + bq * d;       // [bq][d]
  float* sH = sDO + bq * d;        // [d][d+1]
  float* sZ = sH + d * dp;         // [d]
  float* sDen = sZ + d;            // [bq]
  float* sDl = sDen + bq;          // [bq]
  const long long u = blockIdx.y;
  const int i = blockIdx.x;
  const long long row0 = u * D.N + (long long)i * bq;
  float* gHi = gH + (u * D.Tm + i) * (long long)d * d;
  float* gZi = gZ + (u * D.Tm + i) * d;
  if (marg_cnt[u * D.Tm + i] == 0) {
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) gHi[e] = 0.f;
    for (int e = threadIdx.x; e < d; e += blockDim.x) gZi[e] = 0.f;
    for (int e = threadIdx.x; e < bq * d; e += blockDim.x) dqf[row0 * d + e] = 0.f;
    return;
  }
  const HT* Hi = H + (u * D.Tm + i) * (long long)d * d;
  for (int e = threadIdx.x; e < bq * d; e += blockDim.x) {
    sQF[e] = qf[row0 * d + e];
    sDO[e] = dOl[row0 * d + e];
  }
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) sH[(e / d) * dp + e % d] = to_f(Hi[e]);
  for (int a = threadIdx.x; a < d; a += blockDim.x) sZ[a] = Z[(u * D.Tm + i) * d + a];
  for (int r = threadIdx.x; r < bq; r += blockDim.x) sDl[r] = Dl[row0 + r];
  __syncthreads();
  for (int r = threadIdx.x; r < bq; r += blockDim.x) {
    float den = 0.f;
    for (int a = 0; a < d; ++a) den = add_rn(den, mul_rn(sQF[r * d + a], sZ[a]));
    sDen[r] = den;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int a = idx / d, b = idx % d;
    float acc = 0.f;
    for (int r = 0; r < bq; ++r) {
      const float den = sDen[r];
      if (den == 0.f) continue;
      const float qa = div_rn(sQF[r * d + a], den);
      if (qa != 0.f) acc = add_rn(acc, mul_rn(qa, sDO[r * d + b]));
    }
    gHi[idx] = acc;
  }
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < bq; ++r) {
      const float den = sDen[r];
      if (den == 0.f) continue;
      const float qa = div_rn(sQF[r * d + a], den);
      if (qa != 0.f) acc = __fsub_rn(acc, mul_rn(qa, sDl[r]));
    }
    gZi[a] = acc;
  }
  for (int idx = threadIdx.x; idx < bq * d; idx += blockDim.x) {
    const int r = idx / d, a = idx % d;
    const float den = sDen[r];
    float val = 0.f;
    if (den != 0.f) {
      float acc = 0.f;
      for (int b = 0; b < d; ++b) acc = add_rn(acc, mul_rn(sDO[r * d + b], sH[a * dp + b]));
      val = div_rn(__fsub_rn(acc, mul_rn(sDl[r], sZ[a])), den);
    }
    dqf[row0 * d + idx] = val;
  }
}

// Row phase, sparse dQ (backward.cpp:98-119).  grid (Tm, U).
template <typename In>
__global__ void k_bwd_rows_sparse(Dims D, const In* __restrict__ q, const In* __restrict__ k,
                                  const In* __restrict__ v, const In* __restrict__ d_out,
                                  const float* __restrict__ lse, const float* __restrict__ Ds,
                                  const int* __restrict__ crit_cnt,
                                  const int* __restrict__ crit_idx, float* __restrict__ dq) {
  extern __shared__ float sm[];
  const int d = D.d, bq = D.bq, bkv = D.bkv, dp = d + 1;
  float* sQ = sm;                    // [bq][d]
  float* sDO = sQ + bq * d;          // [bq][d]
  float* sK = sDO + bq * d;          // [bkv][d+1]
  float* sV = sK + bkv * dp;         // [bkv][d+1]
  float* sP = sV + bkv * dp;         // [bq][bkv]
  float* sAcc = sP + bq * bkv;       // [bq][d]
  float* sLse = sAcc + bq * d;       // [bq]
  float* sDs = sLse + bq;            // [bq]
  const long long u = blockIdx.y;
  const int i = blockIdx.x;
  const long long row0 = u * D.N + (long long)i * bq;
  for (int e = threadIdx.x; e < bq * d; e += blockDim.x) {
    sQ[e] = to_f(q[row0 * d + e]);
    sDO[e] = to_f(d_out[row0 * d + e]);
    sAcc[e] = 0.f;
  }
  for (int r = threadIdx.x; r < bq; r += blockDim.x) {
    sLse[r] = lse[row0 + r];
    sDs[r] = Ds[row0 + r];
  }
  const int cnt = crit_cnt[u * D.Tm + i];
  const int* list = crit_idx + (u * D.Tm + i) * (long long)D.Tn;
  for (int t = 0; t < cnt; ++t) {
    const long long kv0 = (u * D.N + (long long)list[t] * bkv) * d;
    __syncthreads();
    for (int e = threadIdx.x; e < bkv * d; e += blockDim.x) {
      const int c = e / d, x = e % d;
      sK[c * dp + x] = to_f(k[kv0 + e]);
      sV[c * dp + x] = to_f(v[kv0 + e]);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < bq * bkv; idx += blockDim.x) {
      const int r = idx / bkv, c = idx % bkv;
      float s = 0.f, dpv = 0.f;
      for (int e = 0; e < d; ++e) {
        s = add_rn(s, mul_rn(sQ[r * d + e], sK[c * dp + e]));
        dpv = add_rn(dpv, mul_rn(sDO[r * d + e], sV[c * dp + e]));
      }
      s = mul_rn(s, D.scale_f);
      const float p = expf(s - sLse[r]);
      sP[idx] = mul_rn(mul_rn(p, __fsub_rn(dpv, sDs[r])), D.scale_f);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < bq * d; idx += blockDim.x) {
      const int r = idx / d, e = idx % d;
      float a = sAcc[idx];
      for (int c = 0; c < bkv; ++c) a = add_rn(a, mul_rn(sP[r * bkv + c], sK[c * dp + e]));
      sAcc[idx] = a;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bq * d; e += blockDim.x) dq[row0 * d + e] = sAcc[e];
}

// Column phase, sparse dK/dV (backward.cpp:144-168).  grid (Tn, U); accumulates into the
// block-owned f32 rows of dk/dv (no atomics: each KV block has one owner).
template <typename In>
__global__ void k_bwd_cols_sparse(Dims D, const In* __restrict__ q, const In* __restrict__ k,
                                  const In* __restrict__ v, const In* __restrict__ d_out,
                                  const float* __restrict__ lse, const float* __restrict__ Ds,
                                  const int* __restrict__ ccol_cnt,
                                  const int* __restrict__ ccol_idx, float* __restrict__ dk,
                                  float* __restrict__ dv) {
  extern __shared__ float sm[];
  const int d = D.d, bq = D.bq, bkv = D.bkv, dp = d + 1;
  float* sK = sm;                    // [bkv][d+1]
  float* sV = sK + bkv * dp;         // [bkv][d+1]
  float* sQ = sV + bkv * dp;         // [bq][d]
  float* sDO = sQ + bq * d;          // [bq][d]
  float* sP = sDO + bq * d;          // [bq][bkv]
  float* sdS = sP + bq * bkv;        // [bq][bkv]
  float* sLse = sdS + bq * bkv;      // [bq]
  float* sDs = sLse + bq;            // [bq]
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  const long long kv0 = u * D.N + (long long)j * bkv;
  for (int e = threadIdx.x; e < bkv * d; e += blockDim.x) {
    const int c = e / d, x = e % d;
    sK[c * dp + x] = to_f(k[kv0 * d + e]);
    sV[c * dp + x] = to_f(v[kv0 * d + e]);
  }
  const int cnt = ccol_cnt[u * D.Tn + j];
  const int* list = ccol_idx + (u * D.Tn + j) * (long long)D.Tm;
  for (int t = 0; t < cnt; ++t) {
    const long long row0 = u * D.N + (long long)list[t] * bq;
    __syncthreads();
    for (int e = threadIdx.x; e < bq * d; e += blockDim.x) {
      sQ[e] = to_f(q[row0 * d + e]);
      sDO[e] = to_f(d_out[row0 * d + e]);
    }
    for (int r = threadIdx.x; r < bq; r += blockDim.x) {
      sLse[r] = lse[row0 + r];
      sDs[r] = Ds[row0 + r];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < bq * bkv; idx += blockDim.x) {
      const int r = idx / bkv, c = idx % bkv;
      float s = 0.f, dpv = 0.f;
      for (int e = 0; e < d; ++e) {
        s = add_rn(s, mul_rn(sQ[r * d + e], sK[c * dp + e]));
        dpv = add_rn(dpv, mul_rn(sDO[r * d + e], sV[c * dp + e]));
      }
      s = mul_rn(s, D.scale_f);
      const float p = expf(s - sLse[r]);
      sP[idx] = p;
      sdS[idx] = mul_rn(mul_rn(p, __fsub_rn(dpv, sDs[r])), D.scale_f);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < bkv * d; idx += blockDim.x) {
      const int c = idx / d, e = idx % d;
      float av = dv[kv0 * d + idx], ak = dk[kv0 * d + idx];
      for (int r = 0; r < bq; ++r) {
        av = add_rn(av, mul_rn(sP[r * bkv + c], sDO[r * d + e]));
        ak = add_rn(ak, mul_rn(sdS[r * bkv + c], sQ[r * d + e]));
      }
      dv[kv0 * d + idx] = av;
      dk[kv0 * d + idx] = ak;
    }
  }
}

// Column phase, linear branch (backward.cpp:170-198).  grid (Tn, U).
template <typename In>
__global__ void k_bwd_cols_lin(Dims D, const int8_t* __restrict__ labels,
                               const In* __restrict__ v, const float* __restrict__ kf,
                               const float* __restrict__ gH, const float* __restrict__ gZ,
                               float* __restrict__ dkf, float* __restrict__ dv) {
  extern __shared__ float sm[];
  const int d = D.d, bkv = D.bkv, dp = d + 1;
  float* sHa = sm;                   // [d][d+1]
  float* sZa = sHa + d * dp;         // [d]
  float* sV = sZa + d;               // [bkv][d]
  float* sKF = sV + bkv * d;         // [bkv][d]
  int* slist = reinterpret_cast<int*>(sKF + bkv * d);  // [Tm]
  __shared__ int s_cnt;
  const long long u = blockIdx.y;
  const int j = blockIdx.x;
  const long long kv0 = u * D.N + (long long)j * bkv;
  if (threadIdx.x < 32) {
    const int8_t* lu = labels + u * (long long)D.Tm * D.Tn;
    int base = 0;
    for (int i0 = 0; i0 < D.Tm; i0 += 32) {
      const int i = i0 + threadIdx.x;
      const bool m = i < D.Tm && lu[(long long)i * D.Tn + j] == 0;
      const unsigned b = __ballot_sync(0xffffffffu, m);
      if (m) slist[base + __popc(b & ((1u << threadIdx.x) - 1u))] = i;
      base += __popc(b);
    }
    if (threadIdx.x == 0) s_cnt = base;
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt == 0) {
    for (int e = threadIdx.x; e < bkv * d; e += blockDim.x) dkf[kv0 * d + e] = 0.f;
    return;
  }
  const float* gHu = gH + u * (long long)D.Tm * d * d;
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < cnt; ++p) {
      const float x = gHu[(long long)slist[p] * d * d + idx];
      acc = p == 0 ? x : add_rn(acc, x);
    }
    sHa[(idx / d) * dp + idx % d] = acc;
  }
  const float* gZu = gZ + u * (long long)D.Tm * d;
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < cnt; ++p) {
      const float x = gZu[(long long)slist[p] * d + a];
      acc = p == 0 ? x : add_rn(acc, x);
    }
    sZa[a] = acc;
  }
  for (int e = threadIdx.x; e < bkv * d; e += blockDim.x) {
    sV[e] = to_f(v[kv0 * d + e]);
    sKF[e] = kf[kv0 * d + e];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < bkv * d; idx += blockDim.x) {
    const int t = idx / d, a = idx % d;
    float acc = 0.f;
    for (int b = 0; b < d; ++b) acc = add_rn(acc, mul_rn(sV[t * d + b], sHa[a * dp + b]));
    dkf[kv0 * d + idx] = add_rn(acc, sZa[a]);
    // dv_lin[t][b] with b = a here (same index space)
    const int b = a;
    float lin = 0.f;
    for (int aa = 0; aa < d; ++aa) {
      const float ka = sKF[t * d + aa];
      if (ka == 0.f) continue;
      lin = add_rn(lin, mul_rn(ka, sHa[aa * dp + b]));
    }
    dv[kv0 * d + idx] = add_rn(dv[kv0 * d + idx], lin);
  }
}

// dQ_total = J_phi(Q)^T dQ^phi + dQ (feature_map.cpp:42-73, backward.cpp:211-214); warp/row.
template <typename In>
__global__ void k_vjp_out(Dims D, int phi, const In* __restrict__ x,
                          const float* __restrict__ dfeat, const float* __restrict__ dsparse,
                          In* __restrict__ out) {
  const long long r = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31, d = D.d;
  if (r >= D.U * D.N) return;
  const long long g = r * d;
  if (phi != 2) {
    for (int c = lane; c < d; c += 32) {
      const float xv = to_f(x[g + c]);
      const float gv = dfeat[g + c];
      const float j = phi == 0 ? (xv >= 0.f ? gv : expf(xv) * gv) : (xv > 0.f ? gv : 0.f);
      out[g + c] = from_f<In>(j + dsparse[g + c]);
    }
    return;
  }
  float m = -INFINITY;
  for (int c = lane; c < d; c += 32) m = fmaxf(m, to_f(x[g + c]));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += expf(to_f(x[g + c]) - m);
  s = warp_sum(s);
  float dot = 0.f;
  for (int c = lane; c < d; c += 32) dot += expf(to_f(x[g + c]) - m) / s * dfeat[g + c];
  dot = warp_sum(dot);
  for (int c = lane; c < d; c += 32) {
    const float sv = expf(to_f(x[g + c]) - m) / s;
    out[g + c] = from_f<In>(sv * (dfeat[g + c] - dot) + dsparse[g + c]);
  }
}

template <typename In>
__global__ void k_cast_out(const float* __restrict__ x, In* __restrict__ out, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = from_f<In>(x[e]);
}

size_t rows_sparse_smem(const Dims& D) {
  const int d = D.d, bq = D.bq, bkv = D.bkv;
  return size_t(3 * bq * d + 2 * bkv * (d + 1) + bq * bkv + 2 * bq) * 4;
}
size_t cols_sparse_smem(const Dims& D) {
  const int d = D.d, bq = D.bq, bkv = D.bkv;
  return size_t(2 * bkv * (d + 1) + 2 * bq * d + 2 * bq * bkv + 2 * bq) * 4;
}
size_t cols_lin_smem(const Dims& D) {
  const int d = D.d, bkv = D.bkv;
  return size_t(d * (d + 1) + d + 2 * bkv * d + D.Tm) * 4;
}
size_t rows_lin_smem(const Dims& D) {
  const int d = D.d, bq = D.bq;
  return size_t(2 * bq * d + d * (d + 1) + d + 2 * bq) * 4;
}
size_t prep_smem(const Dims& D) { return size_t(D.d * (D.d + 1) + 8 * D.d) * 4; }

unsigned grid1(long long total, int per) {
  return unsigned(std::max<long long>(1, (total + per - 1) / per));
}

template <typename In>
void forward_t(const Dims& D, const In* q, const In* k, const In* v, const In* w, In* o,
               In* o_s, In* o_l, float* lse, const StateBufs& s, const WorkBufs& wb,
               cudaStream_t st, bool attention = true) {
  const long long rows = D.U * D.N;
  k_phi<In><<<grid1(rows, 8), 256, 0, st>>>(q, wb.qf, rows, D.d, D.phi);
  check_launch("k_phi(q)", st);
  k_phi<In><<<grid1(rows, 8), 256, 0, st>>>(k, wb.kf, rows, D.d, D.phi);
  check_launch("k_phi(k)", st);
  const size_t sum_smem = size_t(2 * D.bkv * D.d) * 4;
  set_smem(k_summaries<In>, sum_smem);
  k_summaries<In><<<dim3(D.Tn, unsigned(D.U)), kThreads, sum_smem, st>>>(
      wb.kf, v, D.N, D.d, D.bkv, D.Tn, wb.h, wb.z);
  check_launch("k_summaries", st);
  const size_t agg_smem = size_t(D.Tn) * 4;
  set_smem(k_aggregate_rows, agg_smem);
  k_aggregate_rows<<<dim3(D.Tm, unsigned(D.U)), kThreads, agg_smem, st>>>(
      s.labels, wb.h, wb.z, D.d, D.Tm, D.Tn, s.H, s.Z);
  check_launch("k_aggregate_rows", st);
  if (!attention) return;  // sla_b200_build_state: the forward state without the outputs
  const FwdSmem L = fwd_smem(D);
  set_smem(k_fwd_generic<In>, L.bytes);
  k_fwd_generic<In><<<dim3(D.Tm, unsigned(D.U)), kThreads, L.bytes, st>>>(
      D, L, q, k, v, w, wb.qf, s.crit_cnt, s.crit_idx, s.marg_cnt, s.H, s.Z, o, o_s, o_l, lse);
  check_launch("k_fwd_generic", st);
}

template <typename In>
void backward_t(const Dims& D, const In* q, const In* k, const In* v, const In* w,
                const In* o_s, const In* o_l, const float* lse, const In* d_out, const In* d_out_l,
                In* dq, In* dk, In* dv, float* dw, const StateBufs& s, const WorkBufs& wb,
                cudaStream_t st) {
  const long long rows = D.U * D.N;
  const size_t nd = size_t(rows) * D.d;
  if (dw) SLAB_CUDA(cudaMemsetAsync(dw, 0, sizeof(float) * size_t(D.H) * D.d * D.d, st));
  SLAB_CUDA(cudaMemsetAsync(wb.dk, 0, sizeof(float) * nd, st));
  SLAB_CUDA(cudaMemsetAsync(wb.dv, 0, sizeof(float) * nd, st));
  prof_mark("", st);
  k_phi<In><<<grid1(rows, 8), 256, 0, st>>>(q, wb.qf, rows, D.d, D.phi);
  check_launch("k_phi(q)", st);
  k_phi<In><<<grid1(rows, 8), 256, 0, st>>>(k, wb.kf, rows, D.d, D.phi);
  check_launch("k_phi(k)", st);
  launch_build_csc(D, s, st);
  const size_t ps = prep_smem(D);
  set_smem(k_bwd_prep<In>, ps);
  k_bwd_prep<In><<<dim3(grid1(D.N, 64), unsigned(D.U)), 256, ps, st>>>(
      D, w, d_out, d_out_l, o_s, o_l, wb.dOl, wb.Ds, wb.Dl);
  check_launch("k_bwd_prep", st);
  if (dw) {  // dproj = O^l^T dO^s (backward.cpp:46)
    const size_t dws = size_t(64 * D.d) * 4;
    set_smem(k_dw<In>, dws);
    k_dw<In><<<dim3(grid1(D.N, 32), unsigned(D.U)), 256, dws, st>>>(D, o_l, d_out, dw);
    check_launch("k_dw", st);
  }
  const size_t rl = rows_lin_smem(D);
  if (s.H) {
    set_smem(k_bwd_rows_lin<float>, rl);
    k_bwd_rows_lin<float><<<dim3(D.Tm, unsigned(D.U)), kThreads, rl, st>>>(
        D, s.marg_cnt, wb.qf, wb.dOl, wb.Dl, s.H, s.Z, wb.gH, wb.gZ, wb.dqf);
  } else {
    set_smem(k_bwd_rows_lin<__nv_bfloat16>, rl);
    k_bwd_rows_lin<__nv_bfloat16><<<dim3(D.Tm, unsigned(D.U)), kThreads, rl, st>>>(
        D, s.marg_cnt, wb.qf, wb.dOl, wb.Dl, s.Hb, s.Z, wb.gH, wb.gZ, wb.dqf);
  }
  check_launch("k_bwd_rows_lin", st);
  const size_t rs = rows_sparse_smem(D);
  set_smem(k_bwd_rows_sparse<In>, rs);
  k_bwd_rows_sparse<In><<<dim3(D.Tm, unsigned(D.U)), kThreads, rs, st>>>(
      D, q, k, v, d_out, lse, wb.Ds, s.crit_cnt, s.crit_idx, wb.dq);
  check_launch("k_bwd_rows_sparse", st);
  const size_t cs = cols_sparse_smem(D);
  set_smem(k_bwd_cols_sparse<In>, cs);
  k_bwd_cols_sparse<In><<<dim3(D.Tn, unsigned(D.U)), kThreads, cs, st>>>(
      D, q, k, v, d_out, lse, wb.Ds, s.ccol_cnt, s.ccol_idx, wb.dk, wb.dv);
  check_launch("k_bwd_cols_sparse", st);
  const size_t cl = cols_lin_smem(D);
  set_smem(k_bwd_cols_lin<In>, cl);
  k_bwd_cols_lin<In><<<dim3(D.Tn, unsigned(D.U)), kThreads, cl, st>>>(
      D, s.labels, v, wb.kf, wb.gH, wb.gZ, wb.dkf, wb.dv);
  check_launch("k_bwd_cols_lin", st);
  k_vjp_out<In><<<grid1(rows, 8), 256, 0, st>>>(D, D.phi, q, wb.dqf, wb.dq, dq);
  check_launch("k_vjp_out(q)", st);
  k_vjp_out<In><<<grid1(rows, 8), 256, 0, st>>>(D, D.phi, k, wb.dkf, wb.dk, dk);
  check_launch("k_vjp_out(k)", st);
  k_cast_out<In><<<unsigned(std::min<long long>(grid1(nd, 256), 148 * 8)), 256, 0, st>>>(
      wb.dv, dv, (long long)nd);
  check_launch("k_cast_out(dv)", st);
}

}  // namespace

bool generic_supported(const Dims& D, std::string* why) {
  const size_t limit = 227 * 1024;
  const size_t need = std::max({fwd_smem(D).bytes, rows_sparse_smem(D), cols_sparse_smem(D),
                                cols_lin_smem(D), rows_lin_smem(D), prep_smem(D),
                                size_t(2 * D.bkv * D.d) * 4});
  if (need > limit) {
    if (why)
      *why = "sla_b200: shape needs " + std::to_string(need) +
             " bytes of shared memory in the generic kernels (limit 232448)";
    return false;
  }
  return true;
}

void generic_forward(const Dims& D, int dtype, const void* q, const void* k, const void* v,
                     const void* w, void* o, void* o_s, void* o_l, float* lse,
                     const StateBufs& s, const WorkBufs& wb, cudaStream_t st, bool attention) {
  if (dtype == 0) {
    using T = __nv_bfloat16;
    forward_t<T>(D, (const T*)q, (const T*)k, (const T*)v, (const T*)w, (T*)o, (T*)o_s,
                 (T*)o_l, lse, s, wb, st, attention);
  } else {
    forward_t<float>(D, (const float*)q, (const float*)k, (const float*)v, (const float*)w,
                     (float*)o, (float*)o_s, (float*)o_l, lse, s, wb, st, attention);
  }
}

void generic_backward(const Dims& D, int dtype, const void* q, const void* k, const void* v,
                      const void* w, const void* o_s, const void* o_l, const float* lse,
                      const void* d_out, const void* d_out_l, void* dq, void* dk, void* dv, float* dw,
                      const StateBufs& s, const WorkBufs& wb, cudaStream_t st) {
  if (dtype == 0) {
    using T = __nv_bfloat16;
    backward_t<T>(D, (const T*)q, (const T*)k, (const T*)v, (const T*)w, (const T*)o_s,
                  (const T*)o_l, lse, (const T*)d_out, (const T*)d_out_l, (T*)dq, (T*)dk, (T*)dv, dw, s,
                  wb, st);
  } else {
    backward_t<float>(D, (const float*)q, (const float*)k, (const float*)v, (const float*)w,
                      (const float*)o_s, (const float*)o_l, lse, (const float*)d_out,
                      (const float*)d_out_l, (float*)dq, (float*)dk, (float*)dv, dw, s, wb, st);
  }
}

// proj_backward's dW = O^l^T dO (backward.cpp:12-22) summed over the batch per head, f32 [H, d, d]
void generic_dw(const Dims& D, int dtype, const void* o_l, const void* d_out, float* dw, cudaStream_t st) {
  SLAB_CUDA(cudaMemsetAsync(dw, 0, sizeof(float) * size_t(D.H) * D.d * D.d, st));
  const size_t dws = size_t(64 * D.d) * 4;
  if (dtype == 0) {
    set_smem(k_dw<__nv_bfloat16>, dws);
    k_dw<__nv_bfloat16><<<dim3(grid1(D.N, 32), unsigned(D.U)), 256, dws, st>>>(
        D, (const __nv_bfloat16*)o_l, (const __nv_bfloat16*)d_out, dw);
  } else {
    set_smem(k_dw<float>, dws);
    k_dw<float><<<dim3(grid1(D.N, 32), unsigned(D.U)), 256, dws, st>>>(D, (const float*)o_l,
                                                                          (const float*)d_out, dw);
  }
  check_launch("k_dw", st);
}

}  // namespace slab
