// classify.cu -- K1+K2: block pooling, compressed-weight prediction and three-way block
// classification, plus the lookup structures every later kernel iterates.
//
// Reference: mask.cpp:40-153 (pool_mean, predict_compressed_weights, classify_mask,
// build_lookup), forward.cpp:174-185 (the mask is computed in f64 on every path).
//
// HBM-bound: Q and K are each read once (vectorised over d, coalesced across threads);
// everything after pooling works on T x d / T x T data that lives in L2.
#include <algorithm>
#include <cfloat>
#include <type_traits>

#include "buffers.hpp"
#include "kernels.hpp"

namespace slab {

// ---------------------------------------------------------------------------------------
// K0: first non-finite entry (forward.cpp:15-25 check_input), flat index via atomicMin.
// ---------------------------------------------------------------------------------------
template <typename In>
__global__ void k_check_finite(const In* __restrict__ x, long long total,
                               long long* __restrict__ slot) {
  long long first = LLONG_MAX;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    if (!isfinite(to_f(x[i]))) {
      first = i;
      break;
    }
  }
  if (first != LLONG_MAX) atomicMin(slot, first);
}

// ---------------------------------------------------------------------------------------
// K1a: block means (mask.cpp:40-55): ascending row sum, then one division, in R.
// grid (T, U), threads over the d columns (coalesced).
// ---------------------------------------------------------------------------------------
template <typename R, typename In>
__global__ void k_pool(const In* __restrict__ x, R* __restrict__ out, long long N, int d, int b,
                       int T, long long n_valid, RowLayout rl) {
  const long long u = blockIdx.y;
  const int g = blockIdx.x;
  // ragged N (SLA_B200_FLAG_RAGGED): the last block's mean is over its valid rows only
  const long long left = n_valid - (long long)g * b;
  const int rows = left < b ? int(left) : b;
  const RowMap rm = row_map(rl, u, N);
  const In* base = x + (rm.base + (long long)g * b * rm.stride) * d;  // rows < `rows` all exist
  const long long rs = rm.stride * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    R acc = R(0);
    for (int r = 0; r < rows; ++r) acc = add_rn(acc, R(to_f(base[r * rs + c])));
    out[(u * T + g) * d + c] = div_rn(acc, R(rows));
  }
}

// K1a for bf16 inputs with d % 4 == 0: Q and K in one launch (blockIdx.z), one warp per block,
// each lane four adjacent columns (8-byte loads, four independent ascending sums), the same
// per-column operation order as k_pool.
template <typename R>
__global__ void __launch_bounds__(32) k_pool2_bf16(const __nv_bfloat16* __restrict__ q,
                                                   const __nv_bfloat16* __restrict__ k,
                                                   R* __restrict__ pq, R* __restrict__ pk, long long Nq,
                                                   long long Nk, int d, int b, int Tq, int Tk,
                                                   long long nq_valid, long long nk_valid, RowLayout rl) {
  pdl_entry();  // launched by launch_pdl
  const long long u = blockIdx.y;
  const int g = blockIdx.x;
  const __nv_bfloat16* x = blockIdx.z ? k : q;
  R* out = blockIdx.z ? pk : pq;
  const long long N = blockIdx.z ? Nk : Nq, n_valid = blockIdx.z ? nk_valid : nq_valid;
  const int T = blockIdx.z ? Tk : Tq;
  if (g >= T) return;
  const long long left = n_valid - (long long)g * b;
  const int rows = left < b ? int(left) : b;
  const RowMap rm = row_map(rl, u, N);
  const __nv_bfloat16* base = x + (rm.base + (long long)g * b * rm.stride) * d;  // rows < `rows` all exist
  const long long rs = rm.stride * d;
  for (int c = 4 * threadIdx.x; c < d; c += 128) {
    R a0 = R(0), a1 = R(0), a2 = R(0), a3 = R(0);
    const __nv_bfloat16* xr = base + c;
    auto acc = [&](const uint2& v) {
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
      const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
      a0 = add_rn(a0, R(f0.x));
      a1 = add_rn(a1, R(f0.y));
      a2 = add_rn(a2, R(f1.x));
      a3 = add_rn(a3, R(f1.y));
    };
    int r = 0;
    for (; r + 16 <= rows; r += 16, xr += 16 * rs) {  // 16 rows' loads in flight, then the ascending sums
      uint2 v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = *reinterpret_cast<const uint2*>(xr + e * rs);
#pragma unroll
      for (int e = 0; e < 16; ++e) acc(v[e]);
    }
    for (; r < rows; ++r, xr += rs) acc(*reinterpret_cast<const uint2*>(xr));
    R* o = out + (u * T + g) * d + c;
    o[0] = div_rn(a0, R(rows));
    o[1] = div_rn(a1, R(rows));
    o[2] = div_rn(a2, R(rows));
    o[3] = div_rn(a3, R(rows));
  }
}

// ---------------------------------------------------------------------------------------
// K1b+K2: one CTA per (unit, block row).  Scores in R with the reference's operation order
// (matmul_nt ascending-k dot, mat.hpp:83-97; then * 1/sqrt(d)), max-shifted softmax with
// the ascending-j normaliser (mask.cpp:65-79), then a bitonic sort of
// (weight desc, column asc) -- exactly std::stable_sort's order from an iota start
// (mask.cpp:105-113) -- and the label / lookup writes (mask.cpp:114-153).
// ---------------------------------------------------------------------------------------
// K1b: pooled scores S = pool(Q) pool(K)^T * (1/sqrt(d)) for all block pairs, tiled 64x64
// per CTA (each thread a 4x4 patch, strided by 16 rows / columns).  Every element is still ONE sequential ascending-c dot
// with separately rounded mul and add (mat.hpp:83-97), so the values are bit-identical to
// the reference's; tiling only shares the pooled rows through shared memory.
// K1b (f64 path): 64 x 64 score tile per CTA of 128 threads, 4 rows x 8 columns per thread
// (12 shared-memory reads per 32 multiply-adds: the tile is FP64-issue bound, not smem bound),
// the pooled rows staged in 32-column chunks by cp.async into two buffers (chunk c+1 lands while
// chunk c is multiplied).  Operation order as mat.hpp:83-97: ascending c, mul and add rounded
// separately, then * 1/sqrt(d).
template <typename R>
__global__ void __launch_bounds__(128) k_scores(const R* __restrict__ pq, const R* __restrict__ pk,
                                                int d, int Tm, int Tn, R inv_sqrt_d,
                                                R* __restrict__ s) {
  pdl_entry();  // launched by launch_pdl
  constexpr int CK = 32, PITCH = CK + 1;
  extern __shared__ __align__(16) unsigned char scores_smem[];  // R [2][64][PITCH] twice
  auto sa = reinterpret_cast<R(*)[64][PITCH]>(scores_smem);
  auto sb = reinterpret_cast<R(*)[64][PITCH]>(scores_smem + sizeof(R) * 2 * 64 * PITCH);
  const long long u = blockIdx.z;
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // rows ty + 16a, columns tx + 8b
  R acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = R(0);
  const R* pqu = pq + u * (long long)Tm * d;
  const R* pku = pk + u * (long long)Tn * d;
  const int nch = (d + CK - 1) / CK;
  auto stage = [&](int ch, int buf) {  // rows past T and columns past d as zeros
    const int c0 = ch * CK;
    for (int e = threadIdx.x; e < 64 * CK; e += 128) {
      const int r = e / CK, c = e % CK;
      R* da = &sa[buf][r][c];
      R* db = &sb[buf][r][c];
      if (i0 + r < Tm && c0 + c < d)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(da))),
                     "l"(pqu + (long long)(i0 + r) * d + c0 + c), "n"(int(sizeof(R)))
                     : "memory");
      else
        *da = R(0);
      if (j0 + r < Tn && c0 + c < d)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(db))),
                     "l"(pku + (long long)(j0 + r) * d + c0 + c), "n"(int(sizeof(R)))
                     : "memory");
      else
        *db = R(0);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nch) {
      stage(ch + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int ck = min(CK, d - ch * CK);
    for (int c = 0; c < ck; ++c) {
      R av[4], bv[8];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[buf][ty + 16 * a][c];
#pragma unroll
      for (int b = 0; b < 8; ++b) bv[b] = sb[buf][tx + 8 * b][c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = add_rn(acc[a][b], mul_rn(av[a], bv[b]));
    }
    __syncthreads();  // buffer buf is restaged two chunks later
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + ty + 16 * a;
    if (i >= Tm) continue;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int j = j0 + tx + 8 * b;
      if (j < Tn) s[(u * Tm + i) * (long long)Tn + j] = mul_rn(acc[a][b], inv_sqrt_d);
    }
  }
}

template <typename R>
__device__ __forceinline__ bool before(R ka, int ia, R kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

template <typename R>
__global__ void k_classify(const R* __restrict__ scores, int Tm,
                           int Tn, int P2, int n1, int n_neg,
                           int8_t* __restrict__ labels, int* __restrict__ crit_cnt,
                           int* __restrict__ crit_idx, int* __restrict__ marg_cnt,
                           double* __restrict__ p_c_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* key = reinterpret_cast<R*>(smem_raw);                   // [P2]
  int* idx = reinterpret_cast<int*>(key + P2);                // [P2]
  int8_t* lab = reinterpret_cast<int8_t*>(idx + P2);          // [Tn]
  __shared__ R red[32];

  const long long u = blockIdx.y;
  const int i = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const R* srow = scores + (u * Tm + i) * (long long)Tn;
  R lmax = -R(INFINITY);
  for (int j = tid; j < Tn; j += nt) {
    const R s = srow[j];
    key[j] = s;
    lmax = s > lmax ? s : lmax;
  }
  // block max (order-independent, exact)
  for (int o = 16; o > 0; o >>= 1) {
    const R other = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmax = other > lmax ? other : lmax;
  }
  if ((tid & 31) == 0) red[tid >> 5] = lmax;
  __syncthreads();
  if (tid == 0) {
    R m = red[0];
    for (int w = 1; w < (nt + 31) / 32; ++w) m = red[w] > m ? red[w] : m;
    red[0] = m;
  }
  __syncthreads();
  const R m = red[0];
  for (int j = tid; j < Tn; j += nt) key[j] = exp_r(key[j] - m);
  __syncthreads();
  if (tid == 0) {  // the reference's sequential normaliser (mask.cpp:73-77)
    R sum = R(0);
    for (int j = 0; j < Tn; ++j) sum = add_rn(sum, key[j]);
    red[1] = sum;
  }
  __syncthreads();
  const R sum = red[1];
  for (int j = tid; j < P2; j += nt) {
    if (j < Tn) {
      key[j] = div_rn(key[j], sum);
      if (p_c_out) p_c_out[(u * Tm + i) * Tn + j] = double(key[j]);
    } else {
      key[j] = -R(1);  // pads sort after every weight (weights are >= 0)
    }
    idx[j] = j;
  }
  __syncthreads();

  // bitonic sort into before-order; pass (k, jj) compares t and t ^ jj for the P2/2 pairs
  // with bit jj of t clear -- indexed by pair so every thread does one exchange per pass
  int lj = 0;
  for (int k = 2; k <= P2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      lj = __ffs(jj) - 1;
      for (int pr = tid; pr < (P2 >> 1); pr += nt) {
        const int t = ((pr >> lj) << (lj + 1)) | (pr & (jj - 1));
        const int x = t | jj;
        const R ka = key[t], kb = key[x];
        const int ia = idx[t], ib = idx[x];
        const bool t_first = before(ka, ia, kb, ib);
        const bool up = (t & k) == 0;
        if (up != t_first) {
          key[t] = kb;
          key[x] = ka;
          idx[t] = ib;
          idx[x] = ia;
        }
      }
      __syncthreads();
    }
  }
  (void)lj;
  for (int r = tid; r < Tn; r += nt) {
    const int j = idx[r];
    lab[j] = r < n1 ? int8_t(1) : (r >= Tn - n_neg ? int8_t(-1) : int8_t(0));
  }
  __syncthreads();
  int8_t* lrow = labels + (u * Tm + i) * (long long)Tn;
  for (int j = tid; j < Tn; j += nt) lrow[j] = lab[j];
  // ascending critical list + marginal count (warp 0)
  if (tid < 32) {
    int base = 0, marg = 0;
    int* crow = crit_idx + (u * Tm + i) * (long long)Tn;
    for (int j0 = 0; j0 < Tn; j0 += 32) {
      const int j = j0 + tid;
      const int l = j < Tn ? lab[j] : -1;
      const unsigned bc = __ballot_sync(0xffffffffu, l == 1);
      const unsigned bm = __ballot_sync(0xffffffffu, l == 0);
      if (l == 1) crow[base + __popc(bc & ((1u << tid) - 1u))] = j;
      base += __popc(bc);
      marg += __popc(bm);
    }
    if (tid == 0) {
      crit_cnt[u * Tm + i] = base;
      marg_cnt[u * Tm + i] = marg;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K2, warp-per-row variant for 32 <= P2 <= 512 (the Wan2.1 shape has T = 512): one warp owns
// a block row, EPL = P2/32 consecutive entries per lane in registers.  Same arithmetic as
// k_classify -- exact max, exp, the reference's sequential ascending normaliser (the running
// sum is handed lane to lane), one rounded division -- and the same bitonic network over
// (weight desc, column asc), with the distance >= EPL passes done by shuffles.  No block
// barriers: a whole row is one warp's registers.
// ---------------------------------------------------------------------------------------
#ifndef SLAB_CLASSIFY_RANK
#define SLAB_CLASSIFY_RANK 1  // 1: k_classify_rank (rank raw scores) for T <= 2048
#endif
// diagnostics: rows that took k_classify_rank's exact P_c path (null: not counted)
static int* g_exact_counter = nullptr;
int* classify_exact_counter() { return g_exact_counter; }
void set_classify_exact_counter(int* p) { g_exact_counter = p; }
#ifndef SLAB_CLASSIFY_SELECT
#define SLAB_CLASSIFY_SELECT 1  // 1: quickselect of the two rank thresholds; 0: full bitonic sort
#endif
template <typename R, int EPL>
__global__ void __launch_bounds__(256) k_classify_warp(const R* __restrict__ scores, long long rows,
                                                       int Tn, int n1, int n_neg,
                                                       int8_t* __restrict__ labels, int* __restrict__ crit_cnt,
                                                       int* __restrict__ crit_idx, int* __restrict__ marg_cnt,
                                                       double* __restrict__ p_c_out,
                                                       __nv_bfloat16* __restrict__ m0, int m0_ld) {
  pdl_entry();  // launched by launch_pdl
  constexpr int P2 = 32 * EPL;
  __shared__ int8_t slab[8][P2];
  __shared__ R ebuf[8][P2 + 1];  // the 8 rows' exponentials for the sequential normaliser
  __shared__ R rsum[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row0 = (long long)blockIdx.x * 8;
  const long long row = row0 + warp;
  const bool active = row < rows;
  const R* srow = scores + (active ? row : 0) * Tn;
  R key[EPL];
  int idx[EPL];
  R m = -R(INFINITY);
#pragma unroll
  for (int r = 0; r < EPL; ++r) {
    const int j = lane * EPL + r;
    key[r] = j < Tn ? srow[j] : -R(INFINITY);
    m = key[r] > m ? key[r] : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const R other = __shfl_xor_sync(0xffffffffu, m, o);
    m = other > m ? other : m;
  }
#pragma unroll
  for (int r = 0; r < EPL; ++r) key[r] = lane * EPL + r < Tn ? exp_r(key[r] - m) : R(0);
  // sequential ascending-j normaliser (mask.cpp:73-77).  The chain of Tn dependent adds is
  // inherent (bit-exact order); lanes 0-7 of warp 0 run the block's 8 chains side by side
  // from shared memory instead of every warp predicating its chain through all 32 lanes.
#pragma unroll
  for (int r = 0; r < EPL; ++r) ebuf[warp][lane * EPL + r] = key[r];
  __syncthreads();
  if (warp == 0 && lane < 8) {
    R acc = R(0);
    if (row0 + lane < rows)
      for (int j = 0; j < Tn; ++j) acc = add_rn(acc, ebuf[lane][j]);
    rsum[lane] = acc;
  }
  __syncthreads();
  if (!active) return;
  const R sum = rsum[warp];
#pragma unroll
  for (int r = 0; r < EPL; ++r) {
    const int j = lane * EPL + r;
    idx[r] = j;
    if (j < Tn) {
      key[r] = div_rn(key[r], sum);
      if (p_c_out) p_c_out[row * Tn + j] = double(key[r]);
    } else {
      key[r] = -R(1);  // pads sort after every weight (weights are >= 0)
    }
  }
#if SLAB_CLASSIFY_SELECT
  // Ranks by selection instead of a full sort.  rank(e) = #(w > w_e) + #(w == w_e, j < j_e) is
  // the position in stable_sort's (weight desc, column asc) order (mask.cpp:91-119), so with
  // v1 = the weight at rank n1 - 1 and v2 = the weight at rank Tn - n_neg,
  //   critical   <=> w > v1, or w == v1 and #(w > v1) + (ties of v1 before e) < n1,
  //   negligible <=> w < v2, or w == v2 and #(w > v2) + (ties of v2 before e) >= Tn - n_neg.
  // Each threshold is a quickselect over exact comparisons (pads carry -1 and never qualify).
  (void)idx;
  constexpr unsigned FULL = 0xffffffffu;
  // candidates are a per-lane bit mask over the lane's EPL weights; pivots come from shared memory
#pragma unroll
  for (int r = 0; r < EPL; ++r) ebuf[warp][lane * EPL + r] = key[r];
  __syncwarp();
  const R* prow = &ebuf[warp][lane * EPL];
  unsigned vmask = 0u;
#pragma unroll
  for (int r = 0; r < EPL; ++r) vmask |= (lane * EPL + r < Tn ? 1u : 0u) << r;
  auto select_desc = [&](int K) -> R {  // the weight at 0-based rank K
    unsigned cm = vmask;
    int k = K;
    for (int it = 0;; ++it) {
      const unsigned has = __ballot_sync(FULL, cm != 0u);
      if (has == 0u) return R(-1);  // no candidate left (only with non-finite weights): never hang
      const int rot = (it * 11) & 31;
      const unsigned rm = rot ? (has >> rot) | (has << (32 - rot)) : has;
      const int src = (__ffs(rm) - 1 + rot) & 31;
      R mv = R(0);
      if (lane == src) mv = prow[__ffs(cm) - 1];
      const R pivot = __shfl_sync(FULL, mv, src);
      unsigned gm = 0u, em = 0u;
#pragma unroll
      for (int r = 0; r < EPL; ++r) {
        gm |= (key[r] > pivot ? 1u : 0u) << r;
        em |= (key[r] == pivot ? 1u : 0u) << r;
      }
      gm &= cm;
      em &= cm;
      const int g = __reduce_add_sync(FULL, __popc(gm));
      const int e = __reduce_add_sync(FULL, __popc(em));
      if (k < g) {
        cm = gm;
      } else if (k < g + e) {
        return pivot;
      } else {
        k -= g + e;
        cm &= ~(gm | em);
      }
    }
  };
  // #(w > v) over the row, and this lane's count of ties w == v before its first element
  auto ties_before = [&](R v, int& gt) -> int {
    int g = 0, t = 0;
#pragma unroll
    for (int r = 0; r < EPL; ++r) {
      g += key[r] > v;
      t += key[r] == v;
    }
    gt = __reduce_add_sync(FULL, g);
    int x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    return x - t;
  };
  int8_t* lab = slab[warp];
  bool crit[EPL], negl[EPL];
#pragma unroll
  for (int r = 0; r < EPL; ++r) crit[r] = negl[r] = false;
  if (n1 > 0) {
    const R v1 = select_desc(n1 - 1);
    int gt1;
    int run = ties_before(v1, gt1);
#pragma unroll
    for (int r = 0; r < EPL; ++r) {
      if (key[r] == v1) crit[r] = gt1 + run++ < n1;
      else crit[r] = key[r] > v1;
    }
  }
  if (n_neg > 0) {
    const R v2 = select_desc(Tn - n_neg);
    int gt2;
    int run = ties_before(v2, gt2);
#pragma unroll
    for (int r = 0; r < EPL; ++r) {
      if (key[r] == v2) negl[r] = gt2 + run++ >= Tn - n_neg;
      else negl[r] = key[r] < v2;
    }
  }
#pragma unroll
  for (int r = 0; r < EPL; ++r) {
    const int j = lane * EPL + r;
    if (j < Tn) lab[j] = crit[r] ? int8_t(1) : (negl[r] ? int8_t(-1) : int8_t(0));
  }
#else
#pragma unroll
  for (int k = 2; k <= P2; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= EPL) {  // partner in lane ^ (jj / EPL), same register
        const int lm = jj / EPL;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          const R ok = __shfl_xor_sync(0xffffffffu, key[r], lm);
          const int oi = __shfl_xor_sync(0xffffffffu, idx[r], lm);
          const int t = (lane * EPL + r) & ~jj;  // lower position of the pair
          const bool up = (t & k) == 0;
          const bool mine_first = before(key[r], idx[r], ok, oi);
          if ((lower == up) != mine_first) {
            key[r] = ok;
            idx[r] = oi;
          }
        }
      } else {  // partner in the same lane
#pragma unroll
        for (int r = 0; r < EPL; ++r) {
          if (r & jj) continue;
          const int x = r | jj;
          const bool up = ((lane * EPL + r) & k) == 0;
          if (up != before(key[r], idx[r], key[x], idx[x])) {
            const R tk = key[r];
            key[r] = key[x];
            key[x] = tk;
            const int ti = idx[r];
            idx[r] = idx[x];
            idx[x] = ti;
          }
        }
      }
    }
  }
  int8_t* lab = slab[warp];
#pragma unroll
  for (int r = 0; r < EPL; ++r) {
    const int e = lane * EPL + r;  // rank
    if (idx[r] < Tn) lab[idx[r]] = e < n1 ? int8_t(1) : (e >= Tn - n_neg ? int8_t(-1) : int8_t(0));
  }
#endif
  __syncwarp();
  int8_t* lrow = labels + row * Tn;
  for (int j = lane; j < Tn; j += 32) lrow[j] = lab[j];
  if (m0) {  // fast path: the marginal indicator row (A operand of H = M0 h), bf16 pairs
    __nv_bfloat162* mrow = reinterpret_cast<__nv_bfloat162*>(m0 + row * m0_ld);
    for (int j2 = lane; j2 < m0_ld / 2; j2 += 32) {
      const int j = 2 * j2;
      mrow[j2] = __floats2bfloat162_rn(j < Tn && lab[j] == 0 ? 1.f : 0.f,
                                       j + 1 < Tn && lab[j + 1] == 0 ? 1.f : 0.f);
    }
  }
  int base = 0, marg = 0;
  int* crow = crit_idx + row * Tn;
  for (int j0 = 0; j0 < Tn; j0 += 32) {
    const int j = j0 + lane;
    const int l = j < Tn ? lab[j] : -1;
    const unsigned bc = __ballot_sync(0xffffffffu, l == 1);
    const unsigned bm = __ballot_sync(0xffffffffu, l == 0);
    if (l == 1) crow[base + __popc(bc & ((1u << lane) - 1u))] = j;
    base += __popc(bc);
    marg += __popc(bm);
  }
  if (lane == 0) {
    crit_cnt[row] = base;
    marg_cnt[row] = marg;
  }
}

// ---------------------------------------------------------------------------------------
// K2 by ranking the raw pooled scores (T <= 2048): one warp per block row, the row in shared
// memory with interleaved ownership (element j = 32 r + lane: conflict-free).
//
// P_c = g(S) with g(s) = round(exp(round(s - m)) / sum) (mask.cpp:65-79) is monotone
// non-decreasing in s, so stable_sort's (P_c desc, j asc) order (mask.cpp:105-113) and the
// (S desc, j asc) order put the same blocks on each side of a rank boundary whenever g
// separates the scores next to it strictly.  Per boundary (rank n1 and rank T - n_neg) the
// kernel finds A = S at rank K - 1 and B = S at rank K by quickselect and checks
//   A > B:   g(A) > g(B);
//   A == B:  g(min{s > A}) > g(A) > g(max{s < A})   (the tie class straddles the boundary),
// where x > y => g(x) > g(y) is guaranteed once exp(x - m) > exp(y - m) (1 + 2^-50): the division
// by the common sum cannot merge values a factor 1 + 2^-50 apart.  Then the labels follow from
// the S-ranks and the row needs neither the T exponentials nor the sequential T-long normaliser.
// Otherwise (near-ties, or P_c requested) the warp computes P_c exactly as k_classify_warp does
// -- max-shifted exp, the ascending sequential normaliser, one rounded division -- and ranks P_c.
// ---------------------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ bool g_separated(R x, R y, R m) {  // x > y: is g(x) > g(y) certain?
  const R ex = exp_r(x - m), ey = exp_r(y - m);
  constexpr R eps = sizeof(R) == 8 ? R(8.8817841970012523e-16) : R(9.5367431640625e-07);  // 2^-50, 2^-20
  constexpr R tiny = sizeof(R) == 8 ? R(2.2250738585072014e-308) : R(1.17549435e-38f);
  if (ey == R(0)) return ex >= tiny;  // p(x) = ex / sum (sum <= T) cannot underflow to 0
  return ex > ey * (R(1) + eps);
}

// position of the n-th (0-based) set bit of m
__device__ __forceinline__ int nth_set_bit(uint64_t m, int n) {
  const uint32_t lo = uint32_t(m);
  const int c = __popc(lo);
  if (n < c) return int(__fns(lo, 0, n + 1));
  return 32 + int(__fns(uint32_t(m >> 32), 0, n - c + 1));
}

// EPL > 0: the row lives in registers (EPL = T / 32 rounded up, compile-time: T <= 512);
// EPL == 0: in shared memory (T <= 2048).  Element j = 32 r + lane either way.
#define SLAB_RANK_FOR(r) _Pragma("unroll (EPL > 0 ? EPL : 1)") for (int r = 0; r < (EPL > 0 ? EPL : E); ++r)
template <typename R, int EPL>
__global__ void __launch_bounds__(256, (EPL > 8 || EPL == 0) ? 2 : 3) k_classify_rank(const R* __restrict__ scores, long long rows, int Tn,
                                                       int n1, int n_neg, int8_t* __restrict__ labels,
                                                       int* __restrict__ crit_cnt, int* __restrict__ crit_idx,
                                                       int* __restrict__ marg_cnt, double* __restrict__ p_c_out,
                                                       __nv_bfloat16* __restrict__ m0, int m0_ld,
                                                       int* __restrict__ exact_rows) {
  pdl_entry();  // launched by launch_pdl
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int E = EPL > 0 ? EPL : (Tn + 31) >> 5;  // elements per lane (<= 64)
  const int Tp = E * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  R* v = reinterpret_cast<R*>(smem_raw) + (size_t)warp * Tp;  // the row (EPL == 0) / exact-path scratch
  const long long row = (long long)blockIdx.x * 8 + warp;
  if (row >= rows) return;
  constexpr unsigned FULL = 0xffffffffu;
  const R* srow = scores + row * Tn;
  R key[EPL > 0 ? EPL : 1] = {};
  auto val = [&](int r) -> R {
    if constexpr (EPL > 0) return key[r];
    else return v[32 * r + lane];
  };
  auto set = [&](int r, R x) {
    if constexpr (EPL > 0) key[r] = x;
    else v[32 * r + lane] = x;
  };
  uint64_t valid = 0;
  R m = -R(INFINITY);
  SLAB_RANK_FOR(r) {
    const int j = 32 * r + lane;
    const R x = j < Tn ? srow[j] : -R(INFINITY);
    set(r, x);
    if (j < Tn) {
      valid |= uint64_t(1) << r;
      m = x > m ? x : m;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const R other = __shfl_xor_sync(FULL, m, o);
    m = other > m ? other : m;
  }
  __syncwarp();
  // The value at 0-based rank K of the valid entries (descending), with #(>) and #(==).  The
  // first step brackets rank K between two quantiles of a 32-entry sample (one per lane, sorted
  // across the warp); then quickselect with pivots drawn from the remaining candidates.
  auto select_desc = [&](int K, int& gt, int& eq) -> R {
    uint64_t cm = valid;
    int k = K, base_gt = 0;
    {
      R smp = (valid & 1u) ? val(0) : -R(INFINITY);
#pragma unroll
      for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          const R o = __shfl_xor_sync(FULL, smp, jj);
          const bool keep_max = ((lane & jj) == 0) == ((lane & kk) == 0);
          smp = keep_max ? (o > smp ? o : smp) : (o < smp ? o : smp);
        }
      const int q = int((long long)K * 32 / Tn);
      const R hi = __shfl_sync(FULL, smp, q > 1 ? q - 2 : 0);
      const R lo = __shfl_sync(FULL, smp, q < 29 ? q + 2 : 31);
      uint64_t gm = 0, bm = 0;
      SLAB_RANK_FOR(r) {
        const R x = val(r);
        gm |= uint64_t(x > hi) << r;
        bm |= uint64_t(x >= lo && x <= hi) << r;
      }
      gm &= cm;
      bm &= cm;
      const int g = __reduce_add_sync(FULL, __popcll(gm));
      const int b = __reduce_add_sync(FULL, __popcll(bm));
      if (k < g) {
        cm = gm;
      } else if (k < g + b) {
        cm = bm;
        k -= g;
        base_gt = g;
      } else {
        cm &= ~(gm | bm);
        k -= g + b;
        base_gt = g + b;
      }
    }
    for (int it = 0;; ++it) {
      const unsigned has = __ballot_sync(FULL, cm != 0u);
      if (has == 0u) {  // only with non-finite scores: never hang
        gt = eq = 0;
        return -R(INFINITY);
      }
      const int rot = (it * 11) & 31;
      const unsigned rm = rot ? (has >> rot) | (has << (32 - rot)) : has;
      const int src = (__ffs(rm) - 1 + rot) & 31;
      R mv = R(0);
      if (lane == src) {
        const int rr = nth_set_bit(cm, __popcll(cm) >> 1);  // the lane's median-index candidate
        if constexpr (EPL > 0) {
#pragma unroll
          for (int r = 0; r < EPL; ++r)
            if (r == rr) mv = key[r];
        } else {
          mv = v[32 * rr + lane];
        }
      }
      const R pivot = __shfl_sync(FULL, mv, src);
      uint64_t gm = 0, em = 0;
      SLAB_RANK_FOR(r) {
        const R x = val(r);
        gm |= uint64_t(x > pivot) << r;
        em |= uint64_t(x == pivot) << r;
      }
      gm &= cm;
      em &= cm;
      const int g = __reduce_add_sync(FULL, __popcll(gm));
      const int e = __reduce_add_sync(FULL, __popcll(em));
      if (k < g) {
        cm = gm;
      } else if (k < g + e) {
        gt = base_gt + g;
        eq = e;
        return pivot;
      } else {
        k -= g + e;
        base_gt += g + e;
        cm &= ~(gm | em);
      }
    }
  };
  auto max_below = [&](R a, bool& found) -> R {  // max{valid x < a}
    R best = -R(INFINITY);
    bool f = false;
    SLAB_RANK_FOR(r) {
      const R x = val(r);
      if (((valid >> r) & 1u) && x < a && (!f || x > best)) {
        best = x;
        f = true;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const R ob = __shfl_xor_sync(FULL, best, o);
      const bool of = __shfl_xor_sync(FULL, f, o);
      if (of && (!f || ob > best)) best = ob;
      f = f || of;
    }
    found = f;
    return best;
  };
  auto min_above = [&](R a) -> R {  // min{valid x > a} (the caller knows one exists)
    R best = R(INFINITY);
    SLAB_RANK_FOR(r) {
      const R x = val(r);
      if (((valid >> r) & 1u) && x > a && x < best) best = x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const R ob = __shfl_xor_sync(FULL, best, o);
      best = ob < best ? ob : best;
    }
    return best;
  };
  // ---- rank boundaries in the S domain, with the separation checks
  const int K1 = n1, K2 = Tn - n_neg;  // in-set sizes: critical, non-negligible
  int g1 = 0, e1 = 0, g2 = 0, e2 = 0;
  R A1 = R(0), A2 = R(0);
  bool exact = p_c_out != nullptr;
  auto boundary_ok = [&](int K, R A, int g, int e) -> bool {  // A = the value at rank K - 1
    if (K >= Tn) return true;  // nothing outside the set
    if (g + e > K) {           // the tie class of A straddles the boundary
      bool ok = true;
      if (g > 0) ok = g_separated(min_above(A), A, m);
      bool f;
      const R lo = max_below(A, f);
      if (f) ok = ok && g_separated(A, lo, m);
      return ok;
    }
    bool f;
    const R B = max_below(A, f);  // the value at rank K
    return !f || g_separated(A, B, m);
  };
  if (!exact) {
    A1 = select_desc(K1 - 1, g1, e1);
    exact = !boundary_ok(K1, A1, g1, e1);
    if (!exact && n_neg > 0) {
      A2 = select_desc(K2 - 1, g2, e2);
      exact = !boundary_ok(K2, A2, g2, e2);
    }
  }
  if (exact) {  // P_c exactly as the reference computes it (mask.cpp:65-79), then rank P_c
    if (exact_rows && lane == 0) atomicAdd(exact_rows, 1);
    SLAB_RANK_FOR(r) {
      const int j = 32 * r + lane;
      const R e = j < Tn ? exp_r(val(r) - m) : R(0);
      if (EPL > 0) set(r, e);
      v[j] = e;  // shared copy for the sequential normaliser
    }
    __syncwarp();
    R sum = R(0);
    if (lane == 0)  // the reference's sequential ascending normaliser (mask.cpp:73-77)
      for (int j = 0; j < Tn; ++j) sum = add_rn(sum, v[j]);
    sum = __shfl_sync(FULL, sum, 0);
    __syncwarp();
    SLAB_RANK_FOR(r) {
      const int j = 32 * r + lane;
      if (j < Tn) {
        const R p = div_rn(val(r), sum);
        set(r, p);
        if (p_c_out) p_c_out[row * Tn + j] = double(p);
      } else {
        set(r, -R(INFINITY));
      }
    }
    __syncwarp();
    A1 = select_desc(K1 - 1, g1, e1);
    if (n_neg > 0) A2 = select_desc(K2 - 1, g2, e2);
  }
  // ---- labels: in-set = {x > A} plus the first K - #(x > A) ties of A in index order; the label
  // row, the marginal indicator row (bf16 0/1, the A operand of H = M0 h) and the ascending
  // critical list are written in the same pass (element j = 32 r + lane: coalesced per r)
  int run1 = 0, run2 = 0, base = 0, marg = 0;
  const unsigned lt = (1u << lane) - 1u;
  int8_t* lrow = labels + row * Tn;
  int* crow = crit_idx + row * Tn;
  __nv_bfloat16* mrow = m0 ? m0 + row * m0_ld : nullptr;
  SLAB_RANK_FOR(r) {
    const int j = 32 * r + lane;
    const bool ok = j < Tn;
    const R x = val(r);
    const bool t1 = ok && x == A1, t2 = ok && n_neg > 0 && x == A2;
    const unsigned b1 = __ballot_sync(FULL, t1), b2 = __ballot_sync(FULL, t2);
    const bool crit = ok && (x > A1 || (t1 && run1 + __popc(b1 & lt) < K1 - g1));
    const bool keep = n_neg == 0 || x > A2 || (t2 && run2 + __popc(b2 & lt) < K2 - g2);
    run1 += __popc(b1);
    run2 += __popc(b2);
    const bool mg = ok && !crit && keep;
    if (ok) lrow[j] = crit ? int8_t(1) : (keep ? int8_t(0) : int8_t(-1));
    if (mrow && j < m0_ld) mrow[j] = __float2bfloat16_rn(mg ? 1.f : 0.f);
    const unsigned bc = __ballot_sync(FULL, crit);
    if (crit) crow[base + __popc(bc & lt)] = j;
    base += __popc(bc);
    marg += __popc(__ballot_sync(FULL, mg));
  }
  if (lane == 0) {
    crit_cnt[row] = base;
    marg_cnt[row] = marg;
  }
}
#undef SLAB_RANK_FOR

// ---------------------------------------------------------------------------------------
// build_lookup for an injected label grid (mask.cpp:121-153); flags invalid labels.
// ---------------------------------------------------------------------------------------
__global__ void k_build_lut(const int8_t* __restrict__ labels, int Tm, int Tn,
                            int* __restrict__ crit_cnt, int* __restrict__ crit_idx,
                            int* __restrict__ marg_cnt, long long* __restrict__ bad) {
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= Tm) return;
  const long long row = (long long)blockIdx.y * Tm + i;
  const int8_t* lrow = labels + row * Tn;
  int* crow = crit_idx + row * Tn;
  int base = 0, marg = 0;
  for (int j0 = 0; j0 < Tn; j0 += 32) {
    const int j = j0 + lane;
    const int l = j < Tn ? lrow[j] : -1;
    if (j < Tn && (l < -1 || l > 1) && bad) atomicMin(bad, row * Tn + j);
    const unsigned bc = __ballot_sync(0xffffffffu, l == 1);
    const unsigned bm = __ballot_sync(0xffffffffu, l == 0);
    if (l == 1) crow[base + __popc(bc & ((1u << lane) - 1u))] = j;
    base += __popc(bc);
    marg += __popc(bm);
  }
  if (lane == 0) {
    crit_cnt[row] = base;
    marg_cnt[row] = marg;
  }
}

// Transposed critical lists (backward.cpp:133-137): per column, ascending rows.
__global__ void k_build_csc(const int8_t* __restrict__ labels, int Tm, int Tn,
                            int* __restrict__ ccol_cnt, int* __restrict__ ccol_idx,
                            int* __restrict__ ccol_marg) {
  pdl_entry();  // launched by launch_pdl
  const long long u = blockIdx.y;
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= Tn) return;
  const int8_t* lu = labels + u * (long long)Tm * Tn;
  int* out = ccol_idx + (u * Tn + j) * (long long)Tm;
  int base = 0, marg = 0;
  for (int i0 = 0; i0 < Tm; i0 += 32) {
    const int i = i0 + lane;
    const int l = i < Tm ? lu[(long long)i * Tn + j] : -1;
    const unsigned b = __ballot_sync(0xffffffffu, l == 1);
    if (l == 1) out[base + __popc(b & ((1u << lane) - 1u))] = i;
    base += __popc(b);
    marg += __popc(__ballot_sync(0xffffffffu, l == 0));
  }
  if (lane == 0) {
    ccol_cnt[u * Tn + j] = base;
    ccol_marg[u * Tn + j] = marg;
  }
}

// Marginal indicator as a bf16 0/1 matrix: the A operand of H = M0 h (fast path).
__global__ void k_build_m0(const int8_t* __restrict__ labels, long long total, int Tn, int ld,
                           __nv_bfloat16* __restrict__ m0) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / ld;
    const int j = int(e % ld);
    m0[e] = __float2bfloat16_rn(j < Tn && labels[row * Tn + j] == 0 ? 1.f : 0.f);
  }
}

// ---------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------
static int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

size_t classify_smem_bytes(const Dims& D, bool f64) {
  const int P2 = next_pow2(D.Tn);
  const size_t rs = f64 ? 8 : 4;
  return rs * P2 + 4 * size_t(P2) + size_t(D.Tn) + 16;
}

template <typename In>
static void check_finite_t(const In* x, long long total, long long* slot, cudaStream_t st) {
  const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 16));
  k_check_finite<In><<<blocks, 256, 0, st>>>(x, total, slot);
  check_launch("k_check_finite", st);
}

void launch_check_finite(const Dims& D, int dtype, const void* x, long long* slot,
                         cudaStream_t st) {
  const long long total = D.U * D.N_valid * D.d;  // the caller's elements (ragged: N_valid rows)
  if (dtype == 0)
    check_finite_t(static_cast<const __nv_bfloat16*>(x), total, slot, st);
  else
    check_finite_t(static_cast<const float*>(x), total, slot, st);
}

template <typename R, typename In>
static bool classify_t(const Dims& D, const In* q, const In* k, const StateBufs& s,
                       const WorkBufs& w, double* p_c, cudaStream_t st, cudaEvent_t after_pool) {
  R* pq = reinterpret_cast<R*>(w.pq);
  R* pk = reinterpret_cast<R*>(w.pk);
  const int pt = D.d < 256 ? ((D.d + 31) / 32) * 32 : 256;
  bool pooled = false;
  if constexpr (std::is_same<In, __nv_bfloat16>::value) {
    if (D.d % 4 == 0 && D.bq == D.bkv) {
      launch_pdl(k_pool2_bf16<R>, dim3(std::max(D.Tm, D.Tn), unsigned(D.U), 2), 32, 0, st, q, k, pq, pk, D.N, D.Nk,
                 D.d, D.bq, D.Tm, D.Tn, D.N_valid, D.Nk_valid, D.rl);
      check_launch("k_pool", st);
      pooled = true;
    }
  }
  if (!pooled) {
    k_pool<R, In><<<dim3(D.Tm, unsigned(D.U)), pt, 0, st>>>(q, pq, D.N, D.d, D.bq, D.Tm, D.N_valid, D.rl);
    check_launch("k_pool(q)", st);
    k_pool<R, In><<<dim3(D.Tn, unsigned(D.U)), pt, 0, st>>>(k, pk, D.Nk, D.d, D.bkv, D.Tn, D.Nk_valid, D.rl);
    check_launch("k_pool(k)", st);
  }
  if (after_pool) SLAB_CUDA(cudaEventRecord(after_pool, st));  // (the caller forks its side stream here)
  const size_t smem = classify_smem_bytes(D, sizeof(R) == 8);
  if (smem > 48 * 1024)
    SLAB_CUDA(cudaFuncSetAttribute(k_classify<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
  R* scores = reinterpret_cast<R*>(w.p_c);
  const int scores_smem = int(sizeof(R)) * 4 * 64 * 33;
  SLAB_CUDA(cudaFuncSetAttribute(k_scores<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, scores_smem));
  launch_pdl(k_scores<R>, dim3((D.Tn + 63) / 64, (D.Tm + 63) / 64, unsigned(D.U)), 128, scores_smem, st,
             (const R*)pq, (const R*)pk, D.d, D.Tm, D.Tn, R(D.inv_sqrt_d), scores);
  check_launch("k_scores", st);
  const int P2 = next_pow2(D.Tn);
  const long long rows = D.U * (long long)D.Tm;
  const unsigned wblocks = unsigned((rows + 7) / 8);
  if (SLAB_CLASSIFY_RANK && D.Tn <= 2048) {  // rank the raw scores (exact P_c only where needed)
    const int E = (D.Tn + 31) / 32;  // the row in registers up to T = 512 (EPL = E rounded up to 2^k)
    auto go = [&](auto kern, int epl) {
      const size_t rsm = size_t(8) * 32 * (epl > 0 ? epl : E) * (sizeof(R) + 1);  // as the kernel carves it
      SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rsm)));
      launch_pdl(kern, wblocks, 256, rsm, st, (const R*)scores, rows, D.Tn, D.n1, D.n_neg, s.labels, s.crit_cnt,
                 s.crit_idx, s.marg_cnt, p_c, s.M0, int(m0_stride(D)), classify_exact_counter());
      check_launch("k_classify", st);
    };
    if (E <= 1) go(k_classify_rank<R, 1>, 1);
    else if (E <= 2) go(k_classify_rank<R, 2>, 2);
    else if (E <= 4) go(k_classify_rank<R, 4>, 4);
    else if (E <= 8) go(k_classify_rank<R, 8>, 8);
    else if (E <= 16) go(k_classify_rank<R, 16>, 16);
    else go(k_classify_rank<R, 0>, 0);
    return true;
  }
  auto warp_rows = [&](auto kern) {
    launch_pdl(kern, wblocks, 256, 0, st, (const R*)scores, rows, D.Tn, D.n1, D.n_neg, s.labels, s.crit_cnt,
               s.crit_idx, s.marg_cnt, p_c, s.M0, int(m0_stride(D)));
    check_launch("k_classify", st);
  };
  switch (P2) {  // one warp per block row while a row fits 16 registers per lane
    case 32: warp_rows(k_classify_warp<R, 1>); return true;
    case 64: warp_rows(k_classify_warp<R, 2>); return true;
    case 128: warp_rows(k_classify_warp<R, 4>); return true;
    case 256: warp_rows(k_classify_warp<R, 8>); return true;
    case 512: warp_rows(k_classify_warp<R, 16>); return true;
    default: break;
  }
  k_classify<R><<<dim3(D.Tm, unsigned(D.U)), 256, smem, st>>>(
      scores, D.Tm, D.Tn, P2, D.n1, D.n_neg, s.labels,
      s.crit_cnt, s.crit_idx, s.marg_cnt, p_c);
  check_launch("k_classify", st);
  return false;
}

bool launch_classify(const Dims& D, int dtype, int mask_precision, const void* q, const void* k,
                     const StateBufs& s, const WorkBufs& w, double* p_c, cudaStream_t st,
                     cudaEvent_t after_pool) {
  // the f32 variant computes 1/sqrt(d) in f32 as well
  if (dtype == 0) {
    auto qb = static_cast<const __nv_bfloat16*>(q);
    auto kb = static_cast<const __nv_bfloat16*>(k);
    if (mask_precision == 0)
      return classify_t<double>(D, qb, kb, s, w, p_c, st, after_pool);
    return classify_t<float>(D, qb, kb, s, w, p_c, st, after_pool);
  } else {
    auto qf = static_cast<const float*>(q);
    auto kf = static_cast<const float*>(k);
    if (mask_precision == 0)
      return classify_t<double>(D, qf, kf, s, w, p_c, st, after_pool);
    return classify_t<float>(D, qf, kf, s, w, p_c, st, after_pool);
  }
}

void launch_build_lut(const Dims& D, const StateBufs& s, long long* bad, cudaStream_t st) {
  const int warps = 8;
  k_build_lut<<<dim3((D.Tm + warps - 1) / warps, unsigned(D.U)), 32 * warps, 0, st>>>(
      s.labels, D.Tm, D.Tn, s.crit_cnt, s.crit_idx, s.marg_cnt, bad);
  check_launch("k_build_lut", st);
}

void launch_build_csc(const Dims& D, const StateBufs& s, cudaStream_t st) {
  const int warps = 8;
  launch_pdl(k_build_csc, dim3((D.Tn + warps - 1) / warps, unsigned(D.U)), 32 * warps, 0, st,
             (const int8_t*)s.labels, D.Tm, D.Tn, s.ccol_cnt, s.ccol_idx, s.ccol_marg);
  check_launch("k_build_csc", st);
}

void launch_build_m0(const Dims& D, const StateBufs& s, cudaStream_t st) {
  const int ld = int(m0_stride(D));
  const long long total = D.U * (long long)D.Tm * ld;
  const int blocks = int(std::min<long long>((total + 255) / 256, 148 * 8));
  k_build_m0<<<blocks, 256, 0, st>>>(s.labels, total, D.Tn, ld, s.M0);
  check_launch("k_build_m0", st);
}

}  // namespace slab
