// attn_bwd.cu -- the fused SLA backward on tcgen05, two deterministic passes that mirror the
// reference's row and column phases (backward.cpp:68-120 and 142-199); no atomics.
//
// k_bwd_rows<D>: one CTA per (unit, query block i)
//   dO^l_i = dO_i W^T (MMA), D^s, D^l row dots, x = phi(q)/den,
//   dH_i = x^T dO^l_i (MMA, written bf16 for the M0^T aggregation GEMM), dZ_i = -x^T D^l,
//   dQ^phi = (dO^l H_i^T - D^l Z_i^T) / den (MMA + epilogue),
//   sparse dQ = sum_j dS_ij K_j over the critical list (S, dP recomputed on tcgen05),
//   dq_total = J_phi(q)^T dQ^phi + dQ written once (backward.cpp:211-214).
// k_bwd_cols<D>: one CTA per (unit, key block j)
//   sparse dV_j += P^T dO_i, dK_j += dS^T Q_i over the critical rows (CSC list),
//   linear dK^phi_j = V_j dH_agg^T + dZ_agg, dV_j += phi(K_j) dH_agg (dH_agg = M0^T dH),
//   dk_total = J_phi(k)^T dK^phi + dK and dv written once.
//
// Warp roles as in the forward: warp 0 TMA, warp 1 MMA (one thread), warps 2-5 compute
// (row = 16*(warp%4) + lane for M=64 tiles).
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

__device__ long long g_bwd_ts[128];  // debug timeline of one CTA (sla_b200_diag_bwd_timeline)

namespace {

__device__ __forceinline__ void ts_mark(bool on, int slot) {  // -DSLAB_TIMELINE builds only
#ifdef SLAB_TIMELINE
  if (on) g_bwd_ts[slot] = clock64();
#else
  (void)on;
  (void)slot;
#endif
}

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(h2[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  v.x = tc::pack_bf16(f[0], f[1]);
  v.y = tc::pack_bf16(f[2], f[3]);
  v.z = tc::pack_bf16(f[4], f[5]);
  v.w = tc::pack_bf16(f[6], f[7]);
  return v;
}
// byte offset of columns [col, col+8) of row r in a K-major SW128 tile (64-column blocks of
// 8 KB); col is an element index, a multiple of 8
__device__ __forceinline__ uint32_t tile_off(int r, int col) {
  return uint32_t(col >> 6) * 8192u + tc::sw128_off(uint32_t(r), uint32_t((col >> 3) & 7));
}

struct BwdParams {
  const int* crit_cnt;
  const int* crit_idx;
  const int* marg_cnt;
  const int* ccol_cnt;
  const int* ccol_idx;
  const float* Z;      // [U, Tm, D]
  const float* lse;    // [U, N]
  const float* Ds;     // [U, N] (rows kernel writes, cols kernel reads)
  float* Ds_out;
  const __nv_bfloat16* o_s;
  const __nv_bfloat16* o_l;
  __nv_bfloat16* gH;   // [U, Tm, D, D] dH_i (rows kernel out)
  float* gZ;           // [U, Tm, D] dZ_i
  const float* gZa;    // [U, Tn, D] dZ_agg (cols kernel in)
  int* has_lin_col;    // unused
  __nv_bfloat16* dq;   // outputs
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  long long N;
  int Tm, Tn, H;
  float scale;         // 1/sqrt(D)
  float scale_log2;    // scale * log2(e)
  int phi;
  const int8_t* labels;
};

// =========================================================================================
// rows pass
// =========================================================================================
// Critical key blocks are consumed in PAIRS: a pair tile stacks K_j1 over K_j2 (128 rows per
// 64-column chunk), so S^T = [K_j1; K_j2] Q_i^T, dP^T = [V_j1; V_j2] dO_i^T and
// dQ_i^T += [K_j1; K_j2]^T dS^T are all M = 128 (or M = d) tcgen05 MMAs at full rate.  P and dS
// are elementwise given lse and D^s, so the transposed layout needs no cross-lane reductions.
template <int D>
struct RowsLayout {
  static constexpr int kT = 64 * D * 2;   // 64-row tile
  static constexpr int kP = 128 * D * 2;  // 128-row pair tile
  static constexpr int oQ = 0, oDO = kT, oDOL = 2 * kT;
  static constexpr int oDL = 3 * kT;            // [64][64] bf16: column 0 = D^l/den (N tail of dH)
  static constexpr int oRing = 3 * kT + 8192;
  static constexpr int kStage = 2 * kP;  // K pair + V pair, or W / H_i (D*D*2)
  static constexpr int kStages = 2;
  static constexpr int oDS = oRing + kStages * kStage;  // 2 x dS^T [128 kv][64 q] (16 KB); X aliases
  static constexpr int oDZ = oDS + 32768;               // floats: zs[D], lse2/ds/dls/mx/inv [64]
  static constexpr int oBar = oDZ + 4 * (D + 5 * 64);
  static constexpr int kBytes = oBar + 256 + 1024;
  static_assert(kBytes <= 232448, "smem");
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    k_bwd_rows(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
               const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
               const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmH,
               BwdParams p) {
  using L = RowsLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sDO = smem + L::oDO;
  uint8_t* sDOL = smem + L::oDOL;
  uint8_t* sDL = smem + L::oDL;
  uint8_t* sRing = smem + L::oRing;
  uint8_t* sDS = smem + L::oDS;
  uint8_t* sX = sDS;  // phi(Q) tile (bf16), dead once dH is formed; aliases the dS buffers
  float* zs = reinterpret_cast<float*>(smem + L::oDZ);  // Z_i staged in smem
  float* s_lse2 = zs + D;      // per query row: lse * log2(e)
  float* s_ds = s_lse2 + 64;   // D^s
  float* s_dls = s_ds + 64;    // D^l / den
  float* s_mx = s_dls + 64;    // softmax-phi statistics of q
  float* s_inv = s_mx + 64;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* qdo_full = bars + 0;
  constexpr int RS = L::kStages;
  uint64_t* ring_full = bars + 16;        // [RS]
  uint64_t* ring_empty = bars + 16 + RS;  // [RS]
  uint64_t* sdp_full = bars + 5;    // [2]
  uint64_t* ds_full = bars + 7;     // [2]
  uint64_t* ds_empty = bars + 9;    // [2]
  uint64_t* dol_done = bars + 11;
  uint64_t* x_ready = bars + 12;
  uint64_t* lin_done = bars + 13;
  uint64_t* dh_read = bars + 14;
  uint64_t* dq_done = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * RS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const long long u = blockIdx.y;
  const long long urow = u * p.Tm + i;
  const int cnt = p.crit_cnt[urow];
  const int* list = p.crit_idx + urow * p.Tn;
  const bool has_lin = p.marg_cnt[urow] > 0;
  const int row0 = int(u * p.N) + i * 64;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(qdo_full, 1);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(ring_full + s, 1);
        tc::mbar_init(ring_empty + s, 1);
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(sdp_full + s, 1);
        tc::mbar_init(ds_full + s, 8);
        tc::mbar_init(ds_empty + s, 1);
      }
      tc::mbar_init(dol_done, 1);
      tc::mbar_init(x_ready, 4);
      tc::mbar_init(lin_done, 1);
      tc::mbar_init(dh_read, 4);
      tc::mbar_init(dq_done, 1);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dQ^T [0,64) and dQ^phi^T [64,128) (M = D), S^T|dP^T pair buffers at 128 and 256 (M = 128);
  // the prologue's dO^l (M = 64) uses [128, 128+D), [dH|dZ] (M = D) uses [256, 256+D+64)
  const uint32_t tDQT = tmem, tQPHIT = tmem + 64, tB0 = tmem + 128, tB1 = tmem + 256;
  const int np = (cnt + 1) >> 1;  // pairs of critical blocks
  const bool dbg = blockIdx.x == 100 && blockIdx.y == 0;
  ts_mark(dbg && threadIdx.x == 0, 30);

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(qdo_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_3d(sQ + c * 8192, &tmQ, qdo_full, 64 * c, row0, 0);
        tc::tma_load_3d(sDO + c * 8192, &tmDO, qdo_full, 64 * c, row0, 0);
      }
      // warm L2 with every K/V tile this block row will stream (the ring is only two pairs deep)
      for (int t = 0; t < cnt; ++t) {
        const int kv_row = int(u * p.N) + list[t] * 64;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_prefetch_3d(&tmK, 64 * c, kv_row, 0);
          tc::tma_prefetch_3d(&tmV, 64 * c, kv_row, 0);
        }
      }
      int item = 0;
      auto acquire = [&](int bytes) -> uint8_t* {
        const int s = item % RS;
        tc::mbar_wait(ring_empty + s, ((item / RS) & 1) ^ 1);
        tc::mbar_expect_tx(ring_full + s, bytes);
        return sRing + s * L::kStage;
      };
      {
        uint8_t* dst = acquire(D * D * 2);
        const int h = int(u % p.H);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tc::tma_load_3d(dst + c * D * 128, &tmW, ring_full + (item % RS), 64 * c, h * D, 0);
        ++item;
      }
      if (has_lin) {
        uint8_t* dst = acquire(D * D * 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(dst + c * D * 128, &tmH, ring_full + (item % RS), 64 * c, int(urow * D), 0);
        ++item;
      }
      for (int pp = 0; pp < np; ++pp) {
        // an odd tail repeats its block (finite data); the compute warps zero its dS rows
        const int r1 = int(u * p.N) + list[2 * pp] * 64;
        const int r2 = int(u * p.N) + list[min(2 * pp + 1, cnt - 1)] * 64;
        uint8_t* dst = acquire(2 * L::kP);
        uint64_t* fb = ring_full + (item % RS);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_3d(dst + c * 16384, &tmK, fb, 64 * c, r1, 0);
          tc::tma_load_3d(dst + c * 16384 + 8192, &tmK, fb, 64 * c, r2, 0);
          tc::tma_load_3d(dst + L::kP + c * 16384, &tmV, fb, 64 * c, r1, 0);
          tc::tma_load_3d(dst + L::kP + c * 16384 + 8192, &tmV, fb, 64 * c, r2, 0);
        }
        ++item;
      }
    }
  } else if (warp == 1) {
    const uint32_t aQ = tc::smem_u32(sQ), aDO = tc::smem_u32(sDO), aDOL = tc::smem_u32(sDOL);
    const uint32_t aR = tc::smem_u32(sRing), aDS = tc::smem_u32(sDS);
    constexpr uint32_t id_nd_kk = tc::idesc_bf16(64, D, false, false);   // A K-major, B K-major
    constexpr uint32_t id_dh = tc::idesc_bf16(D, D + 64, true, true);    // A, B MN-major
    constexpr uint32_t id_qphit = tc::idesc_bf16(D, 64, false, false);   // H (K-major) x dO^l^T
    constexpr uint32_t id_st = tc::idesc_bf16(128, 64, false, false);    // pair x Q^T
    constexpr uint32_t id_dqt = tc::idesc_bf16(D, 64, true, true);       // pair^T x dS^T
    int item = 0;
    auto wait_item = [&]() -> uint32_t {
      const int s = item % RS;
      tc::mbar_wait(ring_full + s, (item / RS) & 1);
      tc::tc_fence_after();
      return aR + s * L::kStage;
    };
    auto kdesc = [](uint32_t base, int kk, int rows) {  // K-major tile with `rows` rows/chunk
      return tc::desc_kmajor(base + (kk >> 2) * rows * 128 + (kk & 3) * 32);
    };
    tc::mbar_wait(qdo_full, 0);
    {  // dO^l = dO W^T  -> B0
      const uint32_t sw = wait_item();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16(tB0, kdesc(aDO, kk, 64), kdesc(sw, kk, D), id_nd_kk, kk > 0);
        tc::mma_commit(ring_empty + (item % RS));
        tc::mma_commit(dol_done);
      }
      __syncwarp();
      ++item;
    }
    tc::mbar_wait(x_ready, 0);
    tc::tc_fence_after();
    if (has_lin) {
      const uint32_t sh = wait_item();
      if (lane == 0) {
        // dQ^phi^T raw = H_i (dO^l/den)^T (M = D over a, N = 64 query rows, K = D over b)
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16(tQPHIT, kdesc(sh, kk, D), kdesc(aDOL, kk, 64), id_qphit, kk > 0);
        // [dH_i | -dZ_i] = phi(Q)^T [dO^l/den | D^l/den] (M = D over a, N = D + 64, K = 64
        // rows) -> columns [128, 128 + D + 64) (B0/B1 are idle until dh_read)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::mma_bf16(tB0, tc::desc_mnmajor(aDS + kk * 2048, 8192), tc::desc_mnmajor(aDOL + kk * 2048, 8192), id_dh,
                       kk > 0);
        tc::mma_commit(ring_empty + (item % RS));
        tc::mma_commit(lin_done);
      }
      __syncwarp();
      ++item;
      tc::mbar_wait(dh_read, 0);  // B1 and the X (= dS) buffers are free again
      tc::tc_fence_after();
    }
    const int item0 = item;
    auto issue_dq = [&](int j) {  // dQ^T += [K_j1; K_j2]^T dS^T  (M = D, N = 64, K = 128)
      tc::mbar_wait(ds_full + (j & 1), (j >> 1) & 1);
      tc::tc_fence_after();
      const int it = item0 + j;
      const uint32_t sk = aR + (it % RS) * L::kStage;
      if (lane == 0) {
        const uint32_t sds = aDS + (j & 1) * 16384;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_bf16(tDQT, tc::desc_mnmajor(sk + kk * 2048, 16384), tc::desc_mnmajor(sds + kk * 2048, 16384),
                       id_dqt, (j | kk) != 0);
        tc::mma_commit(ring_empty + (it % RS));
        tc::mma_commit(ds_empty + (j & 1));
      }
      __syncwarp();
    };
    for (int t = 0; t < np; ++t) {
      const uint32_t skv = wait_item();
      ts_mark(dbg && lane == 0 && t < 16, 32 + t);
      if (lane == 0) {
        const uint32_t tb = (t & 1) ? tB1 : tB0;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          tc::mma_bf16(tb, kdesc(skv, kk, 128), kdesc(aQ, kk, 64), id_st, kk > 0);                // S^T
          tc::mma_bf16(tb + 64, kdesc(skv + L::kP, kk, 128), kdesc(aDO, kk, 64), id_st, kk > 0);  // dP^T
        }
        tc::mma_commit(sdp_full + (t & 1));
      }
      __syncwarp();
      ++item;
      if (t > 0) issue_dq(t - 1);
    }
    if (np > 0) issue_dq(np - 1);
    if (lane == 0) tc::mma_commit(dq_done);
    __syncwarp();
  } else {
    // warps 2-5 (group 0) run the per-row prologue: row r = 16*q4 + (lane & 15), column
    // half lane>>4, lanes 0-15 also own TMEM row r (M = 64 layout).  Warps 6-9 (group 1) join
    // for the pair loop (second 32-column half of every S^T/dP^T row) and the epilogue.
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int r = 16 * q4 + (lane & 15);
    const int h0 = (lane >> 4) * (D / 2);
    const bool valid = lane < 16;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const long long grow = (long long)row0 + r;
    const int tid = threadIdx.x - 64;  // 0..255
    if (grp == 0) {
    for (int a = tid; a < D; a += 128) zs[a] = has_lin ? p.Z[urow * D + a] : 0.f;
    for (int e = tid; e < 64 * 7; e += 128)  // chunks 1..7 of the D^l/den tile are zero
      *reinterpret_cast<uint4*>(sDL + tc::sw128_off(e / 7, 1 + e % 7)) = make_uint4(0, 0, 0, 0);
    named_sync(2, 128);
    tc::mbar_wait(qdo_full, 0);
    // D^s = <dO, O^s> (backward.cpp:48-58)
    float ds_r = 0.f;
#pragma unroll
    for (int c = 0; c < D / 2; c += 8) {
      float f[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(sDO + tile_off(r, h0 + c)), f);
      unpack8(*reinterpret_cast<const uint4*>(p.o_s + grow * D + h0 + c), g);
#pragma unroll
      for (int e = 0; e < 8; ++e) ds_r = fmaf(f[e], g[e], ds_r);
    }
    ds_r += __shfl_xor_sync(0xffffffffu, ds_r, 16);
    if (valid) p.Ds_out[grow] = ds_r;
    // phi(q) (feature_map.cpp:24-40) over this half row, den = phi(q) . Z_i
    float mx = 0.f, inv = 1.f;
    if (p.phi == 2) {
      mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < D / 2; c += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) mx = fmaxf(mx, f[e]);
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      float se = 0.f;
#pragma unroll
      for (int c = 0; c < D / 2; c += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) se += __expf(f[e] - mx);
      }
      se += __shfl_xor_sync(0xffffffffu, se, 16);
      inv = 1.f / se;
    }
    auto phi_of = [&](float x) { return p.phi == 2 ? __expf(x - mx) * inv : phi_elem(p.phi, x); };
    float den = 0.f;
#pragma unroll
    for (int c = 0; c < D / 2; c += 8) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        f[e] = phi_of(f[e]);
        den = fmaf(f[e], zs[h0 + c + e], den);
      }
      *reinterpret_cast<uint4*>(sX + tile_off(r, h0 + c)) = pack8(f);
    }
    den += __shfl_xor_sync(0xffffffffu, den, 16);
    const float inv_den = (has_lin && den != 0.f) ? 1.f / den : 0.f;  // den == 0 -> zero row
    // dO^l (TMEM, lanes 0-15) -> D^l = <dO^l, O^l>, sDOL = dO^l / den, sDL = D^l / den
    tc::mbar_wait(dol_done, 0);
    ts_mark(dbg && threadIdx.x == 64, 0);
    tc::tc_fence_after();
    float dl_r = 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t a[32];
      tc::tmem_ld32(tB0 + lane_base + c0, a);
      tc::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float f[8], g[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * c + e]);
          unpack8(*reinterpret_cast<const uint4*>(p.o_l + grow * D + c0 + 8 * c), g);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            dl_r = fmaf(f[e], g[e], dl_r);
            f[e] *= inv_den;
          }
          *reinterpret_cast<uint4*>(sDOL + tile_off(r, c0 + 8 * c)) = pack8(f);
        }
      }
    }
    const float dls = dl_r * inv_den;  // D^l / den
    if (valid) {
      *reinterpret_cast<uint4*>(sDL + tc::sw128_off(r, 0)) = make_uint4(tc::pack_bf16(dls, 0.f), 0, 0, 0);
      s_lse2[r] = p.lse[grow] * 1.4426950408889634f;
      s_ds[r] = ds_r;
      s_dls[r] = dls;
      s_mx[r] = mx;
      s_inv[r] = inv;
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(x_ready);
    ts_mark(dbg && threadIdx.x == 64, 1);
    // dH_i (bf16, for the M0^T aggregation GEMM) and dZ_i = -(column D of the product)
    __nv_bfloat16* gHi = p.gH + urow * D * D;
    if (has_lin) {
      tc::mbar_wait(lin_done, 0);
      tc::tc_fence_after();
      const int arow = D == 128 ? 32 * q4 + lane : 16 * q4 + lane;
      const bool avalid = D == 128 || lane < 16;
#pragma unroll 1
      for (int c0 = 0; c0 < D + 32; c0 += 32) {
        uint32_t a[32];
        tc::tmem_ld32(tB0 + lane_base + c0, a);
        tc::tmem_ld_wait();
        if (!avalid) continue;
        if (c0 == D) {
          p.gZ[urow * D + arow] = -__uint_as_float(a[0]);
          continue;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * c + e]);
          *reinterpret_cast<uint4*>(gHi + arow * D + c0 + 8 * c) = pack8(f);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(dh_read);
      ts_mark(dbg && threadIdx.x == 64, 2);
    } else {
      for (int e = tid; e < D * D / 8; e += 128) reinterpret_cast<uint4*>(gHi)[e] = make_uint4(0, 0, 0, 0);
      for (int a = tid; a < D; a += 128) p.gZ[urow * D + a] = 0.f;
    }
    }  // group 0 prologue
    named_sync(1, 256);  // per-row staging visible to every compute thread
    ts_mark(dbg && threadIdx.x == 64, 3);
    // sparse dQ over pairs: thread = key row c of the pair (c < 64: block j1, else j2);
    // dS^T[c][r] = P (dP^T - D^s_r) / sqrt(d), P = exp(S^T/sqrt(d) - lse_r)
    const int c = 32 * q4 + lane;
#pragma unroll 1
    for (int t = 0; t < np; ++t) {
      tc::mbar_wait(sdp_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 64 + t);
      const bool live = c < 64 || 2 * t + 1 < cnt;
      const uint32_t tb = ((t & 1) ? tB1 : tB0) + lane_base + 32 * grp;
      uint32_t pk[16];
      {
        uint32_t sv[32], dp[32];
        tc::tmem_ld32(tb, sv);
        tc::tmem_ld32(tb + 64, dp);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int rr = 32 * grp + e;
          const float p0 = ex2f(__uint_as_float(sv[e]) * p.scale_log2 - s_lse2[rr]);
          const float p1 = ex2f(__uint_as_float(sv[e + 1]) * p.scale_log2 - s_lse2[rr + 1]);
          const float d0 = live ? p0 * (__uint_as_float(dp[e]) - s_ds[rr]) * p.scale : 0.f;
          const float d1 = live ? p1 * (__uint_as_float(dp[e + 1]) - s_ds[rr + 1]) * p.scale : 0.f;
          pk[e >> 1] = tc::pack_bf16(d0, d1);
        }
      }
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 80 + t);
      if (t >= 2) tc::mbar_wait(ds_empty + (t & 1), ((t - 2) >> 1) & 1);
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 96 + t);
      uint8_t* drow = sDS + (t & 1) * 16384;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        *reinterpret_cast<uint4*>(drow + tc::sw128_off(c, 4 * grp + ch)) =
            make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ds_full + (t & 1));
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 4 + t);
    }
    // dq_total = J_phi(q)^T dQ^phi + dQ.  The accumulators are transposed (lane = column a);
    // stage them through smem (the idle ring) as [row][a] fp32, then finish row-wise.  For the
    // softmax feature map <phi(q), dQ^phi> = D^l - (D^l/den) den = 0 exactly (O^l = phi(q) H /
    // den), so the Jacobian reduces to phi(q) * dQ^phi.
    tc::mbar_wait(dq_done, 0);
    ts_mark(dbg && threadIdx.x == 64, 20);

    tc::tc_fence_after();
    constexpr int TP = D + 4;  // padded row pitch (floats)
    float* tq = reinterpret_cast<float*>(sRing);
    float* tphi = tq + 64 * TP;
    {
      const int acol = D == 128 ? 32 * q4 + lane : 16 * q4 + lane;
      const bool avalid = D == 128 || lane < 16;
      uint32_t a[32], b[32];
      if (has_lin) tc::tmem_ld32(tQPHIT + lane_base + 32 * grp, a);
      if (cnt > 0) tc::tmem_ld32(tDQT + lane_base + 32 * grp, b);
      tc::tmem_ld_wait();
      if (avalid) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int rq = 32 * grp + e;
          tq[rq * TP + acol] = cnt > 0 ? __uint_as_float(b[e]) : 0.f;
          tphi[rq * TP + acol] = has_lin ? __uint_as_float(a[e]) : 0.f;
        }
      }
    }
    named_sync(1, 256);
    {
      const int rq = tid >> 2, c0 = (tid & 3) * (D / 4);
      const float dlsr = s_dls[rq], mxr = s_mx[rq], invr = s_inv[rq];
#pragma unroll
      for (int cc = 0; cc < D / 4; cc += 8) {
        const int col = c0 + cc;
        float x[8], o[8];
        unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(rq, col)), x);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float g = tphi[rq * TP + col + e] - dlsr * zs[col + e];
          float jg;
          if (p.phi == 2) jg = __expf(x[e] - mxr) * invr * g;
          else if (p.phi == 0) jg = x[e] >= 0.f ? g : __expf(x[e]) * g;
          else jg = x[e] > 0.f ? g : 0.f;
          o[e] = jg + tq[rq * TP + col + e];
        }
        *reinterpret_cast<uint4*>(p.dq + ((long long)row0 + rq) * D + col) = pack8(o);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

// =========================================================================================
// columns pass: critical query blocks in PAIRS (M = 128 S / dP tiles), dV^T / dK^T accumulated
// transposed (M = D) at full tensor rate; linear dK^phi^T and dV^T += dH_agg^T phi(K)^T on the
// tensor core; the epilogue transposes through smem and finishes row-wise.
// =========================================================================================
template <int D>
struct ColsLayout {
  static constexpr int kT = 64 * D * 2;    // 64-row tile
  static constexpr int kP = 128 * D * 2;   // 128-row pair tile
  static constexpr int oK = 0, oV = kT;
  static constexpr int oRing = 2 * kT;
  static constexpr int kStage = 2 * kP;    // Q pair + dO pair, or dH_agg (D*D*2)
  static constexpr int kStages = 2;
  static constexpr int oPD = oRing + kStages * kStage;  // 2 x [P 16 KB | dS 16 KB]; phi(K) aliases
  static constexpr int oZA = oPD + 65536;               // float [D] dZ_agg
  static constexpr int oBar = oZA + 4 * D;
  static constexpr int kBytes = oBar + 256 + 1024;
  static_assert(kBytes <= 232448, "smem");
};

template <int D>
__global__ void __launch_bounds__(320, 1)
    k_bwd_cols(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
               const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
               const __grid_constant__ CUtensorMap tmHa, BwdParams p) {
  using L = ColsLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + L::oK;
  uint8_t* sV = smem + L::oV;
  uint8_t* sRing = smem + L::oRing;
  uint8_t* sPD = smem + L::oPD;
  uint8_t* sKF = sPD;  // phi(K_j), written once the accumulation MMAs have drained the P/dS buffers
  float* zas = reinterpret_cast<float*>(smem + L::oZA);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  constexpr int RS = L::kStages;
  uint64_t* kv_full = bars + 0;
  uint64_t* sdp_full = bars + 1;   // [2]
  uint64_t* pd_full = bars + 3;    // [2]
  uint64_t* pd_empty = bars + 5;   // [2]
  uint64_t* acc_done = bars + 7;
  uint64_t* kf_ready = bars + 8;
  uint64_t* all_done = bars + 9;
  uint64_t* ring_full = bars + 16;        // [RS]
  uint64_t* ring_empty = bars + 16 + RS;  // [RS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * RS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x;
  const long long u = blockIdx.y;
  const long long ucol = u * p.Tn + j;
  const int cnt = p.ccol_cnt[ucol];
  const int np = (cnt + 1) >> 1;
  const int* list = p.ccol_idx + ucol * p.Tm;
  __shared__ int s_lin;
  if (threadIdx.x == 0) s_lin = 0;
  __syncthreads();
  {
    const int8_t* lu = p.labels + u * (long long)p.Tm * p.Tn;
    int any = 0;
    for (int ii = threadIdx.x; ii < p.Tm; ii += blockDim.x) any |= lu[(long long)ii * p.Tn + j] == 0;
    if (any) s_lin = 1;
  }
  __syncthreads();
  const bool has_lin = s_lin != 0;
  const int kv0 = int(u * p.N) + j * 64;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(kv_full, 1);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(ring_full + s, 1);
        tc::mbar_init(ring_empty + s, 1);
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(sdp_full + s, 1);
        tc::mbar_init(pd_full + s, 8);
        tc::mbar_init(pd_empty + s, 1);
      }
      tc::mbar_init(acc_done, 1);
      tc::mbar_init(kf_ready, 8);
      tc::mbar_init(all_done, 1);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dV^T [0,64), dK^T [64,128) (M = D); S|dP pair buffers at 128 and 256 (M = 128);
  // dK^phi^T at [384, 448) (M = D)
  const uint32_t tDVT = tmem, tDKT = tmem + 64, tB0 = tmem + 128, tB1 = tmem + 256, tKPT = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(kv_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_3d(sK + c * 8192, &tmK, kv_full, 64 * c, kv0, 0);
        tc::tma_load_3d(sV + c * 8192, &tmV, kv_full, 64 * c, kv0, 0);
      }
      for (int t = 0; t < cnt; ++t) {  // warm L2 with every Q / dO tile of this column
        const int q_row = int(u * p.N) + list[t] * 64;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_prefetch_3d(&tmQ, 64 * c, q_row, 0);
          tc::tma_prefetch_3d(&tmDO, 64 * c, q_row, 0);
        }
      }
      int item = 0;
      auto acquire = [&](int bytes) -> uint8_t* {
        const int s = item % RS;
        tc::mbar_wait(ring_empty + s, ((item / RS) & 1) ^ 1);
        tc::mbar_expect_tx(ring_full + s, bytes);
        return sRing + s * L::kStage;
      };
      for (int pp = 0; pp < np; ++pp) {
        const int r1 = int(u * p.N) + list[2 * pp] * 64;
        const int r2 = int(u * p.N) + list[min(2 * pp + 1, cnt - 1)] * 64;
        uint8_t* dst = acquire(2 * L::kP);
        uint64_t* fb = ring_full + (item % RS);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_3d(dst + c * 16384, &tmQ, fb, 64 * c, r1, 0);
          tc::tma_load_3d(dst + c * 16384 + 8192, &tmQ, fb, 64 * c, r2, 0);
          tc::tma_load_3d(dst + L::kP + c * 16384, &tmDO, fb, 64 * c, r1, 0);
          tc::tma_load_3d(dst + L::kP + c * 16384 + 8192, &tmDO, fb, 64 * c, r2, 0);
        }
        ++item;
      }
      if (has_lin) {
        uint8_t* dst = acquire(D * D * 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(dst + c * D * 128, &tmHa, ring_full + (item % RS), 64 * c, int(ucol * D), 0);
        ++item;
      }
    }
  } else if (warp == 1) {
    const uint32_t aK = tc::smem_u32(sK), aV = tc::smem_u32(sV), aKF = tc::smem_u32(sKF);
    const uint32_t aR = tc::smem_u32(sRing), aPD = tc::smem_u32(sPD);
    constexpr uint32_t id_s = tc::idesc_bf16(128, 64, false, false);   // pair x K^T
    constexpr uint32_t id_acc = tc::idesc_bf16(D, 64, true, true);     // pair^T x P
    constexpr uint32_t id_kp = tc::idesc_bf16(D, 64, false, false);    // dH_agg x V^T
    constexpr uint32_t id_vl = tc::idesc_bf16(D, 64, true, false);     // dH_agg^T x phi(K)^T
    int item = 0;
    auto wait_item = [&]() -> uint32_t {
      const int s = item % RS;
      tc::mbar_wait(ring_full + s, (item / RS) & 1);
      tc::tc_fence_after();
      return aR + s * L::kStage;
    };
    auto kdesc = [](uint32_t base, int kk, int rows) {
      return tc::desc_kmajor(base + (kk >> 2) * rows * 128 + (kk & 3) * 32);
    };
    tc::mbar_wait(kv_full, 0);
    tc::tc_fence_after();
    auto issue_acc = [&](int t) {  // dV^T += dO_pair^T P, dK^T += Q_pair^T dS  (M = D, K = 128)
      tc::mbar_wait(pd_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t sq = aR + (t % RS) * L::kStage;
      if (lane == 0) {
        const uint32_t sp = aPD + (t & 1) * 32768, sd = sp + 16384;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          tc::mma_bf16(tDVT, tc::desc_mnmajor(sq + L::kP + kk * 2048, 16384), tc::desc_mnmajor(sp + kk * 2048, 16384),
                       id_acc, (t | kk) != 0);
          tc::mma_bf16(tDKT, tc::desc_mnmajor(sq + kk * 2048, 16384), tc::desc_mnmajor(sd + kk * 2048, 16384),
                       id_acc, (t | kk) != 0);
        }
        tc::mma_commit(ring_empty + (t % RS));
        tc::mma_commit(pd_empty + (t & 1));
      }
      __syncwarp();
    };
    for (int t = 0; t < np; ++t) {
      const uint32_t sq = wait_item();
      if (lane == 0) {
        const uint32_t tb = (t & 1) ? tB1 : tB0;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          tc::mma_bf16(tb, kdesc(sq, kk, 128), kdesc(aK, kk, 64), id_s, kk > 0);                // S
          tc::mma_bf16(tb + 64, kdesc(sq + L::kP, kk, 128), kdesc(aV, kk, 64), id_s, kk > 0);   // dP
        }
        tc::mma_commit(sdp_full + (t & 1));
      }
      __syncwarp();
      ++item;
      if (t > 0) issue_acc(t - 1);
    }
    if (np > 0) issue_acc(np - 1);
    if (lane == 0) tc::mma_commit(acc_done);
    __syncwarp();
    if (has_lin) {
      const uint32_t sh = wait_item();
      tc::mbar_wait(kf_ready, 0);
      tc::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          // dK^phi^T raw = dH_agg V^T (M = D over a, N = 64 keys, K = D over b)
          tc::mma_bf16(tKPT, kdesc(sh, kk, D), kdesc(aV, kk, 64), id_kp, kk > 0);
          // dV^T += dH_agg^T phi(K)^T (M = D over b, N = 64 keys, K = D over a)
          tc::mma_bf16(tDVT, tc::desc_mnmajor(sh + kk * 2048, D * 128), kdesc(aKF, kk, 64), id_vl,
                       (np > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(ring_empty + (item % RS));
      }
      __syncwarp();
      ++item;
    }
    if (lane == 0) tc::mma_commit(all_done);
    __syncwarp();
  } else {
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const int tid = threadIdx.x - 64;  // 0..255
    for (int a = tid; a < D; a += 256) zas[a] = has_lin ? p.gZa[ucol * D + a] : 0.f;
    // ---- loop: thread = query row rq of the pair (S / dP lanes), 32 key columns per group
    const int rq = 32 * q4 + lane;
    for (int t = 0; t < np; ++t) {
      const bool live = rq < 64 || 2 * t + 1 < cnt;
      const long long qrow = u * p.N + (long long)list[min(2 * t + (rq >> 6), cnt - 1)] * 64 + (rq & 63);
      const float lse2 = p.lse[qrow] * 1.4426950408889634f;
      const float dsr = p.Ds[qrow];
      tc::mbar_wait(sdp_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t tb = ((t & 1) ? tB1 : tB0) + lane_base + 32 * grp;
      uint32_t pp[16], dd[16];
      {
        uint32_t sv[32], dp[32];
        tc::tmem_ld32(tb, sv);
        tc::tmem_ld32(tb + 64, dp);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float p0 = ex2f(__uint_as_float(sv[e]) * p.scale_log2 - lse2);
          float p1 = ex2f(__uint_as_float(sv[e + 1]) * p.scale_log2 - lse2);
          float d0 = p0 * (__uint_as_float(dp[e]) - dsr) * p.scale;
          float d1 = p1 * (__uint_as_float(dp[e + 1]) - dsr) * p.scale;
          if (!live) p0 = p1 = d0 = d1 = 0.f;
          pp[e >> 1] = tc::pack_bf16(p0, p1);
          dd[e >> 1] = tc::pack_bf16(d0, d1);
        }
      }
      if (t >= 2) tc::mbar_wait(pd_empty + (t & 1), ((t - 2) >> 1) & 1);
      uint8_t* prow = sPD + (t & 1) * 32768;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        *reinterpret_cast<uint4*>(prow + tc::sw128_off(rq, 4 * grp + ch)) =
            make_uint4(pp[4 * ch], pp[4 * ch + 1], pp[4 * ch + 2], pp[4 * ch + 3]);
        *reinterpret_cast<uint4*>(prow + 16384 + tc::sw128_off(rq, 4 * grp + ch)) =
            make_uint4(dd[4 * ch], dd[4 * ch + 1], dd[4 * ch + 2], dd[4 * ch + 3]);
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(pd_full + (t & 1));
    }
    // ---- phi(K_j) rows (4 threads per key row, D/4 columns each): statistics + the bf16 tile
    tc::mbar_wait(kv_full, 0);  // K_j must have landed even when no critical row came by
    const int c = tid >> 2, c0 = (tid & 3) * (D / 4);
    float mx = 0.f, inv = 1.f;
    if (p.phi == 2) {
      mx = -INFINITY;
#pragma unroll
      for (int cc = 0; cc < D / 4; cc += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(c, c0 + cc)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) mx = fmaxf(mx, f[e]);
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      float se = 0.f;
#pragma unroll
      for (int cc = 0; cc < D / 4; cc += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(c, c0 + cc)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) se += __expf(f[e] - mx);
      }
      se += __shfl_xor_sync(0xffffffffu, se, 1);
      se += __shfl_xor_sync(0xffffffffu, se, 2);
      inv = 1.f / se;
    }
    auto phi_of = [&](float x) { return p.phi == 2 ? __expf(x - mx) * inv : phi_elem(p.phi, x); };
    tc::mbar_wait(acc_done, 0);  // the P / dS buffers are free
    if (has_lin) {
#pragma unroll
      for (int cc = 0; cc < D / 4; cc += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(c, c0 + cc)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = phi_of(f[e]);
        *reinterpret_cast<uint4*>(sKF + tile_off(c, c0 + cc)) = pack8(f);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(kf_ready);
    }
    tc::mbar_wait(all_done, 0);
    tc::tc_fence_after();
    // ---- transpose dK^T, dV^T, dK^phi^T (lane = column a) into smem [key row][a]
    constexpr int TP = D + 4;
    float* tk = reinterpret_cast<float*>(sRing);
    float* tv = tk + 64 * TP;
    float* tkp = tv + 64 * TP;
    {
      const int acol = D == 128 ? 32 * q4 + lane : 16 * q4 + lane;
      const bool avalid = D == 128 || lane < 16;
      uint32_t a[32], b[32], e3[32];
      if (np > 0) tc::tmem_ld32(tDKT + lane_base + 32 * grp, a);
      if (np > 0 || has_lin) tc::tmem_ld32(tDVT + lane_base + 32 * grp, b);
      if (has_lin) tc::tmem_ld32(tKPT + lane_base + 32 * grp, e3);
      tc::tmem_ld_wait();
      if (avalid) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int kr = 32 * grp + e;
          tk[kr * TP + acol] = np > 0 ? __uint_as_float(a[e]) : 0.f;
          tv[kr * TP + acol] = (np > 0 || has_lin) ? __uint_as_float(b[e]) : 0.f;
          tkp[kr * TP + acol] = has_lin ? __uint_as_float(e3[e]) : 0.f;
        }
      }
    }
    named_sync(1, 256);
    // ---- dk_total = J_phi(k)^T (dK^phi + dZ_agg) + dK ; dv  (row-wise, 4 threads per row)
    float dot = 0.f;
    if (p.phi == 2 && has_lin) {
#pragma unroll
      for (int cc = 0; cc < D / 4; cc += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(c, c0 + cc)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot = fmaf(phi_of(f[e]), tkp[c * TP + c0 + cc + e] + zas[c0 + cc + e], dot);
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      dot += __shfl_xor_sync(0xffffffffu, dot, 2);
    }
    const long long grow = (long long)kv0 + c;
#pragma unroll
    for (int cc = 0; cc < D / 4; cc += 8) {
      const int col = c0 + cc;
      float f[8], o[8], w8[8];
      unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(c, col)), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float g = has_lin ? tkp[c * TP + col + e] + zas[col + e] : 0.f;
        float jg;
        if (p.phi == 2) jg = phi_of(f[e]) * (g - dot);
        else if (p.phi == 0) jg = f[e] >= 0.f ? g : __expf(f[e]) * g;
        else jg = f[e] > 0.f ? g : 0.f;
        o[e] = jg + tk[c * TP + col + e];
        w8[e] = tv[c * TP + col + e];
      }
      *reinterpret_cast<uint4*>(p.dk + grow * D + col) = pack8(o);
      *reinterpret_cast<uint4*>(p.dv + grow * D + col) = pack8(w8);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int D>
void launch_rows_t(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                   const void* d_out, const __nv_bfloat16* Hb, BwdParams p, cudaStream_t st) {
  CUtensorMap tq, tdo, tk, tv, tw, th;
  const uint64_t rows = uint64_t(Dm.U) * Dm.N;
  make_tmap_bf16(&tq, q, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tdo, d_out, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tk, k, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tv, v, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tw, w, D, uint64_t(Dm.H) * D, 1, D, 0, D);
  make_tmap_bf16(&th, Hb, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);
  auto kern = k_bwd_rows<D>;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RowsLayout<D>::kBytes));
  kern<<<dim3(Dm.Tm, unsigned(Dm.U)), 320, RowsLayout<D>::kBytes, st>>>(tq, tdo, tk, tv, tw, th, p);
  check_launch("k_bwd_rows", st);
}

template <int D>
void launch_cols_t(const Dims& Dm, const void* q, const void* k, const void* v, const void* d_out,
                   const __nv_bfloat16* Ha, BwdParams p, cudaStream_t st) {
  CUtensorMap tq, tdo, tk, tv, th;
  const uint64_t rows = uint64_t(Dm.U) * Dm.N;
  make_tmap_bf16(&tq, q, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tdo, d_out, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tk, k, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tv, v, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&th, Ha, D, uint64_t(Dm.U) * Dm.Tn * D, 1, D, 0, D);
  auto kern = k_bwd_cols<D>;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ColsLayout<D>::kBytes));
  kern<<<dim3(Dm.Tn, unsigned(Dm.U)), 320, ColsLayout<D>::kBytes, st>>>(tq, tdo, tk, tv, th, p);
  check_launch("k_bwd_cols", st);
}

}  // namespace

void launch_bwd_rows(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                     const void* o_s, const void* o_l, const float* lse, const void* d_out, void* dq,
                     const StateBufs& s, __nv_bfloat16* gH, float* gZ, float* Ds, cudaStream_t st) {
  BwdParams p{};
  p.crit_cnt = s.crit_cnt;
  p.crit_idx = s.crit_idx;
  p.marg_cnt = s.marg_cnt;
  p.Z = s.Z;
  p.lse = lse;
  p.Ds_out = Ds;
  p.o_s = static_cast<const __nv_bfloat16*>(o_s);
  p.o_l = static_cast<const __nv_bfloat16*>(o_l);
  p.gH = gH;
  p.gZ = gZ;
  p.dq = static_cast<__nv_bfloat16*>(dq);
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.scale = float(Dm.inv_sqrt_d);
  p.scale_log2 = float(Dm.inv_sqrt_d * 1.4426950408889634);
  p.phi = Dm.phi;
  if (Dm.d == 128)
    launch_rows_t<128>(Dm, q, k, v, w, d_out, s.Hb, p, st);
  else
    launch_rows_t<64>(Dm, q, k, v, w, d_out, s.Hb, p, st);
}

void launch_bwd_cols(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                     const void* d_out, void* dk, void* dv, const StateBufs& s,
                     const __nv_bfloat16* Ha, const float* gZa, const float* Ds, cudaStream_t st) {
  BwdParams p{};
  p.ccol_cnt = s.ccol_cnt;
  p.ccol_idx = s.ccol_idx;
  p.labels = s.labels;
  p.lse = lse;
  p.Ds = Ds;
  p.gZa = gZa;
  p.dk = static_cast<__nv_bfloat16*>(dk);
  p.dv = static_cast<__nv_bfloat16*>(dv);
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.scale = float(Dm.inv_sqrt_d);
  p.scale_log2 = float(Dm.inv_sqrt_d * 1.4426950408889634);
  p.phi = Dm.phi;
  if (Dm.d == 128)
    launch_cols_t<128>(Dm, q, k, v, d_out, Ha, p, st);
  else
    launch_cols_t<64>(Dm, q, k, v, d_out, Ha, p, st);
}

}  // namespace slab

extern "C" int sla_b200_diag_bwd_timeline(long long* host32) {
  return cudaMemcpyFromSymbol(host32, slab::g_bwd_ts, 128 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
