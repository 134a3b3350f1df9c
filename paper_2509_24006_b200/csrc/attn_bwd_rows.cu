// attn_bwd_rows.cu -- the ROW phase of the SLA backward (backward.cpp:46-120, 211-214) as two
// tcgen05 kernels:
//
// k_bwd_lin<D>: one CTA per (unit, query block i), 2 CTAs / SM, 8 compute warps -- the linear branch
//   dO^l_i = dO_i W^T (MMA, backward.cpp:12-22), D^s, D^l (backward.cpp:48-58),
//   x = phi(q), den = phi(q) . Z_i, [dH_i | -dZ_i] = x^T [dO^l/den | D^l/den] (one MMA),
//   dQ^phi^T = H_i (dO^l/den)^T (MMA) - (D^l/den) Z_i  (backward.cpp:70-95).
//   Outputs: D^s, dH_i (bf16, for the M0^T aggregation GEMM), dZ_i, dQ^phi (bf16 rows).
// k_bwd_rows<D>: one CTA per (unit, query block i), 1 CTA / SM -- the sparse dQ
//   critical key blocks in PAIRS: S^T = [K_j1; K_j2] Q^T, dP^T = [V_j1; V_j2] dO^T (M = 128),
//   dS^T = P (dP - D^s) / sqrt(d), dQ^T += [K_j1; K_j2]^T dS^T (M = d) (backward.cpp:98-119),
//   then dq_total = J_phi(q)^T dQ^phi + dQ (backward.cpp:211-214).
//   K pairs and V pairs stream through separate rings (3 and 2 slots): V frees as soon as dP
//   is done, so the tensor pipe keeps S/dP of the next pair queued behind dQ of this one.
#include <algorithm>

#include "bwd_common.cuh"

#ifndef SLAB_ROWS_POLY
#define SLAB_ROWS_POLY 0  // every N-th exponential by ex2_poly; measured: 0 0.620 ms, 4 0.629, 2 0.653
#endif

namespace slab {
namespace {

// CW consecutive TMEM columns of this warp's lane quarter (32x32b shape)
template <int N>
__device__ __forceinline__ void tmem_ld_cw(uint32_t taddr, uint32_t (&r)[N]) {
  static_assert(N == 16 || N == 32, "16 or 32 columns");
  if constexpr (N == 32) tc::tmem_ld32(taddr, r);
  else tc::tmem_ld16(taddr, r);
}

// =========================================================================================
// linear branch
// =========================================================================================
template <int D>
struct LinLayout {
  static constexpr int kT = 64 * D * 2;
  static constexpr int oQ = 0, oDO = kT, oDOL = 2 * kT, oDL = 3 * kT, oX = 3 * kT + 8192;
  static constexpr int oWH = oX + kT;   // W, then H_i (D*D*2)
  static constexpr int oZS = oWH + D * D * 2;
  static constexpr int oRed = oZS + 4 * D + 4 * 64;  // float [5][2][64] row-sum halves
  static constexpr int oBar = oRed + 5 * 128 * 4;
  static constexpr int kBytes = oBar + 128 + 1024;
  static_assert(kBytes <= 116736, "2 CTAs / SM");
};

constexpr int kLinThreads = 64 + 256;  // TMA warp, MMA warp, 8 compute warps

template <int D>
__global__ void __launch_bounds__(kLinThreads, 2)
    k_bwd_lin(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
              const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmH,
              const __grid_constant__ CUtensorMap tmOS, const __grid_constant__ CUtensorMap tmOL,
              const __grid_constant__ CUtensorMap tmGH, BwdParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = LinLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sDO = smem + L::oDO;
  uint8_t* sDOL = smem + L::oDOL;
  uint8_t* sDL = smem + L::oDL;
  uint8_t* sX = smem + L::oX;
  uint8_t* sWH = smem + L::oWH;
  float* zs = reinterpret_cast<float*>(smem + L::oZS);
  float* s_dls = zs + D;
  float* s_red = reinterpret_cast<float*>(smem + L::oRed);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* qdo_full = bars + 0;
  uint64_t* w_full = bars + 1;
  uint64_t* w_free = bars + 2;
  uint64_t* h_full = bars + 3;
  uint64_t* dol_done = bars + 4;
  uint64_t* x_ready = bars + 5;
  uint64_t* lin_done = bars + 6;
  uint64_t* o_full = bars + 7;  // O^s -> sX and O^l -> sDOL (both consumed before being overwritten)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const long long u = blockIdx.y;
  const RowTma rt = row_tma(p.rl, u, p.N);
  const long long urow = u * p.Tm + i;
  const bool has_lin = p.marg_cnt[urow] > 0;
  const int row0 = int(u * p.N) + i * 64;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(qdo_full, 1);
      tc::mbar_init(w_full, 1);
      tc::mbar_init(w_free, 1);
      tc::mbar_init(h_full, 1);
      tc::mbar_init(dol_done, 1);
      tc::mbar_init(x_ready, 8);
      tc::mbar_init(lin_done, 1);
      tc::mbar_init(o_full, 1);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<256>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dO^l (M = 64) at [0, D); then [dH | dZ] (M = D) at [0, D + 64) and dQ^phi^T (M = D) at [192, 256)
  const uint32_t tA = tmem, tQP = tmem + 192;

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(qdo_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_rows(sQ + c * 8192, &tmQ, qdo_full, 64 * c, i * 64, rt);
        tc::tma_load_rows(sDO + c * 8192, &tmDO, qdo_full, 64 * c, i * 64, rt);
      }
      tc::mbar_expect_tx(o_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_rows(sX + c * 8192, &tmOS, o_full, 64 * c, i * 64, rt);
        tc::tma_load_rows(sDOL + c * 8192, &tmOL, o_full, 64 * c, i * 64, rt);
      }
      tc::mbar_expect_tx(w_full, D * D * 2);
      const int h = int(u % p.H);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) tc::tma_load_3d(sWH + c * D * 128, &tmW, w_full, 64 * c, h * D, 0);
      if (has_lin) {
        tc::mbar_wait(w_free, 0);
        tc::mbar_expect_tx(h_full, D * D * 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tc::tma_load_3d(sWH + c * D * 128, &tmH, h_full, 64 * c, int(urow * D), 0);
      }
    }
  } else if (warp == 1) {
    const uint32_t aDO = tc::smem_u32(sDO), aDOL = tc::smem_u32(sDOL), aX = tc::smem_u32(sX);
    const uint32_t aWH = tc::smem_u32(sWH);
    constexpr uint32_t id_dol = tc::idesc_bf16(64, D, false, false);
    constexpr uint32_t id_dh = tc::idesc_bf16(D, D + 64, true, true);
    constexpr uint32_t id_qp = tc::idesc_bf16(D, 64, false, false);
    auto kdesc = [](uint32_t base, int kk, int rows) {
      return tc::desc_kmajor(base + (kk >> 2) * rows * 128 + (kk & 3) * 32);
    };
    tc::mbar_wait(qdo_full, 0);
    tc::mbar_wait(w_full, 0);
    tc::tc_fence_after();
    // dO^l = dO W^T  (whole warp, one elected lane issues; see tc::mma_bf16_w)
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16_w(tA, kdesc(aDO, kk, 64), kdesc(aWH, kk, D), id_dol, kk > 0);
    tc::mma_commit_w(w_free);
    tc::mma_commit_w(dol_done);
    if (has_lin) {
      tc::mbar_wait(x_ready, 0);
      tc::mbar_wait(h_full, 0);
      tc::tc_fence_after();
      // dQ^phi^T raw = H_i (dO^l/den)^T  (M = D over a, N = 64 rows, K = D over b)
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16_w(tQP, kdesc(aWH, kk, D), kdesc(aDOL, kk, 64), id_qp, kk > 0);
      // [dH_i | -dZ_i] = phi(Q)^T [dO^l/den | D^l/den]  (M = D, N = D + 64, K = 64 rows)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc::mma_bf16_w(tA, tc::desc_mnmajor(aX + kk * 2048, 8192), tc::desc_mnmajor(aDOL + kk * 2048, 8192), id_dh, kk > 0);
      tc::mma_commit_w(lin_done);
    }
  } else {
    // 8 compute warps: warps w and w + 4 share TMEM lane quarter q4 (rows 16 q4 .. +15 of the
    // M = 64 layout) and split the columns; 4 threads per row, D/4 columns each
    // (quarter cq = 2 half + lane / 16).  Row sums combine lanes l / l+16 by shuffle and the two
    // warps of a pair through s_red with a 64-thread named barrier per pair.
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = 16 * q4 + (lane & 15);
    const int h0 = (2 * half + (lane >> 4)) * (D / 4);
    const bool valid = lane < 16;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const long long grow = (long long)row0 + r;
    const int tid = threadIdx.x - 64;  // 0..255
    auto pair_sum = [&](float x, int slot) {  // full-row sum of a per-thread partial
      x += __shfl_xor_sync(0xffffffffu, x, 16);
      if (valid) s_red[slot * 128 + half * 64 + r] = x;
      named_sync(2 + q4, 64);
      return s_red[slot * 128 + r] + s_red[slot * 128 + 64 + r];
    };
    auto pair_max = [&](float x, int slot) {
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 16));
      if (valid) s_red[slot * 128 + half * 64 + r] = x;
      named_sync(2 + q4, 64);
      return fmaxf(s_red[slot * 128 + r], s_red[slot * 128 + 64 + r]);
    };
    for (int a = tid; a < D; a += 256) zs[a] = has_lin ? tc::load_sum3(p.Z + urow * 3 * D + a, D) : 0.f;
    for (int e = tid; e < 64 * 7; e += 256)
      *reinterpret_cast<uint4*>(sDL + tc::sw128_off(e / 7, 1 + e % 7)) = make_uint4(0, 0, 0, 0);
    named_sync(1, 256);
    tc::mbar_wait(qdo_full, 0);
    tc::mbar_wait(o_full, 0);
    float ds_r = 0.f;
#pragma unroll
    for (int c = 0; c < D / 4; c += 8) {
      float f[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(sDO + tile_off(r, h0 + c)), f);
      unpack8(*reinterpret_cast<const uint4*>(sX + tile_off(r, h0 + c)), g);
#pragma unroll
      for (int e = 0; e < 8; ++e) ds_r = fmaf(f[e], g[e], ds_r);
    }
    ds_r = pair_sum(ds_r, 0);
    if (valid && half == 0 && !p.ds_external) p.Ds_out[grow] = ds_r;
    named_sync(1, 256);  // O^s (in sX) fully consumed before phi(Q) overwrites it
    float mx = 0.f, inv = 1.f;
    if (p.phi == 2) {
      mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < D / 4; c += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) mx = fmaxf(mx, f[e]);
      }
      mx = pair_max(mx, 1);
      float se = 0.f;
#pragma unroll
      for (int c = 0; c < D / 4; c += 8) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) se += __expf(f[e] - mx);
      }
      inv = 1.f / pair_sum(se, 2);
    }
    float den = 0.f;
#pragma unroll
    for (int c = 0; c < D / 4; c += 8) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(r, h0 + c)), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        f[e] = p.phi == 2 ? __expf(f[e] - mx) * inv : phi_elem(p.phi, f[e]);
        den = fmaf(f[e], zs[h0 + c + e], den);
      }
      *reinterpret_cast<uint4*>(sX + tile_off(r, h0 + c)) = pack8(f);
    }
    den = pair_sum(den, 3);
    const float inv_den = (has_lin && den != 0.f) ? 1.f / den : 0.f;  // den == 0 -> zero row
    tc::mbar_wait(dol_done, 0);
    tc::tc_fence_after();
    float dl_r = 0.f;
#pragma unroll 1
    for (int c0 = 32 * half; c0 < D; c0 += 64) {  // this warp's TMEM column blocks of dO^l
      uint32_t a[32];
      tc::tmem_ld32(tA + lane_base + c0, a);
      tc::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float f[8], g[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * c + e]);
          unpack8(*reinterpret_cast<const uint4*>(sDOL + tile_off(r, c0 + 8 * c)), g);  // O^l row
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            dl_r = fmaf(f[e], g[e], dl_r);
            f[e] *= inv_den;
          }
          *reinterpret_cast<uint4*>(sDOL + tile_off(r, c0 + 8 * c)) = pack8(f);  // same thread, same row
        }
      }
    }
    const float dls = pair_sum(dl_r, 4) * inv_den;  // D^l / den (lanes >= 16 contribute 0)
    if (valid && half == 0) {
      *reinterpret_cast<uint4*>(sDL + tc::sw128_off(r, 0)) = make_uint4(tc::pack_bf16(dls, 0.f), 0, 0, 0);
      s_dls[r] = dls;
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(x_ready);
    named_sync(1, 256);  // s_dls visible
    __nv_bfloat16* gHi = p.gH + urow * D * D;
    __nv_bfloat16* dqp = p.dqphi + (long long)row0 * D;
    if (has_lin) {
      tc::mbar_wait(lin_done, 0);
      tc::tc_fence_after();
      const int arow = D == 128 ? 32 * q4 + lane : 16 * q4 + lane;
      const bool avalid = D == 128 || lane < 16;
#pragma unroll 1
      for (int c0 = 32 * half; c0 < D + 32; c0 += 64) {  // [dH | -dZ] column blocks of this warp
        uint32_t a[32];
        tc::tmem_ld32(tA + lane_base + c0, a);
        tc::tmem_ld_wait();
        if (!avalid) continue;
        if (c0 == D) {
          tc::store_split3(p.z3 + urow * 3 * D + arow, D, -__uint_as_float(a[0]));
          continue;
        }
        // dH_i row arow -> SW128 staging boxes [D rows][64 cols] in the dead Q / dO tiles
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(a[8 * c + e]);
          const int col = c0 + 8 * c;
          tc::sts_u4(tc::smem_u32(sQ) + (col >> 6) * (D * 128) + tc::sw128_off(arow, (col >> 3) & 7), pack8(f));
        }
      }
      tc::fence_proxy_async();
      named_sync(1, 256);
      if (tid == 0) {  // coalesced: one TMA store per 64-column box
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tc::tma_store_3d(&tmGH, sQ + c * (D * 128), 64 * c, int(urow * D), 0);
        tc::bulk_commit();
      }
      // dQ^phi[r][a] = raw^T[a][r] - (D^l/den)_r Z[a]; stage as a row-major bf16 tile in sX
      // (phi(Q) is dead once lin_done fired), then store coalesced rows
      const float za = avalid ? zs[arow] : 0.f;
      {
        const int c0 = 32 * half;  // this warp's 32 query rows
        uint32_t a[32];
        tc::tmem_ld32(tQP + lane_base + c0, a);
        tc::tmem_ld_wait();
        if (avalid) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int rr = c0 + e;
            const float v = __uint_as_float(a[e]) - s_dls[rr] * za;
            *reinterpret_cast<__nv_bfloat16*>(sX + tile_off(rr, arow & ~7) + (arow & 7) * 2) = __float2bfloat16_rn(v);
          }
        }
      }
      named_sync(1, 256);
      for (int e = tid; e < 64 * D / 8; e += 256) {
        const int rr = e / (D / 8), cc = (e % (D / 8)) * 8;
        *reinterpret_cast<uint4*>(dqp + (long long)rr * D + cc) = *reinterpret_cast<const uint4*>(sX + tile_off(rr, cc));
      }
      if (tid == 0) tc::bulk_wait_read<0>();  // dH_i stores have read the staging smem
    } else {
      for (int e = tid; e < D * D / 8; e += 256) reinterpret_cast<uint4*>(gHi)[e] = make_uint4(0, 0, 0, 0);
      for (int a = tid; a < D; a += 256) tc::store_split3(p.z3 + urow * 3 * D + a, D, 0.f);
      for (int e = tid; e < 64 * D / 8; e += 256) reinterpret_cast<uint4*>(dqp)[e] = make_uint4(0, 0, 0, 0);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

// =========================================================================================
// sparse dQ over pairs of critical key blocks
// =========================================================================================
template <int D>
struct RowsLayout {
  static constexpr int kT = 64 * D * 2;   // 64-row tile
  static constexpr int kP = 128 * D * 2;  // 128-row pair tile
  // K-pair and V-pair ring slots (4 / 1 measured 0.85 ms, 2 / 3 0.72 ms, against 0.59 ms for 3 / 2)
  static constexpr int KS = 3, VS = 2;
  static constexpr int oQ = 0, oDO = kT, oDS = 2 * kT;  // dS^T [128 kv][64 q] bf16 (16 KB)
  static constexpr int oK = oDS + 16384;
  static constexpr int oV = oK + KS * kP;
  static constexpr int oSM = oV + VS * kP;  // floats: lse2[64], ds[64]
  static constexpr int oBar = oSM + 512;
  static constexpr int kBytes = oBar + 256 + 1024;
  static_assert(kBytes <= 232448, "smem");
};

// Warps: 0 / 10 TMA producers (K pairs, V pairs), 1 S^T/dP^T issuer, 2-9 softmax-gradient /
// epilogue, 11 dQ^T issuer.  With one issuer in a static order the pass ran 0.706 ms, with two
// 0.678 ms.
// softmax-gradient warps: 8 (32 query columns each per lane quarter) or 16 (16 columns each);
// (16 warps, for latency hiding, measured slower: TMEM-load and barrier traffic grow with them)
#ifndef SLAB_ROWS_PERSIST
#define SLAB_ROWS_PERSIST 1  // one CTA per SM walking the query blocks (0: one CTA per block)
#endif
#ifndef SLAB_ROWS_CW
#define SLAB_ROWS_CW 8  // measured: 8 warps 0.600 ms, 16 warps 0.613
#endif
constexpr int kRowsCW = SLAB_ROWS_CW;
constexpr int kRowsVWarp = 2 + kRowsCW, kRowsDQWarp = 3 + kRowsCW;  // V producer, dQ issuer
constexpr int kRowsThreads = 32 * (kRowsCW + 4);

template <int D>
__global__ void __launch_bounds__(kRowsThreads, 1)
    k_bwd_rows(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
               const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
               BwdParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = RowsLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sDO = smem + L::oDO;
  uint8_t* sDS = smem + L::oDS;
  uint8_t* sK = smem + L::oK;
  uint8_t* sV = smem + L::oV;
  float* s_lse2 = reinterpret_cast<float*>(smem + L::oSM);
  float* s_ds = s_lse2 + 64;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* qdo_full = bars + 0;
  uint64_t* sdp_full = bars + 1;   // [2]
  uint64_t* ds_full = bars + 3;
  uint64_t* ds_empty = bars + 4;
  uint64_t* dq_done = bars + 5;
  uint64_t* sdp_free = bars + 6;   // [2] compute warps have read S^T|dP^T buffer t&1 (2-issuer mode)
  uint64_t* k_full = bars + 8;               // [KS]
  uint64_t* k_empty = k_full + L::KS;        // [KS]
  uint64_t* v_full = k_empty + L::KS;        // [VS]
  uint64_t* v_empty = v_full + L::VS;        // [VS]
  uint64_t* s_full = bars + 18;    // [2] S^T(t) alone is in TMEM (P's exponentials start early)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
  static_assert(8 + 2 * (L::KS + L::VS) <= 18, "barrier slots");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent: CTA b takes the query blocks (work items) b, b + gridDim.x, ... of the [U, Tm]
  // grid (every item has the same n1 critical blocks under a dynamic mask).  Ring slots, TMEM
  // buffers and barrier phases run on G = the CTA's pairs so far (G0) + the item's pair t, so no
  // barrier is re-initialised between items; the per-item barriers (qdo_full, dq_done) take the
  // item count's parity.  With gridDim.x == items every CTA runs one item (the grid launch).
  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(qdo_full, 1);
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(sdp_full + s, 1);
        tc::mbar_init(s_full + s, 1);
        tc::mbar_init(sdp_free + s, kRowsCW);
      }
      tc::mbar_init(ds_full, kRowsCW);
      tc::mbar_init(ds_empty, 1);
      tc::mbar_init(dq_done, 1);
      for (int s = 0; s < L::KS; ++s) {
        tc::mbar_init(k_full + s, 1);
        tc::mbar_init(k_empty + s, 1);
      }
      for (int s = 0; s < L::VS; ++s) {
        tc::mbar_init(v_full + s, 1);
        tc::mbar_init(v_empty + s, 1);
      }
      tc::fence_barrier_init();
      tc::tma_prefetch(&tmK);
      tc::tma_prefetch(&tmV);
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tDQT = tmem, tB0 = tmem + 128, tB1 = tmem + 256;  // dQ^T (M = D); S^T|dP^T pairs
  int G0 = 0;  // pairs this CTA processed before the current item (32-bit: cheap % and / by constants)
  int nit = 0;       // items this CTA processed before the current one
#pragma unroll 1
  for (long long item = blockIdx.x; item < p.items; item += gridDim.x, ++nit) {
  const int i = int(item % p.Tm);
  const long long u = item / p.Tm;
  const RowTma rt = row_tma(p.rl, u, p.N);
  const RowMap rm = row_map(p.rl, u, p.N);
  const long long urow = u * p.Tm + i;
  const int cnt = p.crit_cnt[urow];
  const int* list = p.crit_idx + urow * p.Tn;
  const int np = (cnt + 1) >> 1;
  const int row0 = int(u * p.N) + i * 64;
  const int ip = nit & 1;  // parity of the per-item barriers
  const bool dbg = i == SLAB_DBG_X && u == 6;
  ts_mark(dbg && threadIdx.x == 0, 127);
  cta_mark(threadIdx.x == 0, 0, item);
  if (warp == 0) {
    if (lane == 0) {
      // Q_i / dO_i and pair 0 (K and V) now; the producer loops start at pair 1.  Pair 0's
      // slots were released by the previous item's last MMAs (all complete: dq_done).
      const int l0 = list[0], l1 = list[min(1, p.Tn - 1)];
      const int k0s = G0 % L::KS, v0s = G0 % L::VS;
      tc::mbar_expect_tx(qdo_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_rows(sQ + c * 8192, &tmQ, qdo_full, 64 * c, i * 64, rt);
        tc::tma_load_rows(sDO + c * 8192, &tmDO, qdo_full, 64 * c, i * 64, rt);
      }
      if (np > 0) {
        const int r1 = l0 * 64, r2 = (cnt > 1 ? l1 : l0) * 64;  // key rows within the unit
        ts_mark(dbg, 0);
        ts_mark(dbg, 112);
        tc::mbar_expect_tx(k_full + k0s, L::kP);
        tc::mbar_expect_tx(v_full + v0s, L::kP);
        uint8_t* dk0 = sK + k0s * L::kP;
        uint8_t* dv0 = sV + v0s * L::kP;
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_rows(dk0 + c * 16384, &tmK, k_full + k0s, 64 * c, r1, rt);
          tc::tma_load_rows(dk0 + c * 16384 + 8192, &tmK, k_full + k0s, 64 * c, r2, rt);
        }
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_rows(dv0 + c * 16384, &tmV, v_full + v0s, 64 * c, r1, rt);
          tc::tma_load_rows(dv0 + c * 16384 + 8192, &tmV, v_full + v0s, 64 * c, r2, rt);
        }
      }
    }
    __syncwarp();
  }

  if (warp == 0 || warp == kRowsVWarp) {
#ifdef SLAB_TIMELINE
    if (dbg && warp == 0 && lane == 1) {  // observer: true K / V pair arrival times
      for (int t = 0; t < np && t < 16; ++t) {
        const int G = G0 + t;
        tc::mbar_wait(k_full + G % L::KS, (G / L::KS) & 1);
        g_bwd_ts[80 + t] = clock64();
        tc::mbar_wait(v_full + G % L::VS, (G / L::VS) & 1);
        g_bwd_ts[96 + t] = clock64();
      }
    }
#endif
    // two producer warps (Q/dO + K ring, V ring): one issuing warp's TMA stream caps at ~40 B/cycle
    if (lane == 0) {
      const int pid = warp == 0 ? 0 : 1;
      for (int t = 1; t < np; ++t) {  // pair 0 left before the block barrier
        // an odd tail repeats its block (finite data); the compute warps zero its dS rows
        const int r1 = list[2 * t] * 64;  // key rows within the unit
        const int r2 = list[min(2 * t + 1, cnt - 1)] * 64;
        const int G = G0 + t;
        const int ks = G % L::KS, vs = G % L::VS;
        if (pid == 0) {
          tc::mbar_wait(k_empty + ks, ((G / L::KS) & 1) ^ 1);
          tc::mbar_expect_tx(k_full + ks, L::kP);
          ts_mark(dbg && t < 16, t);
          uint8_t* dk = sK + ks * L::kP;
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            tc::tma_load_rows(dk + c * 16384, &tmK, k_full + ks, 64 * c, r1, rt);
            tc::tma_load_rows(dk + c * 16384 + 8192, &tmK, k_full + ks, 64 * c, r2, rt);
          }
        } else {
          tc::mbar_wait(v_empty + vs, ((G / L::VS) & 1) ^ 1);
          tc::mbar_expect_tx(v_full + vs, L::kP);
          ts_mark(dbg && t < 8, 112 + t);
          uint8_t* dv = sV + vs * L::kP;
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            tc::tma_load_rows(dv + c * 16384, &tmV, v_full + vs, 64 * c, r1, rt);
            tc::tma_load_rows(dv + c * 16384 + 8192, &tmV, v_full + vs, 64 * c, r2, rt);
          }
        }
      }
    }
  } else if (warp == 1) {
    // S^T/dP^T issuer, whole warp converged (see tc::mma_bf16_w).  The tensor pipe is in order;
    // with dQ on its own warp, S/dP(t+2) enters the pipe as soon as buffer t&1 was read, so the
    // softmax-gradient warps find S/dP(t+1) done when they finish pair t.
    const uint64_t dQk = tc::desc_kmajor(tc::smem_u32(sQ)), dDOk = tc::desc_kmajor(tc::smem_u32(sDO));
    const uint64_t dKk = tc::desc_kmajor(tc::smem_u32(sK)), dVk = tc::desc_kmajor(tc::smem_u32(sV));
    constexpr uint32_t id_st = tc::idesc_bf16(128, 64, false, false);  // pair x Q^T
    // K-major SW128 tile of `rows` rows: k-step kk (16 elements) starts at chunk kk/4, +32 B
    auto koff = [](int kk, int rows) { return uint32_t((kk >> 2) * rows * 128 + (kk & 3) * 32); };
    tc::mbar_wait(qdo_full, ip);
    cta_mark(lane == 0, 1, item);
    auto issue_sdp = [&](int t) {
      const int G = G0 + t;
      const int ks = G % L::KS, vs = G % L::VS;
      tc::mbar_wait(k_full + ks, (G / L::KS) & 1);
      tc::tc_fence_after();
      ts_mark(dbg && lane == 0 && t < 16, 16 + t);
      const uint32_t tb = (G & 1) ? tB1 : tB0;
      const uint64_t dk = tc::desc_add(dKk, ks * L::kP), dv = tc::desc_add(dVk, vs * L::kP);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)  // S^T on the K pair alone
        tc::mma_bf16_w(tb, tc::desc_add(dk, koff(kk, 128)), tc::desc_add(dQk, koff(kk, 64)), id_st, kk > 0);
      tc::mma_commit_w(s_full + (G & 1));
      tc::mbar_wait(v_full + vs, (G / L::VS) & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        tc::mma_bf16_w(tb + 64, tc::desc_add(dv, koff(kk, 128)), tc::desc_add(dDOk, koff(kk, 64)), id_st, kk > 0);
      tc::mma_commit_w(sdp_full + (G & 1));
      tc::mma_commit_w(v_empty + vs);
      ts_mark(dbg && lane == 0 && t < 16, 208 + t);
    };
    // S^T/dP^T(t) as soon as its K / V pair landed and the softmax-gradient warps have read
    // TMEM buffer t&1 (sdp_free of t-2); dQ is issued by warp 11 independently
    for (int t = 0; t < np; ++t) {
      const int G = G0 + t;
      if (G >= 2) tc::mbar_wait(sdp_free + (G & 1), ((G - 2) >> 1) & 1);
      issue_sdp(t);
    }
    __syncwarp();
  } else if (warp == kRowsDQWarp) {
    // dQ^T += [K_j1; K_j2]^T dS^T  (M = D, N = 64, K = 128) as soon as dS(t) is in smem
    tc::mbar_wait(qdo_full, ip);
    const uint64_t dKm = tc::desc_mnmajor(tc::smem_u32(sK), 16384);
    const uint64_t dDSm = tc::desc_mnmajor(tc::smem_u32(sDS), 16384);
    constexpr uint32_t id_dqt = tc::idesc_bf16(D, 64, true, true);
    for (int t = 0; t < np; ++t) {
      const int G = G0 + t;
      tc::mbar_wait(ds_full, G & 1);
      tc::tc_fence_after();
      ts_mark(dbg && lane == 0 && t < 16, 64 + t);
      const uint64_t dk = tc::desc_add(dKm, (G % L::KS) * L::kP);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        tc::mma_bf16_w(tDQT, tc::desc_add(dk, kk * 2048), tc::desc_add(dDSm, kk * 2048), id_dqt, (t | kk) != 0);
      tc::mma_commit_w(k_empty + (G % L::KS));
      tc::mma_commit_w(ds_empty);
      ts_mark(dbg && lane == 0 && t < 16, 224 + t);
    }
    tc::mma_commit_w(dq_done);
    __syncwarp();
  } else {
    constexpr int NCT = 32 * kRowsCW;   // compute threads
    constexpr int CW = 256 / kRowsCW;   // query columns per thread in the loop (32 or 16)
    constexpr int TPR = NCT / 64;       // threads per query row in the epilogue (4 or 8)
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const int tid = threadIdx.x - 64;  // 0 .. NCT-1
    // this thread's dQ^phi chunks for the epilogue (written by k_bwd_lin): issued now so their
    // latency hides behind the main loop instead of stalling the final row-wise pass
    constexpr int DQ = D / TPR;
    uint4 gq[DQ / 8];
    {
      const int rq = tid / TPR, sub = tid % TPR;
      const __nv_bfloat16* src = p.dqphi + ((long long)row0 + rq) * D + sub * DQ;
#pragma unroll
      for (int i = 0; i < DQ / 8; ++i)
        gq[i] = *reinterpret_cast<const uint4*>(src + ((8 * i + 8 * sub) & (DQ - 1)));
    }
    if (tid < 64) {  // the caller's lse (0 for rows past a ragged N: their dO is zero-filled)
      const long long cr = rm.row((long long)i * 64 + tid);
      s_lse2[tid] = cr >= 0 ? p.lse[cr] * 1.4426950408889634f : 0.f;
    }
    else if (tid < 128) s_ds[tid - 64] = p.Ds[(long long)row0 + tid - 64] * p.scale;  // D^s / sqrt(d)
    named_sync(1, NCT);
    const int c = 32 * q4 + lane;  // key row of the pair (c < 64: block j1, else j2)
#pragma unroll 1
    for (int t = 0; t < np; ++t) {
      // P = exp2(S log2e / sqrt(d) - lse log2e) from S^T alone, while dP^T may still wait for
      // its V pair; then dS = P (dP - D^s) / sqrt(d).  The per-query constants (lse log2e,
      // D^s / sqrt(d)) are shared-space vector loads.
      const int G = G0 + t;
      tc::mbar_wait(s_full + (G & 1), (G >> 1) & 1);
      tc::tc_fence_after();
      const bool live = c < 64 || 2 * t + 1 < cnt;
      const uint32_t tb = ((G & 1) ? tB1 : tB0) + lane_base + CW * grp;
      const uint32_t a_l = tc::smem_u32(s_lse2) + 4u * uint32_t(CW * grp);
      const uint32_t a_d = tc::smem_u32(s_ds) + 4u * uint32_t(CW * grp);
      uint32_t pk[CW / 2];
      {
        float pf[CW];
        {
          uint32_t sv[CW];
          tmem_ld_cw(tb, sv);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < CW; e += 4) {
            const float4 l4 = tc::lds_f4(a_l + 4u * e);
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // every fourth exponential on the FMA pipe
              const float x = __uint_as_float(sv[e + q]) * p.scale_log2 - lv[q];
              pf[e + q] = tc::poly_slot(e + q, SLAB_ROWS_POLY) ? tc::ex2_poly(x) : ex2f(x);
            }
          }
        }
        tc::mbar_wait(sdp_full + (G & 1), (G >> 1) & 1);
        tc::tc_fence_after();
        ts_mark(dbg && threadIdx.x == 64 && t < 16, 32 + t);
        ts_mark(dbg && lane == 0 && t >= 4 && t < 8 && warp < 10, 192 + 8 * (t - 4) + (warp - 2));
        uint32_t dp[CW];
        tmem_ld_cw(tb + 64, dp);
        tc::tmem_ld_wait();
        tc::tc_fence_before();  // TMEM buffer t&1 may take S/dP(t+2)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(sdp_free + (G & 1));
        ts_mark(dbg && threadIdx.x == 64 && t < 16, 240 + t);
        const float sc = p.scale;
#pragma unroll
        for (int e = 0; e < CW; e += 4) {
          const float4 d4 = tc::lds_f4(a_d + 4u * e);
          const float dv4[4] = {d4.x, d4.y, d4.z, d4.w};
          float dsv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) dsv[q] = pf[e + q] * fmaf(__uint_as_float(dp[e + q]), sc, -dv4[q]);
          pk[e >> 1] = tc::pack_bf16(dsv[0], dsv[1]);
          pk[(e >> 1) + 1] = tc::pack_bf16(dsv[2], dsv[3]);
        }
        if (!live) {  // the repeated block of an odd tail contributes nothing
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) pk[e] = 0u;
        }
      }
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 128 + t);
      if (G >= 1) tc::mbar_wait(ds_empty, (G - 1) & 1);  // dQ of the previous pair has read dS
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 144 + t);
      const uint32_t a_ds_tile = tc::smem_u32(sDS);
#pragma unroll
      for (int ch = 0; ch < CW / 8; ++ch)
        tc::sts_u4(a_ds_tile + tc::sw128_off(c, (CW / 8) * grp + ch), make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]));
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(ds_full);
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 48 + t);
      ts_mark(dbg && lane == 0 && t >= 4 && t < 8 && warp < 10, 160 + 8 * (t - 4) + (warp - 2));
    }
    // dq_total = J_phi(q)^T dQ^phi + dQ: transpose dQ^T through smem (the K ring is idle once
    // dq_done fired), then finish row-wise with 4 threads per query row.  For the softmax
    // feature map <phi(q), dQ^phi> = D^l - (D^l/den) den = 0 exactly (O^l = phi(q) H / den), so
    // the Jacobian reduces to phi(q) * dQ^phi.
    // phi(q) of this thread's quarter row first: it needs only Q_i, so it runs while the last
    // dQ^T MMAs drain.  Chunks are held in the rotated order the row-wise pass walks
    // (slot cc0 <-> columns c0 + ((cc0 + 8 sub) & (DQ - 1))), which spreads its reads of the
    // transposed tile over the banks.
    const int rq = tid / TPR, sub = tid % TPR, c0 = sub * DQ;
    auto rot = [&](int cc0) { return (cc0 + 8 * sub) & (DQ - 1); };
    float x[DQ];
#pragma unroll
    for (int cc0 = 0; cc0 < DQ; cc0 += 8) {
      float t8[8];
      unpack8(*reinterpret_cast<const uint4*>(sQ + tile_off(rq, c0 + rot(cc0))), t8);
#pragma unroll
      for (int e = 0; e < 8; ++e) x[cc0 + e] = t8[e];
    }
    if (p.phi == 2) {  // phi(q) in place, one exp per element
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < DQ; ++e) mx = fmaxf(mx, x[e]);
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float se = 0.f;
#pragma unroll
      for (int e = 0; e < DQ; ++e) {
        x[e] = __expf(x[e] - mx);
        se += x[e];
      }
#pragma unroll
      for (int o = 1; o < TPR; o <<= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const float inv = 1.f / se;
#pragma unroll
      for (int e = 0; e < DQ; ++e) x[e] *= inv;
    }
    tc::mbar_wait(dq_done, ip);
    tc::tc_fence_after();
    ts_mark(dbg && threadIdx.x == 64, 120);
    cta_mark(threadIdx.x == 64, 2, item);
    constexpr int TP = D + 1;  // with the chunk rotation: conflict-free row-wise reads
    float* tq = reinterpret_cast<float*>(sK);
    {
      const int acol = D == 128 ? 32 * q4 + lane : 16 * q4 + lane;
      const bool avalid = D == 128 || lane < 16;
      uint32_t b[CW];
      if (np > 0) tmem_ld_cw(tDQT + lane_base + CW * grp, b);
      tc::tmem_ld_wait();
      if (avalid) {
#pragma unroll
        for (int e = 0; e < CW; ++e) tq[(CW * grp + e) * TP + acol] = np > 0 ? __uint_as_float(b[e]) : 0.f;
      }
    }
    named_sync(1, NCT);
    {
      const long long grow = rm.row((long long)i * 64 + rq);  // -1: past a ragged N
#pragma unroll
      for (int cc0 = 0; cc0 < DQ; cc0 += 8) {
        const int col = c0 + rot(cc0);
        float g[8], o[8];
        unpack8(gq[cc0 / 8], g);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xe = x[cc0 + e];
          float jg;
          if (p.phi == 2) jg = xe * g[e];
          else if (p.phi == 0) jg = xe >= 0.f ? g[e] : __expf(xe) * g[e];
          else jg = xe > 0.f ? g[e] : 0.f;
          o[e] = jg + tq[rq * TP + col + e];
        }
        if (grow >= 0) *reinterpret_cast<uint4*>(p.dq + grow * D + col) = pack8(o);
        if (p.dq_part) {  // SlaGradients::dq and ::dq_feat (f32)
          float4* dqs = reinterpret_cast<float4*>(p.dq_part + grow * D + col);
          float4* dqf = reinterpret_cast<float4*>(p.dqf_part + grow * D + col);
          const float* t = tq + rq * TP + col;
          dqs[0] = make_float4(t[0], t[1], t[2], t[3]);
          dqs[1] = make_float4(t[4], t[5], t[6], t[7]);
          dqf[0] = make_float4(g[0], g[1], g[2], g[3]);
          dqf[1] = make_float4(g[4], g[5], g[6], g[7]);
        }
      }
    }
    ts_mark(dbg && threadIdx.x == 64, 124);
    cta_mark(threadIdx.x == 64, 3, item);
  }
  G0 += np;
  tc::tc_fence_before();
  __syncthreads();  // the item is done: smem (the dQ^T transpose in the K ring) and TMEM are free
  tc::tc_fence_after();
  }  // items
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

void launch_bwd_lin(const Dims& Dm, const void* q, const void* w, const void* o_s, const void* o_l,
                    const void* d_out, const StateBufs& s, __nv_bfloat16* gH, __nv_bfloat16* z3, float* Ds,
                    __nv_bfloat16* dqphi, bool ds_external, cudaStream_t st) {
  BwdParams p{};
  p.ds_external = ds_external;
  p.rl = Dm.rl;
  p.marg_cnt = s.marg_cnt;
  p.Z = s.Z;
  p.Ds_out = Ds;
  p.o_s = static_cast<const __nv_bfloat16*>(o_s);
  p.o_l = static_cast<const __nv_bfloat16*>(o_l);
  p.gH = gH;
  p.z3 = z3;
  p.dqphi = dqphi;
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.phi = Dm.phi;
  CUtensorMap tq, tdo, tw, th, tos, tol, tgh;
  auto go = [&](auto kern, int bytes, auto dd) {
    constexpr int D = decltype(dd)::value;
    make_tmap_rows(&tq, q, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_rows(&tdo, d_out, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_bf16(&tw, w, D, uint64_t(Dm.H) * D, 1, D, 0, D);
    make_tmap_bf16(&th, s.Hb, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);
    make_tmap_rows(&tos, o_s, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_rows(&tol, o_l, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_bf16(&tgh, gH, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);  // dH_i boxes [D rows][64]
    SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    launch_pdl(kern, dim3(Dm.Tm, unsigned(Dm.U)), kLinThreads, bytes, st, tq, tdo, tw, th, tos, tol, tgh, p);
    check_launch("k_bwd_lin", st);
  };
  if (Dm.d == 128)
    go(k_bwd_lin<128>, LinLayout<128>::kBytes, std::integral_constant<int, 128>{});
  else
    go(k_bwd_lin<64>, LinLayout<64>::kBytes, std::integral_constant<int, 64>{});
}

void launch_bwd_rows(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                     const void* d_out, void* dq, const StateBufs& s, const float* Ds,
                     const __nv_bfloat16* dqphi, float* dq_part, float* dqf_part, cudaStream_t st) {
  BwdParams p{};
  p.rl = Dm.rl;
  p.dq_part = dq_part;
  p.dqf_part = dqf_part;
  p.crit_cnt = s.crit_cnt;
  p.crit_idx = s.crit_idx;
  p.lse = lse;
  p.Ds = Ds;
  p.dqphi = const_cast<__nv_bfloat16*>(dqphi);
  p.dq = static_cast<__nv_bfloat16*>(dq);
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.scale = float(Dm.inv_sqrt_d);
  p.scale_log2 = float(Dm.inv_sqrt_d * 1.4426950408889634);
  p.phi = Dm.phi;
  CUtensorMap tq, tdo, tk, tv;
  auto go = [&](auto kern, int bytes, auto dd) {
    constexpr int D = decltype(dd)::value;
    make_tmap_rows(&tq, q, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_rows(&tdo, d_out, D, Dm.U, Dm.N, p.rl, 64);
    make_tmap_rows(&tk, k, D, Dm.U, Dm.Nk, p.rl, 64);
    make_tmap_rows(&tv, v, D, Dm.U, Dm.Nk, p.rl, 64);
    SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const long long items = (long long)Dm.U * Dm.Tm;
    p.items = items;
    const unsigned grid = unsigned(SLAB_ROWS_PERSIST ? std::min<long long>(items, sm_count()) : items);
    launch_pdl(kern, dim3(grid), kRowsThreads, bytes, st, tq, tdo, tk, tv, p);
    check_launch("k_bwd_rows", st);
  };
  if (Dm.d == 128)
    go(k_bwd_rows<128>, RowsLayout<128>::kBytes, std::integral_constant<int, 128>{});
  else
    go(k_bwd_rows<64>, RowsLayout<64>::kBytes, std::integral_constant<int, 64>{});
}

}  // namespace slab

#ifdef SLAB_TIMELINE  // diagnostic accessors: timeline builds only (profiles/ctaprof.py)
extern "C" int sla_b200_diag_rows_ctaprof(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, slab::g_cta_prof, sizeof(slab::g_cta_prof)) == cudaSuccess ? 0 : 1;
}
#endif

#ifdef SLAB_TIMELINE  // diagnostic accessors: timeline builds only (profiles/ctaprof.py)
extern "C" int sla_b200_diag_bwd_timeline(long long* host128) {
  return cudaMemcpyFromSymbol(host128, slab::g_bwd_ts, 256 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
#endif
