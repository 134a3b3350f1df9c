// attn_bwd_cols2.cu -- the COLUMNS pass (backward.cpp:142-199) with row-major accumulators:
// dK_j += dS^T Q_pair and dV_j += P^T dO_pair as M = 64 (key rows) x N = d MMAs, so the
// epilogue reads each key row of dK, dV, dK^phi straight from TMEM (no shared-memory transposes)
// and applies the phi-Jacobian row-wise.  The accumulation MMAs cost 8 x 64 cycles instead of
// 8 x 50 per pair; the loop is bound by the Q / dO stream, not by them.  Selected by
// SLA_B200_COLS=2; otherwise as attn_bwd.cu.
// The rows pass and the linear-branch kernel live in attn_bwd_rows.cu.  Together they mirror
// the reference's deterministic two-phase design (backward.cpp:68-120 and 142-199); no atomics.
//
// k_bwd_cols2<D>: one CTA per (unit, key block j)
//   sparse dV_j += P^T dO_i, dK_j += dS^T Q_i over the critical rows (CSC list),
//   linear dK^phi_j = V_j dH_agg^T + dZ_agg, dV_j += phi(K_j) dH_agg (dH_agg = M0^T dH),
//   dk_total = J_phi(k)^T dK^phi + dK and dv written once.
//
// Warp roles: warps 0 and 10 TMA (Q pairs / dO pairs, since one issuing warp's TMA stream caps
// at ~40 B/cycle), warps 1 and 11 MMA, warps 2-9 compute.
#include <cstdlib>

#include "bwd_common.cuh"

namespace slab {

namespace {

// =========================================================================================
// columns pass: critical query blocks in PAIRS (M = 128 S / dP tiles), dV^T / dK^T accumulated
// transposed (M = D) at full tensor rate; linear dK^phi^T and dV^T += dH_agg^T phi(K)^T on the
// tensor core; the epilogue transposes through smem and finishes row-wise.
// =========================================================================================
// The ring holds slots of one pair tile each: pair t's Q pair is item 2t, its dO pair item 2t+1
// (item n in slot n % kSlots), and dH_agg the last item.  S(t) waits only for the Q pair, dP(t)
// for the dO pair; acc(t) runs dK^T first and releases the Q pair's slot halfway, which is the
// slot dO(t+2) refills.  One P / dS buffer makes room for the fifth slot; P and dS have their own
// full / empty barriers, so dS(t+1) is written once dK^T(t) has read dS(t) and dK^T(t+1) queues
// behind dV^T(t) without a gap.  Measured (C3, k_bwd_cols ms): 4 slots + 2 P/dS buffers 1.008;
// 5 slots + 1 buffer, dK first 0.890; + P from S before dP lands 0.882.
// every N-th exponential by tc::ex2_poly.  Measured before the P / dS barrier split: 0 0.869 ms,
// 2 0.875, 4 0.851; after it: 0 0.840, 3 0.838, 4 0.842, 8 0.847 -- no gain, so off
#ifndef SLAB_COLS_POLY
#define SLAB_COLS_POLY 0
#endif
#ifndef SLAB_COLS_DVFIRST  // 1: acc(t) issues dV^T first, P stored first (measured 0.881 vs 0.838 ms)
#define SLAB_COLS_DVFIRST 0
#endif
// DQ = D/4 consecutive columns of my row half in the M = 64 TMEM layout: threads 0-15 read
// columns [c, c + DQ), threads 16-31 [c + D/2, c + D/2 + DQ) of the same lanes
template <int D>
__device__ __forceinline__ void ld_rowq(uint32_t taddr, uint32_t (&r)[D / 4]);
template <>
__device__ __forceinline__ void ld_rowq<128>(uint32_t taddr, uint32_t (&r)[32]) {
  tc::tmem_ld32_x2<64>(taddr, r);
}
template <>
__device__ __forceinline__ void ld_rowq<64>(uint32_t taddr, uint32_t (&r)[16]) {
  tc::tmem_ld16_x2<32>(taddr, r);
}

template <int D>
struct Cols2Layout {
  static constexpr int kT = 64 * D * 2;    // 64-row tile
  static constexpr int kP = 128 * D * 2;   // 128-row pair tile
  static constexpr int oK = 0, oV = kT;
  static constexpr int oRing = 2 * kT;
  static constexpr int kSlot = kP;         // Q pair, dO pair, or dH_agg (D*D*2 <= kP)
  static constexpr int kSlots = 5;
  static constexpr int oPD = oRing + kSlots * kSlot;  // [P 16 KB | dS 16 KB]; phi(K) aliases
  static constexpr int oZA = oPD + 32768;             // float [D] dZ_agg
  static constexpr int oX = oZA + 4 * D;              // float [2][2][64]: row partials exchanged between warp pairs
  static constexpr int oBar = oX + 1024;
  static constexpr int kBytes = oBar + 256 + 1024;
  static_assert(kBytes <= 232448, "smem");
  static_assert(D * D * 2 <= kSlot && 3 * 64 * (D + 1) * 4 <= kSlots * kSlot, "ring reuse");
};

// Warps: 0 and 10 TMA producers, 1 S/dP issuer, 2-9 softmax-gradient / epilogue, 11 the
// dV / dK accumulation issuer (and the linear-branch MMAs).  Two issuing warps keep one's
// barrier waits from delaying the other's MMAs (1.09 -> 1.04 ms); 4 producer warps and a
// single poll-driven issuer were measured no better.
constexpr int kAccWarp = 11;
constexpr int kColsThreads = 32 * 12;

template <int D>
__global__ void __launch_bounds__(kColsThreads, 1)
    k_bwd_cols2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
               const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
               const __grid_constant__ CUtensorMap tmHa, const __grid_constant__ CUtensorMap tmDKo,
               const __grid_constant__ CUtensorMap tmDVo, BwdParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = Cols2Layout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + L::oK;
  uint8_t* sV = smem + L::oV;
  uint8_t* sRing = smem + L::oRing;
  uint8_t* sPD = smem + L::oPD;
  uint8_t* sKF = sPD;  // phi(K_j), written once the accumulation MMAs have drained the P/dS buffers
  float* zas = reinterpret_cast<float*>(smem + L::oZA);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  constexpr int RS = L::kSlots;
  uint64_t* kv_full = bars + 0;
  uint64_t* sdp_full = bars + 1;   // [2]
  uint64_t* p_full = bars + 3;     // compute warps stored P(t)
  uint64_t* ds_full = bars + 4;    // ... dS(t)
  uint64_t* p_empty = bars + 5;    // dV^T(t) has read P(t)
  uint64_t* ds_empty = bars + 6;   // dK^T(t) has read dS(t)
  uint64_t* acc_done = bars + 7;
  uint64_t* kf_ready = bars + 8;
  uint64_t* all_done = bars + 9;
  uint64_t* sdp_free = bars + 10;  // [2] (2-issuer mode) compute warps have read S|dP buffer t&1
  uint64_t* s_full = bars + 12;    // [2] S(t) alone is in TMEM (P's exponentials start early)
  uint64_t* ring_full = bars + 16;        // [RS]
  uint64_t* ring_empty = bars + 16 + RS;  // [RS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * RS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x;
  const long long u = blockIdx.y;
  const RowTma rt = row_tma(p.rl, u, p.N);
  const RowMap rm = row_map(p.rl, u, p.N);
  const long long ucol = u * p.Tn + j;
  const int cnt = p.ccol_cnt[ucol];
  const int np = (cnt + 1) >> 1;
  const int* list = p.ccol_idx + ucol * p.Tm;
  const bool dbg = blockIdx.x == SLAB_DBG_X && blockIdx.y == 6;
  ts_mark(dbg && threadIdx.x == 0, 127);
  cta_mark(threadIdx.x == 0, 0);
  const bool has_lin = p.ccol_marg[ucol] > 0;  // some marginal row in this column (k_build_csc)
  ts_mark(dbg && threadIdx.x == 0, 126);
  // pair 0's query blocks, loaded alongside cnt so its loads can leave before the TMEM
  // allocation and the block barrier
  int l0 = 0, l1 = 0;
  if (threadIdx.x == 0) {
    l0 = list[0];
    l1 = list[min(1, p.Tm - 1)];
  }

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(kv_full, 1);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(ring_full + s, 1);  // one arrive.expect_tx: the item's producer warp
        tc::mbar_init(ring_empty + s, 1);
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(sdp_full + s, 1);
        tc::mbar_init(s_full + s, 1);
      }
      tc::mbar_init(p_full, 8);
      tc::mbar_init(ds_full, 8);
      tc::mbar_init(p_empty, 1);
      tc::mbar_init(ds_empty, 1);
      tc::mbar_init(acc_done, 1);
      tc::mbar_init(sdp_free, 8);
      tc::mbar_init(sdp_free + 1, 8);
      tc::mbar_init(kf_ready, 8);
      tc::mbar_init(all_done, 1);
      tc::fence_barrier_init();
      // K_j / V_j and pair 0 (items 0 and 1) now; the producer loops start at pair 1
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmDO);
      tc::mbar_expect_tx(kv_full, 2 * L::kT);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_load_rows(sK + c * 8192, &tmK, kv_full, 64 * c, j * 64, rt);
        tc::tma_load_rows(sV + c * 8192, &tmV, kv_full, 64 * c, j * 64, rt);
      }
      if (np > 0) {
        const int r1 = l0 * 64, r2 = (cnt > 1 ? l1 : l0) * 64;  // query rows within the unit
        ts_mark(dbg, 0);
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          tc::mbar_expect_tx(ring_full + it, L::kP);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            tc::tma_load_rows(sRing + it * L::kSlot + c * 16384, it ? &tmDO : &tmQ, ring_full + it, 64 * c, r1, rt);
            tc::tma_load_rows(sRing + it * L::kSlot + c * 16384 + 8192, it ? &tmDO : &tmQ, ring_full + it, 64 * c, r2, rt);
          }
        }
      }
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // dV [0,128), dK [128,256) (M = 64 key rows, N = D); S|dP pair buffers at 256 and 384
  // (M = 128); dK^phi (M = 64) in the first S|dP buffer once the loop is done
  const uint32_t tDVT = tmem, tDKT = tmem + 128, tB0 = tmem + 256, tB1 = tmem + 384, tKPT = tB0;

  if (warp == 0 || (warp >= 10 && warp < kAccWarp)) {
    // No L2 prefetch of the column's Q / dO tiles: prefetches queue in the TMA unit ahead of
    // the ring loads, and a wave's columns share one unit's Q / dO, which stays L2-resident.
    // Two producer warps fill each stage (TMA issue from one warp caps at ~40 B/cycle):
    // pid 0 loads the Q pair (and K_j / V_j), pid 1 the dO pair.
    if (lane == 0) {
      const int pid = warp == 0 ? 0 : 1;
      auto acquire = [&](int item, int bytes) -> uint8_t* {
        const int s = item % RS;
        tc::mbar_wait(ring_empty + s, ((item / RS) & 1) ^ 1);
        tc::mbar_expect_tx(ring_full + s, bytes);
        return sRing + s * L::kSlot;
      };
      const CUtensorMap* tm = pid ? &tmDO : &tmQ;
      for (int pp = 1; pp < np; ++pp) {  // pair 0 left before the block barrier
        const int r1 = list[2 * pp] * 64;  // query rows within the unit
        const int r2 = list[min(2 * pp + 1, cnt - 1)] * 64;
        const int item = 2 * pp + pid;
        uint8_t* dst = acquire(item, L::kP);
        ts_mark(dbg && pid == 0 && pp < 16, pp);
        uint64_t* fb = ring_full + (item % RS);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_rows(dst + c * 16384, tm, fb, 64 * c, r1, rt);
          tc::tma_load_rows(dst + c * 16384 + 8192, tm, fb, 64 * c, r2, rt);
        }
      }
      if (has_lin && pid == 0) {  // dH_agg: the last item, D / 64 chunks of [D rows x 64]
        const int item = 2 * np;
        uint8_t* dst = acquire(item, D * D * 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(dst + c * D * 128, &tmHa, ring_full + (item % RS), 64 * c, int(ucol * D), 0);
      }
    }
  } else if (warp == 1 || warp == kAccWarp) {
    const uint32_t aK = tc::smem_u32(sK), aV = tc::smem_u32(sV), aKF = tc::smem_u32(sKF);
    const uint32_t aR = tc::smem_u32(sRing), aPD = tc::smem_u32(sPD);
    constexpr uint32_t id_s = tc::idesc_bf16(128, 64, false, false);   // pair x K^T
    constexpr uint32_t id_acc = tc::idesc_bf16(64, D, true, true);     // P^T x dO_pair, dS^T x Q_pair
    constexpr uint32_t id_kp = tc::idesc_bf16(64, D, false, false);    // V x dH_agg^T
    constexpr uint32_t id_vl = tc::idesc_bf16(64, D, false, true);     // phi(K) x dH_agg
    auto wait_item = [&](int item) -> uint32_t {
      const int s = item % RS;
      tc::mbar_wait(ring_full + s, (item / RS) & 1);
      tc::tc_fence_after();
      return aR + s * L::kSlot;
    };
    auto kdesc = [](uint32_t base, int kk, int rows) {
      return tc::desc_kmajor(base + (kk >> 2) * rows * 128 + (kk & 3) * 32);
    };
    tc::mbar_wait(kv_full, 0);
    tc::tc_fence_after();
    ts_mark(dbg && lane == 0, 125);
    cta_mark(lane == 0, 1);
    // Whole warp runs the issue loop (warp-uniform operands, one elected lane issues; see
    // tc::mma_bf16_w).  Descriptors: ring slot s at +s*kSlot, k-step kk at +koff / +kk*2048.
    const uint64_t dRk = tc::desc_kmajor(aR), dKk = tc::desc_kmajor(aK), dVk = tc::desc_kmajor(aV);
    const uint64_t dRm = tc::desc_mnmajor(aR, 16384), dPDm = tc::desc_mnmajor(aPD, 16384);
    auto koff = [](int kk, int rows) { return uint32_t((kk >> 2) * rows * 128 + (kk & 3) * 32); };
    // acc(t): dK^T += Q_pair^T dS, then dV^T += dO_pair^T P  (M = D, N = 64 keys, K = 128)
    auto issue_acc = [&](int t) {
      const int sq = (2 * t) % RS, sdo = (2 * t + 1) % RS;
      const uint64_t dq = tc::desc_add(dRm, sq * L::kSlot), ddo = tc::desc_add(dRm, sdo * L::kSlot);
      const uint64_t dp = dPDm, dd = tc::desc_add(dPDm, 16384);
      auto dk = [&] {
        tc::mbar_wait_w(ds_full, t & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // A = dS^T (MN-major [q][key] tile), B = Q_pair (MN-major, d chunks 16 KB apart)
          tc::mma_bf16_w(tDKT, tc::desc_add(dd, kk * 2048), tc::desc_add(dq, kk * 2048), id_acc, (t | kk) != 0);
        tc::mma_commit_w(ring_empty + sq);  // dO(t+2) refills this slot
        tc::mma_commit_w(ds_empty);
      };
      auto dv = [&] {
        tc::mbar_wait_w(p_full, t & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // A = P^T, B = dO_pair
          tc::mma_bf16_w(tDVT, tc::desc_add(dp, kk * 2048), tc::desc_add(ddo, kk * 2048), id_acc, (t | kk) != 0);
        tc::mma_commit_w(ring_empty + sdo);
        tc::mma_commit_w(p_empty);
      };
      if (SLAB_COLS_DVFIRST) {
        dv();
        dk();
      } else {
        dk();
        dv();
      }
    };
    // The tensor pipe executes in issue order; the two issuers interleave S/dP(t+1) and acc(t)
    // in whichever order their inputs become ready.
    if (warp == 1) {
      // S/dP(t) once its ring stage landed and the compute warps have read TMEM buffer t&1
      for (int ts = 0; ts < np; ++ts) {
        const int iq = 2 * ts, ido = 2 * ts + 1;
        if (ts >= 2) tc::mbar_wait(sdp_free + (ts & 1), ((ts - 2) >> 1) & 1);
        tc::mbar_wait(ring_full + iq % RS, (iq / RS) & 1);
        tc::tc_fence_after();
        ts_mark(dbg && lane == 0 && ts < 16, 16 + ts);
        const uint64_t dq = tc::desc_add(dRk, (iq % RS) * L::kSlot), ddo = tc::desc_add(dRk, (ido % RS) * L::kSlot);
        const uint32_t tb = (ts & 1) ? tB1 : tB0;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)  // S = Q_pair K_j^T as soon as the Q pair landed
          tc::mma_bf16_w(tb, tc::desc_add(dq, koff(kk, 128)), tc::desc_add(dKk, koff(kk, 64)), id_s, kk > 0);
        tc::mma_commit_w(s_full + (ts & 1));
        tc::mbar_wait(ring_full + ido % RS, (ido / RS) & 1);
        tc::tc_fence_after();
        ts_mark(dbg && lane == 0 && ts < 16, 80 + ts);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)  // dP = dO_pair V_j^T
          tc::mma_bf16_w(tb + 64, tc::desc_add(ddo, koff(kk, 128)), tc::desc_add(dVk, koff(kk, 64)), id_s, kk > 0);
        tc::mma_commit_w(sdp_full + (ts & 1));
      }
      __syncwarp();
    } else {  // accumulation warp: dK^T(t) / dV^T(t) as soon as dS(t) / P(t) are in smem
      for (int ta = 0; ta < np; ++ta) {
        ts_mark(dbg && lane == 0 && ta < 16, 96 + ta);
        issue_acc(ta);
#ifdef SLAB_TIMELINE
        if (dbg && ta < 16) {  // acc(ta) completion (P(ta+1)'s store waits for it anyway)
          tc::mbar_wait_w(p_empty, ta & 1);
          ts_mark(lane == 0, 64 + ta);
        }
#endif
      }
      tc::mma_commit_w(acc_done);
    }
    __syncwarp();
    if (warp == kAccWarp) {  // the linear part and all_done: same issuing thread as acc
    if (has_lin) {
      const int item = 2 * np;
      const uint32_t sh = wait_item(item);
      // dK^phi raw = V_j dH_agg^T (M = 64 keys, N = D over a, K = D over b): needs only dH_agg
      // and V_j, so it runs while the compute warps still write the phi(K_j) tile
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) tc::mma_bf16_w(tKPT, kdesc(aV, kk, 64), kdesc(sh, kk, D), id_kp, kk > 0);
      tc::mbar_wait(kf_ready, 0);
      tc::tc_fence_after();
      // dV += phi(K_j) dH_agg (M = 64 keys, N = D over b, K = D over a)
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        tc::mma_bf16_w(tDVT, kdesc(aKF, kk, 64), tc::desc_mnmajor(sh + kk * 2048, D * 128), id_vl,
                       (np > 0 || kk > 0) ? 1u : 0u);
      tc::mma_commit_w(ring_empty + (item % RS));
      __syncwarp();
    }
    if (lane == 0) tc::mma_commit(all_done);
    __syncwarp();
    }
  } else {
    const int q4 = warp & 3;
    const int grp = (warp - 2) >> 2;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const int tid = threadIdx.x - 64;  // 0..255
    for (int a = tid; a < D; a += 256) zas[a] = has_lin ? tc::load_sum3(p.gZa + ucol * 3 * D + a, D) : 0.f;
    // ---- loop: thread = query row rq of the pair (S / dP lanes), 32 key columns per group
    const int rq = 32 * q4 + lane;
    // per-query-row lse / D^s of pair t+1 are fetched during pair t (two dependent global
    // loads -- list entry, then the row values -- would otherwise stall every iteration)
    auto row_of = [&](int t) {
      return u * p.N + (long long)list[min(2 * t + (rq >> 6), cnt - 1)] * 64 + (rq & 63);
    };
    float lse_n = 0.f, ds_n = 0.f;
    if (np > 0) {
      const long long r0 = row_of(0);
      const long long c0r = rm.row(r0 - u * p.N);  // the caller's lse in place
      lse_n = c0r >= 0 ? p.lse[c0r] : 0.f;
      ds_n = p.Ds[r0];
    }
    for (int t = 0; t < np; ++t) {
      const bool live = rq < 64 || 2 * t + 1 < cnt;
      const float lse2 = lse_n * 1.4426950408889634f;
      const float dss = ds_n * p.scale;  // D^s / sqrt(d)
      if (t + 1 < np) {
        const long long r1 = row_of(t + 1);
        const long long c1r = rm.row(r1 - u * p.N);
        lse_n = c1r >= 0 ? p.lse[c1r] : 0.f;
        ds_n = p.Ds[r1];
      }
      // P from S alone (the exponentials run while dP(t) may still wait for its dO pair)
      tc::mbar_wait(s_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t tb = ((t & 1) ? tB1 : tB0) + lane_base + 32 * grp;
      uint32_t pp[16], dd[16];
      {
        float pf[32];
        {
          uint32_t sv[32];
          tc::tmem_ld32(tb, sv);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {  // every POLY-th exponential on the FMA pipe
            const float x = __uint_as_float(sv[e]) * p.scale_log2 - lse2;
            pf[e] = tc::poly_slot(e, SLAB_COLS_POLY) ? tc::ex2_poly(x) : ex2f(x);
          }
        }
#pragma unroll
        for (int e = 0; e < 32; e += 2) pp[e >> 1] = tc::pack_bf16(pf[e], pf[e + 1]);
        tc::mbar_wait(sdp_full + (t & 1), (t >> 1) & 1);
        tc::tc_fence_after();
        ts_mark(dbg && threadIdx.x == 64 && t < 16, 32 + t);
        uint32_t dp[32];
        tc::tmem_ld32(tb + 64, dp);
        tc::tmem_ld_wait();
        tc::tc_fence_before();  // TMEM buffer t&1 may take S/dP(t+2)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(sdp_free + (t & 1));
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float d0 = pf[e] * fmaf(__uint_as_float(dp[e]), p.scale, -dss);
          const float d1 = pf[e + 1] * fmaf(__uint_as_float(dp[e + 1]), p.scale, -dss);
          dd[e >> 1] = tc::pack_bf16(d0, d1);
        }
        if (!live) {  // the repeated block of an odd tail contributes nothing
#pragma unroll
          for (int e = 0; e < 16; ++e) pp[e] = dd[e] = 0u;
        }
      }
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 128 + t);
      const uint32_t prow = tc::smem_u32(sPD);
      auto store_ds = [&] {
        if (t >= 1) tc::mbar_wait(ds_empty, (t - 1) & 1);
        ts_mark(dbg && threadIdx.x == 64 && t < 16, 144 + t);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          tc::sts_u4(prow + 16384 + tc::sw128_off(rq, 4 * grp + ch), make_uint4(dd[4 * ch], dd[4 * ch + 1], dd[4 * ch + 2], dd[4 * ch + 3]));
        tc::fence_proxy_async();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(ds_full);
      };
      auto store_p = [&] {
        if (t >= 1) tc::mbar_wait(p_empty, (t - 1) & 1);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          tc::sts_u4(prow + tc::sw128_off(rq, 4 * grp + ch), make_uint4(pp[4 * ch], pp[4 * ch + 1], pp[4 * ch + 2], pp[4 * ch + 3]));
        tc::fence_proxy_async();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full);
      };
      if (SLAB_COLS_DVFIRST) {
        store_p();
        store_ds();
      } else {
        store_ds();
        store_p();
      }
      ts_mark(dbg && threadIdx.x == 64 && t < 16, 48 + t);
    }
    // ---- epilogue, row-wise from TMEM.  Thread: key row r of block j (M = 64 layout: lanes
    // 0-15 of its warp's quarter), column half hh, column quarter grp of that half -> 32 of the D
    // columns; a row's 4 threads combine partials with shfl(16) and the partner warp (smem).
    const int r = 16 * q4 + (lane & 15);
    const int hh = lane >> 4;
    const int col0 = hh * (D / 2) + grp * (D / 4);  // D / 4 columns: 32 (D = 128) or 16 (D = 64)
    constexpr int DQ = D / 4;
    const uint32_t aXc = tc::smem_u32(smem + L::oX);
    int xb = 0;  // exchange buffer parity
    auto row_combine = [&](float v, bool is_max) -> float {
      v = is_max ? fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16)) : v + __shfl_xor_sync(0xffffffffu, v, 16);
      const uint32_t a = aXc + uint32_t((xb * 2 + grp) * 256 + 4 * r);
      if (hh == 0) asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
      named_sync(3 + q4, 64);  // this warp and its partner (same TMEM quarter)
      float o;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(a + (grp ? -256 : 256)));
      xb ^= 1;
      return is_max ? fmaxf(v, o) : v + o;
    };
    tc::mbar_wait(kv_full, 0);  // K_j must have landed even when no critical row came by
    float kf[DQ];
#pragma unroll
    for (int cc = 0; cc < DQ; cc += 8) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(sK + tile_off(r, col0 + cc)), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) kf[cc + e] = f[e];
    }
    if (p.phi == 2) {  // per-row softmax over d (feature_map.cpp:22-40)
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < DQ; ++e) mx = fmaxf(mx, kf[e]);
      mx = row_combine(mx, true);
      float se = 0.f;
#pragma unroll
      for (int e = 0; e < DQ; ++e) {
        kf[e] = __expf(kf[e] - mx);
        se += kf[e];
      }
      const float inv = 1.f / row_combine(se, false);
#pragma unroll
      for (int e = 0; e < DQ; ++e) kf[e] *= inv;
    } else {
#pragma unroll
      for (int e = 0; e < DQ; ++e) kf[e] = phi_elem(p.phi, kf[e]);
    }
    tc::mbar_wait(acc_done, 0);  // the P / dS buffers are free
    ts_mark(dbg && threadIdx.x == 64, 120);
    cta_mark(threadIdx.x == 64, 2);
    if (has_lin) {  // the phi(K_j) tile: A operand of dV += phi(K_j) dH_agg
#pragma unroll
      for (int cc = 0; cc < DQ; cc += 8) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = kf[cc + e];
        *reinterpret_cast<uint4*>(sKF + tile_off(r, col0 + cc)) = pack8(f);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(kf_ready);
    }
    tc::mbar_wait(all_done, 0);
    tc::tc_fence_after();
    ts_mark(dbg && threadIdx.x == 64, 122);
    const uint32_t tcol = lane_base + uint32_t(grp * DQ);  // my columns: hh * D/2 via the x2 offset
    named_sync(1, 256);  // zas (dZ_agg) written by all compute threads at entry
    // ---- dk_total = J_phi(k)^T (dK^phi + dZ_agg) + dK ; dv
    float g[DQ];
    {
      uint32_t t32[DQ];
      if (has_lin) {
        ld_rowq<D>(tKPT + tcol, t32);
        tc::tmem_ld_wait();
      }
#pragma unroll
      for (int e = 0; e < DQ; ++e) g[e] = has_lin ? __uint_as_float(t32[e]) + zas[col0 + e] : 0.f;
    }
    if (p.phi == 2) {  // softmax: J^T g = phi (g - <phi, g>)
      float dot = 0.f;
#pragma unroll
      for (int e = 0; e < DQ; ++e) dot = fmaf(kf[e], g[e], dot);
      dot = row_combine(dot, false);
#pragma unroll
      for (int e = 0; e < DQ; ++e) kf[e] = kf[e] * (g[e] - dot);
    } else if (p.phi == 0) {  // elu1: J = 1 where k >= 0 (phi >= 1) else phi
#pragma unroll
      for (int e = 0; e < DQ; ++e) kf[e] = kf[e] >= 1.f ? g[e] : kf[e] * g[e];
    } else {  // relu: J = 1 where phi > 0
#pragma unroll
      for (int e = 0; e < DQ; ++e) kf[e] = kf[e] > 0.f ? g[e] : 0.f;
    }
    const long long grow = rm.row((long long)j * 64 + r);  // -1: past a ragged N
    {
      uint32_t t32[DQ];
      if (np > 0) {
        ld_rowq<D>(tDKT + tcol, t32);
        tc::tmem_ld_wait();
      }
      if (p.dk_part && grow >= 0) {  // SlaGradients::dk and ::dk_feat (f32)
        float4* dks = reinterpret_cast<float4*>(p.dk_part + grow * D + col0);
        float4* dkf = reinterpret_cast<float4*>(p.dkf_part + grow * D + col0);
#pragma unroll
        for (int e = 0; e < DQ; e += 4) {
          dks[e / 4] = np > 0 ? make_float4(__uint_as_float(t32[e]), __uint_as_float(t32[e + 1]), __uint_as_float(t32[e + 2]),
                                            __uint_as_float(t32[e + 3]))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          dkf[e / 4] = make_float4(g[e], g[e + 1], g[e + 2], g[e + 3]);
        }
      }
      // dk staged as a K-major SW128 tile in the P / dS region (free since all_done: its phi(K)
      // tile has been consumed), stored by TMA (coalesced; rows past a ragged N are clipped)
#pragma unroll
      for (int cc = 0; cc < DQ; cc += 8) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = kf[cc + e] + (np > 0 ? __uint_as_float(t32[cc + e]) : 0.f);
        *reinterpret_cast<uint4*>(sPD + tile_off(r, col0 + cc)) = pack8(o);
      }
    }
    {
      uint32_t t32[DQ];
      const bool any = np > 0 || has_lin;
      if (any) {
        ld_rowq<D>(tDVT + tcol, t32);
        tc::tmem_ld_wait();
      }
#pragma unroll
      for (int cc = 0; cc < DQ; cc += 8) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = any ? __uint_as_float(t32[cc + e]) : 0.f;
        *reinterpret_cast<uint4*>(sPD + 16384 + tile_off(r, col0 + cc)) = pack8(o);
      }
    }
    tc::fence_proxy_async();
    named_sync(1, 256);
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tc::tma_store_rows(&tmDKo, sPD + c * 8192, 64 * c, j * 64, rt);
        tc::tma_store_rows(&tmDVo, sPD + 16384 + c * 8192, 64 * c, j * 64, rt);
      }
      tc::bulk_commit();
      tc::bulk_wait_read<0>();  // smem may be released; the writes complete with the grid
    }
  }
  ts_mark(dbg && threadIdx.x == 64, 124);
  cta_mark(threadIdx.x == 64, 3);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int D>
void launch_cols2_t(const Dims& Dm, const void* q, const void* k, const void* v, const void* d_out,
                   const __nv_bfloat16* Ha, BwdParams p, cudaStream_t st) {
  CUtensorMap tq, tdo, tk, tv, th, tdk, tdv;
  make_tmap_rows(&tq, q, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tdo, d_out, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tk, k, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_rows(&tv, v, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_bf16(&th, Ha, D, uint64_t(Dm.U) * Dm.Tn * D, 1, D, 0, D);
  make_tmap_rows(&tdk, p.dk, D, Dm.U, Dm.Nk, p.rl, 64);  // outputs: key rows (n_kv views: Nk)
  make_tmap_rows(&tdv, p.dv, D, Dm.U, Dm.Nk, p.rl, 64);
  auto kern = k_bwd_cols2<D>;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cols2Layout<D>::kBytes));
  launch_pdl(kern, dim3(Dm.Tn, unsigned(Dm.U)), kColsThreads, Cols2Layout<D>::kBytes, st, tq, tdo, tk, tv, th, tdk, tdv, p);
  check_launch("k_bwd_cols", st);  // same profiler name as attn_bwd.cu
}

}  // namespace

void launch_bwd_cols2(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                     const void* d_out, void* dk, void* dv, const StateBufs& s,
                     const __nv_bfloat16* Ha, const float* gZa, const float* Ds, float* dk_part,
                     float* dkf_part, int* work, cudaStream_t st) {
  BwdParams p{};
  p.rl = Dm.rl;
  p.work = work;  // unused: one CTA per key block (a persistent variant spilled)
  p.dk_part = dk_part;
  p.dkf_part = dkf_part;
  p.ccol_cnt = s.ccol_cnt;
  p.ccol_idx = s.ccol_idx;
  p.ccol_marg = s.ccol_marg;
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
    launch_cols2_t<128>(Dm, q, k, v, d_out, Ha, p, st);
  else
    launch_cols2_t<64>(Dm, q, k, v, d_out, Ha, p, st);
}

}  // namespace slab


#ifdef SLAB_TIMELINE  // diagnostic accessors: timeline builds only (profiles/ctaprof.py)
extern "C" int sla_b200_diag_cols2_ctaprof(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, slab::g_cta_prof, sizeof(slab::g_cta_prof)) == cudaSuccess ? 0 : 1;
}
extern "C" int sla_b200_diag_cols2_timeline(long long* host128) {
  return cudaMemcpyFromSymbol(host128, slab::g_bwd_ts, 256 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
#endif
