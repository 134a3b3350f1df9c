// attn_fwd.cu -- K5: the fused SLA forward for one 64-row query block per CTA on tcgen05.
//
// One kernel handles all three block classes of its block row (forward.cpp:81-172):
//   * marginal: O^l = phi(Q_i) H_i / (phi(Q_i) . Z_i) -- phi(Q_i) is built in smem, the
//     phi(Q_i) H_i product runs on the tensor core (H_i = M0 . h from gemm.cu);
//   * critical: online-softmax FlashAttention loop over the ascending critical list
//     (forward.cpp:29-79), S = Q K_j^T and O += P V_j on tcgen05 with TMEM accumulators;
//   * negligible: never touched;
// and the projection epilogue O = O^s + O^l W (forward.cpp:187-195) accumulates O^l W onto
// the normalised O^s in TMEM.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (one thread), warps 2-5
// softmax / epilogue (row r = 16*(warp%4) + (lane & 15); lanes 0-15 / 16-31 take the two column
// halves through the 16x32bx2 TMEM shape).
// The K/V ring also carries H_i (before the loop) and W (after it) as ring items.
// Lazy rescaling: O is rescaled only when the running max grows by more than 2^8.
#include <cstdlib>

#include "kernels.hpp"
#include "tc.cuh"

#ifndef SLAB_FWD_POLY
#define SLAB_FWD_POLY 0  // every N-th exponential by tc::ex2_poly; measured: 0 best, 4 +0.003 ms, 2 +0.027
#endif

namespace slab {

#ifdef SLAB_TIMELINE
static __device__ long long g_fwd_ts[128];  // -DSLAB_TIMELINE: timeline of one CTA
#endif

namespace {

__device__ __forceinline__ void fts(bool on, int slot) {
#ifdef SLAB_TIMELINE
  if (on) g_fwd_ts[slot] = clock64();
#else
  (void)on;
  (void)slot;
#endif
}

template <int D>
struct FwdLayout {
  static constexpr int kQ = 64 * D * 2;       // Q tile, K-major SW128 (D/64 chunks of 8 KB)
  static constexpr int kTile = 64 * D * 2;    // one K or V tile == one 64-column chunk of H / W
  static constexpr int kSlots = 2;            // per ring; 2 CTAs / SM share the tensor core
  static constexpr int kPX = 16384;           // 2 P buffers (8 KB) == phi(Q) / O^l tile
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + kQ;          // K ring; W chunks after the loop
  static constexpr int oV = oK + kSlots * kTile;  // V ring; H chunks before the loop
  static constexpr int oPX = oV + kSlots * kTile;
  static constexpr int oBar = oPX + kPX;
  static constexpr int oZ = oBar + 256;       // Z_i (f32 [D])
  static constexpr int kBytes = oZ + D * 4 + 1024;
  static_assert(kBytes <= 232448 / 2, "smem: 2 CTAs / SM");
  static_assert(D / 64 <= kSlots, "H/W chunks must fit a ring");
  static_assert(64 * D * 2 <= kPX, "X tile must fit the P region");
};

struct FwdParams {
  const int* crit_cnt;
  const int* crit_idx;
  const int* marg_cnt;
  const float* Z;
  __nv_bfloat16* o;
  __nv_bfloat16* o_s;
  __nv_bfloat16* o_l;
  float* lse;
  long long N;
  int Tm, Tn, H;
  float scale_log2;
  int has_w;
  int phi;
  int kv_last;  // valid keys in the last key block (64 unless ragged N)
  RowLayout rl; // the caller's q, k, v, o, o_s, o_l, lse (read / written in place)
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(192, 2)
    k_attn_fwd(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmH,
               const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
               const __grid_constant__ CUtensorMap tmOs, const __grid_constant__ CUtensorMap tmOl, FwdParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = FwdLayout<D>;
  constexpr int RS = L::kSlots;
  constexpr int NC = D / 64;  // 64-column chunks of H / W
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sK = smem + L::oK;
  uint8_t* sV = smem + L::oV;
  uint8_t* sPX = smem + L::oPX;
  float* sZ = reinterpret_cast<float*>(smem + L::oZ);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars + 0;
  uint64_t* s_full = bars + 5;      // [2]
  uint64_t* p_full = bars + 7;      // [2]
  uint64_t* pv_done = bars + 9;     // [2]
  uint64_t* lin_done = bars + 11;
  uint64_t* x_full = bars + 12;
  uint64_t* o_ready = bars + 13;
  uint64_t* proj_done = bars + 14;
  uint64_t* k_full = bars + 16;     // [RS]
  uint64_t* k_empty = bars + 18;    // [RS]
  uint64_t* v_full = bars + 20;     // [RS]
  uint64_t* v_empty = bars + 22;    // [RS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const long long u = blockIdx.y;
  const RowTma rt = row_tma(p.rl, u, p.N);
  const RowMap rm = row_map(p.rl, u, p.N);
  const long long urow = u * p.Tm + i;
  const int cnt = p.crit_cnt[urow];
  const int* list = p.crit_idx + urow * p.Tn;
  const bool has_lin = p.marg_cnt[urow] > 0;
  const bool has_w = p.has_w != 0;
  const bool dbg = blockIdx.x == 100 && blockIdx.y == 6;
  fts(dbg && threadIdx.x == 0, 127);

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::tma_prefetch(&tmV);
      tc::mbar_init(q_full, 1);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(k_full + s, 1);
        tc::mbar_init(k_empty + s, 1);
        tc::mbar_init(v_full + s, 1);
        tc::mbar_init(v_empty + s, 1);
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(s_full + s, 1);
        tc::mbar_init(p_full + s, 4);
        tc::mbar_init(pv_done + s, 1);
      }
      tc::mbar_init(lin_done, 1);
      tc::mbar_init(x_full, 4);
      tc::mbar_init(o_ready, 4);
      tc::mbar_init(proj_done, 1);
      tc::fence_barrier_init();
      // Q_i leaves before the TMEM allocation and the block barrier (the producer below
      // continues with K(0), H_i, ...)
      tc::mbar_expect_tx(q_full, L::kQ);
#pragma unroll
      for (int c = 0; c < NC; ++c) tc::tma_load_rows(sQ + c * 8192, &tmQ, q_full, 64 * c, i * 64, rt);
    }
    __syncwarp();
    tc::tmem_alloc<256>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem;                // D columns
  const uint32_t tS0 = tmem + 128;         // two 64-column score buffers

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    // Two rings: K slots are released by S(t), V slots by PV(t), so K(t+2) is in flight while
    // PV(t) still waits for P(t).  H_i's chunks go through the V ring (needed before V(0)),
    // W's chunks through the K ring (needed after the last S).
    if (lane == 0) {
      int kit = 0, vit = 0;
      auto take = [&](uint64_t* full, uint64_t* empty, uint8_t* base, int& it, int bytes) -> uint8_t* {
        const int s = it % RS;
        tc::mbar_wait(empty + s, ((it / RS) & 1) ^ 1);
        tc::mbar_expect_tx(full + s, bytes);
        return base + s * L::kTile;
      };
      auto load_kv = [&](const CUtensorMap* tm, uint64_t* full, uint64_t* empty, uint8_t* base, int& it, int t) {
        const int kv_r = list[t] * 64;  // key row within the unit
        uint8_t* dst = take(full, empty, base, it, L::kTile);
#pragma unroll
        for (int c = 0; c < NC; ++c) tc::tma_load_rows(dst + c * 8192, tm, full + (it % RS), 64 * c, kv_r, rt);
        ++it;
      };
      if (cnt > 0) load_kv(&tmK, k_full, k_empty, sK, kit, 0);
      if (has_lin) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint8_t* dst = take(v_full, v_empty, sV, vit, L::kTile);
          tc::tma_load_3d(dst, &tmH, v_full + (vit % RS), 64 * c, int(urow * D), 0);
          ++vit;
        }
      }
      for (int t = 0; t < cnt; ++t) {
        fts(dbg && t < 24, t);
        if (t + 1 < cnt) load_kv(&tmK, k_full, k_empty, sK, kit, t + 1);
        load_kv(&tmV, v_full, v_empty, sV, vit, t);
      }
      if (has_w) {
        const int h = int(u % p.H);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint8_t* dst = take(k_full, k_empty, sK, kit, L::kTile);
          tc::tma_load_3d(dst, &tmW, k_full + (kit % RS), 64 * c, h * D, 0);
          ++kit;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t sQa = tc::smem_u32(sQ), sKa = tc::smem_u32(sK), sVa = tc::smem_u32(sV);
    const uint32_t sPa = tc::smem_u32(sPX);
    constexpr uint32_t id_s = tc::idesc_bf16(64, 64, false, false);
    constexpr uint32_t id_o = tc::idesc_bf16(64, D, false, true);
    constexpr uint32_t id_c = tc::idesc_bf16(64, 64, false, true);  // X . (one 64-col chunk)
    int kit = 0, vit = 0;
    auto wait_slot = [&](uint64_t* full, uint32_t base, int it) -> uint32_t {
      const int s = it % RS;
      tc::mbar_wait(full + s, (it / RS) & 1);
      tc::tc_fence_after();
      return base + s * L::kTile;
    };
    // every lane runs the issue code (warp-uniform operands); one elected lane issues
    const uint64_t dQk = tc::desc_kmajor(sQa), dPk = tc::desc_kmajor(sPa);
    auto koff = [](int kk) { return uint32_t((kk >> 2) * 8192 + (kk & 3) * 32); };
    auto issue_s = [&](int t) {
      const uint32_t sk = wait_slot(k_full, sKa, kit);
      fts(dbg && lane == 0 && t < 24, 24 + t);
      const uint32_t ts = tS0 + 64 * (t & 1);
      const uint64_t dk = tc::desc_kmajor(sk);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        tc::mma_bf16_w(ts, tc::desc_add(dQk, koff(kk)), tc::desc_add(dk, koff(kk)), id_s, kk > 0);
      tc::mma_commit_w(k_empty + (kit % RS));
      tc::mma_commit_w(s_full + (t & 1));
      ++kit;
    };
    // tO[:, 64c:64c+64] (+)= X . chunk_c for the NC chunks at ring items it0.. (H_i or W)
    auto issue_chunks = [&](uint64_t* full, uint64_t* empty, uint32_t base, int& it, bool acc) {
      uint32_t sc[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) sc[c] = wait_slot(full, base, it + c);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const uint64_t dc = tc::desc_mnmajor(sc[c], 8192);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16_w(tO + 64 * c, tc::desc_add(dPk, koff(kk)), tc::desc_add(dc, kk * 2048), id_c, acc || kk > 0);
        tc::mma_commit_w(empty + ((it + c) % RS));
      }
      it += NC;
    };
    auto issue_pv = [&](int j) {
      tc::mbar_wait(p_full + (j & 1), (j >> 1) & 1);
      const uint32_t sv = wait_slot(v_full, sVa, vit);
      const uint64_t dp = tc::desc_add(dPk, (j & 1) * 8192), dv = tc::desc_mnmajor(sv, 8192);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc::mma_bf16_w(tO, tc::desc_add(dp, kk * 32), tc::desc_add(dv, kk * 2048), id_o, (j | kk) != 0);
      tc::mma_commit_w(v_empty + (vit % RS));
      tc::mma_commit_w(pv_done + (j & 1));
      ++vit;
    };
    tc::mbar_wait(q_full, 0);
    if (cnt > 0) issue_s(0);  // S(0) runs while the softmax warps build phi(Q_i)
    if (has_lin) {            // O-region <- phi(Q_i) H_i
      tc::mbar_wait(x_full, 0);
      fts(dbg && lane == 0, 102);
      issue_chunks(v_full, v_empty, sVa, vit, false);
      tc::mma_commit_w(lin_done);
    }
    for (int t = 1; t < cnt; ++t) {
      issue_s(t);
      issue_pv(t - 1);
    }
    if (cnt > 0) issue_pv(cnt - 1);
    if (has_w) {  // O-region (normalised O^s) += O^l W
      tc::mbar_wait(o_ready, 0);
      tc::tc_fence_after();
      issue_chunks(k_full, k_empty, sKa, kit, true);
      tc::mma_commit_w(proj_done);
    }
  } else {
    // ------------------------------------------------------------------ softmax / epilogue
    // Every lane works: row r = 16*q4 + (lane & 15) (the M=64 TMEM layout), and lanes 0-15 /
    // 16-31 take the two column halves through the 16x32bx2 TMEM shape; row reductions need
    // one shfl_xor(16).
    const int q4 = warp & 3;
    const int r = 16 * q4 + (lane & 15);
    const int hh = lane >> 4;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    constexpr int DH = D / 2;                    // columns per half row
    auto dcol = [&](int c0) { return hh * DH + c0; };  // first column of chunk c0 of my half
    if (has_lin) {  // Z_i -> smem (one coalesced row instead of per-thread dependent loads)
      const int tid = threadIdx.x - 64;
      if (tid < D) sZ[tid] = tc::load_sum3(p.Z + urow * 3 * D + tid, D);
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    uint32_t olp[DH / 2];  // my half row of O^l (bf16x2), kept for the projection
    tc::mbar_wait(q_full, 0);
    fts(dbg && threadIdx.x == 64, 96);

    // ---- marginal branch: phi(Q_i) into X, den = phi(q) . Z_i, then O^l = phi(q) H_i / den
    float den = 0.f;
    if (has_lin) {
      // my half row of Q_i -> f32 registers, then phi in place (feature_map.cpp:10-20)
      float x[DH];
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        const int col = dcol(c);
        const uint4 v = *reinterpret_cast<const uint4*>(sQ + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7));
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          x[c + 2 * e] = f.x;
          x[c + 2 * e + 1] = f.y;
        }
      }
      if (p.phi == 2) {  // per-row softmax over d: each exp computed once
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < DH; ++e) mx = fmaxf(mx, x[e]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        float se = 0.f;
#pragma unroll
        for (int e = 0; e < DH; ++e) {
          x[e] = __expf(x[e] - mx);
          se += x[e];
        }
        se += __shfl_xor_sync(0xffffffffu, se, 16);
        const float inv = 1.f / se;
#pragma unroll
        for (int e = 0; e < DH; ++e) x[e] *= inv;
      } else {
#pragma unroll
        for (int e = 0; e < DH; ++e) x[e] = phi_elem(p.phi, x[e]);
      }
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        const int col = dcol(c);
        {  // Z_i from smem as two 16-byte loads per 8 columns
          const float4 z0 = *reinterpret_cast<const float4*>(sZ + col), z1 = *reinterpret_cast<const float4*>(sZ + col + 4);
          den = fmaf(x[c], z0.x, den);
          den = fmaf(x[c + 1], z0.y, den);
          den = fmaf(x[c + 2], z0.z, den);
          den = fmaf(x[c + 3], z0.w, den);
          den = fmaf(x[c + 4], z1.x, den);
          den = fmaf(x[c + 5], z1.y, den);
          den = fmaf(x[c + 6], z1.z, den);
          den = fmaf(x[c + 7], z1.w, den);
        }
        *reinterpret_cast<uint4*>(sPX + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7)) =
            make_uint4(tc::pack_bf16(x[c], x[c + 1]), tc::pack_bf16(x[c + 2], x[c + 3]),
                       tc::pack_bf16(x[c + 4], x[c + 5]), tc::pack_bf16(x[c + 6], x[c + 7]));
      }
      den += __shfl_xor_sync(0xffffffffu, den, 16);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(x_full);
      fts(dbg && threadIdx.x == 64, 97);
      tc::mbar_wait(lin_done, 0);
      tc::tc_fence_after();
      fts(dbg && threadIdx.x == 64, 98);
      const float inv_den = den != 0.f ? 1.f / den : 0.f;  // den == 0 -> zero row (forward.cpp:136)
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t a[32];
        tc::tmem_ld32_x2<DH>(tO + lane_base + c0, a);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 2)
          olp[(c0 + e) >> 1] = tc::pack_bf16(__uint_as_float(a[e]) * inv_den, __uint_as_float(a[e + 1]) * inv_den);
      }
    } else {
#pragma unroll
      for (int e = 0; e < DH / 2; ++e) olp[e] = 0u;
    }

    fts(dbg && threadIdx.x == 64, 99);
    // ---- critical branch: online softmax over the ascending critical list
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < cnt; ++t) {
      tc::mbar_wait(s_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      fts(dbg && threadIdx.x == 64 && t < 24, 48 + t);
      uint32_t sa[32];
      tc::tmem_ld32_x2<32>(tS0 + 64 * (t & 1) + lane_base, sa);  // my 32 of the 64 scores
      tc::tmem_ld_wait();
      if (p.kv_last < 64 && list[t] == p.Tn - 1) {  // ragged N: keys past N get no weight
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (32 * hh + e >= p.kv_last) sa[e] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 32; ++e) mx = fmaxf(mx, __uint_as_float(sa[e]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16)) * p.scale_log2;
      const float m_new = fmaxf(m_used, mx);
      const bool need = t > 0 && m_new > m_used + 8.f;
      if (t == 0) m_used = m_new;
      if (__any_sync(0xffffffffu, need)) {  // rescale O and l (all previous PVs must be done)
        tc::mbar_wait(pv_done + ((t - 1) & 1), ((t - 1) >> 1) & 1);
        tc::tc_fence_after();
        const float alpha = need ? ex2(m_used - m_new) : 1.f;
        if (need) {
          l *= alpha;
          m_used = m_new;
        }
#pragma unroll 1
        for (int c0 = 0; c0 < DH; c0 += 32) {
          uint32_t o[32];
          tc::tmem_ld32_x2<DH>(tO + lane_base + c0, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tc::tmem_st32_x2<DH>(tO + lane_base + c0, o);
        }
        tc::tmem_st_wait();
      }
      if (t >= 2) tc::mbar_wait(pv_done + (t & 1), ((t - 2) >> 1) & 1);  // P buffer free
      const float sc = p.scale_log2;
      float ps = 0.f;
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float x0 = __uint_as_float(sa[e]) * sc - m_used, x1 = __uint_as_float(sa[e + 1]) * sc - m_used;
        const float p0 = tc::poly_slot(e, SLAB_FWD_POLY) ? tc::ex2_poly(x0) : ex2(x0);
        const float p1 = tc::poly_slot(e + 1, SLAB_FWD_POLY) ? tc::ex2_poly(x1) : ex2(x1);
        ps += p0 + p1;
        pk[e >> 1] = tc::pack_bf16(p0, p1);
      }
      l += ps + __shfl_xor_sync(0xffffffffu, ps, 16);
      uint8_t* prow = sPX + (t & 1) * 8192;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(prow + tc::sw128_off(r, 4 * hh + c)) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + (t & 1));
      fts(dbg && threadIdx.x == 64 && t < 24, 72 + t);
    }

    fts(dbg && threadIdx.x == 64, 100);
    // ---- finalize O^s, lse (forward.cpp:68-78); stage O^s / O^l for the projection
    if (cnt > 0) {
      tc::mbar_wait(pv_done + ((cnt - 1) & 1), ((cnt - 1) >> 1) & 1);
      tc::tc_fence_after();
    }
    fts(dbg && threadIdx.x == 64, 103);
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < DH; c0 += 32) {
      uint32_t o[32];
      if (cnt > 0) {
        tc::tmem_ld32_x2<DH>(tO + lane_base + c0, o);
        tc::tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * inv_l);
#pragma unroll
      for (int e = 0; e < 32; e += 8) {
        uint4 v;
        v.x = tc::pack_bf16(__uint_as_float(o[e]), __uint_as_float(o[e + 1]));
        v.y = tc::pack_bf16(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
        v.z = tc::pack_bf16(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5]));
        v.w = tc::pack_bf16(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7]));
        const int col = dcol(c0) + e;  // staged in the dead Q tile, written by TMA below
        tc::sts_u4(tc::smem_u32(sQ) + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7), v);
      }
      if (has_w) tc::tmem_st32_x2<DH>(tO + lane_base + c0, o);
    }
    if (hh == 0) {  // the caller's lse row (none past a ragged N)
      const long long cr = rm.row((long long)i * 64 + r);
      if (cr >= 0) p.lse[cr] = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994531f : kLseSentinel;
    }
    if (has_w) {
      tc::tmem_st_wait();
      // X <- O^l (bf16), the A operand of O^l W: my half row, from registers
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        const int col = dcol(c);
        *reinterpret_cast<uint4*>(sPX + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7)) =
            make_uint4(olp[c >> 1], olp[(c >> 1) + 1], olp[(c >> 1) + 2], olp[(c >> 1) + 3]);
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_ready);
      fts(dbg && threadIdx.x == 64, 104);
      tc::mbar_wait(proj_done, 0);
      tc::tc_fence_after();
      fts(dbg && threadIdx.x == 64, 105);
#pragma unroll 1
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t o[32];
        tc::tmem_ld32_x2<DH>(tO + lane_base + c0, o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 v;
          v.x = tc::pack_bf16(__uint_as_float(o[e]), __uint_as_float(o[e + 1]));
          v.y = tc::pack_bf16(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
          v.z = tc::pack_bf16(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5]));
          v.w = tc::pack_bf16(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7]));
          const int col = dcol(c0) + e;  // staged in the idle V ring, written by TMA below
          tc::sts_u4(tc::smem_u32(sV) + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7), v);
        }
      }
    } else {  // no projection: O^l goes to its staging tile (the P buffers, idle after the last PV)
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        const int col = dcol(c);
        tc::sts_u4(tc::smem_u32(sPX) + (col >> 6) * 8192 + tc::sw128_off(r, (col >> 3) & 7),
                   make_uint4(olp[c >> 1], olp[(c >> 1) + 1], olp[(c >> 1) + 2], olp[(c >> 1) + 3]));
      }
    }
    // O^s (Q tile), O^l (X tile) and O (V ring) leave as whole [64 x 64] boxes: coalesced, where
    // row-per-thread 16-byte stores cost 0.075 ms of the kernel's 0.57
    tc::fence_proxy_async();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 64) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        tc::tma_store_rows(&tmOs, sQ + c * 8192, 64 * c, i * 64, rt);
        tc::tma_store_rows(&tmOl, sPX + c * 8192, 64 * c, i * 64, rt);
        if (has_w) tc::tma_store_rows(&tmO, sV + c * 8192, 64 * c, i * 64, rt);
      }
      tc::bulk_commit();
      tc::bulk_wait_read<0>();  // smem may be released; the writes complete with the grid
    }
  }
  fts(dbg && threadIdx.x == 64, 101);
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

template <int D>
void launch_t(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
              const __nv_bfloat16* Hb, FwdParams p, cudaStream_t st) {
  CUtensorMap tq, tk, tv, th, tw;
  make_tmap_rows(&tq, q, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tk, k, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_rows(&tv, v, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_bf16(&th, Hb, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);
  if (w)
    make_tmap_bf16(&tw, w, D, uint64_t(Dm.H) * D, 1, D, 0, D);
  else
    tw = th;
  CUtensorMap to, tos, tol;  // output boxes [64 rows][64 cols]
  make_tmap_rows(&tos, p.o_s, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tol, p.o_l, D, Dm.U, Dm.N, p.rl, 64);
  if (p.o)
    make_tmap_rows(&to, p.o, D, Dm.U, Dm.N, p.rl, 64);
  else
    to = tos;
  auto kern = k_attn_fwd<D>;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdLayout<D>::kBytes));
  launch_pdl(kern, dim3(Dm.Tm, unsigned(Dm.U)), 192, FwdLayout<D>::kBytes, st, tq, tk, tv, th, tw, to, tos, tol, p);
  check_launch("k_attn_fwd", st);
}

}  // namespace

void launch_attn_fwd(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                     void* o, void* o_s, void* o_l, float* lse, const StateBufs& s, cudaStream_t st) {
  FwdParams p{};
  p.crit_cnt = s.crit_cnt;
  p.crit_idx = s.crit_idx;
  p.marg_cnt = s.marg_cnt;
  p.Z = s.Z;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.o_s = static_cast<__nv_bfloat16*>(o_s);
  p.o_l = static_cast<__nv_bfloat16*>(o_l);
  p.lse = lse;
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.scale_log2 = float(Dm.inv_sqrt_d * 1.4426950408889634);
  p.has_w = (w != nullptr && o != nullptr) ? 1 : 0;
  p.phi = Dm.phi;
  p.kv_last = int(Dm.Nk_valid - (long long)(Dm.Tn - 1) * 64);
  p.rl = Dm.rl;
  // SLA_B200_FWD_PAIR=2: the persistent key-block-pair kernel (attn_fwd_pp.cu) at d = 128.  Off
  // by default: measured 0.86 ms against 0.527 for this kernel (C3), see DESIGN.md section 8.
  static const int pair = [] {
    const char* e = getenv("SLA_B200_FWD_PAIR");
    return e ? atoi(e) : 0;
  }();
  if (Dm.d == 128 && pair == 2)
    launch_attn_fwd_pp(Dm, q, k, v, w, o, o_s, o_l, lse, s, st);
  else if (Dm.d == 128)
    launch_t<128>(Dm, q, k, v, w, s.Hb, p, st);
  else
    launch_t<64>(Dm, q, k, v, w, s.Hb, p, st);
}

}  // namespace slab

#ifdef SLAB_TIMELINE  // diagnostic accessors: timeline builds only (profiles/ctaprof.py)
extern "C" int sla_b200_diag_fwd_timeline(long long* host128) {
  return cudaMemcpyFromSymbol(host128, slab::g_fwd_ts, 128 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
#endif
