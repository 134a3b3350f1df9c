// attn_fwd_pp.cu -- K5 for d = 128, persistent: one CTA per SM walks a contiguous range of
// query blocks, key-block pairs on the tensor core, the epilogue of block n overlapped with the
// critical loop of block n+1.
//
// Algorithm as attn_fwd.cu / attn_fwd_pair.cu (forward.cpp:29-79 critical loop, :81-172 block
// classes, :187-195 projection).  Shapes as attn_fwd_pair.cu: S = Q_i [K_j1; K_j2]^T (M = 64,
// N = 128, 8 x 64 cycles) and O^T += [V_j1; V_j2]^T P^T (M = d, N = 64, 8 x 50 cycles): 456
// tensor cycles per critical tile instead of 656.  What the two-CTA pair kernel lacked was
// buffering (one S buffer, one P buffer, a 5-slot ring: every step waited on the previous one,
// DESIGN.md section 8); one CTA per SM owns all 512 TMEM columns and 227 KB of smem:
//   TMEM  S[2] (128 cols each, double-buffered across pairs), O^T[2] (64 each, alternating query
//         blocks: block n+1 accumulates while block n's epilogue reads), O_l^T (64)
//   smem  Q[2] (per block parity; O^s / O staging at its epilogue), P[2] (per pair parity), X
//         (phi(Q_i), then O^l staging), a 9-slot ring of 16 KB items (K half-pairs, V tiles, and
//         per block H_i's and W's 64-column chunks)
// Warps (480 threads): 0 TMA producer; 1 loop MMA issuer (S one pair ahead of PV, across block
// boundaries); 2-9 softmax (online softmax per pair, 32 scores per thread, lazy rescale, row
// statistics and lse at the end of a block); 10-13 epilogue (phi(Q_i) and den for the linear
// branch, O^s = O^T / l, O^l = O_l^T / den, O = O^s + O^l W, transposed through smem into TMA
// stores); 14 epilogue MMA issuer
// (O_l^T = H_i^T phi(Q_i)^T, the projection).  Every per-block barrier is signalled and waited
// exactly once per block whatever the block's class counts, so the phase bookkeeping is uniform.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

#ifdef SLAB_TIMELINE
static __device__ long long g_fpp_ts[256];
#endif
#ifdef SLAB_PP_DEBUG  // progress words in host-mapped memory, readable while the kernel runs
static __device__ volatile int* g_pp_dbg;
#endif

namespace {

constexpr int kD = 128;
constexpr int kThreads = 480;
constexpr int kRS = 9;  // ring slots
#ifndef SLAB_PP_POLY
#define SLAB_PP_POLY 0  // measured: 0 0.817 ms, 3 0.872, 2 0.907 (and a parity failure at 3)
#endif

struct PPLayout {
  static constexpr int kTile = 16384;
  static constexpr int oQ = 0;                  // 2 x Q
  static constexpr int oP = oQ + 2 * kTile;     // 2 x P
  static constexpr int oX = oP + 2 * kTile;     // phi(Q) / O^l
  static constexpr int oRing = oX + kTile;      // kRS slots
  static constexpr int oBar = oRing + kRS * kTile;
  static constexpr int oRowL = oBar + 512;      // float [64]  1/l of the block in its epilogue
  static constexpr int oDen = oRowL + 256;      // float [64]  1/den
  static constexpr int oAlpha = oDen + 256;     // float [64]  rescale factors
  static constexpr int oZ = oAlpha + 256;       // float [128] Z_i
  static constexpr int oRmax = oZ + 512;        // float [2 pair parities][2 subs][64] partial row maxima
  static constexpr int oLpart = oRmax + 1024;   // float [64] the second warp's partial row sums
  static constexpr int kBytes = oLpart + 256;
  static_assert(kBytes <= 232448, "smem");
};

struct PPParams {
  const int* crit_cnt;
  const int* crit_idx;
  const int* marg_cnt;
  const float* Z;
  float* lse;
  long long N;
  int Tm, Tn, H;
  float scale_log2;
  int has_w;
  int phi;
  int kv_last;
  long long items;  // U * Tm query blocks
  RowLayout rl;
};

__device__ __forceinline__ void fpp_mark(bool on, int slot) {
#ifdef SLAB_TIMELINE
  if (on) g_fpp_ts[slot] = clock64();
#else
  (void)on;
  (void)slot;
#endif
}
// role word: [cta * 8 + role] = (block << 20) | (pair << 8) | step
__device__ __forceinline__ void dbgw(int role, int n, long long g, int step) {
#ifdef SLAB_PP_DEBUG
  g_pp_dbg[blockIdx.x * 8 + role] = (n << 20) | (int(g & 0xfff) << 8) | step;
  __threadfence_system();
#else
  (void)role;
  (void)n;
  (void)g;
  (void)step;
#endif
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void sts_f(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ bool bar_red_or(int id, int n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred pi, po;\n setp.ne.u32 pi, %1, 0;\n bar.red.or.pred po, %2, %3, pi;\n"
      " selp.u32 %0, 1, 0, po;\n}\n"
      : "=r"(r)
      : "r"(uint32_t(v)), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// element (row, col) of a [64 rows][128 cols] bf16 tile stored as two K-major SW128 chunks
__device__ __forceinline__ uint32_t elem_off(int row, int col) {
  return uint32_t(col >> 6) * 8192u + tc::sw128_off(uint32_t(row), uint32_t((col & 63) >> 3)) + uint32_t(col & 7) * 2u;
}
__device__ __forceinline__ uint32_t par(long long k) { return uint32_t(k & 1); }

// One query block's schedule.  Ring items in producer order: K(0), then K(p) and V(p-1) for
// p >= 1 (the issuer runs S one pair ahead of PV), V(np-1), then H_i's and W's two chunks each
// (consumed by the epilogue issuer).
struct Blk {
  long long u;
  int i, cnt, np, last_n;
  bool lin, w;
  const int* list;
  __device__ __forceinline__ void load(const PPParams& p, long long qb) {
    u = qb / p.Tm;
    i = int(qb - u * p.Tm);
    const long long urow = qb;
    cnt = p.crit_cnt[urow];
    list = p.crit_idx + urow * p.Tn;
    lin = p.marg_cnt[urow] > 0;
    w = p.has_w != 0;
    np = (cnt + 1) >> 1;
    last_n = (cnt & 1) ? 1 : 2;
  }
  __device__ __forceinline__ int tiles(int pp) const { return pp + 1 < np ? 2 : last_n; }
  __device__ __forceinline__ int kidx(int pp) const { return pp == 0 ? 0 : 4 * pp - 2; }
  __device__ __forceinline__ int vidx(int pp) const {
    if (pp + 2 <= np) return 4 * pp + 4;
    return np == 1 ? 2 : 4 * np - 2;
  }
  __device__ __forceinline__ int hidx() const { return np == 0 ? 0 : vidx(np - 1) + last_n; }
  __device__ __forceinline__ int widx() const { return hidx() + (lin ? 2 : 0); }
  __device__ __forceinline__ int total() const { return widx() + (w ? 2 : 0); }
};

__global__ void __launch_bounds__(kThreads, 1)
    k_attn_fwd_pp(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmH,
                  const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
                  const __grid_constant__ CUtensorMap tmOs, const __grid_constant__ CUtensorMap tmOl, PPParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = PPLayout;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* full = bars + 0;         // [kRS]
  uint64_t* empty = bars + 9;        // [kRS]
  uint64_t* q_full = bars + 18;      // [2] per block parity
  uint64_t* q_free = bars + 20;      // [2]
  uint64_t* s_full = bars + 22;      // [2] per pair parity
  uint64_t* s_free = bars + 24;      // [2]
  uint64_t* p_full = bars + 26;      // [2]
  uint64_t* pv_done = bars + 28;     // [2]
  uint64_t* ot_done = bars + 30;     // [2] per block parity
  uint64_t* ot_free = bars + 32;     // [2]
  uint64_t* stats = bars + 34;       // softmax wrote the block's 1/l
  uint64_t* stats_free = bars + 35;  // the epilogue read it
  uint64_t* x_full = bars + 36;
  uint64_t* lin_done = bars + 37;
  uint64_t* o_ready = bars + 38;
  uint64_t* proj_done = bars + 39;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 44);
  const uint32_t aS = tc::smem_u32(smem);
  const uint32_t aQ = aS + L::oQ, aP = aS + L::oP, aX = aS + L::oX, aR = aS + L::oRing;
  const uint32_t aRowL = aS + L::oRowL, aDen = aS + L::oDen, aAlpha = aS + L::oAlpha, aZ = aS + L::oZ;
  const uint32_t aRmax = aS + L::oRmax, aLpart = aS + L::oLpart;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // query blocks blockIdx.x + n * gridDim.x: at any time the grid works on ~148 consecutive
  // blocks of one (batch, head) unit, whose K / V stay L2-resident (a contiguous range per CTA
  // would touch every unit at once: 12 x 16.8 MB of K / V at C3, more than L2)
  const int nblk = int((p.items - blockIdx.x + gridDim.x - 1) / gridDim.x);
  auto QB = [&](long long n) { return (long long)blockIdx.x + n * gridDim.x; };
  const bool dbg = blockIdx.x == 7;
  fpp_mark(dbg && threadIdx.x == 0, 255);

  if (warp == 0) {
    if (lane == 0) {
      if (aS & 1023u) __trap();  // SW128 tiles need a 1024-aligned base
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::tma_prefetch(&tmV);
      for (int s = 0; s < kRS; ++s) {
        tc::mbar_init(full + s, 1);
        tc::mbar_init(empty + s, 1);
      }
      for (int s = 0; s < 2; ++s) {
        tc::mbar_init(q_full + s, 1);
        tc::mbar_init(q_free + s, 1);
        tc::mbar_init(s_full + s, 1);
        tc::mbar_init(s_free + s, 8);
        tc::mbar_init(p_full + s, 8);
        tc::mbar_init(pv_done + s, 1);
        tc::mbar_init(ot_done + s, 1);
        tc::mbar_init(ot_free + s, 1);
      }
      tc::mbar_init(stats, 8);
      tc::mbar_init(stats_free, 1);
      tc::mbar_init(x_full, 4);
      tc::mbar_init(lin_done, 1);
      tc::mbar_init(o_ready, 4);
      tc::mbar_init(proj_done, 1);
      tc::fence_barrier_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto tS = [&](long long g) { return tmem + 128u * uint32_t(g & 1); };
  auto tOT = [&](int n) { return tmem + 256u + 64u * uint32_t(n & 1); };
  const uint32_t tLT = tmem + 384;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      long long r = 0;  // ring items issued
      auto take = [&](int bytes) -> uint32_t {
        const int s = int(r % kRS);
        dbgw(1, int(r >> 8), r, 3);
        tc::mbar_wait(empty + s, uint32_t((r / kRS) & 1) ^ 1u);
        dbgw(1, int(r >> 8), r, 4);
        fpp_mark(dbg && r < 32, 160 + int(r));  // ring item r issued
        tc::mbar_expect_tx(full + s, bytes);
        dbgw(1, int(r >> 8), r, 5);
        return aR + uint32_t(s) * L::kTile;
      };
      Blk b, bn;
      if (nblk > 0) bn.load(p, QB(0));
      for (int n = 0; n < nblk; ++n) {
        b = bn;
        if (n + 1 < nblk) bn.load(p, QB(n + 1));  // the next block's counts, ahead of need
        const RowTma rt = row_tma(p.rl, b.u, p.N);
        // key rows of pair pp: list[2pp], list[2pp + 1], fetched one pair ahead of their K load
        // (a dependent global load per item would put ~600 cycles of L2 latency on every issue)
        auto rows_of = [&](int pp, int& r1, int& r2) {
          r1 = pp < b.np ? b.list[2 * pp] * 64 : 0;
          r2 = pp < b.np && b.tiles(pp) == 2 ? b.list[2 * pp + 1] * 64 : 0;
        };
        int a1, a2, b1, b2;  // rows of pair pp-1 (its V pending) and pair pp (its K next)
        rows_of(0, a1, a2);
        rows_of(1, b1, b2);
        dbgw(0, n, r, 1);
        if (n >= 2) tc::mbar_wait(q_free + (n & 1), uint32_t(((n >> 1) - 1) & 1));
        dbgw(0, n, r, 2);
        tc::mbar_expect_tx(q_full + (n & 1), L::kTile);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tc::tma_load_rows(smem + L::oQ + (n & 1) * L::kTile + c * 8192, &tmQ, q_full + (n & 1), 64 * c, b.i * 64, rt);
        auto load_k = [&](int pp, int r1, int r2) {
          const int nt = b.tiles(pp);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t dst = take(nt * 8192);
            uint64_t* fb = full + r % kRS;
            tc::tma_load_rows(smem + (dst - aS), &tmK, fb, 64 * c, r1, rt);
            if (nt == 2) tc::tma_load_rows(smem + (dst - aS) + 8192, &tmK, fb, 64 * c, r2, rt);
            ++r;
          }
        };
        auto load_v = [&](int pp, int r1, int r2) {
          const int nt = b.tiles(pp);
          for (int t = 0; t < nt; ++t) {
            const uint32_t dst = take(L::kTile);
            const int row = t ? r2 : r1;
#pragma unroll
            for (int c = 0; c < 2; ++c) tc::tma_load_rows(smem + (dst - aS) + c * 8192, &tmV, full + r % kRS, 64 * c, row, rt);
            ++r;
          }
        };
        // K(0), then K(p) and V(p-1): a V item follows the K item of the next pair
        if (b.np >= 1) load_k(0, a1, a2);
        for (int pp = 1; pp < b.np; ++pp) {
          int d1, d2;
          rows_of(pp + 1, d1, d2);  // prefetch pair pp+1
          load_k(pp, b1, b2);
          load_v(pp - 1, a1, a2);
          a1 = b1; a2 = b2;
          b1 = d1; b2 = d2;
        }
        if (b.np >= 1) load_v(b.np - 1, a1, a2);
        // H_i and W: chunk 0 in the lower of the two slots (positive LBO)
        auto load_chunks = [&](const CUtensorMap* tm, int row) {
          const bool sw = (r + 1) % kRS < r % kRS;
          for (int t = 0; t < 2; ++t) {
            const uint32_t dst = take(L::kTile);
            tc::tma_load_3d(smem + (dst - aS), tm, full + r % kRS, 64 * (t ^ int(sw)), row, 0);
            ++r;
          }
        };
        if (b.lin) load_chunks(&tmH, int(QB(n) * kD));
        if (b.w) load_chunks(&tmW, int(b.u % p.H) * kD);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ loop MMA issuer
    constexpr uint32_t id_s2 = tc::idesc_bf16(64, 128, false, false);
    constexpr uint32_t id_s1 = tc::idesc_bf16(64, 64, false, false);
    constexpr uint32_t id_t = tc::idesc_bf16(128, 64, true, false);
    const uint64_t dR = tc::desc_kmajor(aR), dP0 = tc::desc_kmajor(aP);
    auto koff = [](int kk) { return uint32_t((kk >> 2) * 8192 + (kk & 3) * 32); };
    // S cursor (block sn, pair sp, global pair sg, ring base sbase) runs ahead of the PV cursor
    Blk sb, pb;
    int sn = 0, sp = 0;
    long long sg = 0, sbase = 0;
    bool s_live = nblk > 0;
    if (s_live) sb.load(p, QB(0));
    auto s_settle = [&]() {  // skip blocks without pairs (their Q phase is still waited, in order)
      while (s_live && sp >= sb.np) {
        if (sb.np == 0) tc::mbar_wait(q_full + (sn & 1), uint32_t((sn >> 1) & 1));
        sbase += sb.total();
        ++sn;
        sp = 0;
        if (sn >= nblk) {
          s_live = false;
          break;
        }
        sb.load(p, QB(sn));
      }
    };
    s_settle();
    auto issue_s = [&]() {
      dbgw(2, sn, sg, 1);
      if (sg >= 2) tc::mbar_wait(s_free + par(sg), uint32_t(((sg >> 1) - 1) & 1));
      dbgw(2, sn, sg, 2);
      if (sp == 0) tc::mbar_wait(q_full + (sn & 1), uint32_t((sn >> 1) & 1));
      dbgw(2, sn, sg, 3);
      const long long n0 = sbase + sb.kidx(sp);
      const int s0 = int(n0 % kRS), s1 = int((n0 + 1) % kRS);
      tc::mbar_wait(full + s0, uint32_t((n0 / kRS) & 1));
      tc::mbar_wait(full + s1, uint32_t(((n0 + 1) / kRS) & 1));
      tc::tc_fence_after();
      fpp_mark(dbg && lane == 0 && sg < 32, 32 + int(sg));  // S(g) issued
      const uint64_t dQ = tc::desc_kmajor(aQ + uint32_t(sn & 1) * L::kTile);
      const uint32_t id = sb.tiles(sp) == 2 ? id_s2 : id_s1;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t a = tc::desc_add(dQ, uint32_t((kk >> 2) * 8192 + (kk & 3) * 32));
        const uint64_t bdesc = tc::desc_add(dR, uint32_t(((kk >> 2) ? s1 : s0) * L::kTile + (kk & 3) * 32));
        tc::mma_bf16_w(tS(sg), a, bdesc, id, kk > 0);
      }
      tc::mma_commit_w(empty + s0);
      tc::mma_commit_w(empty + s1);
      tc::mma_commit_w(s_full + par(sg));
      ++sp;
      ++sg;
      s_settle();
    };
    long long pg = 0, pbase = 0;
    for (int n = 0; n < nblk; ++n) {
      pb.load(p, QB(n));
      dbgw(3, n, pg, 1);
      if (n >= 2) tc::mbar_wait(ot_free + (n & 1), uint32_t(((n >> 1) - 1) & 1));
      for (int pp = 0; pp < pb.np; ++pp, ++pg) {
        while (s_live && sg <= pg + 1) issue_s();
        dbgw(3, n, pg, 2);
        tc::mbar_wait(p_full + par(pg), uint32_t((pg >> 1) & 1));
        dbgw(3, n, pg, 3);
        const int nt = pb.tiles(pp);
        const long long n0 = pbase + pb.vidx(pp);
        const int s0 = int(n0 % kRS), s1 = int((n0 + 1) % kRS);
        tc::mbar_wait(full + s0, uint32_t((n0 / kRS) & 1));
        if (nt == 2) tc::mbar_wait(full + s1, uint32_t(((n0 + 1) / kRS) & 1));
        tc::tc_fence_after();
        fpp_mark(dbg && lane == 0 && pg < 32, 64 + int(pg));  // PV(g) issued
        const uint64_t dv0 = tc::desc_mnmajor(aR + uint32_t(s0) * L::kTile, 8192);
        const uint64_t dv1 = tc::desc_mnmajor(aR + uint32_t(s1) * L::kTile, 8192);
        const uint64_t dP = tc::desc_add(dP0, uint32_t(pg & 1) * L::kTile);
        for (int kk = 0; kk < 4 * nt; ++kk)
          tc::mma_bf16_w(tOT(n), tc::desc_add((kk >> 2) ? dv1 : dv0, (kk & 3) * 2048), tc::desc_add(dP, koff(kk)), id_t,
                         (pp | kk) != 0);
        tc::mma_commit_w(empty + s0);
        if (nt == 2) tc::mma_commit_w(empty + s1);
        tc::mma_commit_w(pv_done + par(pg));
      }
      tc::mma_commit_w(ot_done + (n & 1));  // every PV of block n (none if it has no pair)
      pbase += pb.total();
    }
  } else if (warp >= 2 && warp < 10) {
    // ------------------------------------------------------------------ softmax (8 warps)
    // Two warps per TMEM sub-partition: warp w reads lanes 32 (w % 4).. and column quarter
    // `sub` of each 64-column tile; a row's max is combined over its 4 threads (shfl 16 within the
    // warp, smem with the partner warp)
    const int q4 = warp & 3;
    const int sub = (warp - 2) >> 2;
    const int r = 16 * q4 + (lane & 15);
    const int hh = lane >> 4;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const float sc = p.scale_log2;
    const int pair_bar = 3 + q4;  // this warp and its partner (64 threads)
    long long g = 0;
    Blk b;
    for (int n = 0; n < nblk; ++n) {
      b.load(p, QB(n));
      float m_used = -INFINITY, l = 0.f;
      for (int pp = 0; pp < b.np; ++pp, ++g) {
        if (threadIdx.x == 64) dbgw(4, n, g, 1);
        tc::mbar_wait(s_full + par(g), uint32_t((g >> 1) & 1));
        if (threadIdx.x == 64) dbgw(4, n, g, 2);
        fpp_mark(dbg && threadIdx.x == 64 && g < 32, 96 + int(g));  // S(g) seen
        tc::tc_fence_after();
        uint32_t sa0[32];
        tc::tmem_ld32_x2<64>(tS(g) + lane_base + 32 * sub, sa0);
        tc::tmem_ld_wait();
        const bool stp = dbg && threadIdx.x == 64 && g >= 4 && g < 8;
        const int sbase_ = 128 + 8 * int(g - 4);
        fpp_mark(stp, sbase_ + 0);  // S loaded
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_free + par(g));
        float sa[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) sa[e] = __uint_as_float(sa0[e]);
        const bool live = b.tiles(pp) == 2 || hh == 0;
        const int kvalid = !live ? 0 : ((p.kv_last < 64 && b.list[2 * pp + hh] == p.Tn - 1) ? p.kv_last - 32 * sub : 32);
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (kvalid == 32) {  // the common case: no masked column
#pragma unroll
          for (int e = 0; e < 32; ++e) m4[e & 3] = fmaxf(m4[e & 3], sa[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) m4[e & 3] = fmaxf(m4[e & 3], e < kvalid ? sa[e] : -INFINITY);
        }
        float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const uint32_t rmx = aRmax + uint32_t(((g & 1) * 2 + sub) * 256 + 4 * r);
        if (hh == 0) sts_f(rmx, mx);
        fpp_mark(stp, sbase_ + 1);  // own max
        bar_sync(pair_bar, 64);
        fpp_mark(stp, sbase_ + 2);  // partner max
        mx = fmaxf(mx, lds_f(rmx + (sub ? -256 : 256))) * sc;
        const float m_new = fmaxf(m_used, mx);
        const bool need = pp > 0 && m_new > m_used + 8.f;
        const float m_fin = (pp == 0 || need) ? m_new : m_used;
        float ps0 = 0.f, ps1 = 0.f;
        uint32_t pk[16];
        // every SLAB_PP_POLY-th exponential on the FMA pipe (the MUFU's 16 / clock / SM is the
        // softmax stage's throughput limit: 8192 exponentials per pair)
        auto pexp = [&](int e) {
          const float x = sa[e] * sc - m_fin;
          return tc::poly_slot(e, SLAB_PP_POLY) ? tc::ex2_poly(x) : ex2(x);
        };
        if (kvalid == 32) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float p0 = pexp(e), p1 = pexp(e + 1);
            ps0 += p0;
            ps1 += p1;
            pk[e >> 1] = tc::pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float p0 = e < kvalid ? ex2(sa[e] * sc - m_fin) : 0.f;
            const float p1 = e + 1 < kvalid ? ex2(sa[e + 1] * sc - m_fin) : 0.f;
            ps0 += p0;
            ps1 += p1;
            pk[e >> 1] = tc::pack_bf16(p0, p1);
          }
        }
        fpp_mark(stp, sbase_ + 3);  // exps done
        if (g >= 2) tc::mbar_wait(pv_done + par(g), uint32_t(((g >> 1) - 1) & 1));  // P buffer g&1 is free
        fpp_mark(stp, sbase_ + 4);  // P buffer free
        if (bar_red_or(1, 256, need)) {  // some row's max grew by more than 2^8: rescale O^T columns
          // PV(g-1) (same block: pp > 0) must have landed in O^T before it is scaled
          tc::mbar_wait(pv_done + par(g - 1), uint32_t(((g - 1) >> 1) & 1));
          tc::tc_fence_after();
          const float alpha = need ? ex2(m_used - m_new) : 1.f;
          if (need) l *= alpha;
          if (hh == 0 && sub == 0) sts_f(aAlpha + 4 * r, alpha);
          bar_sync(1, 256);
          uint32_t o[32];  // O^T lanes = output columns, my query columns 32 sub ..
          tc::tmem_ld32(tOT(n) + lane_base + 32 * sub, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 al = tc::lds_f4(aAlpha + 4 * (32 * sub + e));
            o[e] = __float_as_uint(__uint_as_float(o[e]) * al.x);
            o[e + 1] = __float_as_uint(__uint_as_float(o[e + 1]) * al.y);
            o[e + 2] = __float_as_uint(__uint_as_float(o[e + 2]) * al.z);
            o[e + 3] = __float_as_uint(__uint_as_float(o[e + 3]) * al.w);
          }
          tc::tmem_st32(tOT(n) + lane_base + 32 * sub, o);
          tc::tmem_st_wait();
          bar_sync(1, 256);
        }
        fpp_mark(stp, sbase_ + 5);  // vote done
        m_used = m_fin;
        const float ps = ps0 + ps1;
        l += ps + __shfl_xor_sync(0xffffffffu, ps, 16);
        const uint32_t prow = aP + uint32_t(g & 1) * L::kTile + uint32_t(hh) * 8192u;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tc::sts_u4(prow + tc::sw128_off(uint32_t(r), uint32_t(4 * sub + c)),
                     make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
        fpp_mark(stp, sbase_ + 6);  // P stored
        tc::fence_proxy_async();
        fpp_mark(stp, sbase_ + 7);  // fenced
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full + par(g));
        fpp_mark(dbg && threadIdx.x == 64 && g < 32, int(g));  // P(g) stored
      }
      // block statistics for the epilogue (the two partial row sums), the caller's lse
      if (threadIdx.x == 64) dbgw(4, n, g, 3);
      if (n >= 1) tc::mbar_wait(stats_free, uint32_t((n - 1) & 1));
      if (threadIdx.x == 64) dbgw(4, n, g, 4);
      if (sub == 1 && hh == 0) sts_f(aLpart + 4 * r, l);
      bar_sync(1, 256);
      if (sub == 0 && hh == 0) {
        l += lds_f(aLpart + 4 * r);
        sts_f(aRowL + 4 * r, l > 0.f ? 1.f / l : 0.f);
        const long long cr = row_map(p.rl, b.u, p.N).row((long long)b.i * 64 + r);
        if (cr >= 0) p.lse[cr] = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994531f : kLseSentinel;
      }
      bar_sync(1, 256);  // aLpart is rewritten only after the next block's loop
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(stats);
    }
  } else if (warp >= 10 && warp < 14) {
    // ------------------------------------------------------------------ epilogue
    const int q4 = warp & 3;
    const int r = 16 * q4 + (lane & 15);  // row phases (phi(Q))
    const int hh = lane >> 4;
    const int a = 32 * q4 + lane;         // transposed phases: output column
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const int tid = threadIdx.x - 320;
    const bool leader = tid == 0;
    Blk b;
    for (int n = 0; n < nblk; ++n) {
      b.load(p, QB(n));
      const RowTma rt = row_tma(p.rl, b.u, p.N);
      const uint32_t aQn = aQ + uint32_t(n & 1) * L::kTile;
      // ---- linear branch inputs: phi(Q_i) -> X, 1/den (X is free: the previous block's O^l store
      // has been read, see the end of this loop)
      if (leader) dbgw(5, n, 0, 1);
      tc::mbar_wait(q_full + (n & 1), uint32_t((n >> 1) & 1));
      if (leader) dbgw(5, n, 0, 2);
      if (b.lin) {
        if (tid < kD) sts_f(aZ + 4 * tid, tc::load_sum3(p.Z + QB(n) * 3 * kD + tid, kD));
        bar_sync(2, 128);
        auto q8 = [&](int c, float (&f)[8]) {
          const uint4 v = *reinterpret_cast<const uint4*>(smem + (aQn - aS) + elem_off(r, 64 * hh + c));
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 t = __bfloat1622float2(h2[e]);
            f[2 * e] = t.x;
            f[2 * e + 1] = t.y;
          }
        };
        float mx = 0.f, inv = 1.f;
        if (p.phi == 2) {  // per-row softmax over d (feature_map.cpp:22-40)
          mx = -INFINITY;
#pragma unroll 2
          for (int c = 0; c < 64; c += 8) {
            float f[8];
            q8(c, f);
#pragma unroll
            for (int e = 0; e < 8; ++e) mx = fmaxf(mx, f[e]);
          }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
          float se = 0.f;
#pragma unroll 2
          for (int c = 0; c < 64; c += 8) {
            float f[8];
            q8(c, f);
#pragma unroll
            for (int e = 0; e < 8; ++e) se += __expf(f[e] - mx);
          }
          se += __shfl_xor_sync(0xffffffffu, se, 16);
          inv = 1.f / se;
        }
        float den = 0.f;
#pragma unroll 2
        for (int c = 0; c < 64; c += 8) {
          const int col = 64 * hh + c;
          float x[8];
          q8(c, x);
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = p.phi == 2 ? __expf(x[e] - mx) * inv : phi_elem(p.phi, x[e]);
          const float4 z0 = tc::lds_f4(aZ + 4 * col), z1 = tc::lds_f4(aZ + 4 * col + 16);
          den = fmaf(x[0], z0.x, den);
          den = fmaf(x[1], z0.y, den);
          den = fmaf(x[2], z0.z, den);
          den = fmaf(x[3], z0.w, den);
          den = fmaf(x[4], z1.x, den);
          den = fmaf(x[5], z1.y, den);
          den = fmaf(x[6], z1.z, den);
          den = fmaf(x[7], z1.w, den);
          tc::sts_u4(aX + elem_off(r, col), make_uint4(tc::pack_bf16(x[0], x[1]), tc::pack_bf16(x[2], x[3]),
                                                       tc::pack_bf16(x[4], x[5]), tc::pack_bf16(x[6], x[7])));
        }
        den += __shfl_xor_sync(0xffffffffu, den, 16);
        if (hh == 0) sts_f(aDen + 4 * r, den != 0.f ? 1.f / den : 0.f);  // den == 0 -> zero row (forward.cpp:136)
        tc::fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(x_full);
      // ---- O^s = O^T / l once block n's loop is done (O^T complete, 1/l in smem)
      if (leader) dbgw(5, n, 0, 3);
      tc::mbar_wait(stats, uint32_t(n & 1));
      if (leader) dbgw(5, n, 0, 4);
      tc::mbar_wait(ot_done + (n & 1), uint32_t((n >> 1) & 1));
      if (leader) dbgw(5, n, 0, 5);
      tc::tc_fence_after();
      fpp_mark(dbg && leader && n < 32, 192 + n);  // epilogue of block n starts
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t o[32];
        if (b.np > 0) {
          tc::tmem_ld32(tOT(n) + lane_base + c0, o);
          tc::tmem_ld_wait();
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 il = tc::lds_f4(aRowL + 4 * (c0 + e));
          const float sv[4] = {il.x, il.y, il.z, il.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float v = b.np > 0 ? __uint_as_float(o[e + t]) * sv[t] : 0.f;
            o[e + t] = __float_as_uint(v);
            sts_u16(aQn + elem_off(c0 + e + t, a), __bfloat16_as_ushort(__float2bfloat16_rn(v)));
          }
        }
        if (p.has_w) tc::tmem_st32(tOT(n) + lane_base + c0, o);
      }
      if (p.has_w) tc::tmem_st_wait();
      tc::fence_proxy_async();
      tc::tc_fence_before();
      bar_sync(2, 128);
      if (leader) {
        tc::mbar_arrive(stats_free);
#pragma unroll
        for (int c = 0; c < 2; ++c) tc::tma_store_rows(&tmOs, smem + (aQn - aS) + c * 8192, 64 * c, b.i * 64, rt);
        tc::bulk_commit();
      }
      // ---- O^l = O_l^T / den -> X (the projection's B operand and the O^l store's source)
      if (leader) dbgw(5, n, 0, 6);
      tc::mbar_wait(lin_done, uint32_t(n & 1));
      if (leader) dbgw(5, n, 0, 7);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t o[32];
        if (b.lin) {
          tc::tmem_ld32(tLT + lane_base + c0, o);
          tc::tmem_ld_wait();
        }
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 id4 = tc::lds_f4(aDen + 4 * (c0 + e));
          const float sv[4] = {id4.x, id4.y, id4.z, id4.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float v = b.lin ? __uint_as_float(o[e + t]) * sv[t] : 0.f;
            sts_u16(aX + elem_off(c0 + e + t, a), __bfloat16_as_ushort(__float2bfloat16_rn(v)));
          }
        }
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_ready);
      bar_sync(2, 128);
      if (leader) {
#pragma unroll
        for (int c = 0; c < 2; ++c) tc::tma_store_rows(&tmOl, smem + L::oX + c * 8192, 64 * c, b.i * 64, rt);
        tc::bulk_commit();
      }
      // ---- O = O^s + O^l W (accumulated onto O^T by the epilogue issuer) -> the Q slot
      if (leader) dbgw(5, n, 0, 8);
      tc::mbar_wait(proj_done, uint32_t(n & 1));
      if (leader) dbgw(5, n, 0, 9);
      tc::tc_fence_after();
      if (p.has_w) {
        if (leader) tc::bulk_wait_read<1>();  // the O^s store has left the Q slot
        bar_sync(2, 128);
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t o[32];
          tc::tmem_ld32(tOT(n) + lane_base + c0, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            sts_u16(aQn + elem_off(c0 + e, a), __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(o[e]))));
        }
        tc::fence_proxy_async();
      }
      tc::tc_fence_before();
      bar_sync(2, 128);
      if (leader) {
        tc::mbar_arrive(ot_free + (n & 1));  // O^T[n & 1] may take block n+2
        if (p.has_w) {
#pragma unroll
          for (int c = 0; c < 2; ++c) tc::tma_store_rows(&tmO, smem + (aQn - aS) + c * 8192, 64 * c, b.i * 64, rt);
          tc::bulk_commit();
        }
        tc::bulk_wait_read<0>();  // Q slot and X are free
        tc::mbar_arrive(q_free + (n & 1));
        fpp_mark(dbg && n < 31, 224 + n);  // epilogue of block n done
      }
      bar_sync(2, 128);
    }
    if (leader) tc::bulk_wait<0>();
  } else if (warp == 14) {
    // ------------------------------------------------------------------ epilogue MMA issuer
    constexpr uint32_t id_t = tc::idesc_bf16(128, 64, true, false);
    const uint64_t dX = tc::desc_kmajor(aX);
    auto koff = [](int kk) { return uint32_t((kk >> 2) * 8192 + (kk & 3) * 32); };
    Blk b;
    long long base = 0;
    // the two MN-major chunks at ring items n0, n0 + 1 (chunk 0 in the lower slot) times X
    auto chunks_x = [&](long long n0, uint32_t dst, bool acc) {
      const int sa = int(n0 % kRS), sb2 = int((n0 + 1) % kRS);
      tc::mbar_wait(full + sa, uint32_t((n0 / kRS) & 1));
      tc::mbar_wait(full + sb2, uint32_t(((n0 + 1) / kRS) & 1));
      tc::tc_fence_after();
      const int lo = min(sa, sb2), hi = max(sa, sb2);
      const uint64_t dA = tc::desc_mnmajor(aR + uint32_t(lo) * L::kTile, uint32_t((hi - lo) * L::kTile));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) tc::mma_bf16_w(dst, tc::desc_add(dA, kk * 2048), tc::desc_add(dX, koff(kk)), id_t, acc || kk > 0);
      tc::mma_commit_w(empty + sa);
      tc::mma_commit_w(empty + sb2);
    };
    for (int n = 0; n < nblk; ++n) {
      b.load(p, QB(n));
      dbgw(6, n, 0, 1);
      tc::mbar_wait(x_full, uint32_t(n & 1));
      dbgw(6, n, 0, 2);
      // H_i's and W's ring items come after all of block n's V items: wait until block n's PVs
      // are done, so that their slots' full barriers are within one lap (a parity wait issued
      // earlier would take an old phase for the awaited one)
      tc::mbar_wait(ot_done + (n & 1), uint32_t((n >> 1) & 1));
      if (b.lin) chunks_x(base + b.hidx(), tLT, false);  // O_l^T = H_i^T phi(Q_i)^T
      tc::mma_commit_w(lin_done);
      dbgw(6, n, 0, 3);
      tc::mbar_wait(o_ready, uint32_t(n & 1));
      dbgw(6, n, 0, 4);
      if (b.w) chunks_x(base + b.widx(), tOT(n), true);  // O^T (normalised O^s) += W^T O_l^T
      tc::mma_commit_w(proj_done);
      base += b.total();
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

void launch_attn_fwd_pp(const Dims& Dm, const void* q, const void* k, const void* v, const void* w, void* o,
                        void* o_s, void* o_l, float* lse, const StateBufs& s, cudaStream_t st) {
  constexpr int D = kD;
  PPParams p{};
  p.crit_cnt = s.crit_cnt;
  p.crit_idx = s.crit_idx;
  p.marg_cnt = s.marg_cnt;
  p.Z = s.Z;
  p.lse = lse;
  p.N = Dm.N;
  p.Tm = Dm.Tm;
  p.Tn = Dm.Tn;
  p.H = int(Dm.H);
  p.scale_log2 = float(Dm.inv_sqrt_d * 1.4426950408889634);
  p.has_w = (w != nullptr && o != nullptr) ? 1 : 0;
  p.phi = Dm.phi;
  p.kv_last = int(Dm.Nk_valid - (long long)(Dm.Tn - 1) * 64);
  p.items = (long long)Dm.U * Dm.Tm;
  p.rl = Dm.rl;
  CUtensorMap tq, tk, tv, th, tw, to, tos, tol;
  make_tmap_rows(&tq, q, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tk, k, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_rows(&tv, v, D, Dm.U, Dm.Nk, p.rl, 64);
  make_tmap_bf16(&th, s.Hb, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);
  if (w)
    make_tmap_bf16(&tw, w, D, uint64_t(Dm.H) * D, 1, D, 0, D);
  else
    tw = th;
  make_tmap_rows(&tos, o_s, D, Dm.U, Dm.N, p.rl, 64);
  make_tmap_rows(&tol, o_l, D, Dm.U, Dm.N, p.rl, 64);
  if (o)
    make_tmap_rows(&to, o, D, Dm.U, Dm.N, p.rl, 64);
  else
    to = tos;
  static int sms = 0;
  if (!sms) SLAB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = int(std::min<long long>(p.items, sms));
  SLAB_CUDA(cudaFuncSetAttribute(k_attn_fwd_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, PPLayout::kBytes));
  launch_pdl(k_attn_fwd_pp, dim3(grid), kThreads, PPLayout::kBytes, st, tq, tk, tv, th, tw, to, tos, tol, p);
  check_launch("k_attn_fwd", st);
}

}  // namespace slab

#ifdef SLAB_TIMELINE
extern "C" int sla_b200_diag_fpp_timeline(long long* host256) {
  return cudaMemcpyFromSymbol(host256, slab::g_fpp_ts, 256 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
#endif

#ifdef SLAB_PP_DEBUG
extern "C" int sla_b200_diag_pp_debug(void* dev_ptr) {
  return cudaMemcpyToSymbol(slab::g_pp_dbg, &dev_ptr, sizeof(void*)) == cudaSuccess ? 0 : 1;
}
#endif
