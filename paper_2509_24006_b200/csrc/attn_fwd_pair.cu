// attn_fwd_pair.cu -- K5 for d = 128: the fused SLA forward over PAIRS of critical key blocks,
// with the output accumulated transposed.
//
// Same algorithm as attn_fwd.cu (forward.cpp:29-79 critical loop, :81-172 block classes,
// :187-195 projection), different instruction shapes.  On sm_100a an N = 64 tcgen05.mma costs
// 50 cycles whatever M is, and an M = 64 one runs at half rate, so the
// per-tile forward S = Q_i K_j^T (M = 64, N = 64: 8 x 50) plus O += P V_j (M = 64, N = 128,
// K = 64: 4 x 64) costs 656 cycles per critical tile.  Here one step covers two tiles:
//   S   = Q_i [K_j1; K_j2]^T            M = 64,  N = 128, K = d     8 x 64 = 512 cycles
//   O^T += [V_j1; V_j2]^T [P_1 P_2]^T   M = d,   N = 64,  K = 128   8 x 50 = 400 cycles
// 456 cycles per tile (-30 %).  The online softmax stays row-wise (S is row-major in TMEM);
// only the accumulator is transposed (TMEM lane = output column a, TMEM column = query row),
// so the rare lazy rescale and the final 1/l are per-column scalings read from smem, and the
// epilogue transposes through shared memory on its way to the TMA stores.  The linear branch
// is transposed the same way: O_l^T = H_i^T phi(Q_i)^T (M = d, N = 64) lands in its own TMEM
// columns while the critical loop runs, and the projection accumulates W^T O_l^T onto the
// normalised O^s (O = O^s + O^l W).
//
// Warps (224 threads, 2 CTAs / SM): 0 TMA producer (one 5-slot ring of 16 KB items: K half-pairs
// [K_j1; K_j2] per 64-column chunk, V tiles, H_i and W chunks, in consumption order), 1 S issuer,
// 2-5 softmax / epilogue (row r = 16 (warp % 4) + lane % 16, column half lane / 16 of the M = 64
// S layout; transposed phases: output column a = 32 (warp % 4) + lane), 6 the O_l^T / PV /
// projection issuer.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

#ifdef SLAB_TIMELINE  // -DSLAB_TIMELINE: event clocks of one CTA, phase clocks of every CTA
static __device__ long long g_fwp_ts[256];
static __device__ unsigned long long g_fwp_prof[8192][4];
#endif

namespace {

constexpr int kPairD = 128;

__device__ __forceinline__ void fwp_mark(bool on, int slot) {
#ifdef SLAB_TIMELINE
  if (on) g_fwp_ts[slot] = clock64();
#else
  (void)on;
  (void)slot;
#endif
}
__device__ __forceinline__ void fwp_prof(bool on, int slot) {  // [entry, loop start, loop end, exit | smid << 56]
#ifdef SLAB_TIMELINE
  if (on) {
    unsigned long long v = clock64();
    if (slot == 3) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      v |= (unsigned long long)sm << 56;
    }
    g_fwp_prof[(blockIdx.y * gridDim.x + blockIdx.x) & 8191][slot] = v;
  }
#else
  (void)on;
  (void)slot;
#endif
}
constexpr int kPairThreads = 224;
constexpr int kPairSlots = 5;

struct PairLayout {
  static constexpr int kTile = 16384;        // one ring item / one [64 x 128] bf16 tile
  static constexpr int oQ = 0;               // Q_i (K-major, 2 chunks); O^s staging at the end
  static constexpr int oP = oQ + kTile;      // phi(Q_i), then P pairs; O^l staging at the end
  static constexpr int oRing = oP + kTile;   // 5 slots; O staging (slot 0) at the end
  static constexpr int oBar = oRing + kPairSlots * kTile;
  static constexpr int oRow = oBar + 256;    // float [64]: alpha / 1/l per query row (Z_i first)
  static constexpr int oDen = oRow + 256;    // float [64]: 1/den per query row
  static constexpr int kBytes = oDen + 256;
  // two CTAs per SM: 228 KB per SM, 1 KB reserved per CTA; the base is 1024-aligned (checked)
  static_assert(kBytes <= (233472 - 2 * 1024) / 2, "smem: 2 CTAs / SM");
};

struct PairParams {
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
  RowLayout rl;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ float lds_f(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// OR of `v` over the n threads of named barrier `id` (all of them wait)
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
// byte offset of element (row, col) in a [64 rows][128 cols] bf16 tile stored as two K-major
// SW128 chunks of 64 columns (8 KB each)
__device__ __forceinline__ uint32_t elem_off(int row, int col) {
  return uint32_t(col >> 6) * 8192u + tc::sw128_off(uint32_t(row), uint32_t((col & 63) >> 3)) + uint32_t(col & 7) * 2u;
}

// Ring item schedule (producer and consumers agree on it): K(0) a/b, H_i (2 chunks, if the row
// has marginal blocks), then K(p) a/b and V(p-1) for p = 1..np-1, V(np-1), W (2 chunks).
struct Items {
  int h2, np, last_n;
  __device__ __forceinline__ int k(int p) const { return p == 0 ? 0 : 2 + h2 + 4 * (p - 1); }
  __device__ __forceinline__ int hidx() const { return np > 0 ? 2 : 0; }
  __device__ __forceinline__ int v(int p) const {
    if (p + 1 < np) return k(p + 1) + 2;
    return np >= 2 ? k(np - 1) + 4 : 2 + h2;
  }
  __device__ __forceinline__ int w() const { return np == 0 ? h2 : v(np - 1) + last_n; }
  __device__ __forceinline__ int tiles(int p) const { return p + 1 < np ? 2 : last_n; }
};
// Two ring items holding the 64-column chunks of an MN-major A operand (H_i^T or W^T): chunk c
// goes to item n + (c ^ swap) so that chunk 0 sits in the lower slot (the descriptor's LBO is
// a positive distance)
__device__ __forceinline__ bool chunk_swap(int n) { return (n + 1) % kPairSlots < n % kPairSlots; }

__global__ void __maxnreg__(128)
    k_attn_fwd_pair(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmH,
                    const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
                    const __grid_constant__ CUtensorMap tmOs, const __grid_constant__ CUtensorMap tmOl,
                    PairParams p) {
  pdl_entry();  // launched by launch_pdl
  using L = PairLayout;
  constexpr int D = kPairD;
  constexpr int RS = kPairSlots;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sP = smem + L::oP;
  uint8_t* sRing = smem + L::oRing;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* full = bars + 0;       // [RS]
  uint64_t* empty = bars + 5;      // [RS]
  uint64_t* q_full = bars + 10;
  uint64_t* s_full = bars + 11;
  uint64_t* s_free = bars + 12;
  uint64_t* p_full = bars + 13;
  uint64_t* pv_done = bars + 14;
  uint64_t* x_full = bars + 15;
  uint64_t* lin_done = bars + 16;
  uint64_t* o_ready = bars + 17;
  uint64_t* proj_done = bars + 18;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);
  const uint32_t aRow = tc::smem_u32(smem + L::oRow), aDen = tc::smem_u32(smem + L::oDen);

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
  const Items it{has_lin ? 2 : 0, (cnt + 1) >> 1, (cnt & 1) ? 1 : 2};
  const int np = it.np;
  const bool dbg = blockIdx.x == 100 && blockIdx.y == 6;
  fwp_mark(dbg && threadIdx.x == 0, 255);
  fwp_prof(threadIdx.x == 0, 0);

  if (warp == 0) {
    if (lane == 0) {
      if (tc::smem_u32(smem) & 1023u) __trap();  // SW128 tiles need a 1024-aligned base
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::tma_prefetch(&tmV);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(full + s, 1);
        tc::mbar_init(empty + s, 1);
      }
      tc::mbar_init(q_full, 1);
      tc::mbar_init(s_full, 1);
      tc::mbar_init(s_free, 4);
      tc::mbar_init(p_full, 4);
      tc::mbar_init(pv_done, 1);
      tc::mbar_init(x_full, 4);
      tc::mbar_init(lin_done, 1);
      tc::mbar_init(o_ready, 4);
      tc::mbar_init(proj_done, 1);
      tc::fence_barrier_init();
      tc::mbar_expect_tx(q_full, L::kTile);
#pragma unroll
      for (int c = 0; c < 2; ++c) tc::tma_load_rows(sQ + c * 8192, &tmQ, q_full, 64 * c, i * 64, rt);
    }
    __syncwarp();
    tc::tmem_alloc<256>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem;          // S pair: M = 64 layout, 128 columns
  const uint32_t tOT = tmem + 128;   // O^T: lane = output column, 64 query columns
  const uint32_t tLT = tmem + 192;   // O_l^T (unnormalised)

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int n = 0;
      auto take = [&](int bytes) -> uint8_t* {
        const int s = n % RS;
        tc::mbar_wait(empty + s, ((n / RS) & 1) ^ 1);
        tc::mbar_expect_tx(full + s, bytes);
        return sRing + s * L::kTile;
      };
      auto load_k = [&](int pp) {  // two half-pair items: [K_j1; K_j2] of column chunk c
        const int nt = it.tiles(pp);
        const int r1 = list[2 * pp] * 64, r2 = nt == 2 ? list[2 * pp + 1] * 64 : 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint8_t* dst = take(nt * 8192);
          fwp_mark(dbg && pp < 16, c * 16 + pp);  // 0..15 K(p)a issued, 16..31 K(p)b
          tc::tma_load_rows(dst, &tmK, full + n % RS, 64 * c, r1, rt);
          if (nt == 2) tc::tma_load_rows(dst + 8192, &tmK, full + n % RS, 64 * c, r2, rt);
          ++n;
        }
      };
      auto load_v = [&](int pp) {  // one item per tile
        const int nt = it.tiles(pp);
        for (int t = 0; t < nt; ++t) {
          uint8_t* dst = take(L::kTile);
          fwp_mark(dbg && pp < 16, 32 + t * 16 + pp);  // 32..47 V(p)a issued, 48..63 V(p)b
          const int r = list[2 * pp + t] * 64;
#pragma unroll
          for (int c = 0; c < 2; ++c) tc::tma_load_rows(dst + c * 8192, &tmV, full + n % RS, 64 * c, r, rt);
          ++n;
        }
      };
      auto load_chunks = [&](const CUtensorMap* tm, int row) {  // H_i or W: [D rows][64] chunks
        const int n0 = n;
        const bool sw = chunk_swap(n0);
        for (int t = 0; t < 2; ++t) {
          uint8_t* dst = take(L::kTile);
          tc::tma_load_3d(dst, tm, full + n % RS, 64 * (t ^ int(sw)), row, 0);
          ++n;
        }
      };
      if (np > 0) load_k(0);
      if (has_lin) load_chunks(&tmH, int(urow * D));
      for (int pp = 1; pp < np; ++pp) {
        load_k(pp);
        load_v(pp - 1);
      }
      if (np > 0) load_v(np - 1);
      if (has_w) load_chunks(&tmW, int(u % p.H) * D);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ S issuer
    const uint32_t aQ = tc::smem_u32(sQ), aR = tc::smem_u32(sRing);
    constexpr uint32_t id_s2 = tc::idesc_bf16(64, 128, false, false);
    constexpr uint32_t id_s1 = tc::idesc_bf16(64, 64, false, false);
    const uint64_t dQ = tc::desc_kmajor(aQ), dR = tc::desc_kmajor(aR);
    tc::mbar_wait(q_full, 0);
    for (int pp = 0; pp < np; ++pp) {
      if (pp > 0) tc::mbar_wait(s_free, (pp - 1) & 1);  // the compute warps hold S(pp-1)
      const int n0 = it.k(pp);
      const int s0 = n0 % RS, s1 = (n0 + 1) % RS;
      tc::mbar_wait(full + s0, (n0 / RS) & 1);
      tc::mbar_wait(full + s1, ((n0 + 1) / RS) & 1);
      tc::tc_fence_after();
      const uint32_t id = it.tiles(pp) == 2 ? id_s2 : id_s1;
      fwp_mark(dbg && lane == 0 && pp < 16, 64 + pp);  // S(p) issued
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t a = tc::desc_add(dQ, uint32_t((kk >> 2) * 8192 + (kk & 3) * 32));
        const uint64_t b = tc::desc_add(dR, uint32_t(((kk >> 2) ? s1 : s0) * L::kTile + (kk & 3) * 32));
        tc::mma_bf16_w(tS, a, b, id, kk > 0);
      }
      tc::mma_commit_w(empty + s0);
      tc::mma_commit_w(empty + s1);
      tc::mma_commit_w(s_full);
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------------ O_l^T / PV / projection issuer
    const uint32_t aP = tc::smem_u32(sP), aR = tc::smem_u32(sRing);
    constexpr uint32_t id_t = tc::idesc_bf16(128, 64, true, false);  // A MN-major [D x K], B K-major [64 x K]
    const uint64_t dP = tc::desc_kmajor(aP);
    auto koff = [](int kk) { return uint32_t((kk >> 2) * 8192 + (kk & 3) * 32); };
    // O^T-shaped product of the two MN-major chunks at items n0, n0+1 with the B tile in sP
    auto chunks_x_p = [&](int n0, uint32_t dst, bool acc) {
      const int sa = n0 % RS, sb = (n0 + 1) % RS;
      tc::mbar_wait(full + sa, (n0 / RS) & 1);
      tc::mbar_wait(full + sb, ((n0 + 1) / RS) & 1);
      tc::tc_fence_after();
      const int lo = min(sa, sb), hi = max(sa, sb);
      const uint64_t dA = tc::desc_mnmajor(aR + lo * L::kTile, uint32_t((hi - lo) * L::kTile));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) tc::mma_bf16_w(dst, tc::desc_add(dA, kk * 2048), tc::desc_add(dP, koff(kk)), id_t, acc || kk > 0);
      tc::mma_commit_w(empty + sa);
      tc::mma_commit_w(empty + sb);
    };
    if (has_lin) {  // O_l^T = H_i^T phi(Q_i)^T
      tc::mbar_wait(x_full, 0);
      chunks_x_p(it.hidx(), tLT, false);
      tc::mma_commit_w(lin_done);
    }
    for (int pp = 0; pp < np; ++pp) {
      tc::mbar_wait(p_full, pp & 1);
      const int nt = it.tiles(pp), n0 = it.v(pp);
      const int s0 = n0 % RS, s1 = (n0 + 1) % RS;
      tc::mbar_wait(full + s0, (n0 / RS) & 1);
      if (nt == 2) tc::mbar_wait(full + s1, ((n0 + 1) / RS) & 1);
      tc::tc_fence_after();
      fwp_mark(dbg && lane == 0 && pp < 16, 80 + pp);  // PV(p) issued
      const uint64_t dv0 = tc::desc_mnmajor(aR + s0 * L::kTile, 8192), dv1 = tc::desc_mnmajor(aR + s1 * L::kTile, 8192);
      for (int kk = 0; kk < 4 * nt; ++kk)
        tc::mma_bf16_w(tOT, tc::desc_add((kk >> 2) ? dv1 : dv0, (kk & 3) * 2048), tc::desc_add(dP, koff(kk)), id_t,
                       (pp | kk) != 0);
      tc::mma_commit_w(empty + s0);
      if (nt == 2) tc::mma_commit_w(empty + s1);
      tc::mma_commit_w(pv_done);
    }
    if (has_w) {  // O^T (normalised O^s) += W^T O_l^T
      tc::mbar_wait(o_ready, 0);
      fwp_mark(dbg && lane == 0, 249);
      tc::tc_fence_after();
      chunks_x_p(it.w(), tOT, true);
      tc::mma_commit_w(proj_done);
    }
  } else {
    // ------------------------------------------------------------------ softmax / epilogue
    const int q4 = warp & 3;
    const int r = 16 * q4 + (lane & 15);  // query row (row phases)
    const int hh = lane >> 4;             // column half: key tile hh of a pair / features hh*64..
    const int a = 32 * q4 + lane;         // output column (transposed phases)
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const uint32_t aQ = tc::smem_u32(sQ), aP = tc::smem_u32(sP);
    const int tid = threadIdx.x - 64;     // 0..127

    // ---- linear branch: phi(Q_i) -> sP (the B operand of O_l^T), den = phi(q) . Z_i
    float den = 0.f;
    if (has_lin) {
      const uint32_t aZ = aRow;  // Z_i borrows the row-scalar arrays until the loop starts
      if (tid < D) {
        const float z = tc::load_sum3(p.Z + urow * 3 * D + tid, D);
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(aZ + 4 * tid), "f"(z) : "memory");
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::mbar_wait(q_full, 0);
      // my half row (64 features) in three passes over the Q tile in smem, 8 features at a time
      // (registers: the S loop below needs them): max, sum of exponentials, then phi -> sP, den
      auto q8 = [&](int c, float (&f)[8]) {
        const uint4 v = *reinterpret_cast<const uint4*>(sQ + elem_off(r, 64 * hh + c));
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
        tc::sts_u4(aP + elem_off(r, col), make_uint4(tc::pack_bf16(x[0], x[1]), tc::pack_bf16(x[2], x[3]),
                                                     tc::pack_bf16(x[4], x[5]), tc::pack_bf16(x[6], x[7])));
      }
      den += __shfl_xor_sync(0xffffffffu, den, 16);
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(x_full);
      fwp_mark(dbg && tid == 0, 248);
    }

    // ---- critical branch: online softmax over key-block pairs (ascending list)
    float m_used = -INFINITY, l = 0.f;
    const float sc = p.scale_log2;
    for (int pp = 0; pp < np; ++pp) {
      tc::mbar_wait(s_full, pp & 1);
      tc::tc_fence_after();
      fwp_mark(dbg && tid == 0 && pp < 16, 96 + pp);  // S(p) seen by the softmax warps
      if (pp == 0) fwp_prof(tid == 0, 1);
      uint32_t sa0[32], sa1[32];  // my 64 columns of the pair: tile hh, keys 0-31 / 32-63
      tc::tmem_ld32_x2<64>(tS + lane_base, sa0);
      tc::tmem_ld32_x2<64>(tS + lane_base + 32, sa1);
      tc::tmem_ld_wait();
      float sa[64];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        sa[e] = __uint_as_float(sa0[e]);
        sa[32 + e] = __uint_as_float(sa1[e]);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(s_free);  // S(pp+1) may overwrite the buffer
      // valid key columns of my tile: 0 for the missing half of an odd tail, kv_last for the
      // last key block of a ragged N, else 64 (masked keys get no weight)
      const bool live = it.tiles(pp) == 2 || hh == 0;
      const int kvalid = !live ? 0 : (list[2 * pp + hh] == p.Tn - 1 ? p.kv_last : 64);
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 64; ++e) mx = fmaxf(mx, e < kvalid ? sa[e] : -INFINITY);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16)) * sc;
      const float m_new = fmaxf(m_used, mx);
      const bool need = pp > 0 && m_new > m_used + 8.f;
      // this row's reference max after the step is known locally (the CTA vote below only
      // decides whether O^T is rescaled), so P is computed and packed now and the 64 scores die
      const float m_fin = (pp == 0 || need) ? m_new : m_used;
      float ps = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 64; e += 2) {
        const float p0 = e < kvalid ? ex2(sa[e] * sc - m_fin) : 0.f;
        const float p1 = e + 1 < kvalid ? ex2(sa[e + 1] * sc - m_fin) : 0.f;
        ps += p0 + p1;
        pk[e >> 1] = tc::pack_bf16(p0, p1);
      }
      // the P buffer (and O^T) are free once PV(pp-1) completed; phi(Q) must have been consumed
      if (pp > 0) tc::mbar_wait(pv_done, (pp - 1) & 1);
      else if (has_lin) tc::mbar_wait(lin_done, 0);
      fwp_mark(dbg && tid == 0 && pp < 16, 112 + pp);  // PV(p-1) done, P buffer free
      if (bar_red_or(1, 128, need)) {  // some row's max grew by more than 2^8: rescale O^T columns
        tc::tc_fence_after();
        const float alpha = need ? ex2(m_used - m_new) : 1.f;
        if (need) l *= alpha;
        if (hh == 0) asm volatile("st.shared.f32 [%0], %1;" ::"r"(aRow + 4 * r), "f"(alpha) : "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t o[32];
          tc::tmem_ld32(tOT + lane_base + c0, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 al = tc::lds_f4(aRow + 4 * (c0 + e));
            o[e] = __float_as_uint(__uint_as_float(o[e]) * al.x);
            o[e + 1] = __float_as_uint(__uint_as_float(o[e + 1]) * al.y);
            o[e + 2] = __float_as_uint(__uint_as_float(o[e + 2]) * al.z);
            o[e + 3] = __float_as_uint(__uint_as_float(o[e + 3]) * al.w);
          }
          tc::tmem_st32(tOT + lane_base + c0, o);
        }
        tc::tmem_st_wait();
        asm volatile("bar.sync 1, 128;" ::: "memory");  // alpha is read before the next rescale rewrites it
      }
      m_used = m_fin;
      const uint32_t prow = aP + uint32_t(hh) * 8192u;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        tc::sts_u4(prow + tc::sw128_off(uint32_t(r), uint32_t(c)), make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
      l += ps + __shfl_xor_sync(0xffffffffu, ps, 16);
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full);
      fwp_mark(dbg && tid == 0 && pp < 16, 128 + pp);  // P(p) stored
    }
    fwp_prof(tid == 0, 2);

    // ---- epilogue: O^s = O^T / l (transposed into the dead Q tile), O^l = O_l^T / den (into sP),
    // then O = O^s + O^l W on the tensor core (into ring slot 0); lse
    if (np > 0) tc::mbar_wait(pv_done, (np - 1) & 1);
    else if (has_lin) tc::mbar_wait(lin_done, 0);
    tc::tc_fence_after();
    if (hh == 0) {
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(aRow + 4 * r), "f"(l > 0.f ? 1.f / l : 0.f) : "memory");
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(aDen + 4 * r), "f"(den != 0.f ? 1.f / den : 0.f) : "memory");
      const long long cr = rm.row((long long)i * 64 + r);  // the caller's lse row (none past a ragged N)
      if (cr >= 0) p.lse[cr] = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994531f : kLseSentinel;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll 1
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t o[32];
      if (np > 0) {
        tc::tmem_ld32(tOT + lane_base + c0, o);
        tc::tmem_ld_wait();
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float v = np > 0 ? __uint_as_float(o[e]) * lds_f(aRow + 4 * (c0 + e)) : 0.f;
        o[e] = __float_as_uint(v);
        sts_u16(aQ + elem_off(c0 + e, a), __bfloat16_as_ushort(__float2bfloat16_rn(v)));
      }
      if (has_w) tc::tmem_st32(tOT + lane_base + c0, o);
    }
#pragma unroll 1
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t o[32];
      if (has_lin) {
        tc::tmem_ld32(tLT + lane_base + c0, o);
        tc::tmem_ld_wait();
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float v = has_lin ? __uint_as_float(o[e]) * lds_f(aDen + 4 * (c0 + e)) : 0.f;
        sts_u16(aP + elem_off(c0 + e, a), __bfloat16_as_ushort(__float2bfloat16_rn(v)));
      }
    }
    if (has_w) {
      tc::tmem_st_wait();
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_ready);
      fwp_mark(dbg && tid == 0, 250);
      tc::mbar_wait(proj_done, 0);
      tc::tc_fence_after();
      fwp_mark(dbg && tid == 0, 251);
      const uint32_t aO = tc::smem_u32(sRing);  // every ring item has been consumed
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t o[32];
        tc::tmem_ld32(tOT + lane_base + c0, o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          sts_u16(aO + elem_off(c0 + e, a), __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(o[e]))));
      }
    }
    tc::fence_proxy_async();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tc::tma_store_rows(&tmOs, sQ + c * 8192, 64 * c, i * 64, rt);
        tc::tma_store_rows(&tmOl, sP + c * 8192, 64 * c, i * 64, rt);
        if (has_w) tc::tma_store_rows(&tmO, sRing + c * 8192, 64 * c, i * 64, rt);
      }
      tc::bulk_commit();
      tc::bulk_wait_read<0>();
      fwp_mark(dbg, 252);
      fwp_prof(true, 3);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

}  // namespace

void launch_attn_fwd_pair(const Dims& Dm, const void* q, const void* k, const void* v, const void* w, void* o,
                          void* o_s, void* o_l, float* lse, const StateBufs& s, cudaStream_t st) {
  constexpr int D = kPairD;
  PairParams p{};
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
  SLAB_CUDA(cudaFuncSetAttribute(k_attn_fwd_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, PairLayout::kBytes));
  // two CTAs per SM need the largest carveout (the driver otherwise picks 132 KB: one CTA)
  SLAB_CUDA(cudaFuncSetAttribute(k_attn_fwd_pair, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  launch_pdl(k_attn_fwd_pair, dim3(Dm.Tm, unsigned(Dm.U)), kPairThreads, PairLayout::kBytes, st, tq, tk, tv, th, tw, to,
             tos, tol, p);
  check_launch("k_attn_fwd", st);
}

}  // namespace slab

#ifdef SLAB_TIMELINE  // diagnostic accessors: timeline builds only (profiles/fwp_timeline.py)
extern "C" int sla_b200_diag_fwp_timeline(long long* host256) {
  return cudaMemcpyFromSymbol(host256, slab::g_fwp_ts, 256 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
extern "C" int sla_b200_diag_fwp_prof(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, slab::g_fwp_prof, sizeof(slab::g_fwp_prof)) == cudaSuccess ? 0 : 1;
}
#endif
