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
// softmax / epilogue (row r = 16*(warp%4) + lane, lanes 0-15: the M=64 TMEM layout).
// The K/V ring also carries H_i (before the loop) and W (after it) as ring items.
// Lazy rescaling: O is rescaled only when the running max grows by more than 2^8.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {

namespace {

template <int D>
struct FwdLayout {
  static constexpr int kQ = 64 * D * 2;       // Q tile, K-major SW128 (D/64 chunks of 8 KB)
  static constexpr int kTile = 64 * D * 2;    // one K or V tile
  static constexpr int kStage = 2 * kTile;    // K + V; also holds H_i or W (D*D*2 bytes)
  static constexpr int kStages = 2;  // 2 CTAs / SM share the tensor core
  static constexpr int kPX = 16384;           // 2 P buffers (8 KB) == phi(Q) / O^l tile
  static constexpr int oQ = 0;
  static constexpr int oRing = oQ + kQ;
  static constexpr int oPX = oRing + kStages * kStage;
  static constexpr int oBar = oPX + kPX;
  static constexpr int kBytes = oBar + 256 + 1024;
  static_assert(kBytes <= 232448, "smem");
  static_assert(D * D * 2 <= kStage, "H/W must fit a ring stage");
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
               const __grid_constant__ CUtensorMap tmW, FwdParams p) {
  using L = FwdLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sRing = smem + L::oRing;
  uint8_t* sPX = smem + L::oPX;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars + 0;
  constexpr int RS = L::kStages;
  uint64_t* ring_full = bars + 16;        // [RS]
  uint64_t* ring_empty = bars + 16 + RS;  // [RS]
  uint64_t* s_full = bars + 5;      // [2]
  uint64_t* p_full = bars + 7;      // [2]
  uint64_t* pv_done = bars + 9;     // [2]
  uint64_t* lin_done = bars + 11;
  uint64_t* x_full = bars + 12;
  uint64_t* o_ready = bars + 13;
  uint64_t* proj_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * RS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const long long u = blockIdx.y;
  const long long urow = u * p.Tm + i;
  const int cnt = p.crit_cnt[urow];
  const int* list = p.crit_idx + urow * p.Tn;
  const bool has_lin = p.marg_cnt[urow] > 0;
  const bool has_w = p.has_w != 0;
  const int row0 = int(u * p.N) + i * 64;  // row in the [U*N, D] view

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&tmQ);
      tc::tma_prefetch(&tmK);
      tc::tma_prefetch(&tmV);
      tc::mbar_init(q_full, 1);
      for (int s = 0; s < RS; ++s) {
        tc::mbar_init(ring_full + s, 1);
        tc::mbar_init(ring_empty + s, 1);
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
    if (lane == 0) {
      tc::mbar_expect_tx(q_full, L::kQ);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) tc::tma_load_3d(sQ + c * 8192, &tmQ, q_full, 64 * c, row0, 0);
      int item = 0;
      auto acquire = [&](int bytes) -> uint8_t* {
        const int s = item % RS;
        tc::mbar_wait(ring_empty + s, ((item / RS) & 1) ^ 1);
        tc::mbar_expect_tx(ring_full + s, bytes);
        return sRing + s * L::kStage;
      };
      if (has_lin) {
        uint8_t* dst = acquire(D * D * 2);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(dst + c * D * 128, &tmH, ring_full + (item % RS), 64 * c, int(urow * D), 0);
        ++item;
      }
      for (int t = 0; t < cnt; ++t) {
        const int kv_row = int(u * p.N) + list[t] * 64;
        uint8_t* dst = acquire(2 * L::kTile);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tc::tma_load_3d(dst + c * 8192, &tmK, ring_full + (item % RS), 64 * c, kv_row, 0);
          tc::tma_load_3d(dst + L::kTile + c * 8192, &tmV, ring_full + (item % RS), 64 * c, kv_row, 0);
        }
        ++item;
      }
      if (has_w) {
        uint8_t* dst = acquire(D * D * 2);
        const int h = int(u % p.H);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(dst + c * D * 128, &tmW, ring_full + (item % RS), 64 * c, h * D, 0);
        ++item;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t sQa = tc::smem_u32(sQ), sRa = tc::smem_u32(sRing), sPa = tc::smem_u32(sPX);
    constexpr uint32_t id_s = tc::idesc_bf16(64, 64, false, false);
    constexpr uint32_t id_o = tc::idesc_bf16(64, D, false, true);
    int item = 0;
    auto wait_item = [&]() -> uint32_t {
      const int s = item % RS;
      tc::mbar_wait(ring_full + s, (item / RS) & 1);
      tc::tc_fence_after();
      return sRa + s * L::kStage;
    };
    tc::mbar_wait(q_full, 0);
    if (has_lin) {  // O-region <- phi(Q_i) H_i
      tc::mbar_wait(x_full, 0);
      const uint32_t sh = wait_item();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16(tO, tc::desc_kmajor(sPa + (kk >> 2) * 8192 + (kk & 3) * 32),
                       tc::desc_mnmajor(sh + kk * 2048, D * 128), id_o, kk > 0);
        tc::mma_commit(ring_empty + (item % RS));
        tc::mma_commit(lin_done);
      }
      __syncwarp();
      ++item;
    }
    const int item0 = item;
    auto issue_pv = [&](int j) {
      tc::mbar_wait(p_full + (j & 1), (j >> 1) & 1);
      tc::tc_fence_after();
      const int it = item0 + j;
      const uint32_t sv = sRa + (it % RS) * L::kStage + L::kTile;
      if (lane == 0) {
        const uint32_t sp = sPa + (j & 1) * 8192;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc::mma_bf16(tO, tc::desc_kmajor(sp + kk * 32), tc::desc_mnmajor(sv + kk * 2048, 8192), id_o,
                       (j | kk) != 0);
        tc::mma_commit(ring_empty + (it % RS));
        tc::mma_commit(pv_done + (j & 1));
      }
      __syncwarp();
    };
    for (int t = 0; t < cnt; ++t) {
      const uint32_t sk = wait_item();
      if (lane == 0) {
        const uint32_t ts = tS0 + 64 * (t & 1);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16(ts, tc::desc_kmajor(sQa + (kk >> 2) * 8192 + (kk & 3) * 32),
                       tc::desc_kmajor(sk + (kk >> 2) * 8192 + (kk & 3) * 32), id_s, kk > 0);
        tc::mma_commit(s_full + (t & 1));
      }
      __syncwarp();
      ++item;
      if (t > 0) issue_pv(t - 1);
    }
    if (cnt > 0) issue_pv(cnt - 1);
    if (has_w) {  // O-region (normalised O^s) += O^l W
      const uint32_t sw = wait_item();
      tc::mbar_wait(o_ready, 0);
      tc::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16(tO, tc::desc_kmajor(sPa + (kk >> 2) * 8192 + (kk & 3) * 32),
                       tc::desc_mnmajor(sw + kk * 2048, D * 128), id_o, 1);
        tc::mma_commit(ring_empty + (item % RS));
        tc::mma_commit(proj_done);
      }
      __syncwarp();
      ++item;
    }
  } else {
    // ------------------------------------------------------------------ softmax / epilogue
    const int q4 = warp & 3;
    const int r = 16 * q4 + lane;           // row within the block (valid for lane < 16)
    const bool valid = lane < 16;
    const uint32_t lane_base = uint32_t(32 * q4) << 16;
    const long long grow = (long long)row0 + r;  // global row in [U*N, D]
    tc::mbar_wait(q_full, 0);

    // ---- marginal branch: phi(Q_i) into X, den = phi(q) . Z_i, then O^l
    float den = 0.f;
    if (has_lin) {
      const float* Zi = p.Z + urow * D;
      float x[D];
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(sQ + (c >> 3) * 8192 + tc::sw128_off(r & 63, c & 7));
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h2[e]);
          x[8 * c + 2 * e] = f.x;
          x[8 * c + 2 * e + 1] = f.y;
        }
      }
      if (p.phi == 2) {  // per-row softmax over d (feature_map.cpp:10-20)
        float mx = -INFINITY;
#pragma unroll
        for (int a = 0; a < D; ++a) mx = fmaxf(mx, x[a]);
        float sum = 0.f;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          x[a] = __expf(x[a] - mx);
          sum += x[a];
        }
        const float inv = 1.f / sum;
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] *= inv;
      } else {
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = phi_elem(p.phi, x[a]);
      }
#pragma unroll
      for (int a = 0; a < D; ++a) den = fmaf(x[a], __ldg(Zi + a), den);
      if (valid) {
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          uint4 v;
          v.x = tc::pack_bf16(x[8 * c + 0], x[8 * c + 1]);
          v.y = tc::pack_bf16(x[8 * c + 2], x[8 * c + 3]);
          v.z = tc::pack_bf16(x[8 * c + 4], x[8 * c + 5]);
          v.w = tc::pack_bf16(x[8 * c + 6], x[8 * c + 7]);
          *reinterpret_cast<uint4*>(sPX + (c >> 3) * 8192 + tc::sw128_off(r, c & 7)) = v;
        }
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(x_full);
      tc::mbar_wait(lin_done, 0);
      tc::tc_fence_after();
      const float inv_den = den != 0.f ? 1.f / den : 0.f;  // den == 0 -> zero row (forward.cpp:136)
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t a[32];
        tc::tmem_ld32(tO + lane_base + c0, a);
        tc::tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 v;
            v.x = tc::pack_bf16(__uint_as_float(a[e]) * inv_den, __uint_as_float(a[e + 1]) * inv_den);
            v.y = tc::pack_bf16(__uint_as_float(a[e + 2]) * inv_den, __uint_as_float(a[e + 3]) * inv_den);
            v.z = tc::pack_bf16(__uint_as_float(a[e + 4]) * inv_den, __uint_as_float(a[e + 5]) * inv_den);
            v.w = tc::pack_bf16(__uint_as_float(a[e + 6]) * inv_den, __uint_as_float(a[e + 7]) * inv_den);
            *reinterpret_cast<uint4*>(p.o_l + grow * D + c0 + e) = v;
          }
        }
      }
    } else if (valid) {
#pragma unroll
      for (int c = 0; c < D; c += 8)
        *reinterpret_cast<uint4*>(p.o_l + grow * D + c) = make_uint4(0, 0, 0, 0);
    }

    // ---- critical branch: online softmax over the ascending critical list
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < cnt; ++t) {
      tc::mbar_wait(s_full + (t & 1), (t >> 1) & 1);
      tc::tc_fence_after();
      uint32_t sa[32], sb[32];
      const uint32_t ts = tS0 + 64 * (t & 1) + lane_base;
      tc::tmem_ld32(ts, sa);
      tc::tmem_ld32(ts + 32, sb);
      tc::tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 32; ++e) mx = fmaxf(mx, fmaxf(__uint_as_float(sa[e]), __uint_as_float(sb[e])));
      mx *= p.scale_log2;
      const float m_new = fmaxf(m_used, mx);
      const bool need = valid && t > 0 && m_new > m_used + 8.f;
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
        for (int c0 = 0; c0 < D; c0 += 32) {
          uint32_t o[32];
          tc::tmem_ld32(tO + lane_base + c0, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tc::tmem_st32(tO + lane_base + c0, o);
        }
        tc::tmem_st_wait();
      }
      if (t >= 2) tc::mbar_wait(pv_done + (t & 1), ((t - 2) >> 1) & 1);  // P buffer free
      const float sc = p.scale_log2;
      float ps = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float p0 = ex2(__uint_as_float(sa[e]) * sc - m_used);
        const float p1 = ex2(__uint_as_float(sa[e + 1]) * sc - m_used);
        ps += p0 + p1;
        pk[e >> 1] = tc::pack_bf16(p0, p1);
      }
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float p0 = ex2(__uint_as_float(sb[e]) * sc - m_used);
        const float p1 = ex2(__uint_as_float(sb[e + 1]) * sc - m_used);
        ps += p0 + p1;
        pk[16 + (e >> 1)] = tc::pack_bf16(p0, p1);
      }
      l += ps;
      if (valid) {
        uint8_t* prow = sPX + (t & 1) * 8192;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(prow + tc::sw128_off(r, c)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(p_full + (t & 1));
    }

    // ---- finalize O^s, lse (forward.cpp:68-78); stage O^s / O^l for the projection
    if (cnt > 0) {
      tc::mbar_wait(pv_done + ((cnt - 1) & 1), ((cnt - 1) >> 1) & 1);
      tc::tc_fence_after();
    }
    const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t o[32];
      if (cnt > 0) {
        tc::tmem_ld32(tO + lane_base + c0, o);
        tc::tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * inv_l);
      if (valid) {
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 v;
          v.x = tc::pack_bf16(__uint_as_float(o[e]), __uint_as_float(o[e + 1]));
          v.y = tc::pack_bf16(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
          v.z = tc::pack_bf16(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5]));
          v.w = tc::pack_bf16(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7]));
          *reinterpret_cast<uint4*>(p.o_s + grow * D + c0 + e) = v;
        }
      }
      if (has_w) tc::tmem_st32(tO + lane_base + c0, o);
    }
    if (valid) p.lse[grow] = l > 0.f ? (m_used + __log2f(l)) * 0.69314718055994531f : kLseSentinel;
    if (has_w) {
      tc::tmem_st_wait();
      if (valid) {  // X <- O^l (bf16), the A operand of O^l W
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint4 v = *reinterpret_cast<const uint4*>(p.o_l + grow * D + 8 * c);
          *reinterpret_cast<uint4*>(sPX + (c >> 3) * 8192 + tc::sw128_off(r, c & 7)) = v;
        }
      }
      tc::fence_proxy_async();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_ready);
      tc::mbar_wait(proj_done, 0);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t o[32];
        tc::tmem_ld32(tO + lane_base + c0, o);
        tc::tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 v;
            v.x = tc::pack_bf16(__uint_as_float(o[e]), __uint_as_float(o[e + 1]));
            v.y = tc::pack_bf16(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
            v.z = tc::pack_bf16(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5]));
            v.w = tc::pack_bf16(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7]));
            *reinterpret_cast<uint4*>(p.o + grow * D + c0 + e) = v;
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

template <int D>
void launch_t(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
              const __nv_bfloat16* Hb, FwdParams p, cudaStream_t st) {
  CUtensorMap tq, tk, tv, th, tw;
  const uint64_t rows = uint64_t(Dm.U) * Dm.N;
  make_tmap_bf16(&tq, q, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tk, k, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&tv, v, D, rows, 1, D, 0, 64);
  make_tmap_bf16(&th, Hb, D, uint64_t(Dm.U) * Dm.Tm * D, 1, D, 0, D);
  if (w)
    make_tmap_bf16(&tw, w, D, uint64_t(Dm.H) * D, 1, D, 0, D);
  else
    tw = th;
  auto kern = k_attn_fwd<D>;
  SLAB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdLayout<D>::kBytes));
  kern<<<dim3(Dm.Tm, unsigned(Dm.U)), 192, FwdLayout<D>::kBytes, st>>>(tq, tk, tv, th, tw, p);
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
  if (Dm.d == 128)
    launch_t<128>(Dm, q, k, v, w, s.Hb, p, st);
  else
    launch_t<64>(Dm, q, k, v, w, s.Hb, p, st);
}

}  // namespace slab
