// bwd_common.cuh -- helpers shared by the backward kernels (attn_bwd.cu, attn_bwd_rows.cu).
#pragma once

#include "kernels.hpp"
#include "tc.cuh"

#ifndef SLAB_DBG_X
#define SLAB_DBG_X 100  // -DSLAB_TIMELINE: key/query block of the traced CTA (unit 6)
#endif

namespace slab {

// debug timeline of one CTA (-DSLAB_TIMELINE; read by sla_b200_diag_bwd_timeline in attn_bwd_rows.cu)
static __device__ long long g_bwd_ts[256];
// -DSLAB_TIMELINE: per-CTA phase clocks [cta][start, loop start, loop end, end | smid << 56]
static __device__ unsigned long long g_cta_prof[8192][4];

namespace {

__device__ __forceinline__ void ts_mark(bool on, int slot) {  // -DSLAB_TIMELINE builds only
#ifdef SLAB_TIMELINE
  if (on) g_bwd_ts[slot] = clock64();
#else
  (void)on;
  (void)slot;
#endif
}

// per work item (a CTA of a grid launch, or an item of a persistent CTA)
__device__ __forceinline__ void cta_mark(bool on, int slot, long long id) {  // -DSLAB_TIMELINE builds only
#ifdef SLAB_TIMELINE
  if (on) {
    unsigned long long v = clock64();
    if (slot == 3) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      v |= (unsigned long long)sm << 56;
    }
    g_cta_prof[id & 8191][slot] = v;
  }
#else
  (void)on;
  (void)slot;
  (void)id;
#endif
}
__device__ __forceinline__ void cta_mark(bool on, int slot) {
  cta_mark(on, slot, (long long)blockIdx.y * gridDim.x + blockIdx.x);
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
  const int* ccol_marg;
  const float* Z;      // [U, Tm, D]
  const float* lse;    // [U, N]
  const float* Ds;     // [U, N] (rows kernel writes, cols kernel reads)
  float* Ds_out;
  const __nv_bfloat16* o_s;
  const __nv_bfloat16* o_l;
  __nv_bfloat16* gH;   // [U, Tm, D, D] dH_i (linear kernel out)
  __nv_bfloat16* dqphi;  // [U, N, D] dQ^phi (linear kernel out, rows kernel in)
  __nv_bfloat16* z3;   // [U, Tm, 3D] dZ_i in 3 bf16 parts (B operand of dZ_agg = M0^T dZ)
  const float* gZa;    // [U, Tn, 3D] dZ_agg as three partial columns (cols kernel in)
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
  long long items;     // persistent kernels: work items of the launch
  RowLayout rl;        // the caller's q, k, v, dO, o_s, o_l, lse, dq, dk, dv (in place)
  int* work;           // k_bwd_cols: dynamic work counter (zeroed before the launch)
  int ds_external;     // k_bwd_lin: D^s comes from k_rowdot (independent cotangents), not dO . O^s
  // optional SlaGradients parts (backward.hpp:10-16), f32 [U, N, D]; null: not written
  float* dq_part;      // sparse dQ
  float* dqf_part;     // dQ^phi
  float* dk_part;      // sparse dK
  float* dkf_part;     // dK^phi (dK^phi + the broadcast dZ_agg)
};


}  // namespace
}  // namespace slab
