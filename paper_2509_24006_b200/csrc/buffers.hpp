// buffers.hpp -- carving of the caller-owned `state` and `workspace` buffers.
//
// state  (persists forward -> backward; the device SlaForwardState, forward.hpp:33-43):
//   labels     int8  [U, Tm, Tn]     the CompressedMask label grid (mask.hpp:24-51)
//   crit_cnt   int32 [U, Tm]         per-row critical counts
//   crit_idx   int32 [U, Tm, Tn]     ascending critical columns per row (build_lookup)
//   marg_cnt   int32 [U, Tm]         per-row marginal counts
//   H          f32   [U, Tm, d, d]   row_h: aggregated marginal summaries
//   Z          f32   [U, Tm, d]      row_z
// workspace (scratch, no meaning across calls): see the list below.
#pragma once

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace slab {

struct StateBufs {
  int8_t* labels = nullptr;
  int* crit_cnt = nullptr;
  int* crit_idx = nullptr;
  int* marg_cnt = nullptr;
  int* ccol_cnt = nullptr;   // [U, Tn] critical rows per column (CSC, backward)
  int* ccol_idx = nullptr;   // [U, Tn, Tm] ascending critical rows per column
  int* ccol_marg = nullptr;  // [U, Tn] marginal rows per column (backward linear branch)
  float* H = nullptr;
  float* Z = nullptr;
  __nv_bfloat16* Hb = nullptr;   // fast path: H in bf16 [U, Tm, d, d]
  __nv_bfloat16* M0 = nullptr;   // fast path: marginal indicator [U, Tm, Tn] as bf16 0/1
};

struct WorkBufs {
  double* pq = nullptr;      // pooled Q [U, Tm, d] (f64 or f32 storage)
  double* pk = nullptr;      // pooled K [U, Tn, d]
  double* p_c = nullptr;     // optional scratch for weights (unused when caller passes p_c)
  long long* err = nullptr;  // [8] error slots (first non-finite flat index, ...)
  float* qf = nullptr;       // phi(Q) f32 [U, N, d]
  float* kf = nullptr;       // phi(K) f32 [U, N, d]
  float* h = nullptr;        // KV summaries [U, Tn, d, d]
  float* z = nullptr;        // [U, Tn, d]
  float* dOl = nullptr;      // dO W^T  [U, N, d]
  float* Ds = nullptr;       // <dO^s, O^s> [U, N]
  float* Dl = nullptr;       // <dO^l, O^l> [U, N]
  float* gH = nullptr;       // dH_i [U, Tm, d, d]
  float* gZ = nullptr;       // dZ_i [U, Tm, d]
  float* dq = nullptr;       // sparse dQ [U, N, d]
  float* dk = nullptr;       // sparse dK
  float* dv = nullptr;       // dV (both branches)
  float* dqf = nullptr;      // dQ^phi
  float* dkf = nullptr;      // dK^phi
  __nv_bfloat16* hb = nullptr;   // fast path: h in bf16, [U, Tn, d*d]
  __nv_bfloat16* kfb = nullptr;  // fast path: phi(K) in bf16, [U, N, d]
  __nv_bfloat16* hab = nullptr;  // fast path: dH_agg = M0^T dH in bf16, [U, Tn, d*d]
  float* gZa = nullptr;          // fast path: dZ_agg as three partial columns [U, Tn, 3d]
  float* dwp = nullptr;          // fast path: split-K partials of dW [U * N / 64, d, d]
  __nv_bfloat16* dqphi = nullptr;  // fast path: dQ^phi [U, N, d] (linear kernel -> rows kernel)
  __nv_bfloat16* z3b = nullptr;    // fast path: z_j / dZ_i split into 3 bf16 parts [U, T, 3d]
  __nv_bfloat16* wid = nullptr;    // fast path: identity W [H, d, d] (backward with independent cotangents)
  int* work_ctr = nullptr;         // fast path: dynamic work counter of the persistent columns pass
};

// split-K factor of the fast path's dW GEMM: row chunks of 64*c rows, c | N/64, c <= 32
inline int dw_chunk_tiles(const Dims& D) {
  const long long tiles = D.N / 64;
  for (int c = 32; c > 1; c >>= 1)
    if (tiles % c == 0) return c;
  return 1;
}
inline long long dw_chunks(const Dims& D) { return D.N / (64LL * dw_chunk_tiles(D)); }

// Bump allocator: with base == nullptr it only measures.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

inline void carve_state(const Dims& D, bool fast, void* base, StateBufs& s, size_t* bytes) {
  Carver c(base);
  const size_t U = size_t(D.U), Tm = D.Tm, Tn = D.Tn, d = D.d;
  s.labels = c.take<int8_t>(U * Tm * Tn);
  s.crit_cnt = c.take<int>(U * Tm);
  s.crit_idx = c.take<int>(U * Tm * Tn);
  s.marg_cnt = c.take<int>(U * Tm);
  s.ccol_cnt = c.take<int>(U * Tn);
  s.ccol_idx = c.take<int>(U * Tn * Tm);
  s.ccol_marg = c.take<int>(U * Tn);
  s.Z = c.take<float>(U * Tm * d * (fast ? 3 : 1));  // fast path: three partial columns
  if (fast) {
    s.Hb = c.take<__nv_bfloat16>(U * Tm * d * d);
    s.M0 = c.take<__nv_bfloat16>(U * Tm * ((Tn + 7) / 8 * 8));
  } else {
    s.H = c.take<float>(U * Tm * d * d);
  }
  if (bytes) *bytes = c.off + 256;
}

inline void carve_work(const Dims& D, bool fast, void* base, WorkBufs& w, size_t* bytes) {
  Carver c(base);
  const size_t U = size_t(D.U), Tm = D.Tm, Tn = D.Tn, d = D.d, N = size_t(D.N);
  w.err = c.take<long long>(8);
  w.pq = c.take<double>(U * Tm * d);
  w.pk = c.take<double>(U * Tn * d);
  w.p_c = c.take<double>(U * Tm * Tn);  // pooled scores (f64 or f32 storage)
  w.z = c.take<float>(U * Tn * d);
  w.Ds = c.take<float>(U * N);
  w.Dl = c.take<float>(U * N);
  w.gZ = c.take<float>(U * Tm * d);
  if (fast) {  // tcgen05 path: bf16 operands, the backward writes its totals directly
    w.hb = c.take<__nv_bfloat16>(U * (Tm > Tn ? Tm : Tn) * d * d);  // h_j (forward), dH_i (backward)
    w.kfb = c.take<__nv_bfloat16>(U * size_t(D.Nk) * d);
    w.hab = c.take<__nv_bfloat16>(U * Tn * d * d);
    w.gZa = c.take<float>(U * Tn * 3 * d);
    w.dwp = c.take<float>(U * dw_chunks(D) * d * d);
    w.dqphi = c.take<__nv_bfloat16>(U * N * d);
    const size_t T = Tm > Tn ? Tm : Tn;
    w.z3b = c.take<__nv_bfloat16>(U * T * 3 * d);
    w.wid = c.take<__nv_bfloat16>(size_t(D.H) * d * d);
    w.work_ctr = c.take<int>(4);
  } else {  // generic SIMT path: f32 scratch for every intermediate
    w.qf = c.take<float>(U * N * d);
    w.kf = c.take<float>(U * N * d);
    w.dOl = c.take<float>(U * N * d);
    w.gH = c.take<float>(U * Tm * d * d);
    w.dq = c.take<float>(U * N * d);
    w.dk = c.take<float>(U * N * d);
    w.dv = c.take<float>(U * N * d);
    w.dqf = c.take<float>(U * N * d);
    w.dkf = c.take<float>(U * N * d);
    w.h = c.take<float>(U * Tn * d * d);
  }
  if (bytes) *bytes = c.off + 256;
}

}  // namespace slab
