// common.cuh -- shared device helpers and the problem descriptor used by every kernel.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>

namespace slab {

// Row layout of a CALLER tensor [*, rows, row_elems] that the kernels address as (unit u, row r):
//   0: unit-major with the kernels' row count N per unit (flat row u * N + r)
//   1: unit-major ragged, nv rows per unit (SLA_B200_FLAG_RAGGED): rows r >= nv do not exist
//   2: token-major [B, nv, H, .] (SLA_B200_FLAG_BNHD): unit u = b * H + h
// Tensor maps over modes 1 / 2 are 3-D [U][nv][d] / 4-D [B][nv][H][d]: TMA zero-fills the rows
// r >= nv of a box on loads and clips them on stores, so the kernels read and write the caller's
// tensors in place (no padded copies).
struct RowLayout {
  int mode = 0;
  int H = 1;
  long long nv = 0;
};
// element-row index of (u, r) in the caller tensor, -1 when the row does not exist
__host__ __device__ __forceinline__ long long caller_row(const RowLayout& rl, long long u, long long r, long long N) {
  if (rl.mode == 0) return u * N + r;
  if (r >= rl.nv) return -1;
  if (rl.mode == 1) return u * rl.nv + r;
  return ((u / rl.H) * rl.nv + r) * rl.H + (u % rl.H);
}
// The same map for one unit, resolved once per CTA: caller row of kernel row r is
// base + r * stride when r < nv.  Hot loops use this (no per-row layout branches or divisions;
// inlining caller_row into the attention kernels cost 7-8 % of their time).
struct RowMap {
  long long base, stride, nv;
  __host__ __device__ __forceinline__ long long row(long long r) const { return r < nv ? base + r * stride : -1; }
};
__host__ __device__ __forceinline__ RowMap row_map(const RowLayout& rl, long long u, long long N) {
  if (rl.mode == 0) return RowMap{u * N, 1, N};
  if (rl.mode == 1) return RowMap{u * rl.nv, 1, rl.nv};
  return RowMap{(u / rl.H) * rl.nv * rl.H + u % rl.H, rl.H, rl.nv};
}
// 4-D tensor-map coordinates {col, h, y0 + r, z} of unit u's kernel row r (make_tmap_rows
// builds every caller-tensor map as 4-D: [z][rows][h][d]), resolved once per CTA
struct RowTma {
  int h, y0, z;
};
__host__ __device__ __forceinline__ RowTma row_tma(const RowLayout& rl, long long u, long long N) {
  if (rl.mode == 0) return RowTma{0, int(u * N), 0};
  if (rl.mode == 1) return RowTma{0, 0, int(u)};
  return RowTma{int(u % rl.H), 0, int(u / rl.H)};
}

// Derived problem dimensions (resolved once on the host from sla_b200_problem).
struct Dims {
  int64_t U;     // units = batch * heads
  int64_t B, H;  // batch, heads
  int64_t N;     // query rows per unit in the kernels' buffers (sequence length; padded if ragged)
  int64_t Nk;    // key / value rows per unit (== N unless a rectangular problem, sla_b200_problem.n_kv)
  int64_t Nk_valid;  // valid key rows per unit (== Nk unless ragged)
  RowLayout rl;      // layout of the caller's [*, N, d] tensors and lse (mode 0: the kernels' own)
  int64_t N_valid;  // rows per unit in the caller's tensors (== N unless SLA_B200_FLAG_RAGGED)
  bool bnhd;        // caller tensors are [B, N, H, d] (SLA_B200_FLAG_BNHD)
  bool staged;      // ragged or bnhd: kernels run on unit-major zero-padded workspace copies
  int d, bq, bkv;
  int Tm, Tn;    // query / key-value block counts (layout.hpp:10-20)
  int phi;       // 0 elu1, 1 relu, 2 softmax
  int n1, n_neg; // per-row class counts of a dynamic mask (mask.cpp:98-101)
  float scale_f; // T(1)/sqrt(T(d)) with T=float (block_ops.hpp:16)
  double inv_sqrt_d;  // 1.0/sqrt(double(d)) (mask.cpp:63)
};

constexpr float kLseSentinel = -1e30f;  // forward.hpp:18-24 (f32)

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// IEEE round-to-nearest arithmetic that the compiler may not contract into FMA: the
// reference is built for baseline x86-64 (no FMA), so every a*b+c rounds twice.
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double exp_r(double x) { return exp(x); }
__device__ __forceinline__ float exp_r(float x) { return expf(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// feature map phi (feature_map.cpp:24-40), elementwise kinds
__device__ __forceinline__ float phi_elem(int phi, float x) {
  return phi == 0 ? (x >= 0.f ? x + 1.f : expf(x)) : fmaxf(x, 0.f);
}

// host-side launch accounting (gpu_launches in bench.py comes from here) and the optional
// per-kernel event profiler (profiler.cu)
void count_launch(int n = 1);
void prof_mark(const char* name, cudaStream_t st);
bool prof_enabled();  // per-kernel event profiling on (bench.py's breakdown pass)

#define SLAB_CUDA(call)                                                             \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) throw ::slab::CudaError(std::string(#call) + ": " +      \
                                                   cudaGetErrorString(e_));         \
  } while (0)

struct CudaError {
  std::string msg;
  explicit CudaError(std::string m) : msg(std::move(m)) {}
};
struct InvalidArgument {
  std::string msg;
  explicit InvalidArgument(std::string m) : msg(std::move(m)) {}
};
struct RuntimeFailure {
  std::string msg;
  explicit RuntimeFailure(std::string m) : msg(std::move(m)) {}
};

// Programmatic dependent launch: the next kernel of the chain is launched while this one's
// last CTAs still run, and every kernel launched this way starts with griddep_wait() (returns
// once the preceding grid has completed and its writes are visible), so only the launch
// latency and block rasterisation overlap -- never a read of an unfinished result.
#ifndef SLAB_PDL
#define SLAB_PDL 1
#endif
__device__ __forceinline__ void griddep_wait() {
#if SLAB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void griddep_launch() {
#if SLAB_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// prologue of every kernel launched by launch_pdl
__device__ __forceinline__ void pdl_entry() {
  griddep_wait();
  griddep_launch();
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = SLAB_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // errors surface in check_launch
}

// streaming multiprocessors of the current device (persistent grids)
inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline void check_launch(const char* what, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
  prof_mark(what, st);
}

}  // namespace slab
