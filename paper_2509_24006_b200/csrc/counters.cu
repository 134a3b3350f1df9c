// counters.cu -- device accounting from the block LUT:
// flops_report (flops.cpp:7-33) and the forward's ExecCounters (forward.hpp:46-50,
// forward.cpp:117-161) computed from the label grid / counts the classification left in the
// state, plus one pass over Q for the rows whose linear denominator is non-zero.
//
// k_row_stats: one thread per (unit, block row): critical and marginal counts, the number of
//   Four-Russians groups of `g` consecutive key blocks holding a marginal block
//   (aggregation.cpp:118-145).
// k_lin_rows: one warp per query row of a block row with a marginal block: den = phi(q) . Z_i
//   is a sum of non-negative products (phi >= 0, z >= 0), so den != 0 iff some product
//   phi(q)_a Z_i[a] is non-zero (forward.cpp:133-136); per-block-row counts, no atomics.
#include "kernels.hpp"
#include "tc.cuh"

namespace slab {
namespace {

__global__ void k_row_stats(const int8_t* __restrict__ labels, long long rows, int Tn, int g,
                            int4* __restrict__ out) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int8_t* lrow = labels + r * Tn;
  int crit = 0, marg = 0, groups = 0;
  for (int b = 0; b < Tn; b += g) {
    bool hit = false;
    for (int j = b; j < min(b + g, Tn); ++j) {
      const int l = lrow[j];
      crit += l == 1;
      marg += l == 0;
      hit |= l == 0;
    }
    groups += hit;
  }
  out[r] = make_int4(crit, marg, groups, 0);
}

// q: unit-major [U, N, d] (bf16 or f32); Z: [U, Tm, d] f32, or three bf16-split parts
// [U, Tm, 3d] (z3 = 1, the fast path's layout, summed as the consumers do)
template <typename T>
__global__ void k_lin_rows(const T* __restrict__ q, const float* __restrict__ Z, int z3,
                           const int4* __restrict__ stats, int N, int n_valid, int d, int bq,
                           int Tm, int phi, int* __restrict__ lin_rows, RowLayout rl) {
  const int i = blockIdx.x, u = blockIdx.y;
  const long long urow = (long long)u * Tm + i;
  if (threadIdx.x == 0) lin_rows[urow] = 0;
  __syncthreads();
  if (stats[urow].y == 0) return;  // no marginal block: the row is skipped (forward.cpp:130)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float* zi = Z + urow * (long long)(z3 ? 3 * d : d);
  int count = 0;
  for (int rr = warp; rr < bq; rr += nw) {
    const int r = i * bq + rr;
    if (r >= n_valid) break;
    const T* qr = q + caller_row(rl, u, r, N) * d;
    float mx = -INFINITY, se = 0.f;
    if (phi == 2) {  // per-row softmax over the d features (feature_map.cpp:22-40)
      for (int a = lane; a < d; a += 32) mx = fmaxf(mx, to_f(qr[a]));
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int a = lane; a < d; a += 32) se += __expf(to_f(qr[a]) - mx);
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    }
    bool nz = false;
    for (int a = lane; a < d; a += 32) {
      const float x = to_f(qr[a]);
      const float f = phi == 2 ? __expf(x - mx) / se : phi_elem(phi, x);
      const float za = z3 ? tc::load_sum3(zi + a, d) : zi[a];
      nz |= f * za != 0.f;
    }
    count += __any_sync(0xffffffffu, nz) ? 1 : 0;
  }
  if (lane == 0 && count) atomicAdd(lin_rows + urow, count);  // <= bq / 32 adds per block row
}

}  // namespace

void launch_row_stats(const Dims& D, const int8_t* labels, int g, int4* out, cudaStream_t st) {
  const long long rows = D.U * (long long)D.Tm;
  k_row_stats<<<unsigned((rows + 127) / 128), 128, 0, st>>>(labels, rows, D.Tn, g, out);
  check_launch("k_row_stats", st);
}

void launch_lin_rows(const Dims& D, int dtype, const void* q, const float* Z, bool z3,
                     const int4* stats, int* lin_rows, cudaStream_t st) {
  const dim3 grid(unsigned(D.Tm), unsigned(D.U));
  if (dtype == 0)
    k_lin_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(q), Z, z3, stats,
                                                   int(D.N), int(D.N_valid), D.d, D.bq, D.Tm, D.phi, lin_rows, D.rl);
  else
    k_lin_rows<float><<<grid, 256, 0, st>>>(static_cast<const float*>(q), Z, z3, stats, int(D.N),
                                           int(D.N_valid), D.d, D.bq, D.Tm, D.phi, lin_rows, D.rl);
  check_launch("k_lin_rows", st);
}

}  // namespace slab
