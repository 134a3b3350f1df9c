// sla_b200.hpp -- header-only C++ drop-in for the reference operator API, over the C-ABI in
// sla_b200.h.  A caller of the reference swaps `sla::sla_forward(...)` for
// `sla::gpu::sla_forward(...)` (same arguments, same return types, same exceptions):
//
//   reference (namespace sla)                       drop-in (namespace sla::gpu)
//   forward.hpp:63-68   sla_forward                 sla_forward
//   forward.hpp:70-78   sla_forward_with_mask       sla_forward_with_mask
//   forward.hpp:80-83   combine_outputs             combine_outputs
//   backward.hpp:18-23  proj_backward               proj_backward
//   backward.hpp:25-38  sla_backward                sla_backward
//
// Requires the reference headers (sla/forward.hpp, sla/backward.hpp) on the include path, the
// CUDA runtime, and libsla_b200.so at link time.  Host Mat<float> in, host Mat<float> out;
// device buffers are managed here (this is the convenience boundary -- the hot path is the
// device-pointer C-ABI, which performs no allocation).
//
// Precision: by default inputs are rounded to bf16 and run on the tcgen05 fast path
// (b_q = b_kv = 64, d in {64, 128}; outputs within ~1e-2 of the f32 reference).  Set
// sla::gpu::options().fp32 = true for the f32 SIMT kernels (within ~1e-4, any block shape).
//
// sla_backward consumes the SlaForwardState it is given: the state's O^s, O^l and lse are
// uploaded, and the device-side state (lookups, H, Z) is rebuilt from the state's label grid by
// sla_b200_build_state (no attention kernel runs).  combine_outputs and proj_backward run on
// the device (sla_b200_combine_outputs, sla_b200_proj_backward).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "sla/backward.hpp"
#include "sla/forward.hpp"
#include "sla_b200.h"

namespace sla {
namespace gpu {

struct Options {
  bool fp32 = false;         // f32 SIMT kernels instead of the bf16 tcgen05 path
  bool check_finite = true;  // reproduce the reference's non-finite input / output errors
};
inline Options& options() {
  static Options o;
  return o;
}

namespace detail {

inline void throw_status(int rc) {
  if (rc == SLA_B200_OK) return;
  const std::string msg = sla_b200_last_error();
  if (rc == SLA_B200_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("sla::gpu: ") + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 1)); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

inline sla_b200_problem problem(const SlaConfig& cfg, const BlockLayout& layout) {
  sla_b200_problem p{};
  p.batch = 1;
  p.heads = 1;
  p.n = int64_t(layout.n);
  p.d = int64_t(layout.d);
  p.b_q = int64_t(layout.b_q);
  p.b_kv = int64_t(layout.b_kv);
  p.k_h = cfg.k_h;
  p.k_l = cfg.k_l;
  p.phi = int32_t(cfg.phi);
  p.dtype = options().fp32 ? SLA_B200_F32 : SLA_B200_BF16;
  p.mask_precision = SLA_B200_MASK_F64;
  p.flags = options().check_finite ? SLA_B200_FLAG_CHECK_FINITE : 0u;
  return p;
}

inline size_t elem(const sla_b200_problem& p) { return p.dtype == SLA_B200_F32 ? 4 : 2; }

inline void upload(const Mat<float>& m, void* dev, const sla_b200_problem& p) {
  if (p.dtype == SLA_B200_F32) {
    cuda_check(cudaMemcpy(dev, m.data.data(), m.data.size() * 4, cudaMemcpyHostToDevice));
    return;
  }
  std::vector<__nv_bfloat16> h(m.data.size());
  for (size_t i = 0; i < h.size(); ++i) h[i] = __float2bfloat16_rn(m.data[i]);
  cuda_check(cudaMemcpy(dev, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
}

inline Mat<float> download(const void* dev, size_t rows, size_t cols, const sla_b200_problem& p) {
  Mat<float> m(rows, cols);
  if (p.dtype == SLA_B200_F32) {
    cuda_check(cudaMemcpy(m.data.data(), dev, rows * cols * 4, cudaMemcpyDeviceToHost));
    return m;
  }
  std::vector<__nv_bfloat16> h(rows * cols);
  cuda_check(cudaMemcpy(h.data(), dev, h.size() * 2, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < h.size(); ++i) m.data[i] = __bfloat162float(h[i]);
  return m;
}

// One device forward; fills the reference state (outputs, lse, mask) and optionally O.
struct Forward {
  sla_b200_problem p;
  size_t nd, state_bytes = 0, work_bytes = 0;
  DevBuf q, k, v, o_s, o_l, lse, state, work;
  Forward(const sla_b200_problem& pp, const Mat<float>& mq, const Mat<float>& mk, const Mat<float>& mv)
      : p(pp),
        nd(size_t(pp.n * pp.d)),
        q(nd * elem(pp)),
        k(nd * elem(pp)),
        v(nd * elem(pp)),
        o_s(nd * elem(pp)),
        o_l(nd * elem(pp)),
        lse(size_t(pp.n) * 4),
        state(sizes(pp).first),
        work(sizes(pp).second) {
    upload(mq, q.p, p);
    upload(mk, k.p, p);
    upload(mv, v.p, p);
  }
  static std::pair<size_t, size_t> sizes(const sla_b200_problem& p) {
    size_t s = 0, w = 0;
    throw_status(sla_b200_sizes(&p, &s, &w));
    return {s, w};
  }
  void run(const int8_t* host_mask) {
    const size_t grid = size_t(p.n / p.b_q) * size_t(p.n / p.b_kv);
    DevBuf mask(grid);
    if (host_mask) cuda_check(cudaMemcpy(mask.p, host_mask, grid, cudaMemcpyHostToDevice));
    throw_status(sla_b200_forward(&p, q.p, k.p, v.p, nullptr, host_mask ? static_cast<int8_t*>(mask.p) : nullptr,
                                  nullptr, o_s.p, o_l.p, static_cast<float*>(lse.p), state.p, work.p, nullptr));
    cuda_check(cudaDeviceSynchronize());
  }
  // ExecCounters of this forward as the reference counts them for cfg's strategy, added to c
  // (forward.cpp:152-161), from the device LUT (sla_b200_exec_counters)
  void count(const SlaConfig& cfg, ExecCounters* c) const {
    if (!c) return;
    sla_b200_counters e{};
    throw_status(sla_b200_exec_counters(&p, q.p, state.p, static_cast<int>(cfg.aggregation),
                                        static_cast<int>(cfg.group_size), &e, work.p, nullptr));
    c->sparse_block_matmuls += e.sparse_block_matmuls;
    c->linear_row_products += e.linear_row_products;
    c->aggregation.additions += e.additions;
    c->aggregation.subtractions += e.subtractions;
    c->aggregation.lookups += e.lookups;
    c->aggregation.table_build_additions += e.table_build_additions;
  }
  SlaForwardState<float> state_of() const {
    SlaForwardState<float> st;
    const size_t n = size_t(p.n), d = size_t(p.d);
    st.sparse_out = download(o_s.p, n, d, p);
    st.linear_out = download(o_l.p, n, d, p);
    st.row_lse.resize(n);
    cuda_check(cudaMemcpy(st.row_lse.data(), lse.p, n * 4, cudaMemcpyDeviceToHost));
    const int8_t* dl = nullptr;
    throw_status(sla_b200_state_labels(&p, state.p, &dl));
    const size_t tm = size_t(p.n / p.b_q), tn = size_t(p.n / p.b_kv);
    std::vector<int8_t> labels(tm * tn);
    cuda_check(cudaMemcpy(labels.data(), dl, labels.size(), cudaMemcpyDeviceToHost));
    st.mask = build_lookup(tm, tn, std::move(labels));
    return st;
  }
};

}  // namespace detail

// forward.cpp:174-185 -- the mask is re-predicted from the live q, k.
inline SlaForwardState<float> sla_forward(const Mat<float>& q, const Mat<float>& k, const Mat<float>& v,
                                          const SlaConfig& cfg, const BlockLayout& layout, unsigned = 1,
                                          ExecCounters* counters = nullptr) {
  validate_config(cfg);
  detail::Forward f(detail::problem(cfg, layout), q, k, v);
  f.run(nullptr);
  f.count(cfg, counters);
  return f.state_of();
}

// forward.cpp:81-172 -- injected label grid.
inline SlaForwardState<float> sla_forward_with_mask(const Mat<float>& q, const Mat<float>& k,
                                                    const Mat<float>& v, const CompressedMask& mask,
                                                    const SlaConfig& cfg, const BlockLayout& layout,
                                                    unsigned = 1, ExecCounters* counters = nullptr) {
  if (mask.t_m != layout.t_m || mask.t_n != layout.t_n)
    throw std::invalid_argument("sla_forward: mask does not match layout");
  detail::Forward f(detail::problem(cfg, layout), q, k, v);
  f.run(mask.labels.data());
  f.count(cfg, counters);
  return f.state_of();
}

// a block size for calls that only need N x d row work (combine / proj_backward)
inline BlockLayout row_layout(size_t n, size_t d) {
  size_t b = 64;
  while (n % b) b >>= 1;
  return make_block_layout(n, d, b, b);
}

// forward.cpp:187-195 -- O = O^l W + O^s on the device (f32 accumulation).
inline Mat<float> combine_outputs(const SlaForwardState<float>& state, const OutputProjection<float>& proj) {
  const size_t n = state.sparse_out.rows, d = state.sparse_out.cols;
  if (!state.linear_out.same_shape(state.sparse_out) || proj.w.rows != d || proj.w.cols != d)
    throw std::invalid_argument("combine_outputs: shape mismatch");
  SlaConfig cfg;
  const sla_b200_problem p = detail::problem(cfg, row_layout(n, d));
  const size_t es = detail::elem(p);
  detail::DevBuf os(n * d * es), ol(n * d * es), w(d * d * es), o(n * d * es);
  detail::upload(state.sparse_out, os.p, p);
  detail::upload(state.linear_out, ol.p, p);
  detail::upload(proj.w, w.p, p);
  detail::throw_status(sla_b200_combine_outputs(&p, os.p, ol.p, w.p, o.p, nullptr));
  detail::cuda_check(cudaDeviceSynchronize());
  return detail::download(o.p, n, d, p);
}

// backward.cpp:12-22 -- (dO^s, dO^l, dW) = (dO, dO W^T, O^l^T dO) on the device.
inline std::tuple<Mat<float>, Mat<float>, Mat<float>> proj_backward(const Mat<float>& d_out,
                                                                    const Mat<float>& linear_out,
                                                                    const Mat<float>& w) {
  if (!d_out.same_shape(linear_out)) throw std::invalid_argument("proj_backward: shape mismatch");
  const size_t n = d_out.rows, d = d_out.cols;
  SlaConfig cfg;
  const sla_b200_problem p = detail::problem(cfg, row_layout(n, d));
  const size_t es = detail::elem(p);
  size_t sb = 0, wbytes = 0;
  detail::throw_status(sla_b200_sizes(&p, &sb, &wbytes));
  detail::DevBuf dout(n * d * es), ol(n * d * es), wd(d * d * es), dol(n * d * es), dw(d * d * 4), work(wbytes);
  detail::upload(d_out, dout.p, p);
  detail::upload(linear_out, ol.p, p);
  detail::upload(w, wd.p, p);
  detail::throw_status(sla_b200_proj_backward(&p, dout.p, ol.p, wd.p, dol.p, static_cast<float*>(dw.p), work.p,
                                              nullptr));
  detail::cuda_check(cudaDeviceSynchronize());
  Mat<float> dwm(d, d);
  detail::cuda_check(cudaMemcpy(dwm.data.data(), dw.p, d * d * 4, cudaMemcpyDeviceToHost));
  return {d_out, detail::download(dol.p, n, d, p), std::move(dwm)};
}

// backward.hpp:25-38 -- gradients through both branches from independent cotangents dO^s, dO^l
// (sla_b200_backward_split), with the component gradients (backward.hpp:10-16) and
// dproj = O^l^T dO^s (backward.cpp:46).  The caller's state is the one consumed.
inline SlaGradients<float> sla_backward(const SlaForwardState<float>& state, const Mat<float>& q,
                                        const Mat<float>& k, const Mat<float>& v,
                                        const Mat<float>& d_out_sparse, const Mat<float>& d_out_linear,
                                        const SlaConfig& cfg, const BlockLayout& layout, unsigned = 1,
                                        ExecCounters* = nullptr) {
  const size_t n = layout.n, d = layout.d;
  if (state.row_lse.size() != n || state.mask.t_m != layout.t_m || state.mask.t_n != layout.t_n)
    throw std::invalid_argument("sla_backward: state does not match layout");
  if (d_out_sparse.rows != n || d_out_sparse.cols != d || d_out_linear.rows != n || d_out_linear.cols != d)
    throw std::invalid_argument("sla_backward: cotangent shape mismatch");
  validate_config(cfg);
  const sla_b200_problem p = detail::problem(cfg, layout);
  const size_t es = detail::elem(p), grid = layout.t_m * layout.t_n;
  size_t sb = 0, wbytes = 0;
  detail::throw_status(sla_b200_sizes(&p, &sb, &wbytes));
  detail::DevBuf q_(n * d * es), k_(n * d * es), v_(n * d * es), os(n * d * es), ol(n * d * es), lse(n * 4),
      mask(grid), st(sb), work(wbytes), dos(n * d * es), dol(n * d * es), dq(n * d * es), dk(n * d * es),
      dv(n * d * es), dw(d * d * 4), pq(n * d * 4), pk(n * d * 4), pqf(n * d * 4), pkf(n * d * 4);
  detail::upload(q, q_.p, p);
  detail::upload(k, k_.p, p);
  detail::upload(v, v_.p, p);
  detail::upload(state.sparse_out, os.p, p);
  detail::upload(state.linear_out, ol.p, p);
  detail::upload(d_out_sparse, dos.p, p);
  detail::upload(d_out_linear, dol.p, p);
  detail::cuda_check(cudaMemcpy(lse.p, state.row_lse.data(), n * 4, cudaMemcpyHostToDevice));
  detail::cuda_check(cudaMemcpy(mask.p, state.mask.labels.data(), grid, cudaMemcpyHostToDevice));
  detail::throw_status(sla_b200_build_state(&p, q_.p, k_.p, v_.p, static_cast<int8_t*>(mask.p), st.p, work.p,
                                            nullptr));
  sla_b200_grad_parts parts{static_cast<float*>(pq.p), static_cast<float*>(pk.p), static_cast<float*>(pqf.p),
                            static_cast<float*>(pkf.p)};
  detail::throw_status(sla_b200_backward_split(&p, q_.p, k_.p, v_.p, os.p, ol.p, static_cast<float*>(lse.p),
                                               dos.p, dol.p, dq.p, dk.p, dv.p, static_cast<float*>(dw.p), &parts,
                                               st.p, work.p, nullptr));
  detail::cuda_check(cudaDeviceSynchronize());
  SlaGradients<float> g;
  g.dq_total = detail::download(dq.p, n, d, p);
  g.dk_total = detail::download(dk.p, n, d, p);
  g.dv = detail::download(dv.p, n, d, p);
  g.dproj = Mat<float>(d, d);
  detail::cuda_check(cudaMemcpy(g.dproj.data.data(), dw.p, d * d * 4, cudaMemcpyDeviceToHost));
  sla_b200_problem pf = p;
  pf.dtype = SLA_B200_F32;
  g.dq = detail::download(pq.p, n, d, pf);
  g.dk = detail::download(pk.p, n, d, pf);
  g.dq_feat = detail::download(pqf.p, n, d, pf);
  g.dk_feat = detail::download(pkf.p, n, d, pf);
  return g;
}

}  // namespace gpu
}  // namespace sla
