// ref_capi.cpp -- extern "C" entry points over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY; built by oracle/Makefile into oracle/_ref/libsla_ref.so
// from the sources under /root/reference/proj/core, which are never copied here).
//
// Used by tests/ to pin the C restatement (sla_oracle.c) and to generate the golden
// fixtures, and by bench.py --impl reference / cpu_baseline as the reference's own CPU
// path.  Each call runs the reference's public API exactly as its callers do
// (tools/sla_main.cpp:111-215, core/src/finetune.cpp:24-68):
//   sla_forward[_with_mask] -> combine_outputs -> proj_backward -> sla_backward.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sla/backward.hpp"
#include "sla/flops.hpp"
#include "sla/forward.hpp"
#include "sla/mask.hpp"

namespace {

void put_err(const std::string& msg, char* err, std::size_t len) {
  if (!err || !len) return;
  std::strncpy(err, msg.c_str(), len - 1);
  err[len - 1] = 0;
}

template <typename T>
sla::Mat<T> load(const T* p, std::size_t r, std::size_t c) {
  return sla::Mat<T>(r, c, std::vector<T>(p, p + r * c));
}

template <typename T>
void store(const sla::Mat<T>& m, T* p) {
  if (p) std::memcpy(p, m.data.data(), sizeof(T) * m.data.size());
}

template <typename T>
int run(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv, double kh, double kl,
        int phi, unsigned threads, const T* q, const T* k, const T* v, const T* w,
        const std::int8_t* labels_in, const T* d_out, std::int8_t* labels_out, T* o_s, T* o_l,
        T* o, T* lse, T* dq_total, T* dk_total, T* dv, T* dw, T* dq, T* dk, T* dq_feat,
        T* dk_feat, char* err, std::size_t errlen) {
  try {
    sla::SlaConfig cfg;
    cfg.k_h = kh;
    cfg.k_l = kl;
    cfg.phi = static_cast<sla::FeatureMapKind>(phi);
    cfg.dtype = sizeof(T) == 4 ? sla::Dtype::f32 : sla::Dtype::f64;
    const auto layout = sla::make_block_layout(n, d, bq, bkv);
    const auto mq = load(q, n, d), mk = load(k, n, d), mv = load(v, n, d);
    sla::SlaForwardState<T> st;
    if (labels_in) {
      sla::validate_config(cfg);
      auto mask = sla::build_lookup(layout.t_m, layout.t_n,
                                    std::vector<std::int8_t>(labels_in, labels_in + layout.t_m * layout.t_n));
      st = sla::sla_forward_with_mask(mq, mk, mv, mask, cfg, layout, threads);
    } else {
      st = sla::sla_forward(mq, mk, mv, cfg, layout, threads);
    }
    if (labels_out) std::memcpy(labels_out, st.mask.labels.data(), st.mask.labels.size());
    store(st.sparse_out, o_s);
    store(st.linear_out, o_l);
    if (lse) std::memcpy(lse, st.row_lse.data(), sizeof(T) * n);
    if (!w) return 0;
    sla::OutputProjection<T> proj{load(w, d, d)};
    if (o) store(sla::combine_outputs(st, proj), o);
    if (!d_out) return 0;
    auto [dos, dol, dproj] = sla::proj_backward(load(d_out, n, d), st.linear_out, proj.w);
    auto g = sla::sla_backward(st, mq, mk, mv, dos, dol, cfg, layout, threads);
    store(g.dq_total, dq_total);
    store(g.dk_total, dk_total);
    store(g.dv, dv);
    store(dproj, dw);
    store(g.dq, dq);
    store(g.dk, dk);
    store(g.dq_feat, dq_feat);
    store(g.dk_feat, dk_feat);
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(e.what(), err, errlen);
    return 2;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

}  // namespace

extern "C" {

int ref_run_f32(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv, double kh,
                double kl, int phi, unsigned threads, const float* q, const float* k,
                const float* v, const float* w, const std::int8_t* labels_in, const float* d_out,
                std::int8_t* labels_out, float* o_s, float* o_l, float* o, float* lse,
                float* dq_total, float* dk_total, float* dv, float* dw, float* dq, float* dk,
                float* dq_feat, float* dk_feat, char* err, std::size_t errlen) {
  return run<float>(n, d, bq, bkv, kh, kl, phi, threads, q, k, v, w, labels_in, d_out,
                    labels_out, o_s, o_l, o, lse, dq_total, dk_total, dv, dw, dq, dk, dq_feat,
                    dk_feat, err, errlen);
}

int ref_run_f64(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv, double kh,
                double kl, int phi, unsigned threads, const double* q, const double* k,
                const double* v, const double* w, const std::int8_t* labels_in,
                const double* d_out, std::int8_t* labels_out, double* o_s, double* o_l,
                double* o, double* lse, double* dq_total, double* dk_total, double* dv,
                double* dw, double* dq, double* dk, double* dq_feat, double* dk_feat, char* err,
                std::size_t errlen) {
  return run<double>(n, d, bq, bkv, kh, kl, phi, threads, q, k, v, w, labels_in, d_out,
                     labels_out, o_s, o_l, o, lse, dq_total, dk_total, dv, dw, dq, dk, dq_feat,
                     dk_feat, err, errlen);
}

// mask.cpp:57-81 on f64 inputs
int ref_predict(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv, const double* q,
                const double* k, double* p_c, char* err, std::size_t errlen) {
  try {
    const auto layout = sla::make_block_layout(n, d, bq, bkv);
    auto w = sla::predict_compressed_weights(load(q, n, d), load(k, n, d), layout);
    store(w.p_c, p_c);
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(e.what(), err, errlen);
    return 2;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// mask.cpp:91-119
int ref_classify(std::size_t t_m, std::size_t t_n, const double* p_c, double kh, double kl,
                 std::int8_t* labels, char* err, std::size_t errlen) {
  try {
    sla::CompressedWeights w{load(p_c, t_m, t_n)};
    auto m = sla::classify_mask(w, kh, kl);
    std::memcpy(labels, m.labels.data(), m.labels.size());
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(e.what(), err, errlen);
    return 2;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// forward.cpp:81-172 with ExecCounters (forward.hpp:46-50) on an injected label grid, one
// aggregation strategy (config.hpp:19-31: 0 direct, 1 complement, 2 Four-Russians, 3 auto).
// out: sparse_block_matmuls, linear_row_products, additions, subtractions, lookups,
// table_build_additions.
int ref_exec_counters(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv, int phi,
                      int aggregation, std::size_t group_size, const float* q, const float* k,
                      const float* v, const std::int8_t* labels, std::uint64_t* out, char* err,
                      std::size_t errlen) {
  try {
    sla::SlaConfig cfg;
    cfg.phi = static_cast<sla::FeatureMapKind>(phi);
    cfg.dtype = sla::Dtype::f32;
    cfg.aggregation = static_cast<sla::AggregationKind>(aggregation);
    cfg.group_size = group_size;
    const auto layout = sla::make_block_layout(n, d, bq, bkv);
    auto mask = sla::build_lookup(layout.t_m, layout.t_n,
                                  std::vector<std::int8_t>(labels, labels + layout.t_m * layout.t_n));
    sla::ExecCounters c;
    sla::sla_forward_with_mask(load(q, n, d), load(k, n, d), load(v, n, d), mask, cfg, layout, 1, &c);
    const std::uint64_t r[6] = {c.sparse_block_matmuls, c.linear_row_products,
                                c.aggregation.additions, c.aggregation.subtractions,
                                c.aggregation.lookups, c.aggregation.table_build_additions};
    std::memcpy(out, r, sizeof(r));
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(e.what(), err, errlen);
    return 2;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

// flops.cpp:7-33.  out: full, sparse, linear, proj, mask, sla_total; out_f: ratio, sparsity.
int ref_flops_report(std::size_t n, std::size_t d, std::size_t bq, std::size_t bkv,
                     const std::int8_t* labels, std::uint64_t* out, double* out_f, char* err,
                     std::size_t errlen) {
  try {
    const auto layout = sla::make_block_layout(n, d, bq, bkv);
    auto mask = sla::build_lookup(layout.t_m, layout.t_n,
                                  std::vector<std::int8_t>(labels, labels + layout.t_m * layout.t_n));
    const auto r = sla::flops_report(layout, mask);
    const std::uint64_t u[6] = {r.full_flops, r.sparse_flops, r.linear_flops, r.proj_flops,
                                r.mask_flops, r.sla_total};
    std::memcpy(out, u, sizeof(u));
    out_f[0] = r.ratio;
    out_f[1] = r.sparsity;
    return 0;
  } catch (const std::invalid_argument& e) {
    put_err(e.what(), err, errlen);
    return 2;
  } catch (const std::exception& e) {
    put_err(e.what(), err, errlen);
    return 1;
  }
}

}  // extern "C"
