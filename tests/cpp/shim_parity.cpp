// Drop-in demonstration: the reference's own training-step call sequence
// (core/src/finetune.cpp:44-61) run twice -- once through namespace sla (the reference CPU
// library) and once through namespace sla::gpu (include/sla_b200.hpp over libsla_b200.so) --
// on identical bf16-representable inputs.  Prints one JSON line of max-norm relative diffs.
#include <cstdio>
#include <algorithm>
#include <cmath>

#include "sla/backward.hpp"
#include "sla/forward.hpp"
#include "sla/rng.hpp"
#include "sla_b200.hpp"

using namespace sla;

static MatF bf16_mat(SplitMix64& rng, size_t r, size_t c, double sd) {
  MatF m(r, c);
  for (auto& x : m.data) x = __bfloat162float(__float2bfloat16_rn(float(sd * rng.gaussian())));
  return m;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? size_t(atoi(argv[1])) : 1024, d = argc > 2 ? size_t(atoi(argv[2])) : 64;
  SlaConfig cfg;
  cfg.k_h = 5;
  cfg.k_l = 10;
  cfg.phi = FeatureMapKind::feat_softmax;
  const auto layout = make_block_layout(n, d, 64, 64);
  SplitMix64 rng(2024);
  MatF q = bf16_mat(rng, n, d, 1.0), k = bf16_mat(rng, n, d, 1.0), v = bf16_mat(rng, n, d, 1.0);
  MatF w = bf16_mat(rng, d, d, 0.1), dout = bf16_mat(rng, n, d, 1.0);

  // reference
  cfg.aggregation = argc > 3 ? static_cast<AggregationKind>(atoi(argv[3])) : AggregationKind::direct;
  ExecCounters c_ref, c_gpu;
  auto st = sla::sla_forward(q, k, v, cfg, layout, 8, &c_ref);
  auto o = sla::combine_outputs(st, OutputProjection<float>{w});
  auto [ds, dl, dw] = sla::proj_backward(dout, st.linear_out, w);
  auto g = sla::sla_backward(st, q, k, v, ds, dl, cfg, layout, 8);

  // drop-in (same calls, namespace sla::gpu)
  auto st2 = sla::gpu::sla_forward(q, k, v, cfg, layout, 1, &c_gpu);
  auto o2 = sla::gpu::combine_outputs(st2, OutputProjection<float>{w});
  auto [ds2, dl2, dw2] = sla::gpu::proj_backward(dout, st2.linear_out, w);
  auto g2 = sla::gpu::sla_backward(st2, q, k, v, ds2, dl2, cfg, layout);

  // backward.hpp:25-38 takes independent cotangents: linearity in (dO^s, dO^l)
  // (backward_test.cpp:160-190) through the drop-in, with cotangents unrelated through W
  MatF a_s = bf16_mat(rng, n, d, 1.0), a_l = bf16_mat(rng, n, d, 1.0);
  MatF b_s = bf16_mat(rng, n, d, 1.0), b_l = bf16_mat(rng, n, d, 1.0);
  const float ca = 0.75f, cb = -1.25f;  // the mixed cotangents are rounded to bf16 on upload
  MatF mix_s(n, d), mix_l(n, d);
  for (size_t e = 0; e < a_s.data.size(); ++e) {
    mix_s.data[e] = ca * a_s.data[e] + cb * b_s.data[e];
    mix_l.data[e] = ca * a_l.data[e] + cb * b_l.data[e];
  }
  auto ga = sla::gpu::sla_backward(st2, q, k, v, a_s, a_l, cfg, layout);
  auto gb = sla::gpu::sla_backward(st2, q, k, v, b_s, b_l, cfg, layout);
  auto gm = sla::gpu::sla_backward(st2, q, k, v, mix_s, mix_l, cfg, layout);
  auto lin_err = [&](const MatF& ma, const MatF& mb, const MatF& mm) {
    MatF comb(ma.rows, ma.cols);
    for (size_t e = 0; e < comb.data.size(); ++e) comb.data[e] = ca * ma.data[e] + cb * mb.data[e];
    return rel_diff(mm, comb, 1.0);
  };
  double linearity = 0.0;
  for (double x : {lin_err(ga.dq_total, gb.dq_total, gm.dq_total), lin_err(ga.dk_total, gb.dk_total, gm.dk_total),
                   lin_err(ga.dv, gb.dv, gm.dv)})
    linearity = std::max(linearity, x);
  // the same independent cotangents through the reference
  auto gr = sla::sla_backward(st, q, k, v, a_s, a_l, cfg, layout, 8);

  const bool labels_equal = st.mask.labels == st2.mask.labels;
  const bool counters_equal =
      c_ref.sparse_block_matmuls == c_gpu.sparse_block_matmuls &&
      c_ref.linear_row_products == c_gpu.linear_row_products &&
      c_ref.aggregation.additions == c_gpu.aggregation.additions &&
      c_ref.aggregation.subtractions == c_gpu.aggregation.subtractions &&
      c_ref.aggregation.lookups == c_gpu.aggregation.lookups &&
      c_ref.aggregation.table_build_additions == c_gpu.aggregation.table_build_additions;
  std::printf(
      "{\"n\": %zu, \"d\": %zu, \"labels_equal\": %s, \"counters_equal\": %s, \"o\": %.3e, \"o_s\": %.3e, \"o_l\": %.3e, "
      "\"dq_total\": %.3e, \"dk_total\": %.3e, \"dv\": %.3e, \"dw\": %.3e, \"dproj\": %.3e, \"dl\": %.3e, "
      "\"dq\": %.3e, \"dk\": %.3e, \"dq_feat\": %.3e, \"dk_feat\": %.3e, "
      "\"split_dq_total\": %.3e, \"split_dk_total\": %.3e, \"split_dv\": %.3e, \"split_dproj\": %.3e, "
      "\"linearity\": %.3e}\n",
      n, d, labels_equal ? "true" : "false", counters_equal ? "true" : "false", rel_diff(o2, o, 1.0), rel_diff(st2.sparse_out, st.sparse_out, 1.0),
      rel_diff(st2.linear_out, st.linear_out, 1.0), rel_diff(g2.dq_total, g.dq_total, 1.0),
      rel_diff(g2.dk_total, g.dk_total, 1.0), rel_diff(g2.dv, g.dv, 1.0), rel_diff(dw2, dw, 1.0),
      rel_diff(g2.dproj, g.dproj, 1.0), rel_diff(dl2, dl, 1.0), rel_diff(g2.dq, g.dq, 1.0), rel_diff(g2.dk, g.dk, 1.0),
      rel_diff(g2.dq_feat, g.dq_feat, 1.0), rel_diff(g2.dk_feat, g.dk_feat, 1.0),
      rel_diff(ga.dq_total, gr.dq_total, 1.0), rel_diff(ga.dk_total, gr.dk_total, 1.0), rel_diff(ga.dv, gr.dv, 1.0),
      rel_diff(ga.dproj, gr.dproj, 1.0), linearity);
  return labels_equal && counters_equal ? 0 : 1;
}
