/*
 * sla_oracle.h -- CPU restatement of the SLA reference path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the CUDA product path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It is never on the product path.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj/core); see the citation on each declaration.  All math is
 * IEEE f64 with the reference's loop order (sequential ascending sums, mul and add
 * rounded separately -- the reference is built for baseline x86-64, which has no FMA).
 *
 * Parity pinned: tests/test_oracle.py checks this file against the reference's own
 * known-answer tests (tests/*_test.cpp) and against golden vectors produced by the
 * reference itself (oracle/_ref, tests/golden/make_golden.py).
 */
#ifndef SLA_ORACLE_H
#define SLA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- fixture generator: include/sla/rng.hpp:22-64 ---------------------------------- */
uint64_t orc_rng_next(uint64_t* state);
double orc_rng_uniform(uint64_t* state);                        /* (0,1]            */
void orc_rng_gaussian(uint64_t* state, double* out, size_t count, double stddev);
void orc_rng_uniform_range(uint64_t* state, double* out, size_t count, double lo, double hi);
/* tests/test_support.hpp:99-116 random_mask (labels only) */
void orc_random_mask(uint64_t* state, size_t t_m, size_t t_n, double p_critical,
                     double p_marginal, int allow_empty_critical, int8_t* labels);

/* ---- layout / config validation: layout.cpp:8-26, config.cpp:7-19 ------------------- */
/* returns 0 ok, 2 invalid (message copied into err if non-NULL) */
int orc_validate(size_t n, size_t d, size_t b_q, size_t b_kv, double k_h, double k_l,
                 char* err, size_t err_len);

/* ---- mask stage: mask.cpp:40-153 ------------------------------------------------------ */
int orc_pool_mean(const double* x, size_t rows, size_t cols, size_t b, double* out);
int orc_predict(const double* q, const double* k, size_t n, size_t d, size_t b_q,
                size_t b_kv, double* p_c /* T_m x T_n */);
int orc_predict_ragged(const double* q, const double* k, size_t n, size_t d, size_t b, double* p_c);
/* pooled, scaled scores before the softmax (same op order as predict) */
int orc_scores(const double* q, const double* k, size_t n, size_t d, size_t b_q,
               size_t b_kv, double* s /* T_m x T_n */);
void orc_counts(size_t t_n, double k_h, double k_l, size_t* n1, size_t* n_neg);
int orc_classify(const double* p_c, size_t t_m, size_t t_n, double k_h, double k_l,
                 int8_t* labels);

/* ---- feature map: feature_map.cpp:10-73 ----------------------------------------------- */
void orc_phi(const double* x, size_t rows, size_t d, int phi, double* out);
void orc_phi_vjp(const double* x, size_t rows, size_t d, int phi, const double* d_phi,
                 double* out);

/* ---- summaries / aggregation: summaries.cpp:17-42, aggregation.cpp:40-56 ------------- */
void orc_summaries(const double* k_feat, const double* v, size_t n, size_t d, size_t b_kv,
                   double* h /* T_n x d x d */, double* z /* T_n x d */);
/* direct aggregation over an ascending index list (first term copied, then adds) */
void orc_aggregate_direct(const double* h, const double* z, size_t d, const uint32_t* idx,
                          size_t count, double* h_out, double* z_out);

/* ---- forward: forward.cpp:29-195 -------------------------------------------------------- */
/* block_rows: NULL => all block rows; else only the listed block rows are written.
 * row_h/row_z may be NULL.  Returns 0 / 2 (invalid) / 1 (non-finite output). */
int orc_forward(const double* q, const double* k, const double* v, const int8_t* labels,
                size_t n, size_t d, size_t b_q, size_t b_kv, int phi,
                const int32_t* block_rows, size_t n_block_rows, double* o_s, double* o_l,
                double* lse, double* row_h, double* row_z);
void orc_combine(const double* o_s, const double* o_l, const double* w, size_t n, size_t d,
                 double* o);

/* ---- backward: backward.cpp:12-216 ----------------------------------------------------- */
void orc_proj_backward(const double* d_out, const double* o_l, const double* w, size_t n,
                       size_t d, double* d_out_s, double* d_out_l, double* dw);
int orc_backward(const double* q, const double* k, const double* v, const int8_t* labels,
                 const double* o_s, const double* o_l, const double* lse,
                 const double* row_h, const double* row_z, const double* d_out_s,
                 const double* d_out_l, size_t n, size_t d, size_t b_q, size_t b_kv, int phi,
                 double* dq, double* dk, double* dv, double* dq_feat, double* dk_feat,
                 double* dproj, double* dq_total, double* dk_total);

/* ---- accounting: flops.cpp:7-33 --------------------------------------------------------- */
void orc_flops(size_t n, size_t d, size_t b_q, size_t b_kv, const int8_t* labels,
               uint64_t out[6] /* full, sparse, linear, proj, mask, total */);

#ifdef __cplusplus
}
#endif
#endif
