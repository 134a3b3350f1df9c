/*
 * sla_b200.h -- C-ABI of the B200-native SLA (Sparse-Linear Attention) operator.
 *
 * Drop-in boundary for the reference's C++ operator API (namespace sla, reference paths
 * relative to /root/reference/proj/core):
 *
 *   reference                                         replaced by
 *   ------------------------------------------------  ------------------------------------
 *   make_block_layout        layout.cpp:8-26          sla_b200_validate
 *   validate_config          config.cpp:7-19          sla_b200_validate
 *   predict_compressed_weights + classify_mask
 *                            mask.cpp:57-119          sla_b200_classify
 *   sla_forward              forward.hpp:63-68        sla_b200_forward (mask_in == NULL)
 *   sla_forward_with_mask    forward.hpp:70-78        sla_b200_forward (mask_in != NULL)
 *   combine_outputs          forward.hpp:80-83        fused: sla_b200_forward writes o;
 *                                                     standalone: sla_b200_combine_outputs
 *   proj_backward            backward.hpp:18-23       fused into sla_b200_backward[_ex];
 *                                                     standalone: sla_b200_proj_backward
 *   sla_backward             backward.hpp:25-38       sla_b200_backward_split (independent
 *                                                     dO^s, dO^l, as the reference takes them)
 *   SlaGradients parts       backward.hpp:10-16       sla_b200_grad_parts, on both paths
 *   SlaForwardState          forward.hpp:33-43        the caller-owned `state` buffer
 *   std::invalid_argument / std::runtime_error        status 2 / 1 + sla_b200_last_error()
 *
 * Plain C: no CUDA or C++ types cross this boundary.  Pointers are DEVICE pointers unless
 * the function name ends in _host.  `stream` is a cudaStream_t passed as void*.
 * No device allocation happens inside any call; the caller provides `state` (persists
 * from forward to backward, like SlaForwardState) and `workspace` (scratch) buffers of
 * the sizes sla_b200_sizes() reports.  Calls are stream-ordered and re-entrant per stream.
 *
 * Layout: a problem is B*H independent (batch, head) "units"; every [*, N, d] tensor is
 * unit-major and per-unit row-major N x d (the reference Mat layout, mat.hpp:11-18).
 * W is per head, [H, d, d] indexed [in][out] as in OutputProjection (forward.hpp:27-30);
 * dW is accumulated over the batch per head.
 */
#ifndef SLA_B200_H
#define SLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLA_B200_ABI_VERSION 2

/* status codes: mirror the reference CLI exit codes (tools/sla_main.cpp:564-570) */
#define SLA_B200_OK 0
#define SLA_B200_ERR_RUNTIME 1 /* std::runtime_error analogue (CUDA error, non-finite out) */
#define SLA_B200_ERR_INVALID 2 /* std::invalid_argument analogue (shape, config, input)   */

/* feature map phi -- same order as sla::FeatureMapKind (config.hpp:12-16) */
#define SLA_B200_PHI_ELU1 0
#define SLA_B200_PHI_RELU 1
#define SLA_B200_PHI_SOFTMAX 2

/* element type of q/k/v/w/d_out and of the o, o_s, o_l, dq, dk, dv outputs */
#define SLA_B200_BF16 0
#define SLA_B200_F32 1

/* arithmetic of the classification stage (K1+K2).  F64 reproduces the reference bit for
 * bit (mask.hpp:56-58 computes the mask in f64 on every path); F32 is the north-star fp32
 * variant whose rare disagreements lie on near-ties. */
#define SLA_B200_MASK_F64 0
#define SLA_B200_MASK_F32 1

/* flags */
#define SLA_B200_FLAG_CHECK_FINITE 1u /* reject non-finite q/k/v with "(r, c)" (forward.cpp:15-25)
                                         and non-finite outputs (forward.cpp:164-170); syncs  */
#define SLA_B200_FLAG_GENERIC 2u      /* force the shape-generic SIMT kernels                 */
/* Ragged N (an extension; the reference rejects N % b != 0, layout.cpp:12-17, and so does this
 * library without the flag).  With it, T = ceil(N / b) and the last block holds r = N - (T-1) b
 * rows: its pooled mean is over those r rows, keys >= N take no part in either branch (no
 * softmax weight, no phi(K) summary), and only rows < N are read or written.  For N % b == 0
 * the results are identical to the unflagged call.  tcgen05 path only (bf16, b_q = b_kv = 64). */
#define SLA_B200_FLAG_RAGGED 4u
/* Token-major tensors: q, k, v, o, o_s, o_l, dO, dq, dk, dv are [B, N, H, d] and lse is [B, N, H]
 * (the layout a DiT's fused QKV projection produces) instead of the unit-major [B, H, N, d].
 * Staged through unit-major copies in the workspace; tcgen05 path only. */
#define SLA_B200_FLAG_BNHD 8u

typedef struct sla_b200_problem {
  int64_t batch;    /* B                                  */
  int64_t heads;    /* H                                  */
  int64_t n;        /* sequence length N (multiple of b_q and b_kv unless FLAG_RAGGED) */
  int64_t d;        /* head dimension                     */
  int64_t b_q;      /* rows per query block               */
  int64_t b_kv;     /* rows per key/value block           */
  double k_h;       /* percent critical per row, (0, 100] */
  double k_l;       /* percent negligible per row, [0, 100) */
  int32_t phi;      /* SLA_B200_PHI_*                     */
  int32_t dtype;    /* SLA_B200_BF16 | SLA_B200_F32       */
  int32_t mask_precision; /* SLA_B200_MASK_*              */
  uint32_t flags;   /* SLA_B200_FLAG_*                    */
  /* Rectangular view (ABI 2; 0 = n): key / value rows per unit when they differ from the query
   * rows n -- a partitioned execution in which this call owns a range of query blocks against a
   * range of key blocks (paper_2509_24006_b200/runner.py: sub-head and sequence sharding).
   * One unit (batch = heads = 1), tcgen05 path only.  T_m = n / b_q, T_n = n_kv / b_kv. */
  int64_t n_kv;
} sla_b200_problem;

/* Per-call execution summary (the device analogue of ExecCounters, forward.hpp:46-50). */
typedef struct sla_b200_info {
  int32_t path;              /* 0 = generic SIMT kernels, 1 = tcgen05 fast path         */
  int32_t n1, n_neg;         /* per-row class counts of the dynamic mask (mask.cpp:98-101) */
  int32_t t_m, t_n;
  int64_t gpu_launches;      /* kernels launched by the last call on this thread        */
} sla_b200_info;

/* flops_report (flops.cpp:7-33) of one (batch, head) unit, computed from the device LUT. */
typedef struct sla_b200_flops {
  uint64_t full_flops;   /* 4 N^2 d                                              */
  uint64_t sparse_flops; /* 4 b_q b_kv d x critical blocks                       */
  uint64_t linear_flops; /* 2 d^2 per row of a block row with a marginal block, + N d */
  uint64_t proj_flops;   /* 2 N d^2                                              */
  uint64_t mask_flops;   /* 2 N d + 2 T_m T_n d                                  */
  uint64_t sla_total;    /* sparse + linear + proj + mask                        */
  double ratio;          /* sla_total / full_flops                               */
  double sparsity;       /* 1 - critical block fraction                          */
} sla_b200_flops;

/* ExecCounters (forward.hpp:46-50) of a forward, summed over units, as the reference's
 * sla_forward_with_mask counts them for the given aggregation strategy. */
typedef struct sla_b200_exec_counters {
  uint64_t sparse_block_matmuls;   /* 2 per critical block (score + weight-value)        */
  uint64_t linear_row_products;    /* rows with a marginal block and phi(q) . Z_i != 0    */
  uint64_t additions;              /* AggCounters (aggregation.hpp:14-19)                 */
  uint64_t subtractions;
  uint64_t lookups;
  uint64_t table_build_additions;
} sla_b200_counters;

/* Aggregation strategies of the counting (config.hpp:19-31).  The device always computes
 * H = M0 h as one tensor-core GEMM -- arithmetic-equivalent to every strategy -- so the strategy
 * only selects which of the reference's counts are reported. */
#define SLA_B200_AGG_DIRECT 0
#define SLA_B200_AGG_COMPLEMENT 1
#define SLA_B200_AGG_FOUR_RUSSIANS 2
#define SLA_B200_AGG_AUTO 3 /* resolve_strategy with thresholds 0.25 / 0.75, per unit */

/* flops_report of every unit (per_unit: [B*H]) from the LUT in `state` (after
 * sla_b200_classify or sla_b200_forward).  Synchronises `stream`.  Ragged N counts the N
 * valid rows (full / proj / mask flops, and the valid rows of each covered block row). */
int sla_b200_flops_report(const sla_b200_problem* p, const void* state, sla_b200_flops* per_unit,
                          void* workspace, void* stream);

/* ExecCounters of the forward that filled `state` (q: that forward's Q, for the linear-row
 * denominators; group_size: the Four-Russians g, 1..20).  Synchronises `stream`. */
int sla_b200_exec_counters(const sla_b200_problem* p, const void* q, const void* state,
                           int aggregation, int group_size, sla_b200_counters* out,
                           void* workspace, void* stream);

/* Thread-local message of the last non-OK status; carries the reference's fragments. */
const char* sla_b200_last_error(void);
int sla_b200_abi_version(void);

/* make_block_layout + validate_config (+ kernel support limits). */
int sla_b200_validate(const sla_b200_problem* p);

/* Bytes of the persistent forward->backward state and of the scratch workspace. */
int sla_b200_sizes(const sla_b200_problem* p, size_t* state_bytes, size_t* workspace_bytes);

/* Info about how a problem will run (no device work). */
int sla_b200_query(const sla_b200_problem* p, sla_b200_info* info);
int64_t sla_b200_last_launch_count(void);

/* K1+K2: block classification of Q, K (predict_compressed_weights + classify_mask).
 * labels: [B*H, T_m, T_n] int8 in {-1,0,1}.  p_c: optional [B*H, T_m, T_n] f64 weights. */
int sla_b200_classify(const sla_b200_problem* p, const void* q, const void* k, int8_t* labels,
                      double* p_c, void* state, void* workspace, void* stream);

/* Fused forward.  mask_in == NULL: dynamic mask from q, k (sla_forward); else the given
 * label grid (sla_forward_with_mask; rows may have zero critical blocks).
 * w may be NULL (then o may be NULL): projection skipped.  Outputs o = o_s + o_l W,
 * o_s (sparse branch), o_l (linear branch) in p->dtype; lse f32 [B*H, N] with the
 * reference sentinel -1e30 on rows without critical mass.  o may be NULL (projection output
 * not wanted); o_s and o_l are required on the tcgen05 path (they leave the kernel by TMA) and
 * may be NULL on the generic path only if the caller will not run the backward. */
int sla_b200_forward(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                     const void* w, const int8_t* mask_in, void* o, void* o_s, void* o_l,
                     float* lse, void* state, void* workspace, void* stream);

/* Fused backward of O = O^s + O^l W from the combined cotangent d_out
 * (proj_backward + sla_backward: dO^s = dO, dO^l = dO W^T computed in the linear-branch kernel).
 * dq, dk are the composed totals dq_total / dk_total (backward.cpp:211-214); dv accumulates both
 * branches; dw f32 [H, d, d]. */
int sla_b200_backward(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                      const void* w, const void* o_s, const void* o_l, const float* lse,
                      const void* d_out, void* dq, void* dk, void* dv, float* dw,
                      const void* state, void* workspace, void* stream);

/* Optional component gradients of SlaGradients (backward.hpp:10-16), f32 [B*H, N, d]; all four
 * or none.  Both paths: the tcgen05 kernels write them from their epilogues (dq_feat there is
 * the bf16 dQ^phi the row kernels consume). */
typedef struct sla_b200_grad_parts {
  float* dq_sparse;  /* SlaGradients::dq      */
  float* dk_sparse;  /* SlaGradients::dk      */
  float* dq_feat;    /* SlaGradients::dq_feat */
  float* dk_feat;    /* SlaGradients::dk_feat */
} sla_b200_grad_parts;

int sla_b200_backward_ex(const sla_b200_problem* p, const void* q, const void* k,
                         const void* v, const void* w, const void* o_s, const void* o_l,
                         const float* lse, const void* d_out, void* dq, void* dk, void* dv,
                         float* dw, const sla_b200_grad_parts* parts, const void* state,
                         void* workspace, void* stream);

/* sla_backward with independent cotangents (backward.hpp:25-38, backward.cpp:24-216): the sparse
 * branch takes d_out_sparse (dO^s), the linear branch d_out_linear (dO^l) as given -- they need
 * not be related through W.  dw (optional, f32 [H, d, d]) = O^l^T dO^s summed over the batch, the
 * reference's SlaGradients::dproj (backward.cpp:46).  parts: optional component gradients. */
int sla_b200_backward_split(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                            const void* o_s, const void* o_l, const float* lse, const void* d_out_sparse,
                            const void* d_out_linear, void* dq, void* dk, void* dv, float* dw,
                            const sla_b200_grad_parts* parts, const void* state, void* workspace,
                            void* stream);

/* combine_outputs (forward.cpp:187-195): o = o_s + o_l W[h], f32 accumulation, on the device. */
int sla_b200_combine_outputs(const sla_b200_problem* p, const void* o_s, const void* o_l, const void* w,
                             void* o, void* stream);

/* proj_backward (backward.cpp:12-22) on the device: d_out_linear = d_out W[h]^T and
 * dw (f32 [H, d, d]) = O^l^T d_out summed over the batch.  dO^s is d_out itself. */
int sla_b200_proj_backward(const sla_b200_problem* p, const void* d_out, const void* o_l, const void* w,
                           void* d_out_linear, float* dw, void* workspace, void* stream);

/* The device half of a SlaForwardState from its label grid (build_lookup + summaries +
 * aggregation, forward.cpp:81-130) without the attention kernel: lets a caller that holds the
 * forward's outputs (O^s, O^l, lse) run sla_b200_backward_split on them. */
int sla_b200_build_state(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                         const int8_t* mask, void* state, void* workspace, void* stream);

/* The backward in two phases, for partitioned execution (n_kv views; runner.py):
 *   rows (backward.cpp:46-120): for this call's query rows -- dq_total, dW partial (optional,
 *     over these rows only), and the row summaries the column phase needs: ds_out = D^s
 *     (f32 [U, N]), dh_out = dH_i (bf16 [U, T_m, d, d]), dz_out = dZ_i as three bf16 parts
 *     (bf16 [U, T_m, 3 d]).  d_out_linear NULL: dO^l = d_out W^T; else the given dO^l (w unused).
 *   cols (backward.cpp:122-199): for this call's key blocks against EVERY query row of the unit
 *     (n = all rows, n_kv = these keys): lse, ds, dh, dz of all rows, the label grid of all rows
 *     restricted to these key blocks ([U, T_m, T_n]); writes dk_total and dv of these keys.
 *     `state` is scratch for this view (labels, column lists, M0). */
int sla_b200_backward_rows(const sla_b200_problem* p, const void* q, const void* k, const void* v, const void* w,
                           const void* o_s, const void* o_l, const float* lse, const void* d_out,
                           const void* d_out_linear, void* dq, float* dw, float* ds_out, void* dh_out, void* dz_out,
                           const void* state, void* workspace, void* stream);
int sla_b200_backward_cols(const sla_b200_problem* p, const void* q, const void* k, const void* v, const float* lse,
                           const void* d_out, const float* ds, const void* dh, const void* dz, const int8_t* labels,
                           void* dk, void* dv, void* state, void* workspace, void* stream);

/* Per-kernel CUDA-event profiler of this library's own launches (bench/diagnostics).
 * sla_b200_profiler(1) clears and enables, (0) disables.  The report is text lines
 * "<kernel> <total_ms> <launches>"; returns the bytes needed (including the NUL). */
int sla_b200_profiler(int enable);
size_t sla_b200_profiler_report(char* buf, size_t len);

/* Device pointer to the int8 label grid held in `state` after classify/forward. */
int sla_b200_state_labels(const sla_b200_problem* p, const void* state, const int8_t** labels);

#ifdef __cplusplus
}
#endif
#endif /* SLA_B200_H */
