// kernels.hpp -- host launchers of every kernel family (declared here, defined per .cu).
#pragma once

#include "buffers.hpp"

namespace slab {

// classify.cu
size_t classify_smem_bytes(const Dims& D, bool f64);
void launch_check_finite(const Dims& D, int dtype, const void* x, long long* slot,
                         cudaStream_t st);
// returns true when it also wrote the fast path's marginal indicator M0 (s.M0 non-null)
bool launch_classify(const Dims& D, int dtype, int mask_precision, const void* q, const void* k,
                     const StateBufs& s, const WorkBufs& w, double* p_c, cudaStream_t st,
                     cudaEvent_t after_pool = nullptr);
void launch_build_lut(const Dims& D, const StateBufs& s, long long* bad, cudaStream_t st);
void launch_build_csc(const Dims& D, const StateBufs& s, cudaStream_t st);
void launch_build_m0(const Dims& D, const StateBufs& s, cudaStream_t st);
// diagnostics (diag.cu): a device int counting the rows k_classify_rank resolved by exact P_c
int* classify_exact_counter();
void set_classify_exact_counter(int* p);
// counters.cu: device accounting from the LUT (flops_report, ExecCounters)
void launch_row_stats(const Dims& D, const int8_t* labels, int g, int4* out, cudaStream_t st);
void launch_lin_rows(const Dims& D, int dtype, const void* q, const float* Z, bool z3,
                     const int4* stats, int* lin_rows, cudaStream_t st);

// generic.cu -- shape-generic SIMT kernels (fp32 math, any b_q, b_kv, d within smem limits)
bool generic_supported(const Dims& D, std::string* why);
// attention == false: only the state (summaries, H, Z) -- sla_b200_build_state
void generic_forward(const Dims& D, int dtype, const void* q, const void* k, const void* v,
                     const void* w, void* o, void* o_s, void* o_l, float* lse,
                     const StateBufs& s, const WorkBufs& wb, cudaStream_t st, bool attention = true);
// d_out_l == null: dO^l = dO W^T (combined cotangent); else the given dO^l.  dw may be null.
void generic_backward(const Dims& D, int dtype, const void* q, const void* k, const void* v,
                      const void* w, const void* o_s, const void* o_l, const float* lse,
                      const void* d_out, const void* d_out_l, void* dq, void* dk, void* dv, float* dw,
                      const StateBufs& s, const WorkBufs& wb, cudaStream_t st);
void generic_dw(const Dims& D, int dtype, const void* o_l, const void* d_out, float* dw, cudaStream_t st);
// out = (add ? add : 0) + x M with M = W[h] (transpose_w = false) or W[h]^T, f32 accumulation;
// combine_outputs (forward.cpp:187-195) and proj_backward's dO W^T (backward.cpp:12-22)
void launch_rowmat(const Dims& D, int dtype, const void* x, const void* w, bool transpose_w,
                   const void* add, void* out, cudaStream_t st);
// D^s = <dO^s, O^s> per row (backward.cpp:48-58) for independent cotangents
void launch_rowdot(const Dims& D, const void* a, const void* b, float* out, cudaStream_t st);

// gemm.cu -- batched tcgen05 GEMM (bf16 in, f32 accumulate)
struct GemmArgs {
  const void* A;
  const void* B;
  void* C;
  int batch, M, N, K;
  bool a_mn, b_mn, out_f32;
  long long lda, ldb, ldc;          // row strides in elements
  long long a_batch, b_batch, c_batch;  // batch strides in elements
  const char* name;
  // Caller tensors read in place (RowLayout mode 1 / 2, M- / N-major operands only): batch b is
  // K-row chunk b % rpu of unit b / rpu -- rows (b % rpu) * K + k of a [U][nv][d] or
  // [B][nv][H][d] tensor, rows >= nv zero-filled by TMA.  `units` = U.
  RowLayout a_rl, b_rl;
  int a_rpu = 1, b_rpu = 1;
  long long units = 1;
};
void launch_gemm(const GemmArgs& g, cudaStream_t st);

// fast path (tcgen05) -- b_q = b_kv = 64, d in {64, 128}, bf16
inline long long m0_stride(const Dims& D) { return (D.Tn + 7) / 8 * 8; }  // 16-byte rows for TMA
void launch_attn_fwd(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                     void* o, void* o_s, void* o_l, float* lse, const StateBufs& s, cudaStream_t st);
// attn_fwd_pp.cu: d = 128, persistent (one CTA per SM), key-block pairs, overlapped epilogue
void launch_attn_fwd_pp(const Dims& Dm, const void* q, const void* k, const void* v, const void* w, void* o,
                        void* o_s, void* o_l, float* lse, const StateBufs& s, cudaStream_t st);
void fast_summaries(const Dims& Dm, const void* k, const void* v, const WorkBufs& wb, cudaStream_t st);
void fast_aggregate(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, bool m0_ready, cudaStream_t st);
void fast_aggregate_h(const Dims& Dm, const StateBufs& s, const WorkBufs& wb, cudaStream_t st);
void launch_bwd_lin(const Dims& Dm, const void* q, const void* w, const void* o_s, const void* o_l,
                    const void* d_out, const StateBufs& s, __nv_bfloat16* gH, __nv_bfloat16* z3, float* Ds,
                    __nv_bfloat16* dqphi, bool ds_external, cudaStream_t st);
void launch_bwd_rows(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                     const void* d_out, void* dq, const StateBufs& s, const float* Ds,
                     const __nv_bfloat16* dqphi, float* dq_part, float* dqf_part, cudaStream_t st);
void launch_bwd_cols2(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                      const void* d_out, void* dk, void* dv, const StateBufs& s,
                      const __nv_bfloat16* Ha, const float* gZa, const float* Ds, float* dk_part,
                      float* dkf_part, int* work, cudaStream_t st);
void launch_bwd_cols(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                     const void* d_out, void* dk, void* dv, const StateBufs& s,
                     const __nv_bfloat16* Ha, const float* gZa, const float* Ds, float* dk_part,
                     float* dkf_part, int* work, cudaStream_t st);
bool fast_supported(const Dims& D, int dtype);
// A side stream with fork / join events: work that only depends on the call's inputs runs
// there, concurrent with latency-bound kernels on the caller's stream (s == nullptr: none).
struct SideFork {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr, mid = nullptr, join3 = nullptr;
};
// side.s set: the caller already queued the summaries on side.s (completion: side.join); the
// Z aggregation then runs there beside the H aggregation.  Otherwise everything runs on st.
void fast_forward(const Dims& D, const void* q, const void* k, const void* v, const void* w,
                  void* o, void* o_s, void* o_l, float* lse, const StateBufs& s,
                  const WorkBufs& wb, bool m0_ready, const SideFork& side, cudaStream_t st);
// RAII join of a side-stream fork: if an exception leaves the region between the fork and its
// join, the side stream's queued work is still joined into the caller's stream, so the caller
// never reuses buffers that work reads or writes, and a graph capture never ends with an
// unjoined fork.
struct SideJoin {
  cudaStream_t side, main;
  cudaEvent_t ev = nullptr;
  SideJoin(const SideFork& f, cudaStream_t m) : side(f.s), main(m) {}
  SideJoin(cudaStream_t s, cudaStream_t m) : side(s), main(m) {}
  void arm(cudaEvent_t e) { ev = e; }
  void release() { ev = nullptr; }
  ~SideJoin() {
    if (ev && side) {
      cudaEventRecord(ev, side);
      cudaStreamWaitEvent(main, ev, 0);
    }
  }
  SideJoin(const SideJoin&) = delete;
  SideJoin& operator=(const SideJoin&) = delete;
};
// optional SlaGradients parts (backward.hpp:10-16), f32 [U, N, d]; all null or all set
struct GradParts {
  float* dq = nullptr;
  float* dk = nullptr;
  float* dq_feat = nullptr;
  float* dk_feat = nullptr;
};
// d_out_l == null: combined cotangent d_out with dO^l = dO W^T (proj_backward fused);
// else independent cotangents d_out (= dO^s) and d_out_l (sla_backward, backward.hpp:25-38),
// w unused.  dw (= O^l^T dO^s, backward.cpp:46) may be null.
void fast_backward(const Dims& D, const void* q, const void* k, const void* v, const void* w,
                   const void* o_s, const void* o_l, const float* lse, const void* d_out,
                   const void* d_out_l, void* dq, void* dk, void* dv, float* dw,
                   const GradParts& parts, const StateBufs& s, const WorkBufs& wb, cudaStream_t st,
                   const SideFork& side);
void launch_dw_fast(const Dims& Dm, const void* o_l, const void* d_out, float* dw, const WorkBufs& wb,
                    cudaStream_t st);
// the two phases of fast_backward on their own, for partitioned execution (sla_b200_backward_rows /
// _cols): rows writes dH_i, dZ_i parts and D^s to caller buffers; cols takes them for every query
// row (and the state's labels) and produces dK / dV of its key blocks
void fast_backward_rows(const Dims& Dm, const void* q, const void* k, const void* v, const void* w,
                        const void* o_s, const void* o_l, const float* lse, const void* d_out,
                        const void* d_out_l, void* dq, float* dw, const StateBufs& s, const WorkBufs& wb,
                        __nv_bfloat16* gH, __nv_bfloat16* z3, float* Ds, cudaStream_t st);
void fast_backward_cols(const Dims& Dm, const void* q, const void* k, const void* v, const float* lse,
                        const void* d_out, const float* Ds, const __nv_bfloat16* gH, const __nv_bfloat16* z3,
                        void* dk, void* dv, const StateBufs& s, const WorkBufs& wb, cudaStream_t st);

}  // namespace slab
