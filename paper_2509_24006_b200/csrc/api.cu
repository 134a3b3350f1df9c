// api.cu -- the extern "C" boundary (include/sla_b200.h): validation with the reference's
// messages, buffer carving, path dispatch, error mapping to the reference's exception
// classes (status 2 = std::invalid_argument, 1 = std::runtime_error).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/sla_b200.h"
#include "buffers.hpp"
#include "kernels.hpp"

namespace slab {

thread_local std::string g_last_error;
thread_local long long g_launches = 0;
void count_launch(int n) { g_launches += n; }

namespace {

size_t round_half_up(double x) { return size_t(std::floor(x + 0.5)); }

// make_block_layout (layout.cpp:8-26) + validate_config (config.cpp:7-19) + support limits
Dims resolve(const sla_b200_problem* p) {
  if (!p) throw InvalidArgument("sla_b200: null problem");
  if (p->batch < 1 || p->heads < 1) throw InvalidArgument("sla_b200: batch and heads must be >= 1");
  if (p->n <= 0 || p->d <= 0 || p->b_q <= 0 || p->b_kv <= 0)
    throw InvalidArgument("make_block_layout: all sizes must be positive");
  const bool ragged = (p->flags & SLA_B200_FLAG_RAGGED) && (p->n % p->b_q != 0 || p->n % p->b_kv != 0);
  const bool bnhd = p->flags & SLA_B200_FLAG_BNHD;
  if ((ragged || bnhd) &&
      (p->b_q != 64 || p->b_kv != 64 || p->dtype != SLA_B200_BF16 || (p->flags & SLA_B200_FLAG_GENERIC) ||
       (p->d != 64 && p->d != 128)))
    throw InvalidArgument(std::string("sla_b200: ") + (ragged ? "ragged N" : "the [B, N, H, d] layout") +
                          " needs the tcgen05 path (bf16, b_q = b_kv = 64, d in {64, 128})");
  if (!ragged) {
    if (p->n % p->b_q != 0)
      throw InvalidArgument("make_block_layout: b_q=" + std::to_string(p->b_q) +
                            " does not divide N=" + std::to_string(p->n));
    if (p->n % p->b_kv != 0)
      throw InvalidArgument("make_block_layout: b_kv=" + std::to_string(p->b_kv) +
                            " does not divide N=" + std::to_string(p->n));
  }
  if (p->n_kv < 0) throw InvalidArgument("make_block_layout: all sizes must be positive");
  if (p->n_kv > 0 && p->n_kv != p->n) {  // rectangular: a query-row range against a key range
    if (p->batch * p->heads != 1 || ragged || bnhd || (p->flags & (SLA_B200_FLAG_GENERIC | SLA_B200_FLAG_CHECK_FINITE)) ||
        p->dtype != SLA_B200_BF16 || p->b_q != 64 || p->b_kv != 64 || (p->d != 64 && p->d != 128))
      throw InvalidArgument("sla_b200: n_kv != n (a partitioned view) needs one unit on the tcgen05 path "
                            "(bf16, b_q = b_kv = 64, d in {64, 128}, no staging or finiteness checks)");
    if (p->n_kv % p->b_kv != 0)
      throw InvalidArgument("make_block_layout: b_kv=" + std::to_string(p->b_kv) +
                            " does not divide N=" + std::to_string(p->n_kv));
  }
  if (!(p->k_h > 0.0 && p->k_h <= 100.0)) throw InvalidArgument("config: k_h must be in (0, 100]");
  if (!(p->k_l >= 0.0 && p->k_l < 100.0)) throw InvalidArgument("config: k_l must be in [0, 100)");
  if (p->k_h + p->k_l > 100.0) throw InvalidArgument("config: k_h + k_l must be <= 100");
  if (p->phi < 0 || p->phi > 2) throw InvalidArgument("unknown feature map");
  if (p->dtype != SLA_B200_BF16 && p->dtype != SLA_B200_F32)
    throw InvalidArgument("unknown dtype");
  if (p->mask_precision != SLA_B200_MASK_F64 && p->mask_precision != SLA_B200_MASK_F32)
    throw InvalidArgument("unknown mask precision");
  Dims D{};
  D.B = p->batch;
  D.H = p->heads;
  D.U = p->batch * p->heads;
  D.N_valid = p->n;
  D.bnhd = bnhd;
  D.staged = ragged || bnhd;
  // the caller's [*, N, d] tensors and lse, addressed in place by the kernels (RowLayout)
  D.rl.mode = bnhd ? 2 : (ragged ? 1 : 0);
  D.rl.H = int(p->heads);
  D.rl.nv = p->n;
  D.N = ragged ? (p->n + 63) / 64 * 64 : p->n;
  D.Nk = p->n_kv > 0 ? p->n_kv : D.N;
  D.Nk_valid = p->n_kv > 0 ? p->n_kv : D.N_valid;
  D.d = int(p->d);
  D.bq = int(p->b_q);
  D.bkv = int(p->b_kv);
  D.Tm = int(D.N / p->b_q);
  D.Tn = int(D.Nk / p->b_kv);
  D.phi = p->phi;
  if (D.Tn > 8192 || D.Tm > 65535)
    throw InvalidArgument("sla_b200: at most 8192 key blocks per row are supported");
  if (p->d > 1024) throw InvalidArgument("sla_b200: d > 1024 is not supported");
  // mask.cpp:98-101
  size_t n1 = std::max<size_t>(1, round_half_up(p->k_h * double(D.Tn) / 100.0));
  n1 = std::min<size_t>(n1, size_t(D.Tn));
  size_t nn = round_half_up(p->k_l * double(D.Tn) / 100.0);
  nn = std::min<size_t>(nn, size_t(D.Tn) - n1);
  D.n1 = int(n1);
  D.n_neg = int(nn);
  D.scale_f = 1.0f / sqrtf(float(D.d));
  D.inv_sqrt_d = 1.0 / std::sqrt(double(D.d));
  if (classify_smem_bytes(D, p->mask_precision == 0) > 227 * 1024)
    throw InvalidArgument("sla_b200: too many key blocks for the classification kernel");
  return D;
}

bool use_fast(const sla_b200_problem* p, const Dims& D) {
  return !(p->flags & SLA_B200_FLAG_GENERIC) && fast_supported(D, p->dtype);
}

void require_supported(const sla_b200_problem* p, const Dims& D) {
  if (use_fast(p, D)) return;
  std::string why;
  if (!generic_supported(D, &why)) throw InvalidArgument(why);
}

// counts_launches: the call launches kernels, so sla_b200_last_launch_count() restarts at 0
// (queries such as sla_b200_state_labels leave the previous call's count readable)
template <typename F>
int guarded(F&& f, bool counts_launches = true) {
  try {
    g_last_error.clear();
    if (counts_launches) g_launches = 0;
    f();
    return SLA_B200_OK;
  } catch (const InvalidArgument& e) {
    g_last_error = e.msg;
    return SLA_B200_ERR_INVALID;
  } catch (const RuntimeFailure& e) {
    g_last_error = e.msg;
    return SLA_B200_ERR_RUNTIME;
  } catch (const CudaError& e) {
    g_last_error = "sla_b200: CUDA error: " + e.msg;
    return SLA_B200_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SLA_B200_ERR_RUNTIME;
  }
}

void buffers(const sla_b200_problem* p, const Dims& D, const void* state, void* work,
             StateBufs& s, WorkBufs& w) {
  if (!state || !work) throw InvalidArgument("sla_b200: state and workspace are required");
  const bool fast = use_fast(p, D);
  carve_state(D, fast, const_cast<void*>(state), s, nullptr);
  carve_work(D, fast, work, w, nullptr);
}

long long read_slot(long long* slot, cudaStream_t st) {
  long long v = 0;
  SLAB_CUDA(cudaMemcpyAsync(&v, slot, sizeof(v), cudaMemcpyDeviceToHost, st));
  SLAB_CUDA(cudaStreamSynchronize(st));
  return v;
}

void reset_slot(long long* slot, cudaStream_t st) {
  const long long big = LLONG_MAX;
  SLAB_CUDA(cudaMemcpyAsync(slot, &big, sizeof(big), cudaMemcpyHostToDevice, st));
}

// forward.cpp:15-25 check_input: "<name> has non-finite entry at (r, c)"
void check_inputs(const sla_b200_problem* p, const Dims& D, const WorkBufs& w,
                  std::initializer_list<std::pair<const char*, const void*>> xs, cudaStream_t st) {
  for (auto& [name, x] : xs) {
    reset_slot(w.err, st);
    launch_check_finite(D, p->dtype, x, w.err, st);
    const long long bad = read_slot(w.err, st);
    if (bad != LLONG_MAX) {
      const long long per = D.N_valid * D.d;  // the caller's rows (ragged: N_valid per unit)
      const long long u = bad / per, rc = bad % per;
      std::string msg = std::string("sla_forward: ") + name + " has non-finite entry at (" +
                        std::to_string(rc / D.d) + ", " + std::to_string(rc % D.d) + ")";
      if (D.U > 1) msg += " in unit " + std::to_string(u);
      throw InvalidArgument(msg);
    }
  }
}

// returns true when the fast path's marginal indicator M0 was written along with the labels
// SLA_B200_NO_SIDE=1: every kernel on the caller's stream (A/B runs of the side-stream overlap)
bool side_streams_enabled() {
  static const bool on = [] {
    const char* e = getenv("SLA_B200_NO_SIDE");
    return !(e && e[0] == '1');
  }();
  return on;
}

// A non-blocking side stream (and fork / join events) per device and host thread.  The forward
// runs the mask-independent key summaries there while the classification chain, which is
// latency- and FP64-bound and leaves most of each SM idle, runs on the caller's stream.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr, mid = nullptr, join3 = nullptr;
};

SideStream& side_stream() {
  thread_local std::unordered_map<int, SideStream> per_dev;  // created on first use per device
  int dev = 0;
  SLAB_CUDA(cudaGetDevice(&dev));
  SideStream& x = per_dev[dev];
  if (!x.s) {
    SLAB_CUDA(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
    SLAB_CUDA(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
    SLAB_CUDA(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
    SLAB_CUDA(cudaEventCreateWithFlags(&x.join2, cudaEventDisableTiming));
    SLAB_CUDA(cudaEventCreateWithFlags(&x.mid, cudaEventDisableTiming));
    SLAB_CUDA(cudaEventCreateWithFlags(&x.join3, cudaEventDisableTiming));
  }
  return x;
}

bool classify_into_state(const sla_b200_problem* p, const Dims& D, const void* q, const void* k,
                         const int8_t* mask_in, double* p_c, const StateBufs& s,
                         const WorkBufs& w, cudaStream_t st, cudaEvent_t after_pool = nullptr) {
  if (mask_in) {
    const size_t bytes = size_t(D.U) * D.Tm * D.Tn;
    if (mask_in != s.labels)
      SLAB_CUDA(cudaMemcpyAsync(s.labels, mask_in, bytes, cudaMemcpyDeviceToDevice, st));
    const bool check = p->flags & SLA_B200_FLAG_CHECK_FINITE;
    if (check) reset_slot(w.err + 1, st);
    if (after_pool) SLAB_CUDA(cudaEventRecord(after_pool, st));
    launch_build_lut(D, s, check ? w.err + 1 : nullptr, st);
    if (check && read_slot(w.err + 1, st) != LLONG_MAX)
      throw InvalidArgument("build_lookup: label must be -1, 0 or 1");
    return false;
  }
  return launch_classify(D, p->dtype, p->mask_precision, q, k, s, w, p_c, st, after_pool);
}

}  // namespace
}  // namespace slab

using namespace slab;

extern "C" {

const char* sla_b200_last_error(void) { return g_last_error.c_str(); }
int sla_b200_abi_version(void) { return SLA_B200_ABI_VERSION; }
int64_t sla_b200_last_launch_count(void) { return g_launches; }

int sla_b200_validate(const sla_b200_problem* p) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
  }, false);
}

int sla_b200_sizes(const sla_b200_problem* p, size_t* state_bytes, size_t* workspace_bytes) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    StateBufs s;
    WorkBufs w;
    const bool fast = use_fast(p, D);
    carve_state(D, fast, nullptr, s, state_bytes);
    carve_work(D, fast, nullptr, w, workspace_bytes);
  }, false);
}

int sla_b200_query(const sla_b200_problem* p, sla_b200_info* info) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!info) return;
    info->path = use_fast(p, D) ? 1 : 0;
    info->n1 = D.n1;
    info->n_neg = D.n_neg;
    info->t_m = D.Tm;
    info->t_n = D.Tn;
    info->gpu_launches = g_launches;
  }, false);
}

int sla_b200_classify(const sla_b200_problem* p, const void* q, const void* k, int8_t* labels,
                      double* p_c, void* state, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    StateBufs s;
    WorkBufs w;
    buffers(p, D, state, workspace, s, w);
    if (p->flags & SLA_B200_FLAG_CHECK_FINITE) check_inputs(p, D, w, {{"Q", q}, {"K", k}}, st);
    launch_classify(D, p->dtype, p->mask_precision, q, k, s, w, p_c, st);
    if (labels && labels != s.labels)
      SLAB_CUDA(cudaMemcpyAsync(labels, s.labels, size_t(D.U) * D.Tm * D.Tn,
                                cudaMemcpyDeviceToDevice, st));
  });
}

int sla_b200_forward(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                     const void* w, const int8_t* mask_in, void* o, void* o_s, void* o_l,
                     float* lse, void* state, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!q || !k || !v || !lse) throw InvalidArgument("sla_forward: q, k, v and lse are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    StateBufs s;
    WorkBufs wb;
    buffers(p, D, state, workspace, s, wb);
    const bool check = p->flags & SLA_B200_FLAG_CHECK_FINITE;
    if (check) check_inputs(p, D, wb, {{"Q", q}, {"K", k}, {"V", v}}, st);
    const bool fast = use_fast(p, D);
    if (fast && (!o_s || !o_l))  // the tcgen05 forward stores both branch outputs by TMA
      throw InvalidArgument("sla_forward: o_s and o_l are required on the tcgen05 path");
    // fork: phi(K), z and h = phi(K)^T V on the side stream, concurrent with classification.
    // Not under the per-kernel profiler (one event sequence) nor with the finiteness checks
    // (host syncs that may throw between fork and join).
    const bool fork = fast && !check && !prof_enabled() && side_streams_enabled();
    SideStream* ss = fork ? &side_stream() : nullptr;
    SideJoin guard(fork ? ss->s : nullptr, st);
    // the side stream forks after the pooling kernel: phi(K) / summaries and the pooling are
    // both HBM-bound, the scores and rank kernels after it are not
    const bool m0_ready = classify_into_state(p, D, q, k, mask_in, nullptr, s, wb, st, fork ? ss->fork : nullptr);
    if (fork) {
      SLAB_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
      guard.arm(ss->join);
      fast_summaries(D, k, v, wb, ss->s);
      SLAB_CUDA(cudaEventRecord(ss->join, ss->s));
    }
    if (fast) {
      SideFork side;
      if (fork) {
        side.s = ss->s;
        side.join = ss->join;
        side.mid = ss->mid;
        side.join3 = ss->join3;
      }
      fast_forward(D, q, k, v, w, o, o_s, o_l, lse, s, wb, m0_ready, side, st);
    } else {
      generic_forward(D, p->dtype, q, k, v, w, o, o_s, o_l, lse, s, wb, st);
    }
    guard.release();
    if (check) {  // forward.cpp:164-170
      const long long per = D.N * D.d;
      for (const void* out : {static_cast<const void*>(o_s), static_cast<const void*>(o_l)}) {
        if (!out) continue;
        reset_slot(wb.err, st);
        launch_check_finite(D, p->dtype, out, wb.err, st);
        const long long bad = read_slot(wb.err, st);
        if (bad != LLONG_MAX) {
          const long long r = (bad % per) / D.d, c = bad % D.d;
          throw RuntimeFailure("sla_forward: non-finite output at row " + std::to_string(r) +
                               ", col " + std::to_string(c) + " (block row " +
                               std::to_string(r / D.bq) + ")");
        }
      }
    }
  });
}

}  // extern "C"

namespace slab {
namespace {

// proj_backward + sla_backward (d_out_l == null: combined cotangent d_out and W), or sla_backward
// alone with independent cotangents d_out (= dO^s) and d_out_l (backward.hpp:25-38)
void backward_impl(const sla_b200_problem* p, const void* q, const void* k, const void* v, const void* w,
                   const void* o_s, const void* o_l, const float* lse, const void* d_out, const void* d_out_l,
                   void* dq, void* dk, void* dv, float* dw, const sla_b200_grad_parts* parts,
                   const void* state, void* workspace, void* stream) {
  const Dims D = resolve(p);
  require_supported(p, D);
  if (!q || !k || !v || !o_s || !o_l || !lse || !d_out || !dq || !dk || !dv || (!d_out_l && (!w || !dw)))
    throw InvalidArgument("sla_backward: all tensors are required");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  prof_mark("", st);
  StateBufs s;
  WorkBufs wb;
  buffers(p, D, state, workspace, s, wb);
  const bool fast = use_fast(p, D);
  GradParts gp;
  if (parts) {
    gp = GradParts{parts->dq_sparse, parts->dk_sparse, parts->dq_feat, parts->dk_feat};
    if (!gp.dq || !gp.dk || !gp.dq_feat || !gp.dk_feat)
      throw InvalidArgument("sla_backward: gradient parts are all-or-none");
    if (D.staged) throw InvalidArgument("sla_backward: gradient parts are not available for ragged / [B, N, H, d] layouts");
  }
  if (fast) {
    SideFork side;
    if (!prof_enabled() && side_streams_enabled()) {  // the per-kernel profiler times one event sequence
      SideStream& ss = side_stream();
      side.s = ss.s;
      side.fork = ss.fork;
      side.join = ss.join;
      side.join2 = ss.join2;
      side.mid = ss.mid;
      side.join3 = ss.join3;
    }
    fast_backward(D, q, k, v, w, o_s, o_l, lse, d_out, d_out_l, dq, dk, dv, dw, gp, s, wb, st, side);
  } else {
    generic_backward(D, p->dtype, q, k, v, w, o_s, o_l, lse, d_out, d_out_l, dq, dk, dv, dw, s, wb, st);
    if (parts) {
      const size_t bytes = sizeof(float) * size_t(D.U) * D.N * D.d;
      SLAB_CUDA(cudaMemcpyAsync(gp.dq, wb.dq, bytes, cudaMemcpyDeviceToDevice, st));
      SLAB_CUDA(cudaMemcpyAsync(gp.dk, wb.dk, bytes, cudaMemcpyDeviceToDevice, st));
      SLAB_CUDA(cudaMemcpyAsync(gp.dq_feat, wb.dqf, bytes, cudaMemcpyDeviceToDevice, st));
      SLAB_CUDA(cudaMemcpyAsync(gp.dk_feat, wb.dkf, bytes, cudaMemcpyDeviceToDevice, st));
    }
  }
}

}  // namespace
}  // namespace slab

extern "C" {

int sla_b200_backward_ex(const sla_b200_problem* p, const void* q, const void* k,
                         const void* v, const void* w, const void* o_s, const void* o_l,
                         const float* lse, const void* d_out, void* dq, void* dk, void* dv,
                         float* dw, const sla_b200_grad_parts* parts, const void* state,
                         void* workspace, void* stream) {
  return guarded([&] {
    backward_impl(p, q, k, v, w, o_s, o_l, lse, d_out, nullptr, dq, dk, dv, dw, parts, state, workspace, stream);
  });
}

int sla_b200_backward(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                      const void* w, const void* o_s, const void* o_l, const float* lse,
                      const void* d_out, void* dq, void* dk, void* dv, float* dw,
                      const void* state, void* workspace, void* stream) {
  return sla_b200_backward_ex(p, q, k, v, w, o_s, o_l, lse, d_out, dq, dk, dv, dw, nullptr,
                              state, workspace, stream);
}

int sla_b200_backward_split(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                            const void* o_s, const void* o_l, const float* lse, const void* d_out_sparse,
                            const void* d_out_linear, void* dq, void* dk, void* dv, float* dw,
                            const sla_b200_grad_parts* parts, const void* state, void* workspace,
                            void* stream) {
  return guarded([&] {
    if (!d_out_linear) throw InvalidArgument("sla_backward: cotangent shape mismatch");
    backward_impl(p, q, k, v, nullptr, o_s, o_l, lse, d_out_sparse, d_out_linear, dq, dk, dv, dw, parts,
                  state, workspace, stream);
  });
}

int sla_b200_backward_rows(const sla_b200_problem* p, const void* q, const void* k, const void* v, const void* w,
                           const void* o_s, const void* o_l, const float* lse, const void* d_out,
                           const void* d_out_linear, void* dq, float* dw, float* ds_out, void* dh_out, void* dz_out,
                           const void* state, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!use_fast(p, D) || D.staged)
      throw InvalidArgument("sla_b200_backward_rows: the tcgen05 path without staging only");
    if (!q || !k || !v || !o_s || !o_l || !lse || !d_out || !dq || !ds_out || !dh_out || !dz_out ||
        (!d_out_linear && !w))
      throw InvalidArgument("sla_backward: all tensors are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    StateBufs s;
    WorkBufs wb;
    buffers(p, D, state, workspace, s, wb);
    fast_backward_rows(D, q, k, v, w, o_s, o_l, lse, d_out, d_out_linear, dq, dw, s, wb,
                       static_cast<__nv_bfloat16*>(dh_out), static_cast<__nv_bfloat16*>(dz_out), ds_out, st);
  });
}

int sla_b200_backward_cols(const sla_b200_problem* p, const void* q, const void* k, const void* v, const float* lse,
                           const void* d_out, const float* ds, const void* dh, const void* dz, const int8_t* labels,
                           void* dk, void* dv, void* state, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!use_fast(p, D) || D.staged)
      throw InvalidArgument("sla_b200_backward_cols: the tcgen05 path without staging only");
    if (!q || !k || !v || !lse || !d_out || !ds || !dh || !dz || !labels || !dk || !dv)
      throw InvalidArgument("sla_backward: all tensors are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    StateBufs s;
    WorkBufs wb;
    buffers(p, D, state, workspace, s, wb);
    if (labels != s.labels)
      SLAB_CUDA(cudaMemcpyAsync(s.labels, labels, size_t(D.U) * D.Tm * D.Tn, cudaMemcpyDeviceToDevice, st));
    fast_backward_cols(D, q, k, v, lse, d_out, ds, static_cast<const __nv_bfloat16*>(dh),
                       static_cast<const __nv_bfloat16*>(dz), dk, dv, s, wb, st);
  });
}

int sla_b200_combine_outputs(const sla_b200_problem* p, const void* o_s, const void* o_l, const void* w,
                             void* o, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (D.staged) throw InvalidArgument("combine_outputs: staged layouts are fused into sla_b200_forward only");
    if (!o_s || !o_l || !w || !o) throw InvalidArgument("combine_outputs: all tensors are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    launch_rowmat(D, p->dtype, o_l, w, false, o_s, o, st);
  });
}

int sla_b200_proj_backward(const sla_b200_problem* p, const void* d_out, const void* o_l, const void* w,
                           void* d_out_linear, float* dw, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (D.staged) throw InvalidArgument("proj_backward: staged layouts are fused into sla_b200_backward only");
    if (!d_out || !o_l || !w || !d_out_linear || !dw) throw InvalidArgument("proj_backward: shape mismatch");
    if (!workspace) throw InvalidArgument("sla_b200: state and workspace are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    launch_rowmat(D, p->dtype, d_out, w, true, nullptr, d_out_linear, st);  // dO^l = dO W^T
    if (use_fast(p, D)) {
      WorkBufs wb;
      carve_work(D, true, workspace, wb, nullptr);
      launch_dw_fast(D, o_l, d_out, dw, wb, st);  // dW = O^l^T dO
    } else {
      generic_dw(D, p->dtype, o_l, d_out, dw, st);
    }
  });
}

int sla_b200_build_state(const sla_b200_problem* p, const void* q, const void* k, const void* v,
                         const int8_t* mask, void* state, void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (D.staged) throw InvalidArgument("sla_b200_build_state: staged layouts are not supported");
    if (!q || !k || !v || !mask) throw InvalidArgument("sla_b200_build_state: q, k, v and mask are required");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    prof_mark("", st);
    StateBufs s;
    WorkBufs wb;
    buffers(p, D, state, workspace, s, wb);
    const bool m0_ready = classify_into_state(p, D, q, k, mask, nullptr, s, wb, st);
    if (use_fast(p, D)) {
      fast_summaries(D, k, v, wb, st);
      fast_aggregate(D, s, wb, m0_ready, st);
    } else {
      generic_forward(D, p->dtype, q, k, v, nullptr, nullptr, nullptr, nullptr, nullptr, s, wb, st, false);
    }
  });
}

// Per-row LUT statistics (critical, marginal, Four-Russians groups hit) and, when q is given,
// per-block-row linear row products, copied to the host.  Scratch: the pooled-Q area of the
// workspace (U * Tm * d doubles >= 20 bytes per block row), idle outside classification.
struct RowStats {
  std::vector<int4> rows;
  std::vector<int> lin;
};

RowStats row_stats(const sla_b200_problem* p, const Dims& D, const void* q, const void* state,
                   void* workspace, int g, cudaStream_t st) {
  StateBufs s;
  WorkBufs w;
  buffers(p, D, state, workspace, s, w);
  const size_t rows = size_t(D.U) * D.Tm;
  int4* dstats = reinterpret_cast<int4*>(w.pq);
  int* dlin = reinterpret_cast<int*>(dstats + rows);
  launch_row_stats(D, s.labels, g, dstats, st);
  RowStats r;
  r.rows.resize(rows);
  if (q) {
    launch_lin_rows(D, p->dtype, q, s.Z, use_fast(p, D), dstats, dlin, st);
    r.lin.resize(rows);
    SLAB_CUDA(cudaMemcpyAsync(r.lin.data(), dlin, rows * sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  SLAB_CUDA(cudaMemcpyAsync(r.rows.data(), dstats, rows * sizeof(int4), cudaMemcpyDeviceToHost, st));
  SLAB_CUDA(cudaStreamSynchronize(st));
  return r;
}

int sla_b200_flops_report(const sla_b200_problem* p, const void* state, sla_b200_flops* per_unit,
                          void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!per_unit) throw InvalidArgument("flops_report: per_unit is required");
    const RowStats r = row_stats(p, D, nullptr, state, workspace, 1, static_cast<cudaStream_t>(stream));
    const uint64_t n = uint64_t(D.N_valid), d = uint64_t(D.d);
    for (long long u = 0; u < D.U; ++u) {  // flops.cpp:10-32
      uint64_t crit = 0, marg = 0, covered = 0;
      for (int i = 0; i < D.Tm; ++i) {
        const int4 x = r.rows[size_t(u) * D.Tm + i];
        crit += uint64_t(x.x);
        marg += uint64_t(x.y);
        if (x.y > 0) covered += uint64_t(std::min<long long>(D.bq, D.N_valid - (long long)i * D.bq));
      }
      sla_b200_flops& f = per_unit[u];
      f.full_flops = 4 * n * n * d;
      f.sparse_flops = 4 * uint64_t(D.bq) * uint64_t(D.bkv) * d * crit;
      f.linear_flops = 2 * covered * d * d + (marg > 0 ? n * d : 0);
      f.proj_flops = 2 * n * d * d;
      f.mask_flops = 2 * n * d + 2 * uint64_t(D.Tm) * uint64_t(D.Tn) * d;
      f.sla_total = f.sparse_flops + f.linear_flops + f.proj_flops + f.mask_flops;
      f.ratio = double(f.sla_total) / double(f.full_flops);
      f.sparsity = 1.0 - double(crit) / (double(D.Tm) * double(D.Tn));
    }
  });
}

int sla_b200_exec_counters(const sla_b200_problem* p, const void* q, const void* state,
                           int aggregation, int group_size, sla_b200_counters* out,
                           void* workspace, void* stream) {
  return guarded([&] {
    const Dims D = resolve(p);
    require_supported(p, D);
    if (!q || !out) throw InvalidArgument("exec_counters: q and out are required");
    if (aggregation < SLA_B200_AGG_DIRECT || aggregation > SLA_B200_AGG_AUTO)
      throw InvalidArgument("exec_counters: unknown aggregation strategy");
    const int g = group_size >= 1 && group_size <= 20 ? group_size : 1;
    const RowStats r = row_stats(p, D, q, state, workspace, g, static_cast<cudaStream_t>(stream));
    *out = sla_b200_counters{};
    for (long long u = 0; u < D.U; ++u) {
      uint64_t crit = 0, marg = 0;
      for (int i = 0; i < D.Tm; ++i) {
        crit += uint64_t(r.rows[size_t(u) * D.Tm + i].x);
        marg += uint64_t(r.rows[size_t(u) * D.Tm + i].y);
      }
      int kind = aggregation;  // resolve_strategy (aggregation.cpp:147-156), config.hpp:30-31
      if (kind == SLA_B200_AGG_AUTO) {
        const double frac = double(marg) / (double(D.Tm) * double(D.Tn));
        kind = frac <= 0.25 ? SLA_B200_AGG_DIRECT
                            : (frac >= 0.75 ? SLA_B200_AGG_COMPLEMENT : SLA_B200_AGG_FOUR_RUSSIANS);
      }
      if (kind == SLA_B200_AGG_FOUR_RUSSIANS) {
        if (group_size < 1) throw InvalidArgument("four russians: g must be >= 1");
        if (group_size > 20) throw InvalidArgument("four russians: g > 20 would need a 2^g table");
        for (int b = 0; b < D.Tn; b += g)  // Gray-code table walk (aggregation.cpp:95-108)
          out->table_build_additions += (uint64_t(1) << std::min(g, D.Tn - b)) - 1;
      }
      out->sparse_block_matmuls += 2 * crit;  // forward.cpp:46 + 123-124
      for (int i = 0; i < D.Tm; ++i) {
        const size_t row = size_t(u) * D.Tm + i;
        const int4 x = r.rows[row];
        out->linear_row_products += uint64_t(r.lin[row]);
        if (kind == SLA_B200_AGG_DIRECT) {  // aggregation.cpp:40-56: the first term is a copy
          out->additions += x.y > 0 ? uint64_t(x.y - 1) : 0;
        } else if (kind == SLA_B200_AGG_COMPLEMENT) {  // aggregation.cpp:58-70
          out->subtractions += uint64_t(D.Tn - x.y);
        } else {  // aggregation.cpp:118-145
          out->lookups += uint64_t(x.z);
          out->additions += x.z > 0 ? uint64_t(x.z - 1) : 0;
        }
      }
    }
  });
}

int sla_b200_state_labels(const sla_b200_problem* p, const void* state, const int8_t** labels) {
  return guarded([&] {
    const Dims D = resolve(p);
    StateBufs s;
    carve_state(D, use_fast(p, D), const_cast<void*>(state), s, nullptr);
    if (labels) *labels = s.labels;
  }, false);
}

}  // extern "C"
