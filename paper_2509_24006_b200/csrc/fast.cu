// fast.cu -- tcgen05 fast path (b_q = b_kv = 64, d in {64, 128}, bf16).  Placeholder
// dispatch until the kernels land: every problem takes the generic path.
#include "kernels.hpp"

namespace slab {

bool fast_supported(const Dims&, int) { return false; }

void fast_forward(const Dims&, const void*, const void*, const void*, const void*, void*, void*,
                  void*, float*, const StateBufs&, const WorkBufs&, cudaStream_t) {
  throw RuntimeFailure("sla_b200: fast path not built");
}

void fast_backward(const Dims&, const void*, const void*, const void*, const void*, const void*,
                   const void*, const float*, const void*, void*, void*, void*, float*,
                   const StateBufs&, const WorkBufs&, cudaStream_t) {
  throw RuntimeFailure("sla_b200: fast path not built");
}

}  // namespace slab
