// Dual-pair r = 2 comb kernel instantiations (comb2d_kernel, ap_dual_kernels.cuh): w = 4*L.
#include "ap_dual_kernels.cuh"

namespace apk {

template <int L, int K>
static KernelFn pick(bool dense) {
  return dense ? &comb2d_kernel<L, K, true> : &comb2d_kernel<L, K, false>;
}

KernelFn pick_r2_dual(int l, int k, bool dense) {
#define AP_D(L, K) \
  if (l == L && k == K) return pick<L, K>(dense);
  AP_D(8, 1) AP_D(8, 2) AP_D(16, 1) AP_D(16, 2) AP_D(32, 1) AP_D(32, 2)
#undef AP_D
  return nullptr;
}

}  // namespace apk
