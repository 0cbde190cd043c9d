// Dual-pair comb kernel instantiations (ap_dual_kernels.cuh), long lanes (R = 32).
#include "ap_dual_kernels.cuh"

namespace apk {

template <int L, int R, int K>
static KernelFn pick(bool dense, bool hf) {
  if (dense) return hf ? &combd_kernel<L, R, K, true, true> : &combd_kernel<L, R, K, true, false>;
  return hf ? &combd_kernel<L, R, K, false, true> : &combd_kernel<L, R, K, false, false>;
}

KernelFn pick_dual_a(int l, int r, int k, bool dense, bool hf) {
#define AP_D(L, R, K) \
  if (l == L && r == R && k == K) return pick<L, R, K>(dense, hf);
  AP_D(4, 32, 2) AP_D(4, 32, 1) AP_D(8, 32, 2) AP_D(8, 32, 1)
#undef AP_D
  return nullptr;
}

}  // namespace apk
