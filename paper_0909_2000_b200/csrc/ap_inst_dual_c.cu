// Dual-pair comb kernel instantiations (ap_dual_kernels.cuh): the windows 32, 96, 192, 384, 512,
// 768 and 1024 (W = L*R).
#include "ap_dual_kernels.cuh"

namespace apk {

template <int L, int R, int K>
static KernelFn pick(bool dense, bool hf) {
  if (dense) return hf ? &combd_kernel<L, R, K, true, true> : &combd_kernel<L, R, K, true, false>;
  return hf ? &combd_kernel<L, R, K, false, true> : &combd_kernel<L, R, K, false, false>;
}

KernelFn pick_dual_c(int l, int r, int k, bool dense, bool hf) {
#define AP_D(L, R, K) \
  if (l == L && r == R && k == K) return pick<L, R, K>(dense, hf);
  AP_D(4, 8, 2) AP_D(4, 24, 2) AP_D(8, 24, 2) AP_D(16, 24, 2) AP_D(32, 24, 2) AP_D(16, 32, 2) AP_D(32, 32, 2)
#undef AP_D
  return nullptr;
}

}  // namespace apk
