// Dual-pair comb kernel instantiations (ap_dual_kernels.cuh) with lane groups that do not tile
// the warp (L = 5, 10, 15: 30 of 32 lanes work, the rest form an idle phantom group):
// the windows 80, 100, 120, 160, 200, 240, 300, 320.
#include "ap_dual_kernels.cuh"

namespace apk {

template <int L, int R, int K>
static KernelFn pick(bool dense, bool hf) {
  if (dense) return hf ? &combd_kernel<L, R, K, true, true> : &combd_kernel<L, R, K, true, false>;
  return hf ? &combd_kernel<L, R, K, false, true> : &combd_kernel<L, R, K, false, false>;
}

KernelFn pick_dual_d(int l, int r, int k, bool dense, bool hf) {
#define AP_D(L, R, K) \
  if (l == L && r == R && k == K) return pick<L, R, K>(dense, hf);
  AP_D(5, 20, 1) AP_D(10, 20, 1) AP_D(5, 16, 2) AP_D(5, 24, 2) AP_D(5, 32, 2) AP_D(10, 32, 2)
  AP_D(15, 20, 1) AP_D(10, 24, 2)
#undef AP_D
  return nullptr;
}

}  // namespace apk
