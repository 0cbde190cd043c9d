// Dual-pair comb kernel instantiations (ap_dual_kernels.cuh), R <= 16 rows per lane.
#include "ap_dual_kernels.cuh"

namespace apk {

template <int L, int R, int K>
static KernelFn pick(bool dense, bool hf) {
  if (dense) return hf ? &combd_kernel<L, R, K, true, true> : &combd_kernel<L, R, K, true, false>;
  return hf ? &combd_kernel<L, R, K, false, true> : &combd_kernel<L, R, K, false, false>;
}

KernelFn pick_dual_a(int l, int r, int k, bool dense, bool hf);
KernelFn pick_dual_c(int l, int r, int k, bool dense, bool hf);
KernelFn pick_dual_d(int l, int r, int k, bool dense, bool hf);
KernelFn pick_dual(int l, int r, int k, bool dense, bool hf) {
  if (KernelFn f = pick_dual_c(l, r, k, dense, hf)) return f;
  if (KernelFn f = pick_dual_d(l, r, k, dense, hf)) return f;
  if (r == 32) return pick_dual_a(l, r, k, dense, hf);
#define AP_D(L, R, K) \
  if (l == L && r == R && k == K) return pick<L, R, K>(dense, hf);
  AP_D(8, 16, 2) AP_D(8, 16, 1) AP_D(16, 16, 2) AP_D(16, 16, 1) AP_D(8, 8, 2) AP_D(8, 8, 1) AP_D(4, 16, 2)
#undef AP_D
  return nullptr;
}

}  // namespace apk
