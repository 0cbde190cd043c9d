// Instantiations of the r = 2 specialised comb kernel (comb2_kernel): shapes
// (L lanes, RR real rows per lane, K bands).  The host picks one whose blown
// row count R = 2*RR divides W = 2w (see ap_capi.cu kShapes2).  The fp16-key
// (HF) variants of the RR >= 8 shapes live in ap_inst_r2hf.cu.
#include "ap_kernels.cuh"

namespace apk {

KernelFn pick_r2_hf(int l, int rr, int k, bool dense);

template <int L, int RR, int K>
static KernelFn pick(bool dense) {
  return dense ? &comb2_kernel<L, RR, K, true, false> : &comb2_kernel<L, RR, K, false, false>;
}

KernelFn pick_r2(int l, int rr, int k, bool dense, bool hf) {
  if (hf) return pick_r2_hf(l, rr, k, dense);
#define AP_R2(L, RR, K) \
  if (l == L && rr == RR && k == K) return pick<L, RR, K>(dense);
  AP_R2(4, 25, 5) AP_R2(8, 8, 2) AP_R2(8, 8, 4) AP_R2(16, 4, 2) AP_R2(16, 8, 4) AP_R2(32, 8, 4)
  AP_R2(8, 16, 4) AP_R2(16, 16, 4) AP_R2(32, 16, 4) AP_R2(32, 4, 2)
  AP_R2(8, 20, 4) AP_R2(16, 10, 2) AP_R2(32, 5, 1) AP_R2(4, 25, 1) AP_R2(32, 4, 1) AP_R2(16, 4, 1)
  AP_R2(10, 10, 2) AP_R2(5, 20, 4) AP_R2(10, 10, 1) AP_R2(5, 20, 1)
#undef AP_R2
  return nullptr;
}

}  // namespace apk
