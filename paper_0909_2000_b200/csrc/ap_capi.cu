// ap_capi.cu — host side of the C ABI (include/alignplot_b200.h).
//
// Replaces the reference driver compute_plot (runner.cpp:78-131): validation
// (model.cpp:46-61) before any device work, then per device: H2D of the raw
// x slice (rows plus a w-1 halo) and of y, the code-stream
// kernels (fused $-interleave), the fused comb+extract kernel and either the
// dense D2H or the deterministic threshold compaction (scoring.cpp:30-39).
// Rows shard over devices in contiguous blocks; concatenating the blocks in
// device order is the global row-major order, so the only cross-device step
// is the gather of per-device hit counts.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/alignplot_b200.h"
#include "ap_aux_kernels.cuh"
#include "ap_kernels.cuh"
#include "ap_wide_kernels.cuh"
#include "ap_dual_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? AP_NOMEM : AP_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                     \
    }                                                                                     \
  } while (0)

// ---- kernel shape table ---------------------------------------------------
using apk::KernelFn;

// Instantiated shapes: (L lanes per strip pair, R rows per lane, K bands per lane).
struct ShapeDef { int L, R, K; };
constexpr ShapeDef kShapes[] = {
    {4, 32, 2}, {4, 32, 4},
    {8, 8, 2},  {8, 16, 2},  {8, 16, 4},  {8, 24, 2},  {8, 32, 2},  {8, 32, 4},
    {16, 8, 2}, {16, 16, 2}, {16, 16, 4}, {16, 24, 2}, {16, 32, 2}, {16, 32, 4},
    {32, 8, 2}, {32, 16, 2}, {32, 16, 4}, {32, 24, 2}, {32, 32, 2}, {32, 32, 4},
};

KernelFn pick_kernel(int l, int r, int k, bool dense, bool xm, bool hf = false) {
  if (hf) return xm ? nullptr : apk::pick_ghf(l, r, k, dense);
  switch (l) {
    case 4: return apk::pick_l4(r, k, dense, xm);
    case 8: return apk::pick_l8(r, k, dense, xm);
    case 16: return apk::pick_l16(r, k, dense, xm);
    case 32: return apk::pick_l32(r, k, dense, xm);
  }
  return nullptr;
}

// fp16 keys (HF kernels) need the rebase step to stay >= 128 columns
bool ghf_ok(uint32_t W, int l, int k) { return W + uint32_t(l * k) <= apk::kHfMaxSpan; }

constexpr size_t kSmemPerSm = 227 * 1024;


struct Shape {
  int L = 0, R = 0, K = 2;
  bool r2 = false;   // r = 2 specialised kernel (comb2_kernel); R = 2*RR then
  bool xm = false;   // masks computed in registers (no table)
  bool hf = false;   // fp16 keys: one cell op per row (r = 2: a mismatch min; generic: V' of one row in 4) on the FMA pipe
  bool dual = false; // two strip pairs per lane group sharing the mask table (combd_kernel: r = 1, h = 1, W = L*R)
  uint32_t ring = 0;
  size_t smem = 0;
  int warps_per_sm = 0;
};

// Cost per strip pair and column: L lanes x (3 ops per row pair [6 with computed
// masks] + ~14 per-step overhead) + ~25 extraction ops, scaled up when fewer than
// 16 warps per SM fit (registers from the compiled kernel, table in shared memory).
// Dual-pair shapes (combd_kernel, ap_dual_kernels.cuh), in order of preference per window:
// usable when W == L*R exactly (LCS plots with h = 1).
constexpr ShapeDef kDualShapes[] = {
    {4, 32, 2}, {8, 32, 2}, {8, 16, 2}, {16, 16, 1}, {4, 16, 2}, {8, 8, 2},
    {4, 32, 1}, {8, 32, 1}, {8, 16, 1}, {16, 16, 2}, {8, 8, 1},
    {4, 8, 2}, {4, 24, 2}, {8, 24, 2}, {16, 24, 2}, {32, 24, 2}, {16, 32, 2}, {32, 32, 2},
    // lane groups that do not tile the warp (30 of 32 lanes work): windows 80, 100, 120, 160, 200, 240,
    // 300, 320 (9-33% faster than the single-pair kernel; <20,20,1> for 400 and <25,20,1> for 500 were not)
    {5, 20, 1}, {10, 20, 1}, {5, 16, 2}, {5, 24, 2}, {5, 32, 2}, {10, 32, 2}, {15, 20, 1}, {10, 24, 2},
};

bool dual_shape_fits(uint32_t W, uint32_t sigma, bool dense, int l, int r, int k, int hf, Shape* out,
                     size_t smem_limit = kSmemPerSm / 2) {
  if (uint32_t(l * r) != W) return false;
  if (hf < 0) hf = ghf_ok(W, l, k);
  if (hf && !ghf_ok(W, l, k)) return false;
  if (!apk::pick_dual(l, r, k, dense, hf)) return false;
  const uint32_t ring = apk::ring_slots(W, apk::kChunk, l);
  const size_t smem = apk::combd_smem_per_warp(l, r, k, sigma, ring);
  if (smem > smem_limit) return false;
  out->L = l; out->R = r; out->K = k; out->xm = false; out->hf = hf; out->dual = true; out->r2 = false;
  out->ring = ring;
  out->smem = smem * apk::kWarpsPerCta;   // shapes are recorded for 4-warp CTAs (rescaled by the plan)
  out->warps_per_sm = 0;
  return true;
}

bool choose_shape(uint32_t W, uint32_t sigma, bool dense, Shape* out, bool dual_ok = false) {
  // tuning override: AP_SHAPE="L,R,K[,xm[,hf[,dual]]]" (hf default: the automatic choice)
  if (const char* env = std::getenv("AP_SHAPE")) {
    int l = 0, r = 0, k = 0, xm = 0, hf = -1, dual = 0;
    const int nf = std::sscanf(env, "%d,%d,%d,%d,%d,%d", &l, &r, &k, &xm, &hf, &dual);
    if (nf >= 6 && dual && dual_ok && !xm && dual_shape_fits(W, sigma, dense, l, r, k, hf, out)) return true;
    if (hf < 0) hf = !xm && ghf_ok(W, l, k) && pick_kernel(l, r, k, dense, false, true);
    if (nf >= 3 && (!hf || ghf_ok(W, l, k)) && pick_kernel(l, r, k, dense, xm, hf) && uint32_t(l * r) >= W) {
      const uint32_t ring = apk::ring_slots(W, apk::kChunk, l);
      out->L = l; out->R = r; out->K = k; out->xm = xm; out->hf = hf; out->ring = ring;
      out->smem = apk::kWarpsPerCta * apk::comb_smem_per_warp(l, r, xm ? 0 : sigma, ring);
      out->warps_per_sm = 0;
      return out->smem <= kSmemPerSm - 1024;
    }
  }
  if (dual_ok && !std::getenv("AP_NO_DUAL") && !std::getenv("AP_SHAPE")) {
    // first the measured order among shapes whose table leaves >= 8 warps per SM; a larger
    // alphabet's table crowds the warps out, and with 2-6 resident warps the K = 2 shapes (four
    // chains per lane) win: sigma = 60, w = 128: combd<8,16,2> 17.1 ms at 2 warps/SM against
    // combd<4,32,1> 22.8 and the single-pair computed-mask kernel 23.0 (tools/sigma_cmp.sh); past
    // ~90 KB per warp the single-pair kernel wins (sigma = 120, w = 64: 10.5 against 13.4-16.4)
    for (const ShapeDef& d : kDualShapes)
      if (dual_shape_fits(W, sigma, dense, d.L, d.R, d.K, -1, out, kSmemPerSm / 8 - 1024)) return true;
    // (among those the 8-lane groups measured best: sigma = 60, w = 64: <8,8,2> 8.6 ms, <4,16,2> 9.6;
    // sigma = 20, w = 256: <8,32,2> 20.4, <16,16,2> 22.1)
    for (int pass = 0; pass < 3; ++pass)
      for (const ShapeDef& d : kDualShapes) {
        const int cls = d.K == 2 ? (d.L == 8 ? 0 : 1) : 2;
        if (cls == pass && dual_shape_fits(W, sigma, dense, d.L, d.R, d.K, -1, out, 90 * 1024)) return true;
      }
  }
  out->dual = false;
  double best = 1e30;
  for (int xm = 0; xm < 2; ++xm) {
    for (const ShapeDef& d : kShapes) {
      if (uint32_t(d.L * d.R) < W) continue;
      const bool hf = !xm && ghf_ok(W, d.L, d.K) && pick_kernel(d.L, d.R, d.K, dense, false, true);
      KernelFn fn = pick_kernel(d.L, d.R, d.K, dense, xm, hf);
      if (!fn) continue;
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(fn)) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      const uint32_t ring = apk::ring_slots(W, apk::kChunk, d.L);
      const size_t smem = apk::kWarpsPerCta * apk::comb_smem_per_warp(d.L, d.R, xm ? 0 : sigma, ring);
      if (smem > kSmemPerSm - 1024) continue;
      const int by_regs = 65536 / (std::max(fa.numRegs, 1) * 32 * apk::kWarpsPerCta);
      const int by_smem = int(kSmemPerSm / (smem + 1024));
      const int ctas = std::min({by_regs, by_smem, 16});
      if (ctas < 1) continue;
      const int warps = ctas * apk::kWarpsPerCta;
      double cost = double(d.L) * ((xm ? 6.0 : 3.0) * d.R + 14.0) + 25.0;
      // long lanes (R = 32) hide latency with ILP: only penalise below 8 warps per SM
      // (B200: comb<8,32,4> at 8 warps beats comb<16,16,4> at 16 warps on C5 by 3%)
      if (warps < 8) cost *= 8.0 / warps;
      cost *= d.K == 4 && d.L >= 8 ? 0.95 : 1.0;   // 4 bands: more ILP per lane (measured ~5% faster)
      // (L = 4: comb<4,32,2> beats comb<4,32,4> and comb<8,16,4> on C3 by 2-5% on B200)
      if (cost < best) {
        best = cost;
        out->L = d.L;
        out->R = d.R;
        out->K = d.K;
        out->xm = xm;
        out->hf = hf;
        out->ring = ring;
        out->smem = smem;
        out->warps_per_sm = warps;
      }
    }
  }
  return best < 1e29;
}

// r = 2 specialised shapes (L, RR real rows per lane, K bands): usable when
// RR divides w and w/RR <= L (idle trailing lanes are padding).
struct Shape2Def { int L, RR, K; };

constexpr Shape2Def kShapes2[] = {
    {4, 25, 5}, {8, 8, 2}, {8, 8, 4}, {16, 4, 2}, {16, 8, 4}, {32, 8, 4},
    {8, 16, 4}, {16, 16, 4}, {32, 16, 4}, {32, 4, 2},
    {8, 20, 4}, {16, 10, 2}, {32, 5, 1}, {4, 25, 1}, {32, 4, 1}, {16, 4, 1},
    {10, 10, 2}, {5, 20, 4}, {10, 10, 1}, {5, 20, 1},
};

// r = 2 dual-pair shape (comb2d_kernel): 4 real rows per lane, w = 4*L exactly
bool dual2_shape_fits(uint32_t w, uint32_t sigma_y, bool dense, int l, int k, Shape* out) {
  if (l <= 0 || w != uint32_t(4 * l) || !apk::pick_r2_dual(l, k, dense)) return false;
  const uint32_t ring = apk::ring_slots(2 * w, 2 * apk::kChunk, l);
  const size_t smem = apk::comb2d_smem_per_warp(l, sigma_y, ring);
  if (smem > kSmemPerSm / 8) return false;   // keep at least 8 warps per SM
  out->L = l; out->R = 8; out->K = k; out->xm = false; out->r2 = true; out->hf = false; out->dual = true;
  out->ring = ring;
  out->smem = smem * apk::kWarpsPerCta;   // rescaled to the launch's one-warp CTAs by the plan
  out->warps_per_sm = 0;
  return true;
}

bool choose_shape2(uint32_t w, uint32_t sigma_y, bool dense, Shape* out, bool dual_ok = false) {
  if (std::getenv("AP_NO_R2")) return false;
  const uint32_t W = 2 * w;
  out->dual = false;
  if (dual_ok) {
    if (const char* env = std::getenv("AP_SHAPE2")) {   // "L,4,K,0,1": forced dual shape
      int l = 0, rr = 0, k = 0, hf = 0, dual = 0;
      if (std::sscanf(env, "%d,%d,%d,%d,%d", &l, &rr, &k, &hf, &dual) == 5 && dual && rr == 4 &&
          dual2_shape_fits(w, sigma_y, dense, l, k, out))
        return true;
    }
    // not chosen automatically: on C4 it runs at 53.8-54.8 ms per 16384 rows against 53.4 for
    // comb2<16,4,2> (same instruction count: what the shared code feed saves, the second pair's
    // selects, moves and ring stores cost; profiles/ab_r02.md)
  }
  // fp16 keys need W + 2*VB <= kHfMaxSpan (VB = virtual bands down the strip)
  auto hf_ok = [&](int rr, int k) { return W + 2 * (w / uint32_t(rr)) * uint32_t(k) <= apk::kHfMaxSpan; };
  // tuning override: AP_SHAPE2="L,RR,K[,hf]" (hf: 0/1, default: the automatic choice)
  if (const char* env = std::getenv("AP_SHAPE2")) {
    int l = 0, rr = 0, k = 0, hf = -1;
    const int nf = std::sscanf(env, "%d,%d,%d,%d", &l, &rr, &k, &hf);
    if (nf >= 3 && rr > 0 && w % rr == 0 && w / rr <= uint32_t(l)) {
      if (hf < 0) hf = apk::pick_r2(l, rr, k, dense, true) && hf_ok(rr, k);
      if ((!hf || hf_ok(rr, k)) && apk::pick_r2(l, rr, k, dense, hf)) {
      const uint32_t ring = apk::ring_slots(W, 2 * apk::kChunk, l);
      out->L = l; out->R = 2 * rr; out->K = k; out->xm = false; out->r2 = true; out->hf = hf; out->ring = ring;
      out->smem = apk::kWarpsPerCta *
                  apk::comb_smem_per_warp(l, k * apk::r2_band_words(rr / k), sigma_y, ring, 2 * apk::kChunk);
      out->warps_per_sm = 0;
      return out->smem <= kSmemPerSm - 1024;
      }
    }
  }
  double best = 1e30;
  for (const Shape2Def& d : kShapes2) {
    if (w % d.RR || w / d.RR > uint32_t(d.L)) continue;
    const bool hf = apk::pick_r2(d.L, d.RR, d.K, dense, true) && hf_ok(d.RR, d.K);
    KernelFn fn = apk::pick_r2(d.L, d.RR, d.K, dense, hf);
    if (!fn) continue;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(fn)) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    const int bw = apk::r2_band_words(d.RR / d.K);
    const uint32_t ring = apk::ring_slots(W, 2 * apk::kChunk, d.L);
    const size_t smem = apk::kWarpsPerCta * apk::comb_smem_per_warp(d.L, d.K * bw, sigma_y, ring, 2 * apk::kChunk);
    if (smem > kSmemPerSm - 1024) continue;
    const int by_regs = 65536 / (std::max(fa.numRegs, 1) * 32 * apk::kWarpsPerCta);
    const int by_smem = int(kSmemPerSm / (smem + 1024));
    const int ctas = std::min({by_regs, by_smem, 16});
    if (ctas < 1) continue;
    const int warps = ctas * apk::kWarpsPerCta;
    // per lane and raw column: 6 ALU ops per real row + ~30 fixed (shuffles,
    // codes, extraction); the long-chain shapes hide latency with ILP, so only
    // penalise occupancy below 8 warps per SM (fit to B200 sweeps, tools/shape_sweep2.sh)
    const double lanes_per_group = 32.0 / (32 / d.L);   // idle lanes of a non-dividing L count too
    double cost = lanes_per_group * (6.0 * d.RR + 30.0) + 50.0;
    if (warps < 16) cost *= 16.0 / warps;
    if (cost < best) {
      best = cost;
      out->L = d.L;
      out->R = 2 * d.RR;
      out->K = d.K;
      out->xm = false;
      out->r2 = true;
      out->hf = hf;
      out->ring = ring;
      out->smem = smem;
      out->warps_per_sm = warps;
    }
  }
  return best < 1e29;
}

}  // namespace

// ---- context ----------------------------------------------------------------
// Launch plan for (W, w, r, sigma, dense): kernel shape, function, occupancy.
struct LaunchPlan {
  Shape sh;
  int wpc = apk::kWarpsPerCta;   // warps per CTA of the launches
  bool spec = false;
  apk::KernelFn fn = nullptr;
  int per_sm = 0;
};

struct ap_ctx {
  int device = 0;
  int sms = 0;
  std::map<uint64_t, LaunchPlan> plans;   // cached per (w, r, sigma, dense) and env overrides
  std::map<uint64_t, uint32_t> last_sigma;   // y alphabet size of the last call per (w, r, output)
  cudaStream_t stream = nullptr;
  cudaStream_t stream_copy = nullptr;   // D2H of finished row blocks (overlaps the comb kernel)
  cudaStream_t stream_b = nullptr;      // second compute stream (compute-bound streamed plots)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  static constexpr int kMaxBlocks = 32;
  cudaEvent_t ev_blk[kMaxBlocks] = {};
  cudaEvent_t ev_cp[kMaxBlocks] = {};   // copy-done events (AP_TRACE timelines)
  cudaEvent_t ev_join = nullptr;
  std::mutex mu;
  // scratch (grown on demand)
  uint8_t *d_x = nullptr, *d_y = nullptr, *d_xcode = nullptr, *d_ycode = nullptr, *d_map = nullptr;
  size_t cap_x = 0, cap_y = 0, cap_xcode = 0, cap_ycode = 0, cap_ycol = 0;
  uint32_t* d_ycol = nullptr;
  uint32_t* d_small = nullptr;   // [0] sigma, [1] zero flag, [2] speculative-launch abort flag
  uint32_t* h_small = nullptr;   // pinned mirror
  uint16_t* d_out = nullptr;
  size_t cap_out = 0;
  uint16_t* d_out16 = nullptr;   // packed-kernel scores before widening to int32
  size_t cap_out16 = 0;
  uint4* d_stage = nullptr;
  size_t cap_stage = 0;
  unsigned long long* d_cursor = nullptr;
  uint32_t* d_tasks = nullptr;   // per-launch task counters (AP_DYN_TASKS)
  unsigned long long* h_cursor = nullptr;  // pinned
  uint32_t* d_segc = nullptr;
  size_t cap_segc = 0;
  unsigned long long* d_offs = nullptr;
  size_t cap_offs = 0;
  unsigned long long* d_tsum = nullptr;   // scan tile sums / offsets
  size_t cap_tsum = 0;
  int32_t* d_wkeys = nullptr;   // large-window path: per-strip start keys
  size_t cap_wkeys = 0;
  uint8_t* d_wok = nullptr;     // large-window path: per-strip extraction flags
  size_t cap_wok = 0;
  cudaMemPool_t pool = nullptr;   // per-call list buffers of the host API (stream-ordered, cached)
  // pinned bounce ring for device-to-host copies into pageable memory (allocated on first use)
  static constexpr int kMaxBounceSlots = 16;
  char* h_bounce = nullptr;
  int bounce_slots = 0;
  cudaEvent_t ev_bounce[kMaxBounceSlots] = {};
  // the staged list of the last thresholded run_device (placed by place_list)
  struct ListState {
    size_t nrec = 0;
    uint32_t seg_stride = 0, S = 0, S2 = 0, split_row = 0, r = 1, row_global0 = 0;
  } list;
  float last_ms = 0.f;
  int last_launches = 0;
  char last_kernel[64] = "";
};

namespace {

template <typename T>
int grow(T** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return AP_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  size_t bytes = std::max<size_t>(need, 1) * sizeof(T);
  CK(cudaMalloc(reinterpret_cast<void**>(p), bytes));
  *cap = need;
  return AP_OK;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

std::mutex g_ctx_mu;
std::vector<ap_ctx*> g_ctx;

int get_ctx(int device, ap_ctx** out) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (g_ctx.empty()) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      return fail(AP_NODEV, "no CUDA device available (the engine has no CPU fallback)");
    }
    g_ctx.assign(n, nullptr);
  }
  if (device < 0 || device >= int(g_ctx.size())) return fail(AP_NODEV, "device %d not present", device);
  if (!g_ctx[device]) {
    ap_ctx* c = nullptr;
    int rc = ap_ctx_create(device, &c);
    if (rc) return rc;
    g_ctx[device] = c;
  }
  *out = g_ctx[device];
  return AP_OK;
}

int check_cfg(size_t m, size_t n, const ap_config* cfg) {
  if (!cfg) return fail(AP_INVALID, "null config");
  if (cfg->window_w == 0) return fail(AP_CONFIG, "window size must be positive");
  if (cfg->step_h == 0) return fail(AP_CONFIG, "step size must be positive");
  if (cfg->blowup_r != 1 && cfg->blowup_r != 2)
    return fail(AP_CONFIG, "blowup factor must be 1 (LCS) or 2 (alignment score)");
  if (cfg->window_w > m || cfg->window_w > n)
    return fail(AP_EMPTY, "no window of size %zu fits inputs of lengths %zu and %zu",
                size_t(cfg->window_w), m, n);
  if (cfg->window_w * cfg->blowup_r > AP_MAX_BLOWN_WINDOW)
    return fail(AP_CONFIG, "blown windows up to %d are supported (sea16 bound, model.cpp:57-59; got %zu)",
                AP_MAX_BLOWN_WINDOW, size_t(cfg->window_w * cfg->blowup_r));
  if (n * cfg->blowup_r > 0x7FFFFFF0ull) return fail(AP_CONFIG, "y too long for the CUDA engine");
  return AP_OK;
}

// Rows [rb, re) of the grid, clamped.
int row_range(size_t rows, const ap_config* cfg, size_t* rb, size_t* re) {
  *rb = cfg->row_begin;
  *re = cfg->row_end ? std::min<size_t>(cfg->row_end, rows) : rows;
  if (*rb > *re) return fail(AP_INVALID, "row_begin > row_end");
  if (*re - *rb > 0xFFFFFFF0ull) return fail(AP_INVALID, "too many rows in one call");
  return AP_OK;
}

// ---- device-to-host copies of finished output ranges ----------------------------
// A copy into pageable host memory is staged by the driver at ~21 GB/s on B200 hosts (57 GB/s
// pinned, profiles/README_r02.md); callers of the host API (numpy arrays, std::vector) usually
// pass pageable memory.  So pageable destinations go through a pinned ring of slots: the calling
// thread issues slot-sized D2H copies on the copy stream as slots free up, and T host threads
// copy finished slots to their destination in parallel (piece i -> slot i mod 2T -> thread
// i mod T, so a thread only ever waits for copies it will itself release).
struct CopyRange {
  char* dst;
  const char* src;
  size_t bytes;
  cudaEvent_t ready;   // the range is complete once this event fires (nullptr: already)
};

constexpr size_t kBounceSlotBytes = size_t(8) << 20;

bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// All ranges copied when it returns.  Ranges must all be pinned or all pageable.
int copy_out(ap_ctx* c, const std::vector<CopyRange>& rg) {
  if (rg.empty()) return AP_OK;
  size_t total = 0;
  for (const CopyRange& r : rg) total += r.bytes;
  // below ~32 MB the ring's thread start-up costs more than the driver's staged copy saves
  // (C1's 7.5 MB plot: 1.09 ms through the ring vs 0.68 ms direct)
  if (total < (size_t(32) << 20) || host_pinned(rg[0].dst) || std::getenv("AP_NO_BOUNCE")) {
    for (const CopyRange& r : rg) {
      if (r.ready) CK(cudaStreamWaitEvent(c->stream_copy, r.ready, 0));
      CK(cudaMemcpyAsync(r.dst, r.src, r.bytes, cudaMemcpyDeviceToHost, c->stream_copy));
    }
    CK(cudaStreamSynchronize(c->stream_copy));
    return AP_OK;
  }
  if (!c->h_bounce) {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    c->bounce_slots = int(std::min<unsigned>(ap_ctx::kMaxBounceSlots, 2 * std::min(8u, hw / 2)));
    CK(cudaMallocHost(reinterpret_cast<void**>(&c->h_bounce), size_t(c->bounce_slots) * kBounceSlotBytes));
    for (int k = 0; k < c->bounce_slots; ++k) CK(cudaEventCreateWithFlags(&c->ev_bounce[k], cudaEventDisableTiming));
  }
  struct Piece { char* dst; const char* src; size_t bytes; cudaEvent_t ready; };
  std::vector<Piece> pcs;
  for (const CopyRange& r : rg)
    for (size_t off = 0; off < r.bytes; off += kBounceSlotBytes)
      pcs.push_back({r.dst + off, r.src + off, std::min(kBounceSlotBytes, r.bytes - off), off ? nullptr : r.ready});
  const size_t S = size_t(c->bounce_slots), T = S / 2, P = pcs.size();
  std::mutex m;
  std::condition_variable cv;
  size_t issued = 0;
  std::vector<size_t> freed(S);            // piece index that may use slot s next
  for (size_t s2 = 0; s2 < S; ++s2) freed[s2] = s2;
  std::atomic<int> err{AP_OK};
  std::string err_msg;
  auto worker = [&](size_t t) {
    cudaSetDevice(c->device);
    for (size_t i = t; i < P; i += T) {
      {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return issued > i || err.load() != AP_OK; });
      }
      if (err.load() != AP_OK) return;
      const size_t s2 = i % S;
      if (cudaEventSynchronize(c->ev_bounce[s2]) != cudaSuccess) {
        std::lock_guard<std::mutex> lk(m);
        err = AP_CUDA;
        err_msg = cudaGetErrorString(cudaGetLastError());
        cv.notify_all();
        return;
      }
      std::memcpy(pcs[i].dst, c->h_bounce + s2 * kBounceSlotBytes, pcs[i].bytes);
      {
        std::lock_guard<std::mutex> lk(m);
        freed[s2] = i + S;
      }
      cv.notify_all();
    }
  };
  std::vector<std::thread> th;
  for (size_t t = 0; t < std::min(T, P); ++t) th.emplace_back(worker, t);
  for (size_t i = 0; i < P && err.load() == AP_OK; ++i) {
    const size_t s2 = i % S;
    {
      std::unique_lock<std::mutex> lk(m);
      cv.wait(lk, [&] { return freed[s2] >= i || err.load() != AP_OK; });
    }
    if (err.load() != AP_OK) break;
    cudaError_t e = cudaSuccess;
    if (pcs[i].ready) e = cudaStreamWaitEvent(c->stream_copy, pcs[i].ready, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(c->h_bounce + s2 * kBounceSlotBytes, pcs[i].src, pcs[i].bytes, cudaMemcpyDeviceToHost,
                          c->stream_copy);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_bounce[s2], c->stream_copy);
    std::lock_guard<std::mutex> lk(m);
    if (e != cudaSuccess) {
      err = AP_CUDA;
      err_msg = cudaGetErrorString(e);
    } else {
      issued = i + 1;
    }
    cv.notify_all();
  }
  for (auto& t : th) t.join();
  if (err.load() != AP_OK) return fail(err.load(), "device-to-host copy: %s", err_msg.c_str());
  return AP_OK;
}

// bytes per dense output entry: 0 = uint16 half-units, 1 = PGM pixels, 2 = uint8 half-units,
// 3 = int32 half-units (PlotGrid's own type, model.hpp:95-114)
size_t out_elem(int out_kind) { return out_kind == 0 ? 2 : out_kind == 3 ? 4 : 1; }

// Thresholded runs: size the staging and the per-(row, segment) count buffers, zero the cursor.
// Staging (one 16-B record per hit) is sized so a call normally stages every hit in one
// pass: the grid's cell count bounds it, the caller's capacity is a floor, and otherwise it
// takes up to 2^28 records (4 GiB) within an eighth of free device memory.  A list longer
// than the staging still comes out exact: the kernel counts every hit, the staging grows to
// the exact size and the comb re-runs (rare).
int stage_prepare(ap_ctx* c, size_t nrows, size_t cols, size_t cap, size_t seg_stride, bool zero_counts,
                  cudaStream_t st, bool count_only = false) {
  int rc;
  const size_t cells_ub = count_only ? 1 : nrows * cols + 1;   // a count-only call stages nothing
  size_t target = std::max(std::min(cells_ub, size_t(1) << 28), std::min(cap, cells_ub));
  if (c->cap_stage < target) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); fr = 0; }
    target = std::min(target, std::max<size_t>(fr / 8 / sizeof(uint4), std::min(cap, cells_ub)));
    target = std::max<size_t>(target, std::min<size_t>(cells_ub, 1 << 16));
    if (c->cap_stage < target && (rc = grow(&c->d_stage, &c->cap_stage, target))) return rc;
  }
  const size_t nc = nrows * seg_stride;
  if ((rc = grow(&c->d_segc, &c->cap_segc, nc))) return rc;
  if ((rc = grow(&c->d_offs, &c->cap_offs, nc + 1))) return rc;
  if ((rc = grow(&c->d_tsum, &c->cap_tsum, (nc + apk::kScanTile - 1) / apk::kScanTile + 1))) return rc;
  if (zero_counts) CK(cudaMemsetAsync(c->d_segc, 0, nc * sizeof(uint32_t), st));
  CK(cudaMemsetAsync(c->d_cursor, 0, sizeof(unsigned long long), st));
  return AP_OK;
}

// Exclusive scan of the nc per-(row, segment) hit counts into 64-bit offsets (the total at
// offs[nc]), then the staged-record cursor and the total to the host (h_cursor[0], [1]).
int scan_counts(ap_ctx* c, size_t nc, cudaStream_t st) {
  const size_t ntiles = (nc + apk::kScanTile - 1) / apk::kScanTile;
  apk::scan_tile_sums_kernel<<<unsigned(ntiles), apk::kScanThreads, 0, st>>>(c->d_segc, nc, c->d_tsum);
  apk::scan_tile_offsets_kernel<<<1, apk::kScanThreads, 0, st>>>(c->d_tsum, ntiles, c->d_offs + nc);
  apk::scan_tiles_kernel<<<unsigned(ntiles), apk::kScanThreads, 0, st>>>(c->d_segc, nc, c->d_tsum, c->d_offs);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->h_cursor, c->d_cursor, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_cursor + 1, c->d_offs + nc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  c->last_launches += 3;
  return AP_OK;
}

// The large-window path (W = w*r > AP_PACKED_WINDOW, up to 65534; ap_wide_kernels.cuh): one
// CTA per strip combs it band by band with exact 32-bit keys, then one CTA per strip
// extracts its row.  Strips run in batches bounded by the key scratch (~2 GiB).  Code
// streams are already built (x codes, the $-interleaved y stream, $ code `sent`).
int run_wide(ap_ctx* c, const ap_config* cfg, size_t nrows, size_t row_global0, bool dense, void* d_out,
             cudaStream_t st, size_t* nrec_out, size_t* total_out, size_t cap, int out_kind, void* host_out,
             uint32_t sent, size_t n, uint32_t sigma_y, bool count_only) {
  const uint32_t w = uint32_t(cfg->window_w), h = uint32_t(cfg->step_h), r = cfg->blowup_r;
  const uint32_t W = w * r;
  const size_t N = n * r;
  const size_t cols = n - w + 1;
  int rc;
  // Warps per CTA: enough to hold the strip in one band (512 rows per warp), at most 32 with
  // computed masks and at most 8 with the mask table (alphabets of <= 8 codes, 2 KB per code and
  // warp; 4096-row bands, several CTAs per SM).
  const uint32_t codes = sigma_y + (r == 2 ? 1u : 0u);
  const bool tbl = !std::getenv("AP_WIDE_NO_TABLE") && codes <= 8;
  const uint32_t warps = std::min<uint32_t>(tbl ? 8u : apk::kWideMaxWarps,
                                            (W + 32 * apk::kWideRows - 1) / (32 * apk::kWideRows));
  const size_t wsmem = (tbl ? size_t(codes) * 32 * apk::kWideRows * 4 * warps : 0) +
                       size_t(warps) * apk::kWideRing * 4;
  // Packed pairs (two strips per register, 16-bit keys) when the rebase step stays >= 96 columns:
  // every seaweed a later window can count must survive a rebase (ap_wide_kernels.cuh)
  const int32_t rebase_at = 0x7000, rebase_by = rebase_at - int32_t(W) - 64 * int32_t(warps) - 64;
  const bool packed = tbl && rebase_by >= 96 && !std::getenv("AP_WIDE_NO_PACK");
  const uint32_t band_rows = warps * 32 * apk::kWideRows;
  apk::WideParams p{};
  p.xcode = c->d_xcode;
  p.ycode = c->d_ycode;
  p.h = h;
  p.w = w;
  p.r = r;
  p.W = W;
  p.N = uint32_t(N);
  p.sent_code = sent;
  p.band_rows = band_rows;
  p.bands = (W + band_rows - 1) / band_rows;
  p.tbl_codes = codes;
  p.rebase_at = uint32_t(rebase_at);
  p.rebase_by = uint32_t(std::max(rebase_by, 0));
  const void* wfn = packed ? reinterpret_cast<const void*>(&apk::wide2_comb_kernel)
                            : tbl ? reinterpret_cast<const void*>(&apk::wide_comb_kernel<true>)
                                  : reinterpret_cast<const void*>(&apk::wide_comb_kernel<false>);
  CK(cudaFuncSetAttribute(wfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(wsmem)));
  p.cols = uint32_t(cols);
  p.row_global0 = uint32_t(row_global0);
  p.out = static_cast<uint16_t*>(d_out);
  p.out8 = static_cast<uint8_t*>(d_out);
  p.out32 = static_cast<int32_t*>(d_out);
  p.out_kind = uint32_t(out_kind);
  p.pgm_threshold = cfg->threshold_half;
  p.has_pgm_threshold = cfg->has_threshold ? 1u : 0u;
  p.dense = dense ? 1u : 0u;
  if (!dense) {
    if ((rc = stage_prepare(c, nrows, cols, cap, 1, false, st, count_only))) return rc;
    p.t_half = cfg->threshold_half;
    p.stage = c->d_stage;
    p.cursor = c->d_cursor;
    p.stage_cap = count_only ? 0 : c->cap_stage;
    p.seg_counts = c->d_segc;
  }
  size_t batch = std::max<size_t>(2, std::min<size_t>(nrows, (size_t(2) << 30) / (5 * N)));
  batch += batch & 1;   // whole strip pairs per launch (packed kernel)
  if ((rc = grow(&c->d_wkeys, &c->cap_wkeys, batch * N))) return rc;
  if ((rc = grow(&c->d_wok, &c->cap_wok, batch * N))) return rc;
  p.keys = c->d_wkeys;
  p.ok = c->d_wok;
  CK(cudaEventRecord(c->ev0, st));
  auto launch_all = [&]() -> int {
    for (size_t r0 = 0; r0 < nrows; r0 += batch) {
      apk::WideParams q = p;
      q.strips = uint32_t(std::min(batch, nrows - r0));
      q.row0 = uint32_t(r0);
      q.xcode = c->d_xcode + r0 * h;
      if (packed) apk::wide2_comb_kernel<<<(q.strips + 1) / 2, warps * 32, wsmem, st>>>(q);
      else if (tbl) apk::wide_comb_kernel<true><<<q.strips, warps * 32, wsmem, st>>>(q);
      else apk::wide_comb_kernel<false><<<q.strips, warps * 32, wsmem, st>>>(q);
      CK(cudaGetLastError());
      apk::wide_extract_kernel<<<q.strips, apk::kWideExtThreads, 0, st>>>(q);
      CK(cudaGetLastError());
      c->last_launches += 2;
    }
    return AP_OK;
  };
  if ((rc = launch_all())) return rc;
  CK(cudaEventRecord(c->ev1, st));
  std::snprintf(c->last_kernel, sizeof(c->last_kernel), "combw<%u,%d,%s>", warps, apk::kWideRows,
                packed ? "table,packed" : tbl ? "table" : "computed");
  if (dense) {
    if (host_out) {
      CK(cudaEventRecord(c->ev_join, st));
      if ((rc = copy_out(c, {{static_cast<char*>(host_out), static_cast<const char*>(d_out),
                              nrows * cols * out_elem(out_kind), c->ev_join}})))
        return rc;
    }
    CK(cudaStreamSynchronize(st));
    return AP_OK;
  }
  if ((rc = scan_counts(c, nrows, st))) return rc;
  CK(cudaStreamSynchronize(st));
  const size_t nrec = c->h_cursor[0], total = c->h_cursor[1];
  if (nrec != total) return fail(AP_CUDA, "threshold bookkeeping mismatch (%zu staged vs %zu counted)", nrec, total);
  if (nrec > c->cap_stage && !count_only) {   // staging overflowed: grow to the exact size and recompute (rare)
    if ((rc = grow(&c->d_stage, &c->cap_stage, nrec))) return rc;
    p.stage = c->d_stage;
    p.stage_cap = c->cap_stage;
    CK(cudaMemsetAsync(c->d_cursor, 0, sizeof(unsigned long long), st));
    if ((rc = launch_all())) return rc;
  }
  c->list.nrec = count_only ? 0 : nrec;
  c->list.seg_stride = 1;
  c->list.S = uint32_t(N + 1);   // one segment per row
  c->list.S2 = uint32_t(N + 1);
  c->list.split_row = uint32_t(nrows);
  c->list.r = r;
  c->list.row_global0 = uint32_t(row_global0);
  *nrec_out = nrec;
  *total_out = total;
  return AP_OK;
}

// Enqueue the whole pipeline for local rows [0, nrows) whose x windows start
// at d_x (already offset to the first row).  dense: writes d_out.
// out_kind (dense only): 0 = uint16 half-units into d_out, 1 = uint8 PGM pixels
// (io.cpp:136-153 fused; cfg->has_threshold renders cells below it black).
#ifndef AP_STREAM_GROWTH
#define AP_STREAM_GROWTH 1.2
#endif

// Thresholded runs (dense = false) stage the hits and leave them in c->list for place_list;
// `cap` is the caller's list capacity (a lower bound for the staging size).  count_only: the
// caller wants the count alone, so a staging overflow is not re-run (the count is exact anyway).
int run_device(ap_ctx* c, const uint8_t* d_x, size_t mx, const uint8_t* d_y, size_t n,
               const ap_config* cfg, size_t nrows, size_t row_global0, bool dense,
               void* d_out, cudaStream_t st, size_t* nrec_out, size_t* total_out,
               size_t cap, int out_kind = 0, void* host_out = nullptr, bool allow_spec = true,
               bool count_only = false) {
  const uint32_t w = uint32_t(cfg->window_w), h = uint32_t(cfg->step_h), r = cfg->blowup_r;
  const uint32_t W = w * r;
  const size_t N = n * r;
  const size_t cols = n - w + 1;
  c->last_launches = 0;
  if (nrows == 0) {
    if (nrec_out) *nrec_out = 0;
    if (total_out) *total_out = 0;
    return AP_OK;
  }

  int rc;
  // The plan depends on y's alphabet size.  Speculative alphabet: when this context has run
  // the same (w, r, output) before, plan for that call's alphabet size without waiting for
  // this one's -- a plan for more codes than y has is still exact (unused table codes; the $
  // code stays above every real code) -- and let the comb kernel verify on the device: if y
  // has more codes, every warp exits and flags the launch, and the call re-runs synchronously.
  // This removes the host round trip between the alphabet pass and the comb (C1: ~20 us).
  const bool overrides = std::getenv("AP_SHAPE") || std::getenv("AP_SHAPE2") || std::getenv("AP_NO_R2") ||
                         std::getenv("AP_NO_DUAL") || std::getenv("AP_DUAL");
  const uint64_t skey = (uint64_t(w) << 20) | (uint64_t(r) << 18) | (uint64_t(out_kind) << 2) | (dense ? 1 : 0);
  const auto spec_hit = c->last_sigma.find(skey);
  const bool wide = W > AP_PACKED_WINDOW;   // the large-window path plans nothing by sigma
  if (dense && out_kind == 3 && !wide) {
    // int32 half-units on the packed kernels (scores < 2^16): uint16 into scratch, widened on the device
    if ((rc = grow(&c->d_out16, &c->cap_out16, nrows * cols))) return rc;
    if ((rc = run_device(c, d_x, mx, d_y, n, cfg, nrows, row_global0, true, c->d_out16, st, nullptr, nullptr, 0, 0,
                         nullptr, allow_spec)))
      return rc;
    apk::widen_kernel<<<unsigned(std::min<size_t>((nrows * cols + 255) / 256, size_t(c->sms) * 32)), 256, 0, st>>>(
        c->d_out16, nrows * cols, static_cast<int32_t*>(d_out));
    CK(cudaGetLastError());
    c->last_launches += 1;
    if (host_out) {
      CK(cudaEventRecord(c->ev_join, st));
      if ((rc = copy_out(c, {{static_cast<char*>(host_out), static_cast<const char*>(d_out), nrows * cols * 4,
                              c->ev_join}})))
        return rc;
    }
    CK(cudaStreamSynchronize(st));
    return AP_OK;
  }
  const bool speculate = !wide && allow_spec && !overrides && !std::getenv("AP_NO_SPEC") &&
                         spec_hit != c->last_sigma.end();
  // small inputs take the fused single-CTA code-stream kernel (one launch) when speculating
  const bool fused_codes = speculate && mx + N <= (size_t(1) << 20);
  uint32_t sigma_y;
  if (!fused_codes) {
    // alphabet of y -> dense codes
    apk::alphabet_kernel<<<1, 1024, 0, st>>>(d_y, n, c->d_map, c->d_small, c->d_small + 1);
    CK(cudaGetLastError());
  }
  if (speculate) {
    sigma_y = spec_hit->second;
    if (!fused_codes) CK(cudaMemsetAsync(c->d_small + 2, 0, sizeof(uint32_t), st));
  } else {
    CK(cudaMemcpyAsync(c->h_small, c->d_small, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    sigma_y = c->h_small[0];
    c->last_sigma[skey] = sigma_y;
  }
  // after the call's own final synchronisation: did a speculative launch hold?  (1 = re-run)
  auto spec_failed = [&]() -> int {
    if (!speculate) return 0;
    if (c->h_small[2]) {
      c->last_sigma[skey] = c->h_small[0];
      return 1;
    }
    if (c->h_small[0] != sigma_y) c->last_sigma[skey] = c->h_small[0];   // plan the next call exactly
    return 0;
  };
  const uint32_t sent = sigma_y;
  const uint32_t sigma = sigma_y + (r == 2 ? 1 : 0);
  if (wide) {
    int q;
    const size_t ytot = (N + 256 + 31) / 32 * 32;
    if ((q = grow(&c->d_xcode, &c->cap_xcode, mx))) return q;
    if ((q = grow(&c->d_ycode, &c->cap_ycode, ytot))) return q;
    apk::xcode_kernel<<<std::min<size_t>((mx + 255) / 256, 4096), 256, 0, st>>>(d_x, mx, c->d_map, c->d_xcode);
    apk::ycode_kernel<<<std::min<size_t>((ytot + 255) / 256, 4096), 256, 0, st>>>(d_y, n, r, sent, c->d_map,
                                                                                  c->d_ycode, ytot, nullptr);
    CK(cudaGetLastError());
    c->last_launches += 3;
    return run_wide(c, cfg, nrows, row_global0, dense, d_out, st, nrec_out, total_out, cap, out_kind, host_out,
                    sent, n, sigma_y, count_only);
  }

  // launch plan (shape choice, function attributes, occupancy), cached per context;
  // tuning overrides (AP_SHAPE, AP_SHAPE2, AP_NO_R2) bypass the cache
  // the dual-pair kernel (two strip pairs per lane group) needs LCS strips one character apart
  // and enough (pair, segment) tasks to fill the GPU with half as many pair groups (C1 does not:
  // 0.049 -> 0.058 ms); AP_DUAL=1 forces it for eligible plots
  const size_t max_nseg = std::max<size_t>(1, (N - W + 1) / std::max<size_t>(4 * W, 256));
  const char* dual_env = std::getenv("AP_DUAL");
  const bool dual_ok = h == 1 &&
                       (dual_env ? std::atoi(dual_env) != 0 : ((nrows + 1) / 2) * max_nseg >= size_t(16) * 12 * c->sms);
  const uint64_t pkey = (uint64_t(w) << 20) | (uint64_t(r) << 18) | (uint64_t(sigma_y) << 2) | (dual_ok ? 2 : 0) |
                        (dense ? 1 : 0);
  LaunchPlan plan;
  auto hit = overrides ? c->plans.end() : c->plans.find(pkey);
  if (hit != c->plans.end()) {
    plan = hit->second;
  } else {
    plan.spec = r == 2 && choose_shape2(w, sigma_y, dense, &plan.sh, dual_ok);
    if (!plan.spec && !choose_shape(W, sigma, dense, &plan.sh, dual_ok && r == 1))
      return fail(AP_CONFIG, "alphabet of %u codes with blown window %u does not fit the engine's tables",
                  sigma, W);
    plan.fn = plan.spec ? (plan.sh.dual ? apk::pick_r2_dual(plan.sh.L, plan.sh.K, dense)
                                        : apk::pick_r2(plan.sh.L, plan.sh.R / 2, plan.sh.K, dense, plan.sh.hf))
              : plan.sh.dual ? apk::pick_dual(plan.sh.L, plan.sh.R, plan.sh.K, dense, plan.sh.hf)
                        : pick_kernel(plan.sh.L, plan.sh.R, plan.sh.K, dense, plan.sh.xm, plan.sh.hf);
    if (!plan.fn) return fail(AP_CONFIG, "no kernel instantiation for L=%d R=%d", plan.sh.L, plan.sh.R);
    // warps per CTA, as compiled into the kernel (ap_kernels.cuh kGenericWpc / r2_wpc)
    plan.wpc = plan.spec ? apk::r2_wpc(plan.sh.R / 2) : apk::kGenericWpc;
    plan.sh.smem = plan.sh.smem / apk::kWarpsPerCta * plan.wpc;   // shapes are sized for 4-warp CTAs
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(plan.fn),
                            cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.sh.smem)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&plan.per_sm, plan.fn, plan.wpc * 32, plan.sh.smem));
    if (plan.per_sm < 1) return fail(AP_CONFIG, "kernel L=%d R=%d does not fit an SM", plan.sh.L, plan.sh.R);
    if (!overrides) c->plans[pkey] = plan;
  }
  const Shape& sh = plan.sh;
  const bool spec = plan.spec;
  if (spec)
    std::snprintf(c->last_kernel, sizeof(c->last_kernel), "%s<%d,%d,%d,%s>", sh.dual ? "comb2d" : "comb2", sh.L,
                  sh.R / 2, sh.K, sh.hf ? "fp16" : "int");
  else
    std::snprintf(c->last_kernel, sizeof(c->last_kernel), "%s<%d,%d,%d,%s,%s>", sh.dual ? "combd" : "comb", sh.L,
                  sh.R, sh.K, sh.xm ? "computed" : "table", sh.hf ? "fp16" : "int");
  // the dynamic-smem limit is a per-function attribute and other plans may have
  // lowered it since this plan was cached
  CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(plan.fn),
                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(sh.smem)));

  // code streams: the specialised r = 2 kernel reads raw y codes (the $ columns
  // are implicit); the generic kernel reads the $-interleaved stream
  if ((rc = grow(&c->d_xcode, &c->cap_xcode, mx))) return rc;
  const size_t ylen = spec ? n : N;
  const size_t ytot = (ylen + 256 + 31) / 32 * 32;
  if ((rc = grow(&c->d_ycode, &c->cap_ycode, ytot))) return rc;
  // column-word stream: generic kernels, both dual kernels, and the unrolled r = 2 shapes' feed
  const bool r2_ycol = spec && !sh.dual && apk::r2_ycol_feed(sh.R / 2, sh.K);
  const bool want_ycol = !spec || sh.dual || r2_ycol;
  if (want_ycol && (rc = grow(&c->d_ycol, &c->cap_ycol, 2 * ytot))) return rc;   // ytot: multiple of 32
  // column words: the code in both halves, or for the dual-pair kernel its table offset
  const uint32_t ycol_mult = r2_ycol ? uint32_t(sh.R / 2 * 128) : !sh.dual ? 0x00010001u
                             : spec   ? uint32_t(apk::r2d_nq(sh.L) * 16)
                                      : uint32_t(apk::dual_cs(sh.L, sh.R) * 16);
  if (fused_codes) {
    apk::codes_small_kernel<<<1, 1024, 0, st>>>(d_x, mx, d_y, n, spec ? 1 : r, sent, c->d_map, c->d_small,
                                                c->d_xcode, c->d_ycode, ytot, want_ycol ? c->d_ycol : nullptr, ycol_mult);
    CK(cudaGetLastError());
    c->last_launches += 1;
  } else {
    apk::xcode_kernel<<<std::min<size_t>((mx + 255) / 256, 4096), 256, 0, st>>>(d_x, mx, c->d_map,
                                                                                 c->d_xcode);
    CK(cudaGetLastError());
    apk::ycode_kernel<<<std::min<size_t>((ytot + 255) / 256, 4096), 256, 0, st>>>(
        d_y, n, spec ? 1 : r, sent, c->d_map, c->d_ycode, ytot, want_ycol ? c->d_ycol : nullptr, ycol_mult);
    CK(cudaGetLastError());
    c->last_launches += 3;
  }

  KernelFn fn = plan.fn;
  const int per_sm = plan.per_sm;
  const int wpc = plan.wpc;
  const size_t total_warps = size_t(c->sms) * per_sm * wpc;

  // column segments: enough independent (strip pair, segment) tasks for ~4
  // waves, each segment at least 4 windows wide to bound the W-1 overlap.
  const int G = 32 / sh.L * (sh.dual ? 2 : 1);   // strip pairs per warp
  const size_t npairs = (nrows + 1) / 2;
  const size_t ngroups = (npairs + G - 1) / G;
  const size_t out_cols_eff = (N - W) + 1;  // window starts in effective columns (stride 1)
  size_t nseg = 1;
  const size_t want = 4 * total_warps;
  if (ngroups < want) nseg = (want + ngroups - 1) / ngroups;
  const size_t min_seg = std::max<size_t>(4 * W, 256);
  nseg = std::min(nseg, std::max<size_t>(1, out_cols_eff / min_seg));
  // segments of at most 2^18 effective columns: long tasks make the grid's drain long (C4:
  // nseg 1 -> 2 -0.8%, C5: 1 -> 4 -1%; the W-1 overlap stays below 0.4% at the BASELINE windows)
  nseg = std::max(nseg, (out_cols_eff + (size_t(1) << 18) - 1) >> 18);
  if (const char* e = std::getenv("AP_NSEG")) nseg = std::max<size_t>(1, std::strtoull(e, nullptr, 10));   // tuning
  size_t S = (out_cols_eff + nseg - 1) / nseg;
  // segment starts aligned for 16-B vector loads of the code stream (raw codes
  // for the r = 2 kernel: blown starts multiple of 64)
  const size_t salign = spec ? 64 : 32;
  S = (S + salign - 1) / salign * salign;
  nseg = (out_cols_eff + S - 1) / S;

  apk::CombParams p{};
  p.xcode = c->d_xcode;
  p.ycode = c->d_ycode;
  p.ycol = c->d_ycol;
  p.ycol_zero = want_ycol ? c->d_ycol + ytot : nullptr;
  p.rows = uint32_t(nrows);
  p.xlen = uint32_t(mx);
  p.h = h;
  p.w = w;
  p.r = r;
  p.W = W;
  p.N = uint32_t(N);
  p.sigma = spec ? sigma_y : (sh.xm ? 0 : sigma);
  p.one = 1u;
  p.minus_one = 0xFFFFFFFFu;
  p.sigma_dev = c->d_small;
  p.sigma_cap = speculate ? sigma_y : 0xFFFFFFFFu;
  p.abort_flag = c->d_small + 2;
  p.sent_code = sent;
  p.S = uint32_t(S);
  p.nseg = uint32_t(nseg);
  p.g_split = uint32_t(ngroups);   // no short tail tasks unless set below
  p.nseg2 = p.nseg;
  p.S2 = p.S;
  // The last ~wave of work as tasks of half the segment width.  The dynamic task counter
  // hands them out last, so the grid drains on short tasks instead of leaving SMs idle while
  // the last full-length tasks finish (C2: 5.92 -> 5.56 ms; halves beat quarters, 5.61, and
  // a two-wave tail, 5.58).  Launches of at least two waves; the streamed dense host path has
  // short tasks of its own.  AP_TAIL_SPLIT=1 disables it (tuning).
  size_t tail_div = 2;
  if (const char* e = std::getenv("AP_TAIL_SPLIT")) tail_div = size_t(std::max(1, std::atoi(e)));
  if (!(dense && host_out) && tail_div > 1 && ngroups * nseg >= 2 * total_warps && S / tail_div >= 2 * W) {
    size_t S2 = std::max<size_t>((S / tail_div + salign - 1) / salign * salign, std::max<size_t>(2 * W, salign));
    const size_t nseg2 = (out_cols_eff + S2 - 1) / S2;
    double tail_waves = 1.0;
    if (const char* e = std::getenv("AP_TAIL_WAVES")) tail_waves = std::atof(e);
    const size_t g2 = std::min(ngroups, std::max<size_t>(1, size_t(tail_waves * double(total_warps) / double(nseg2))));
    p.g_split = uint32_t(ngroups - g2);
    p.nseg2 = uint32_t(nseg2);
    p.S2 = uint32_t(S2);
  }
  p.seg_stride = std::max(p.nseg, p.nseg2);
  const size_t split_row = size_t(p.g_split) * 2 * G;   // first local row of the short-task groups
  p.ring = sh.ring;
  p.cols = uint32_t(cols);
  p.row_global0 = uint32_t(row_global0);
  p.out = static_cast<uint16_t*>(d_out);
  p.out8 = static_cast<uint8_t*>(d_out);
  p.out_kind = uint32_t(out_kind);
  p.pgm_threshold = cfg->threshold_half;
  p.has_pgm_threshold = cfg->has_threshold ? 1u : 0u;

  const size_t ntasks = size_t(p.g_split) * nseg + (ngroups - p.g_split) * p.nseg2;
  const size_t ctas_needed = (ntasks + wpc - 1) / wpc;
  const size_t grid = std::min<size_t>(ctas_needed, size_t(c->sms) * per_sm);

  if (!dense) {
    // with a tail split the rows of the long-task groups leave counts nseg..seg_stride-1 unset
    if ((rc = stage_prepare(c, nrows, cols, cap, p.seg_stride, p.seg_stride != p.nseg, st, count_only))) return rc;
    // the kernel tests h >= t in biased 16-bit halves: |h| <= 2048, so clamping t
    // to +-0x4000 keeps every comparison exact
    p.t_half = std::min<int32_t>(0x4000, std::max<int32_t>(-0x4000, cfg->threshold_half));
    p.stage = c->d_stage;
    p.cursor = c->d_cursor;
    p.stage_cap = count_only ? 0 : c->cap_stage;
    p.seg_counts = c->d_segc;
  }

  p.task_counter = c->d_tasks + 62;
  if (AP_DYN_TASKS) CK(cudaMemsetAsync(c->d_tasks, 0, 64 * sizeof(uint32_t), st));
  CK(cudaEventRecord(c->ev0, st));
  if (dense && host_out) {
    // Dense output to the host: the plot streams out row block by row block while later
    // blocks comb (copy stream), so the end-to-end time is about max(comb, D2H) plus the
    // exposed ends.  The comb costs ~0.057 ps per blown cell, the D2H (PCIe, ~57 GB/s)
    // ~17.5 ps per byte on B200:
    //  * D2H-bound (uint16 output, W*r < ~600; C2): e2e = (time to the first finished
    //    block) + D2H + ~50 us per copy.  Short tasks (segments of ~max(1024, 4W) columns:
    //    ~0.2 ms per task on C2 instead of ~1.3 ms; the extra W-1 overlap fits in the D2H
    //    time) on one stream, in row blocks of round(1.2^k) full waves (equal tasks, so a
    //    block ends without a ragged tail; a block's comb fits in the previous block's D2H,
    //    so the copy engine never idles): the first copy starts after one task time.
    //    (Swept on B200, AP_STREAM_S / AP_STREAM_GROWTH: 1024 / 1.2 best, 10.37 ms; 2048 /
    //    1.3 10.57; 4096 / 1.45 10.63; two-stream equal blocks 11.07.)
    //  * compute-bound (1-byte output): normal segments, ~16 equal row blocks of at least
    //    half a wave alternating over two compute streams (consecutive blocks overlap), so
    //    only the last block's copy is exposed.
    const size_t elem = out_elem(out_kind);
    const bool d2h_bound = double(elem) * 17.5 > 0.057 * double(W) * double(r);
    size_t Ss = d2h_bound ? std::max<size_t>(1024, 4 * size_t(W)) : S;
    if (const char* e = std::getenv("AP_STREAM_S")) Ss = std::max<size_t>(2 * W, std::strtoull(e, nullptr, 10));   // tuning
    double growth = AP_STREAM_GROWTH;
    if (const char* e = std::getenv("AP_STREAM_GROWTH")) growth = std::max(1.0, std::atof(e));   // tuning
    Ss = std::min(Ss, S);
    Ss = std::max<size_t>((Ss + salign - 1) / salign * salign, salign);
    const size_t nseg_s = (out_cols_eff + Ss - 1) / Ss;
    size_t blk_g0[ap_ctx::kMaxBlocks + 1];
    size_t nblk = 0;
    if (d2h_bound) {
      const size_t wave_groups = std::max<size_t>(1, total_warps / nseg_s);   // pair groups per wave
      size_t g = 0;
      double waves = 1.0;
      while (g < ngroups && nblk < size_t(ap_ctx::kMaxBlocks)) {
        blk_g0[nblk++] = g;
        const size_t wk = std::max<size_t>(1, size_t(waves + 0.5));
        g = (nblk == size_t(ap_ctx::kMaxBlocks)) ? ngroups : std::min(ngroups, g + wk * wave_groups);
        waves *= growth;
      }
    } else {
      const size_t nb = std::min<size_t>({std::max<size_t>(ntasks / std::max<size_t>(total_warps / 2, 1), 1),
                                          std::max<size_t>(ngroups, 1), 16});
      const size_t gpb = (ngroups + nb - 1) / nb;
      for (size_t g = 0; g < ngroups; g += gpb) blk_g0[nblk++] = g;
    }
    blk_g0[nblk] = ngroups;
    if (!d2h_bound) {
      CK(cudaEventRecord(c->ev_join, st));                    // code streams ready
      CK(cudaStreamWaitEvent(c->stream_b, c->ev_join, 0));
    }
    for (size_t k = 0; k < nblk; ++k) {
      const size_t r0 = std::min(nrows, blk_g0[k] * 2 * G), r1 = std::min(nrows, blk_g0[k + 1] * 2 * G);
      cudaStream_t sk = (!d2h_bound && (k & 1)) ? c->stream_b : st;
      apk::CombParams pk = p;
      pk.xcode = c->d_xcode + r0 * h;
      pk.xlen = uint32_t(mx - r0 * h);
      pk.rows = uint32_t(r1 - r0);
      pk.row_global0 = uint32_t(row_global0 + r0);
      pk.out = p.out + (out_kind == 0 ? r0 * cols : 0);
      pk.out8 = p.out8 + (out_kind == 0 ? 0 : r0 * cols);
      pk.S = uint32_t(Ss);
      pk.nseg = uint32_t(nseg_s);
      const size_t tk = ((r1 - r0 + 1) / 2 + G - 1) / G * nseg_s;
      const size_t gk = std::min<size_t>((tk + wpc - 1) / wpc, size_t(c->sms) * per_sm);
      pk.task_counter = c->d_tasks + k;
      fn<<<dim3(unsigned(gk)), dim3(wpc * 32), sh.smem, sk>>>(pk);
      CK(cudaGetLastError());
      CK(cudaEventRecord(c->ev_blk[k], sk));
      c->last_launches += 1;
    }
    // every block's kernel is enqueued before the first copy: a copy to pageable host memory
    // returns only when it is done, which would otherwise hold back the next block's launch
    std::vector<CopyRange> ranges;
    for (size_t k = 0; k < nblk; ++k) {
      const size_t r0 = std::min(nrows, blk_g0[k] * 2 * G), r1 = std::min(nrows, blk_g0[k + 1] * 2 * G);
      ranges.push_back({static_cast<char*>(host_out) + r0 * cols * elem,
                        static_cast<const char*>(d_out) + r0 * cols * elem, (r1 - r0) * cols * elem, c->ev_blk[k]});
    }
    if ((rc = copy_out(c, ranges))) return rc;
    if (!d2h_bound) {
      CK(cudaEventRecord(c->ev_join, c->stream_b));           // join the second stream
      CK(cudaStreamWaitEvent(st, c->ev_join, 0));
    }
    CK(cudaEventRecord(c->ev1, st));
    if (std::getenv("AP_TRACE")) {
      for (size_t k = 0; k < nblk; ++k) CK(cudaEventRecord(c->ev_cp[k], c->stream_copy));
      CK(cudaStreamSynchronize(c->stream_copy));
      for (size_t k = 0; k < nblk; ++k) {
        float tb = 0.f;
        cudaEventElapsedTime(&tb, c->ev0, c->ev_blk[k]);
        std::fprintf(stderr, "[ap trace] block %zu groups [%zu,%zu) comb done %.3f ms\n", k, blk_g0[k], blk_g0[k + 1], tb);
      }
      float tc = 0.f;
      cudaEventElapsedTime(&tc, c->ev0, c->ev_cp[nblk - 1]);
      std::fprintf(stderr, "[ap trace] copies done %.3f ms (nseg %zu, S %zu)\n", tc, nseg_s, Ss);
    }
    if (speculate) CK(cudaMemcpyAsync(c->h_small, c->d_small, 12, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(c->stream_copy));
    CK(cudaStreamSynchronize(st));
    if (spec_failed())
      return run_device(c, d_x, mx, d_y, n, cfg, nrows, row_global0, dense, d_out, st, nrec_out, total_out,
                        cap, out_kind, host_out, false, count_only);
    return AP_OK;
  }
  fn<<<dim3(unsigned(grid)), dim3(wpc * 32), sh.smem, st>>>(p);
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev1, st));
  c->last_launches += 1;

  if (!dense) {
    // deterministic row-major placement: exclusive scan of (row, segment) counts
    // (64-bit offsets and total: lists past 2^32 cells count exactly)
    if ((rc = scan_counts(c, nrows * p.seg_stride, st))) return rc;
    if (speculate) CK(cudaMemcpyAsync(c->h_small, c->d_small, 12, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (spec_failed())
      return run_device(c, d_x, mx, d_y, n, cfg, nrows, row_global0, dense, d_out, st, nrec_out, total_out,
                        cap, out_kind, host_out, false, count_only);
    const size_t nrec = c->h_cursor[0];
    const size_t total = c->h_cursor[1];
    if (nrec != total) return fail(AP_CUDA, "threshold bookkeeping mismatch (%zu staged vs %zu counted)", nrec, total);
    if (nrec > c->cap_stage && !count_only) {
      // staging overflowed: grow to the exact size and recompute (rare)
      if ((rc = grow(&c->d_stage, &c->cap_stage, nrec))) return rc;
      p.stage = c->d_stage;
      p.stage_cap = c->cap_stage;
      CK(cudaMemsetAsync(c->d_cursor, 0, sizeof(unsigned long long), st));
      p.task_counter = c->d_tasks + 63;
      fn<<<dim3(unsigned(grid)), dim3(wpc * 32), sh.smem, st>>>(p);
      CK(cudaGetLastError());
      c->last_launches += 1;
    }
    c->list.nrec = count_only ? 0 : nrec;
    c->list.seg_stride = p.seg_stride;
    c->list.S = uint32_t(S);
    c->list.S2 = p.S2;
    c->list.split_row = uint32_t(split_row);
    c->list.r = r;
    c->list.row_global0 = uint32_t(row_global0);
    *nrec_out = nrec;
    *total_out = total;
  } else {
    // a dense device call completes before returning (a speculative plan is verified here)
    if (speculate) CK(cudaMemcpyAsync(c->h_small, c->d_small, 12, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (spec_failed())
      return run_device(c, d_x, mx, d_y, n, cfg, nrows, row_global0, dense, d_out, st, nrec_out, total_out,
                        cap, out_kind, host_out, false, count_only);
  }
  return AP_OK;
}

// Place the list staged by the last thresholded run_device on c in row-major order
// (apply_threshold, scoring.cpp:30-39): the first min(total, cap) cells into the device
// arrays (rows/cols/halves, or ap_cell records when cells != nullptr).  Enqueued on st.
int place_list(ap_ctx* c, cudaStream_t st, uint32_t* rows, uint32_t* cols, uint16_t* halves, int32_t* halves32,
               apk::CellRec* cells, size_t cap) {
  const ap_ctx::ListState& l = c->list;
  if (!l.nrec || !cap) return AP_OK;
  const size_t blocks = std::min<size_t>((l.nrec + 255) / 256, size_t(c->sms) * 16);
  apk::place_kernel<<<unsigned(blocks), 256, 0, st>>>(c->d_stage, l.nrec, c->d_offs, l.seg_stride, l.S, l.S2,
                                                        l.split_row, l.r, l.row_global0, rows, cols, halves,
                                                        halves32, cells, cap);
  CK(cudaGetLastError());
  c->last_launches += 1;
  return AP_OK;
}

// Half-unit scores lie in [0, 2w] (r = 1) or [0, 2w] with w <= 32767 (r = 2, W <= 65534), so
// the uint16 entry points hold every score except LCS plots with w > 32767 (sea16 allows up to
// 65534): those need the int32 forms (ap_plot_dense_i32, ap_plot_threshold_into / _cells).
int check_u16(const ap_config* cfg) {
  if (cfg && 2 * cfg->window_w > 65535 && cfg->blowup_r == 1)
    return fail(AP_CONFIG, "scores of w = %zu reach %zu half-units, beyond uint16: use the int32 entry points",
                size_t(cfg->window_w), size_t(2 * cfg->window_w));
  return AP_OK;
}

}  // namespace

extern "C" {

int ap_grid_dims(size_t m, size_t n, size_t w, size_t h, size_t* rows, size_t* cols) {
  if (!rows || !cols) return fail(AP_INVALID, "null output pointer");
  if (w == 0 || h == 0) return fail(AP_CONFIG, "window and step must be positive");
  if (w > m || w > n)
    return fail(AP_EMPTY, "no window of size %zu fits inputs of lengths %zu and %zu", w, m, n);
  *rows = (m - w) / h + 1;
  *cols = n - w + 1;
  return AP_OK;
}

int ap_validate(size_t m, size_t n, const ap_config* cfg) { return check_cfg(m, n, cfg); }

const char* ap_last_error(void) { return g_err.c_str(); }

int ap_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int ap_ctx_create(int device, ap_ctx** out) {
  if (!out) return fail(AP_INVALID, "null ctx pointer");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return fail(AP_NODEV, "no CUDA device available (the engine has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(AP_NODEV, "device %d not present", device);
  DevGuard dg(device);
  ap_ctx* c = new ap_ctx();
  c->device = device;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  c->sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->stream_copy, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->stream_b, cudaStreamNonBlocking));
  for (auto& e : c->ev_blk) CK(cudaEventCreate(&e));
  for (auto& e : c->ev_cp) CK(cudaEventCreate(&e));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CK(cudaEventCreate(&c->ev0));
  CK(cudaEventCreate(&c->ev1));
  CK(cudaMalloc(&c->d_small, 64));
  CK(cudaMalloc(&c->d_tasks, 64 * sizeof(uint32_t)));
  CK(cudaMallocHost(&c->h_small, 64));
  CK(cudaMalloc(&c->d_map, 256));
  CK(cudaMalloc(&c->d_cursor, 16));
  CK(cudaMallocHost(&c->h_cursor, 32));
  {
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    CK(cudaMemPoolCreate(&c->pool, &pp));
    uint64_t keep = ~uint64_t(0);   // keep freed list buffers for the next call
    CK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = c;
  return AP_OK;
}

int ap_ctx_destroy(ap_ctx* c) {
  if (!c) return AP_OK;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto& p : g_ctx)
      if (p == c) p = nullptr;
  }
  DevGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  for (void* p : {(void*)c->d_x, (void*)c->d_y, (void*)c->d_xcode, (void*)c->d_ycode, (void*)c->d_ycol, (void*)c->d_map,
                  (void*)c->d_small, (void*)c->d_tasks, (void*)c->d_out, (void*)c->d_stage, (void*)c->d_cursor,
                  (void*)c->d_segc, (void*)c->d_offs, (void*)c->d_tsum, (void*)c->d_wkeys, (void*)c->d_wok,
                  (void*)c->d_out16})
    if (p) cudaFree(p);
  if (c->pool) {
    cudaStreamSynchronize(c->stream_copy);
    cudaMemPoolDestroy(c->pool);
  }
  if (c->h_bounce) cudaFreeHost(c->h_bounce);
  for (int k = 0; k < c->bounce_slots; ++k) cudaEventDestroy(c->ev_bounce[k]);
  if (c->h_small) cudaFreeHost(c->h_small);
  if (c->h_cursor) cudaFreeHost(c->h_cursor);
  cudaStreamSynchronize(c->stream_copy);
  cudaStreamSynchronize(c->stream_b);
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  for (auto& e : c->ev_blk) cudaEventDestroy(e);
  for (auto& e : c->ev_cp) cudaEventDestroy(e);
  cudaEventDestroy(c->ev_join);
  cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->stream_copy);
  cudaStreamDestroy(c->stream_b);
  delete c;
  return AP_OK;
}

float ap_ctx_last_kernel_ms(ap_ctx* c) {
  if (!c) return -1.f;
  DevGuard dg(c->device);
  float ms = -1.f;
  if (cudaEventElapsedTime(&ms, c->ev0, c->ev1) != cudaSuccess) {
    cudaGetLastError();
    return -1.f;
  }
  return ms;
}

int ap_ctx_last_launches(ap_ctx* c) { return c ? c->last_launches : 0; }

const char* ap_ctx_last_kernel(ap_ctx* c) { return c ? c->last_kernel : ""; }

int ap_ctx_plot_dense_device(ap_ctx* c, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                             const ap_config* cfg, uint16_t* d_out, void* stream) {
  if (!c || !d_x || !d_y || !d_out) return fail(AP_INVALID, "null argument");
  int rc = check_cfg(m, n, cfg);
  if (rc || (rc = check_u16(cfg))) return rc;
  size_t rows, cols, rb, re;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, &cols);
  if ((rc = row_range(rows, cfg, &rb, &re))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  DevGuard dg(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const size_t off = rb * cfg->step_h;
  return run_device(c, d_x + off, m - off, d_y, n, cfg, re - rb, rb, true, d_out, st, nullptr, nullptr, 0);
}

int ap_ctx_plot_dense_u8_device(ap_ctx* c, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                                const ap_config* cfg, uint8_t* d_out, void* stream) {
  if (!c || !d_x || !d_y || !d_out) return fail(AP_INVALID, "null argument");
  int rc = check_cfg(m, n, cfg);
  if (rc) return rc;
  if (cfg->window_w > 127)
    return fail(AP_CONFIG, "uint8 half-units need w <= 127 (scores up to 2w), got w = %zu", size_t(cfg->window_w));
  size_t rows, cols, rb, re;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, &cols);
  if ((rc = row_range(rows, cfg, &rb, &re))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  DevGuard dg(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const size_t off = rb * cfg->step_h;
  return run_device(c, d_x + off, m - off, d_y, n, cfg, re - rb, rb, true, d_out, st, nullptr, nullptr, 0, 2);
}

int ap_ctx_plot_dense_i32_device(ap_ctx* c, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                                 const ap_config* cfg, int32_t* d_out, void* stream) {
  if (!c || !d_x || !d_y || !d_out) return fail(AP_INVALID, "null argument");
  int rc = check_cfg(m, n, cfg);
  if (rc) return rc;
  size_t rows, cols, rb, re;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, &cols);
  if ((rc = row_range(rows, cfg, &rb, &re))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  DevGuard dg(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const size_t off = rb * cfg->step_h;
  return run_device(c, d_x + off, m - off, d_y, n, cfg, re - rb, rb, true, d_out, st, nullptr, nullptr, 0, 3);
}

int ap_ctx_plot_pgm_device(ap_ctx* c, const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n,
                           const ap_config* cfg, uint8_t* d_pixels, void* stream) {
  if (!c || !d_x || !d_y || !d_pixels) return fail(AP_INVALID, "null argument");
  int rc = check_cfg(m, n, cfg);
  if (rc) return rc;
  size_t rows, cols, rb, re;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, &cols);
  if ((rc = row_range(rows, cfg, &rb, &re))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  DevGuard dg(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const size_t off = rb * cfg->step_h;
  return run_device(c, d_x + off, m - off, d_y, n, cfg, re - rb, rb, true, d_pixels, st, nullptr, nullptr, 0,
                    1);
}

int ap_ctx_plot_threshold_device(ap_ctx* c, const uint8_t* d_x, size_t m, const uint8_t* d_y,
                                 size_t n, const ap_config* cfg, uint64_t* count, uint32_t* d_rows,
                                 uint32_t* d_cols, uint16_t* d_halves, size_t cap, void* stream) {
  if (!c || !d_x || !d_y || !count) return fail(AP_INVALID, "null argument");
  if (cap && (!d_rows || !d_cols || !d_halves)) return fail(AP_INVALID, "null output arrays");
  int rc = check_cfg(m, n, cfg);
  if (rc || (rc = check_u16(cfg))) return rc;
  size_t rows, cols, rb, re;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, &cols);
  if ((rc = row_range(rows, cfg, &rb, &re))) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  DevGuard dg(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const size_t off = rb * cfg->step_h;
  size_t nrec = 0, total = 0;
  rc = run_device(c, d_x + off, m - off, d_y, n, cfg, re - rb, rb, false, nullptr, st, &nrec, &total, cap, 0, nullptr,
                  true, cap == 0);
  if (rc) return rc;
  if ((rc = place_list(c, st, d_rows, d_cols, d_halves, nullptr, nullptr, cap))) return rc;
  CK(cudaStreamSynchronize(st));
  *count = total;
  if (total > cap) return fail(AP_CAPACITY, "%zu cells pass the threshold, capacity %zu", total, cap);
  return AP_OK;
}

}  // extern "C"

namespace {

bool has_sentinel(const uint8_t* p, size_t n) { return std::memchr(p, 0, n) != nullptr; }

static_assert(sizeof(ap_cell) == sizeof(apk::CellRec) && offsetof(ap_cell, half) == offsetof(apk::CellRec, half),
              "ap_cell and the placement kernel's record must share a layout");

// One device's contiguous block of grid rows [r0, r1).
struct Shard {
  int dev = 0;
  size_t r0 = 0, r1 = 0;
  ap_ctx* ctx = nullptr;
  size_t total = 0;        // hits of this shard (thresholded runs)
  size_t kept = 0;         // entries placed into `list` (<= total)
  char* list = nullptr;    // the shard's row-major list in device memory (ctx pool)
  int rc = AP_OK;
  std::string err;
};

// Shared prologue of the host API: validation before any device work (runner.cpp:81 order),
// the row range, and the row shards over devices.
int plan_shards(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg, size_t* rb,
                size_t* re, size_t* cols, std::vector<Shard>* sh) {
  if (!x || !y || !cfg) return fail(AP_INVALID, "null argument");
  int rc = check_cfg(m, n, cfg);
  if (rc) return rc;
  if (has_sentinel(x, m) || has_sentinel(y, n))
    return fail(AP_CONFIG, "sequence contains the reserved sentinel code 0");
  size_t rows;
  ap_grid_dims(m, n, cfg->window_w, cfg->step_h, &rows, cols);
  if ((rc = row_range(rows, cfg, rb, re))) return rc;
  const int ndev_real = ap_device_count();
  // AP_SHARDS_PER_DEVICE=k (testing): let one physical GPU stand in for k shard
  // devices, so the multi-device split/gather path runs on a single-GPU box.
  int per_dev = 1;
  if (const char* env = std::getenv("AP_SHARDS_PER_DEVICE")) per_dev = std::max(1, std::atoi(env));
  const int ndev_avail = ndev_real * per_dev;
  if (ndev_avail <= 0) return fail(AP_NODEV, "no CUDA device available (the engine has no CPU fallback)");
  int ndev = cfg->n_devices <= 1 ? 1 : std::min(cfg->n_devices, ndev_avail);
  int cur = 0;
  cudaGetDevice(&cur);
  const size_t nr = *re - *rb;
  if (size_t(ndev) > nr) ndev = int(std::max<size_t>(nr, 1));
  sh->assign(ndev, Shard());
  for (int d = 0; d < ndev; ++d) {
    Shard& s = (*sh)[d];
    s.dev = ndev == 1 ? cur : d % std::max(ndev_real, 1);
    s.r0 = *rb + nr * d / ndev;
    s.r1 = *rb + nr * (d + 1) / ndev;
    if ((rc = get_ctx(s.dev, &s.ctx))) return rc;
  }
  return AP_OK;
}

// Run fn(shard) for every shard, one host thread per shard when there are several
// (so devices overlap); returns the first failure.
template <typename F>
int for_shards(std::vector<Shard>& sh, F fn) {
  if (sh.size() == 1) {
    sh[0].rc = fn(sh[0]);
    if (sh[0].rc) sh[0].err = g_err;
  } else {
    std::vector<std::thread> th;
    for (auto& s : sh)
      th.emplace_back([&fn, &s]() {
        s.rc = fn(s);
        if (s.rc) s.err = g_err;
      });
    for (auto& t : th) t.join();
  }
  for (auto& s : sh)
    if (s.rc) return fail(s.rc, "%s", s.err.c_str());
  return AP_OK;
}

// H2D of a shard's x slice (its rows plus the w-1 halo) and of y into the context.
int upload_shard(ap_ctx* c, const Shard& s, const uint8_t* x, const uint8_t* y, size_t n, const ap_config* cfg,
                 cudaStream_t st, size_t* mx) {
  const size_t x0 = s.r0 * cfg->step_h, x1 = (s.r1 - 1) * cfg->step_h + cfg->window_w;
  int q;
  if ((q = grow(&c->d_x, &c->cap_x, x1 - x0))) return q;
  if ((q = grow(&c->d_y, &c->cap_y, n))) return q;
  CK(cudaMemcpyAsync(c->d_x, x + x0, x1 - x0, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_y, y, n, cudaMemcpyHostToDevice, st));
  *mx = x1 - x0;
  return AP_OK;
}

// Dense host API body: every shard streams its row block straight to its offset in out.
int host_dense(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg, void* out,
               int out_kind) {
  size_t rb, re, cols;
  std::vector<Shard> sh;
  int rc = plan_shards(x, m, y, n, cfg, &rb, &re, &cols, &sh);
  if (rc) return rc;
  if (!out && re > rb) return fail(AP_INVALID, "null output");
  const size_t elem = out_elem(out_kind);
  return for_shards(sh, [&](Shard& s) -> int {
    const size_t nrows = s.r1 - s.r0;
    if (nrows == 0) return AP_OK;
    ap_ctx* c = s.ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DevGuard dg(c->device);
    cudaStream_t st = c->stream;
    size_t mx = 0;
    int q;
    if ((q = upload_shard(c, s, x, y, n, cfg, st, &mx))) return q;
    if ((q = grow(&c->d_out, &c->cap_out, nrows * cols * (out_kind == 3 ? 2 : 1)))) return q;
    if ((q = run_device(c, c->d_x, mx, c->d_y, n, cfg, nrows, s.r0, true, c->d_out, st, nullptr, nullptr, 0,
                        out_kind, static_cast<char*>(out) + (s.r0 - rb) * cols * elem)))
      return q;
    CK(cudaStreamSynchronize(st));
    return AP_OK;
  });
}

// Where the thresholded host API delivers the list.
struct ListDest {
  uint32_t* rows = nullptr;
  uint32_t* cols = nullptr;
  uint16_t* halves = nullptr;
  int32_t* halves32 = nullptr;         // callback form: int32 scores
  ap_cell* cells = nullptr;            // array-of-structs form instead of rows / cols / halves
  size_t cap = 0;
  ap_list_alloc_fn alloc = nullptr;    // callback form: called once with the total
  void* user = nullptr;
};

// Thresholded host API body (apply_threshold(compute_plot(...)), scoring.cpp:30-39, fused).
// One comb per shard: phase 1 combs each shard and places its list in device memory owned by
// the call (the context lock is released after it, so concurrent calls cannot overwrite it);
// phase 2 gathers the per-shard counts into global offsets -- the path's only cross-device
// step -- and copies each shard's list straight to its offset in the caller's buffer.
int host_list(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg, uint64_t* count,
              ListDest dst) {
  size_t rb, re, cols;
  std::vector<Shard> sh;
  int rc = plan_shards(x, m, y, n, cfg, &rb, &re, &cols, &sh);
  if (rc) return rc;
  const size_t esz = dst.cells ? sizeof(ap_cell) : 2 * sizeof(uint32_t) + (dst.alloc ? 4 : 2);
  // entries a shard may need: its list starts at a global offset >= 0
  const size_t cap_any = dst.alloc ? ~size_t(0) : dst.cap;
  auto free_lists = [&]() {
    for (auto& s : sh)
      if (s.list) {
        DevGuard dg(s.ctx->device);
        cudaFreeAsync(s.list, s.ctx->stream);
        s.list = nullptr;
      }
  };
  rc = for_shards(sh, [&](Shard& s) -> int {
    const size_t nrows = s.r1 - s.r0;
    if (nrows == 0) return AP_OK;
    ap_ctx* c = s.ctx;
    std::lock_guard<std::mutex> lk(c->mu);
    DevGuard dg(c->device);
    cudaStream_t st = c->stream;
    size_t mx = 0, nrec = 0, total = 0;
    int q;
    if ((q = upload_shard(c, s, x, y, n, cfg, st, &mx))) return q;
    if ((q = run_device(c, c->d_x, mx, c->d_y, n, cfg, nrows, s.r0, false, nullptr, st, &nrec, &total, 0, 0, nullptr,
                        true, cap_any == 0)))
      return q;
    s.total = total;
    s.kept = std::min(total, cap_any);
    if (s.kept) {
      CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&s.list), s.kept * esz, c->pool, st));
      uint32_t* lr = reinterpret_cast<uint32_t*>(s.list);
      if ((q = place_list(c, st, dst.cells ? nullptr : lr, dst.cells ? nullptr : lr + s.kept,
                          dst.cells || dst.alloc ? nullptr : reinterpret_cast<uint16_t*>(lr + 2 * s.kept),
                          dst.alloc ? reinterpret_cast<int32_t*>(lr + 2 * s.kept) : nullptr,
                          dst.cells ? reinterpret_cast<apk::CellRec*>(s.list) : nullptr, s.kept)))
        return q;
    }
    CK(cudaStreamSynchronize(st));
    return AP_OK;
  });
  if (rc) {
    free_lists();
    return rc;
  }
  // phase 2: global offsets (exclusive prefix of the shard counts, in row order)
  std::vector<uint64_t> offs(sh.size());
  uint64_t total = 0;
  for (size_t d = 0; d < sh.size(); ++d) {
    offs[d] = total;
    total += sh[d].total;
  }
  if (count) *count = total;
  size_t cap = dst.cap;
  if (dst.alloc) {
    if (dst.alloc(dst.user, total, &dst.rows, &dst.cols, &dst.halves32) != 0) {
      free_lists();
      return fail(AP_INVALID, "list allocation callback failed for %llu cells", (unsigned long long)total);
    }
    if (total && (!dst.rows || !dst.cols || !dst.halves32)) {
      free_lists();
      return fail(AP_INVALID, "list allocation callback returned null arrays");
    }
    cap = total;
  }
  rc = for_shards(sh, [&](Shard& s) -> int {
    const size_t d = size_t(&s - sh.data());
    if (offs[d] >= cap || !s.kept) return AP_OK;
    const size_t k = std::min<size_t>(s.kept, cap - offs[d]);
    DevGuard dg(s.ctx->device);
    if (dst.cells) {
      CK(cudaMemcpy(dst.cells + offs[d], s.list, k * sizeof(ap_cell), cudaMemcpyDeviceToHost));
    } else {
      const uint32_t* lr = reinterpret_cast<const uint32_t*>(s.list);
      CK(cudaMemcpy(dst.rows + offs[d], lr, k * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(dst.cols + offs[d], lr + s.kept, k * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      if (dst.alloc)
        CK(cudaMemcpy(dst.halves32 + offs[d], lr + 2 * s.kept, k * sizeof(int32_t), cudaMemcpyDeviceToHost));
      else
        CK(cudaMemcpy(dst.halves + offs[d], lr + 2 * s.kept, k * sizeof(uint16_t), cudaMemcpyDeviceToHost));
    }
    return AP_OK;
  });
  free_lists();
  if (rc) return rc;
  if (total > cap)
    return fail(AP_CAPACITY, "%llu cells pass the threshold, capacity %zu", (unsigned long long)total, cap);
  return AP_OK;
}

}  // namespace

extern "C" {

int ap_plot_dense(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                  uint16_t* out_half) {
  if (int rc = check_u16(cfg)) return rc;
  if (cfg && cfg->has_threshold) {
    ap_config c = *cfg;   // the dense grid is never filtered (compute_plot, runner.cpp:78-131)
    c.has_threshold = 0;
    return host_dense(x, m, y, n, &c, out_half, 0);
  }
  return host_dense(x, m, y, n, cfg, out_half, 0);
}

int ap_plot_dense_i32(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                      int32_t* out_half) {
  if (cfg && cfg->has_threshold) {
    ap_config c = *cfg;
    c.has_threshold = 0;
    return host_dense(x, m, y, n, &c, out_half, 3);
  }
  return host_dense(x, m, y, n, cfg, out_half, 3);
}

int ap_plot_pgm(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                uint8_t* pixels) {
  return host_dense(x, m, y, n, cfg, pixels, 1);
}

int ap_plot_dense_u8(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                     uint8_t* out_half) {
  if (cfg && cfg->window_w > 127)
    return fail(AP_CONFIG, "uint8 half-units need w <= 127 (scores up to 2w), got w = %zu", size_t(cfg->window_w));
  if (cfg && cfg->has_threshold) {
    ap_config c = *cfg;
    c.has_threshold = 0;
    return host_dense(x, m, y, n, &c, out_half, 2);
  }
  return host_dense(x, m, y, n, cfg, out_half, 2);
}

int ap_plot_threshold(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                      uint64_t* count, uint32_t* rows, uint32_t* cols, uint16_t* halves, size_t cap) {
  if (!count) return fail(AP_INVALID, "null count");
  if (cap && (!rows || !cols || !halves)) return fail(AP_INVALID, "null output arrays");
  if (!cfg || !cfg->has_threshold) return fail(AP_INVALID, "ap_plot_threshold needs has_threshold");
  if (int rc = check_u16(cfg)) return rc;
  ListDest d;
  d.rows = rows;
  d.cols = cols;
  d.halves = halves;
  d.cap = cap;
  return host_list(x, m, y, n, cfg, count, d);
}

int ap_plot_threshold_into(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                           ap_list_alloc_fn alloc, void* user, uint64_t* count) {
  if (!alloc) return fail(AP_INVALID, "null allocation callback");
  if (!cfg || !cfg->has_threshold) return fail(AP_INVALID, "ap_plot_threshold_into needs has_threshold");
  ListDest d;
  d.alloc = alloc;
  d.user = user;
  return host_list(x, m, y, n, cfg, count, d);
}

int ap_plot_threshold_cells(const uint8_t* x, size_t m, const uint8_t* y, size_t n, const ap_config* cfg,
                            uint64_t* count, ap_cell* cells, size_t cap) {
  if (!count) return fail(AP_INVALID, "null count");
  if (cap && !cells) return fail(AP_INVALID, "null output array");
  if (!cfg || !cfg->has_threshold) return fail(AP_INVALID, "ap_plot_threshold_cells needs has_threshold");
  ListDest d;
  d.cells = cells;
  d.cap = cap;
  return host_list(x, m, y, n, cfg, count, d);
}

}  // extern "C"
