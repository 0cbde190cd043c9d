// ap_wide_kernels.cuh — the large-window path: blown windows W = w*r above the packed
// kernels' 1024 (up to the reference sea16 bound W <= 65534, model.cpp:57-59,
// lane_kernel.cpp:117-123).
//
// The packed kernels (ap_kernels.cuh) hold a strip pair in one warp's registers with
// 16-bit start keys, which caps W at 32 lanes x 32 rows.  Here one CTA combs one strip:
//
//  * Keys are exact 32-bit starts (key = start column + 1 for top seaweeds, 0 for the
//    left boundary, seaweed_scalar.cpp:21-22), one strip per register: no rebasing, no
//    span limit.  Cell (seaweed_scalar.cpp:26-32, exchange iff match or start(V) > start(T)):
//        TM = T ^ (match ? 0x80000000 : 0)      (= T + INT_MIN for T < 2^31)
//        d  = max_s32(TM, V)                    seaweed leaving downwards
//        V' = V ^ T ^ d                         seaweed leaving to the right
//    with match from the codes on the FMA pipe: (x - y)^2 - 1 < 0 iff x == y.
//  * Rows: thread v of the CTA owns R consecutive rows of a band of HB = threads * R rows;
//    a strip of W rows is combed band by band (top padding rows never match, and a
//    never-matching row passes every top seaweed straight down, so padding is exact).
//    A band's bottom keys overwrite its top keys in place (keys[c]): column c's top is
//    read long before its bottom is written.
//  * Wavefront: lane l of warp w combs column s - l at its step s; seaweeds move lane to
//    lane by SHFL, warp to warp through a shared-memory ring with a two-chunk lag (warp w
//    combs its chunk k - 2w in macro step k; __syncthreads between macro steps).
//
// Window extraction (wide_extract_kernel) is two prefix sums instead of a heap
// (seaweed_scalar.cpp:65-99): with a(e) = [bottom seaweed at column e is countable, i.e.
// start(e) >= e - W + 1] and ok[st] = a(e) scattered at the seaweed's start,
//     count(0) = sum_{e < W} a(e),   count(K+1) = count(K) + a(K + W) - ok[K],
// LLCS(K) = W - count(K), reported for K = r * col and converted to half-units
// (runner.cpp:31-35, scoring.cpp:26-28).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apk {

constexpr int kWideRows = 16;       // rows per thread
constexpr int kWideChunk = 32;      // steps per macro step
constexpr int kWideRing = 128;      // warp-to-warp ring slots (columns)
constexpr int kWideMaxWarps = 32;
constexpr uint32_t kPadCode = 0x1FFu;   // x rows that never match (padding, bytes absent from y)
constexpr uint32_t kOffCode = 0x3FFu;   // y columns outside [0, N) (never match)

struct WideParams {
  const uint8_t* xcode;   // mapped x codes of the launch's first row (0xFF: absent from y)
  const uint8_t* ycode;   // effective ($-interleaved for r = 2) y codes, N entries
  int32_t* keys;          // [strips][N] start keys (scratch)
  uint8_t* ok;            // [strips][N] extraction flags (scratch)
  uint32_t strips;        // strips (grid rows) in this launch
  uint32_t h, w, r, W, N;
  uint32_t sent_code;     // $ code (r = 2)
  uint32_t bands, band_rows;   // bands per strip, rows per band (= threads * kWideRows)
  uint32_t tbl_codes;          // TBL kernel: table codes (the y alphabet, plus $ for r = 2)
  uint32_t rebase_at, rebase_by;   // packed kernel: relative-key bound and rebase step
  uint32_t cols;          // grid columns
  uint32_t row0;          // launch row offset within the call (output row = row0 + strip)
  uint32_t row_global0;   // global grid row of the call's row 0
  // dense output
  uint16_t* out;
  uint8_t* out8;
  int32_t* out32;
  uint32_t out_kind;      // 0 = u16 half-units, 1 = PGM pixels, 2 = u8 half-units, 3 = int32 half-units
  int32_t pgm_threshold;
  uint32_t has_pgm_threshold;
  // thresholded output (the packed kernels' staging format; one segment per row)
  uint32_t dense;
  int32_t t_half;
  uint4* stage;
  unsigned long long* cursor;
  unsigned long long stage_cap;
  uint32_t* seg_counts;   // [rows] hits per row
};

// One CTA per strip; blockDim.x = 32 * warps.
// TBL = true (alphabets of <= 8 codes, host-selected): 8-warp CTAs, several per SM, whose masks
// come from a per-band table M[code][quad][thread] of int32 words (INT_MIN on a match, 0
// otherwise; one LDS.128 per 4 rows, conflict-free); the cell is max(T + M, V) in one VIADDMNMX
// plus the LOP3 -- 2 ALU ops per cell instead of 3 ALU + 2 FMA with computed masks.
template <bool TBL>
__global__ void __launch_bounds__(TBL ? 256 : 1024, 1) wide_comb_kernel(const WideParams p) {
  // dynamic shared memory: TBL's table [codes][kWideRows / 4][threads] uint4, then the
  // warp-to-warp rings [warps][kWideRing]
  extern __shared__ __align__(16) unsigned char wsm[];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  int32_t* ring = reinterpret_cast<int32_t*>(wsm + (TBL ? size_t(p.tbl_codes) * kWideRows * 4 * blockDim.x : 0));
  const uint32_t strip = blockIdx.x;
  const uint32_t N = p.N;
  int32_t* keys = p.keys + size_t(strip) * N;
  const uint8_t* xrow = p.xcode + size_t(strip) * p.h;
  const uint32_t rshift = p.r - 1;
  const uint32_t nch = (N + 31 + kWideChunk - 1) / kWideChunk;
  const uint32_t nmacro = nch + 2 * (nwarps - 1);
  const uint32_t pad = p.bands * p.band_rows - p.W;   // never-matching rows above the strip
  uint4* tb4 = reinterpret_cast<uint4*>(wsm);
  constexpr int QW = kWideRows / 4;
  const uint32_t code_stride = uint32_t(QW) * blockDim.x;   // uint4 per code

  for (uint32_t b = 0; b < p.bands; ++b) {
    // x codes of this thread's rows
    int32_t xr[kWideRows];
#pragma unroll
    for (int rho = 0; rho < kWideRows; ++rho) {
      const int32_t i = int32_t(b * p.band_rows + tid * kWideRows + rho) - int32_t(pad);   // blown strip row
      uint32_t code = kPadCode;
      if (i >= 0) {
        if (p.r == 2 && !(i & 1)) {
          code = p.sent_code;
        } else {
          code = xrow[uint32_t(i) >> rshift];
          if (code == 0xFFu) code = kPadCode;
        }
      }
      xr[rho] = int32_t(code);
    }
    __syncthreads();    // the previous band's last bottom keys are written, its table reads done
    if constexpr (TBL) {
      for (uint32_t a = 0; a < p.tbl_codes; ++a)
#pragma unroll
        for (int q = 0; q < QW; ++q) {
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) wv[k] = xr[4 * q + k] == int32_t(a) ? 0x80000000u : 0u;
          tb4[a * code_stride + uint32_t(q) * blockDim.x + tid] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      __syncthreads();
    }
    int32_t V[kWideRows];
#pragma unroll
    for (int rho = 0; rho < kWideRows; ++rho) V[rho] = 0;   // left-boundary seaweeds
    int32_t tout = 0;   // seaweed leaving this thread's bottom row at the previous step

    for (uint32_t k = 0; k < nmacro; ++k) {
      const int32_t lc = int32_t(k) - 2 * int32_t(warp);
      if (lc >= 0 && uint32_t(lc) < nch) {
        for (int u = 0; u < kWideChunk; ++u) {
          const int32_t s = lc * kWideChunk + u;          // this warp's local step
          const int32_t c = s - int32_t(lane);            // column of this lane
          const bool valid = c >= 0 && c < int32_t(N);
          const int32_t yc = valid ? int32_t(__ldg(p.ycode + c)) : int32_t(kOffCode);
          const int32_t sh = __shfl_up_sync(0xFFFFFFFFu, tout, 1);
          int32_t t = sh;
          if (lane == 0) {
            // column s enters this warp: the strip's top (band 0: fresh key s + 1), the previous
            // band's bottom (keys[s]) or the warp above's bottom lane (ring)
            if (s < int32_t(N)) {
              t = warp == 0 ? (b == 0 ? s + 1 : keys[s]) : ring[(warp - 1) * kWideRing + (s & (kWideRing - 1))];
            } else {
              t = 0;
            }
          }
          if constexpr (TBL) {
            // off-grid columns (c outside [0, N)) read code 0's words: t and V are still 0 there, so
            // max(0 + M, 0) = 0 whatever M is
            const uint4* tq = tb4 + uint32_t(valid ? yc : 0) * code_stride + tid;
#pragma unroll
            for (int q = 0; q < QW; ++q) {
              const uint4 m4 = tq[q * blockDim.x];
              const uint32_t m[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const int rho = 4 * q + kk;
                const int32_t d = __viaddmax_s32(t, int32_t(m[kk]), V[rho]);   // max(T + INT_MIN on a match, V)
                V[rho] = V[rho] ^ t ^ d;
                t = d;
              }
            }
          } else {
#pragma unroll
            for (int rho = 0; rho < kWideRows; ++rho) {
              int32_t dd, q1, tm, d;
              asm("mad.lo.s32 %0, %1, -1, %2;" : "=r"(dd) : "r"(yc), "r"(xr[rho]));   // x - y (FMA pipe)
              asm("mad.lo.s32 %0, %1, %1, -1;" : "=r"(q1) : "r"(dd));                 // < 0 iff x == y
              asm("lop3.b32 %0, %1, %2, 0x80000000, 0x78;" : "=r"(tm) : "r"(t), "r"(q1));   // t ^ (q1 & 0x80000000)
              d = max(tm, V[rho]);
              V[rho] = V[rho] ^ t ^ d;
              t = d;
            }
          }
          tout = t;
          if (lane == 31 && valid) {
            if (warp + 1 < nwarps) ring[warp * kWideRing + (c & (kWideRing - 1))] = t;
            else keys[c] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Packed variant (alphabets of <= 8 codes and W up to ~28K; host-selected): one CTA per strip
// PAIR (grid rows 2p, 2p+1 of the launch, same y columns) with both strips' 16-bit start keys in
// one register and the packed kernels' cell -- VIADDMNMX.S16x2 + LOP3 for two cells -- from table
// words carrying both strips' match bits (15, 31).  Keys are relative to a CTA-wide base and are
// rebased (saturating at 0) at macro-step boundaries by every thread at once, so all keys in
// flight (registers, the warp-to-warp ring) shift together; p.rebase_by keeps every seaweed a
// later window can count unsaturated (host: by = 0x7000 - W - 64 * warps - 64).  The bottom keys
// leave as absolute int32 starts (+1) per strip, as the 32-bit kernel writes them.
__global__ void __launch_bounds__(256, 1) wide2_comb_kernel(const WideParams p) {
  extern __shared__ __align__(16) unsigned char wsm[];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  const uint32_t sa = 2 * blockIdx.x, sb = sa + 1;
  const bool has_b = sb < p.strips;
  const uint32_t N = p.N;
  int32_t* keys_a = p.keys + size_t(sa) * N;
  int32_t* keys_b = p.keys + size_t(has_b ? sb : sa) * N;
  const uint8_t* xa_row = p.xcode + size_t(sa) * p.h;
  const uint8_t* xb_row = p.xcode + size_t(has_b ? sb : sa) * p.h;
  const uint32_t rshift = p.r - 1;
  const uint32_t nch = (N + 31 + kWideChunk - 1) / kWideChunk;
  const uint32_t nmacro = nch + 2 * (nwarps - 1);
  const uint32_t pad = p.bands * p.band_rows - p.W;
  constexpr int QW = kWideRows / 4;
  uint4* tb4 = reinterpret_cast<uint4*>(wsm);
  const uint32_t code_stride = uint32_t(QW) * blockDim.x;
  uint32_t* ring = reinterpret_cast<uint32_t*>(wsm + size_t(p.tbl_codes) * kWideRows * 4 * blockDim.x);
  const uint32_t by2 = p.rebase_by * 0x00010001u;

  for (uint32_t b = 0; b < p.bands; ++b) {
    uint32_t xa[kWideRows], xb[kWideRows];
#pragma unroll
    for (int rho = 0; rho < kWideRows; ++rho) {
      const int32_t i = int32_t(b * p.band_rows + tid * kWideRows + rho) - int32_t(pad);
      uint32_t ca = kPadCode, cb = kPadCode;
      if (i >= 0) {
        if (p.r == 2 && !(i & 1)) {
          ca = p.sent_code;
          cb = has_b ? p.sent_code : kPadCode;
        } else {
          ca = xa_row[uint32_t(i) >> rshift];
          cb = has_b ? xb_row[uint32_t(i) >> rshift] : kPadCode;
          if (ca == 0xFFu) ca = kPadCode;
          if (cb == 0xFFu) cb = kPadCode;
        }
      }
      xa[rho] = ca;
      xb[rho] = cb;
    }
    __syncthreads();   // the previous band's bottom keys are written, its table reads done
    for (uint32_t a = 0; a < p.tbl_codes; ++a)
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        uint32_t wv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          wv[k] = (xa[4 * q + k] == a ? 0x00008000u : 0u) | (xb[4 * q + k] == a ? 0x80000000u : 0u);
        tb4[a * code_stride + uint32_t(q) * blockDim.x + tid] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    __syncthreads();
    uint32_t V[kWideRows];
#pragma unroll
    for (int rho = 0; rho < kWideRows; ++rho) V[rho] = 0u;
    uint32_t tout = 0u;
    int32_t kbase = 0;   // key = absolute start + 1 - kbase (0: left boundary or saturated)

    for (uint32_t k = 0; k < nmacro; ++k) {
      if (int32_t(32 * (k + 2)) - kbase >= int32_t(p.rebase_at)) {   // uniform over the CTA
#pragma unroll
        for (int rho = 0; rho < kWideRows; ++rho) V[rho] = __vmaxu2(V[rho], by2) - by2;
        tout = __vmaxu2(tout, by2) - by2;
        for (uint32_t q = tid; q < nwarps * kWideRing; q += blockDim.x) ring[q] = __vmaxu2(ring[q], by2) - by2;
        kbase += int32_t(p.rebase_by);
        __syncthreads();
      }
      const int32_t lc = int32_t(k) - 2 * int32_t(warp);
      if (lc >= 0 && uint32_t(lc) < nch) {
        // branch-free per step: codes by clamped loads (the stream has >= 256 pad bytes) and a
        // select; the column entering this warp is formed by every lane (warp-uniform branches,
        // broadcast loads) and taken by lane 0 with one select
        auto code_at = [&](int32_t cc) -> uint32_t {
          const uint32_t v = uint32_t(__ldg(p.ycode + min(max(cc, 0), int32_t(N))));
          return cc >= 0 && cc < int32_t(N) ? v : 0u;
        };
        const int32_t c0 = lc * kWideChunk - int32_t(lane);
        uint32_t yc_next = code_at(c0 + 1);
        uint4 mq[QW];
        {
          const uint4* tq = tb4 + code_at(c0) * code_stride + tid;
#pragma unroll
          for (int q = 0; q < QW; ++q) mq[q] = tq[q * blockDim.x];
        }
        const uint32_t* ring_in = ring + (warp ? warp - 1 : 0) * kWideRing;
        uint32_t* ring_out = ring + warp * kWideRing;
        const bool last_warp = warp + 1 == nwarps;
#pragma unroll 2
        for (int u = 0; u < kWideChunk; ++u) {
          const int32_t s = lc * kWideChunk + u;
          const int32_t c = s - int32_t(lane);
          const bool valid = c >= 0 && c < int32_t(N);
          const uint32_t yc_after = code_at(c + 2);
          const uint32_t sh = __shfl_up_sync(0xFFFFFFFFu, tout, 1);
          uint32_t inj;                      // the seaweed pair entering this warp at column s
          if (warp != 0) {
            inj = ring_in[s & (kWideRing - 1)];
          } else if (b == 0) {
            inj = uint32_t(s + 1 - kbase) * 0x00010001u;   // fresh: >= 1 (host bound on rebase_by)
          } else {
            const int32_t sc = min(s, int32_t(N) - 1);
            inj = uint32_t(max(keys_a[sc] - kbase, 0)) | (uint32_t(max(keys_b[sc] - kbase, 0)) << 16);
          }
          uint32_t t = lane == 0 ? (s < int32_t(N) ? inj : 0u) : sh;
          // off-grid columns: t and V are 0, and max(0 + M, 0) = 0 whatever M is
          uint4 mcur[QW];
#pragma unroll
          for (int q = 0; q < QW; ++q) mcur[q] = mq[q];
          {
            const uint4* tq = tb4 + yc_next * code_stride + tid;   // the next step's words
#pragma unroll
            for (int q = 0; q < QW; ++q) mq[q] = tq[q * blockDim.x];
          }
          yc_next = yc_after;
#pragma unroll
          for (int q = 0; q < QW; ++q) {
            const uint4 m4 = mcur[q];
            const uint32_t m[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint32_t& v = V[4 * q + kk];
              const uint32_t d = __viaddmax_s16x2(t, m[kk], v);   // max(T + A, V): A = -32768 on a match
              v = v ^ t ^ d;
              t = d;
            }
          }
          tout = t;
          if (!last_warp) {
            if (lane == 31 && valid) ring_out[c & (kWideRing - 1)] = t;
          } else if (lane == 31 && valid) {
            const uint32_t ka = t & 0xFFFFu, kb = t >> 16;
            keys_a[c] = ka ? int32_t(ka) + kbase : 0;
            if (has_b) keys_b[c] = kb ? int32_t(kb) + kbase : 0;
          }
        }
      }
      __syncthreads();
    }
  }
}

// One CTA per strip: flags, then count(K) by a block-wide scan over K, then the output.
constexpr int kWideExtThreads = 512;

__device__ __forceinline__ uint32_t wide_block_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[kWideExtThreads / 32];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= uint32_t(off)) incl += u;
  }
  if (lane == 31) ws[wid] = incl;
  __syncthreads();
  uint32_t base = 0, all = 0;
#pragma unroll
  for (int k = 0; k < kWideExtThreads / 32; ++k) {
    base += uint32_t(k) < wid ? ws[k] : 0u;
    all += ws[k];
  }
  __syncthreads();
  *total = all;
  return base + incl - v;
}

__global__ void __launch_bounds__(kWideExtThreads) wide_extract_kernel(const WideParams p) {
  const uint32_t strip = blockIdx.x;
  const uint32_t N = p.N, W = p.W;
  const int32_t* keys = p.keys + size_t(strip) * N;
  uint8_t* ok = p.ok + size_t(strip) * N;
  const uint32_t row = p.row0 + strip;        // row within the call
  // countable: start = key - 1 >= e - W + 1 (key 0 = left boundary: never)
  auto countable = [&](uint32_t e) -> uint32_t {
    const int32_t st = keys[e] - 1;
    return st >= 0 && st >= int32_t(e) - int32_t(W) + 1 ? 1u : 0u;
  };
  for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) ok[e] = 0;
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < N; e += blockDim.x)
    if (countable(e)) ok[keys[e] - 1] = 1;
  __syncthreads();
  // count(0)
  uint32_t c0 = 0;
  for (uint32_t e = threadIdx.x; e < W; e += blockDim.x) c0 += countable(e);
  uint32_t count;
  wide_block_scan(c0, &count);
  const int32_t kh = int32_t(2 * W) - (p.r == 2 ? int32_t(2 * p.w) : 0);   // half = kh - 2 * count
  const uint32_t nwin = N - W + 1;   // window starts K in effective columns
  uint32_t hits_row = 0;
  // count(K) = count(0) + sum_{K' < K} delta(K'),  delta(K') = a(K' + W) - ok[K']
  for (uint32_t K0 = 0; K0 < nwin; K0 += blockDim.x) {
    const uint32_t K = K0 + threadIdx.x;
    const bool in = K < nwin;
    const int32_t delta = (in && K + 1 < nwin) ? int32_t(countable(K + W)) - int32_t(ok[K]) : 0;
    // exclusive scan of delta over the tile, as biased unsigned sums (exact mod 2^32)
    uint32_t tot;
    const uint32_t ex = wide_block_scan(uint32_t(delta), &tot);
    const uint32_t cnt = count + ex;   // count(K)
    count += tot;
    const bool report = in && !(K & (p.r - 1));
    const uint32_t col = K >> (p.r - 1);
    const int32_t half = kh - 2 * int32_t(cnt);
    if (p.dense) {
      if (report) {
        const size_t o = size_t(row) * p.cols + col;
        if (p.out_kind == 0) {
          p.out[o] = uint16_t(half);
        } else if (p.out_kind == 3) {
          p.out32[o] = half;
        } else if (p.out_kind == 2) {
          p.out8[o] = uint8_t(half);
        } else {   // write_pgm (io.cpp:136-153): (255 * clamp(h, 0, 2w) + w) / 2w, cut -> 0
          const int32_t full = 2 * int32_t(p.w);
          const bool cut = p.has_pgm_threshold && half < p.pgm_threshold;
          p.out8[o] = uint8_t(cut ? 0 : (255 * min(max(half, 0), full) + full / 2) / full);
        }
      }
    } else {
      const uint32_t hit = report && half >= p.t_half ? 1u : 0u;
      uint32_t nhit;
      const uint32_t rank = wide_block_scan(hit, &nhit);
      if (nhit) {
        __shared__ unsigned long long base;
        if (threadIdx.x == 0) base = atomicAdd(p.cursor, (unsigned long long)nhit);
        __syncthreads();
        if (hit) {
          const unsigned long long pos = base + rank;
          if (pos < p.stage_cap)
            p.stage[pos] = make_uint4(p.row_global0 + row, col, uint32_t(half), hits_row + rank);
        }
        __syncthreads();
      }
      hits_row += nhit;
    }
  }
  if (!p.dense && threadIdx.x == 0) p.seg_counts[row] = hits_row;
}

}  // namespace apk
