// ap_aux_kernels.cuh — the small kernels around the comb kernel (included by
// ap_capi.cu only): code streams (fused $-interleave), alphabet mapping and the
// deterministic placement of thresholded records.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apk {

// K1: effective y code stream (fused $-interleave, scoring.cpp:5-17):
// ycode[c] = r == 2 ? (c odd ? map[y[c/2]] : sent) : map[y[c]]; pad with 0.
// With ycol != nullptr also the generic kernel's column words ycol[c] =
// ycode[c] * ycol_mult followed by `total` zero words (what lanes j != 0 read); ycol_mult is
// 0x10001 (the code in both halves) or, for the dual-pair kernel, the table's byte stride per code.
__global__ void ycode_kernel(const uint8_t* __restrict__ y, size_t n, uint32_t r, uint32_t sent,
                             const uint8_t* __restrict__ map, uint8_t* __restrict__ ycode,
                             size_t total, uint32_t* __restrict__ ycol, uint32_t ycol_mult = 0x00010001u) {
  for (size_t c = blockIdx.x * size_t(blockDim.x) + threadIdx.x; c < total;
       c += size_t(gridDim.x) * blockDim.x) {
    const size_t N = n * r;
    uint8_t v = 0;
    if (c < N) v = (r == 2) ? ((c & 1) ? map[y[c >> 1]] : uint8_t(sent)) : map[y[c]];
    ycode[c] = v;
    if (ycol) {
      ycol[c] = uint32_t(v) * ycol_mult;
      ycol[total + c] = 0u;
    }
  }
}

// x codes: map[x[i]] (0xFF for bytes absent from y).
__global__ void xcode_kernel(const uint8_t* __restrict__ x, size_t m, const uint8_t* __restrict__ map,
                             uint8_t* __restrict__ xcode) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < m;
       i += size_t(gridDim.x) * blockDim.x)
    xcode[i] = map[x[i]];
}

// Alphabet of y: presence bitmap -> dense codes (map[b] = rank of b among the
// bytes present in y, 0xFF if absent), sigma -> out[0], "byte 0 present" -> out[1].
// One CTA of 1024 threads; the ranks come from a ballot prefix over 8 warps.
__global__ void alphabet_kernel(const uint8_t* __restrict__ y, size_t n, uint8_t* __restrict__ map,
                                uint32_t* __restrict__ sigma_out, uint32_t* __restrict__ zero_flag) {
  __shared__ uint32_t present[256];
  __shared__ uint32_t wsum[8];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) present[b] = 0;
  __syncthreads();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) present[y[i]] = 1;
  __syncthreads();
  const uint32_t b = threadIdx.x, lane = b & 31u, wid = b >> 5;
  const uint32_t pr = b < 256 ? present[b] : 0u;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pr);
  if (b < 256 && lane == 0) wsum[wid] = __popc(bal);
  __syncthreads();
  if (b < 256) {
    uint32_t base = 0;
    for (uint32_t k = 0; k < wid; ++k) base += wsum[k];
    map[b] = pr ? uint8_t(base + __popc(bal & ((1u << lane) - 1u))) : uint8_t(0xFF);
    if (b == 255) *sigma_out = base + __popc(bal);
    if (b == 0) *zero_flag = pr;
  }
}

// Fused code streams for small inputs (one launch instead of alphabet + xcode + ycode:
// C1-sized plots are launch-bound): one CTA builds the alphabet map in shared memory
// (as alphabet_kernel), writes sigma / the zero flag, clears the speculation abort flag,
// then maps x and y like xcode_kernel and ycode_kernel.
__global__ void codes_small_kernel(const uint8_t* __restrict__ x, size_t m, const uint8_t* __restrict__ y,
                                   size_t n, uint32_t r, uint32_t sent, uint8_t* __restrict__ map,
                                   uint32_t* __restrict__ small, uint8_t* __restrict__ xcode,
                                   uint8_t* __restrict__ ycode, size_t total, uint32_t* __restrict__ ycol,
                                   uint32_t ycol_mult = 0x00010001u) {
  __shared__ uint32_t present[256];
  __shared__ uint32_t wsum[8];
  __shared__ uint8_t smap[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) present[b] = 0;
  __syncthreads();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) present[y[i]] = 1;
  __syncthreads();
  const uint32_t b = threadIdx.x, lane = b & 31u, wid = b >> 5;
  const uint32_t pr = b < 256 ? present[b] : 0u;
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, pr);
  if (b < 256 && lane == 0) wsum[wid] = __popc(bal);
  __syncthreads();
  if (b < 256) {
    uint32_t base = 0;
    for (uint32_t k = 0; k < wid; ++k) base += wsum[k];
    const uint8_t code = pr ? uint8_t(base + __popc(bal & ((1u << lane) - 1u))) : uint8_t(0xFF);
    smap[b] = code;
    map[b] = code;
    if (b == 255) small[0] = base + __popc(bal);
    if (b == 0) { small[1] = pr; small[2] = 0u; }
  }
  __syncthreads();
  for (size_t i = threadIdx.x; i < m; i += blockDim.x) xcode[i] = smap[x[i]];
  const size_t N = n * r;
  for (size_t c = threadIdx.x; c < total; c += blockDim.x) {
    uint8_t v = 0;
    if (c < N) v = (r == 2) ? ((c & 1) ? smap[y[c >> 1]] : uint8_t(sent)) : smap[y[c]];
    ycode[c] = v;
    if (ycol) {
      ycol[c] = uint32_t(v) * ycol_mult;
      ycol[total + c] = 0u;
    }
  }
}

// ---- exclusive scan of the per-(row, segment) hit counts --------------------
// uint32 counts -> uint64 offsets (offs[i] = sum of counts[0, i), offs[n] = total), so lists
// longer than 2^32 cells (a count-only query on C4 / C5 at a low threshold) place and count
// exactly.  Three launches: tile sums, one CTA scanning the tile sums, tile scans.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;                     // counts per thread
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* total) {
  __shared__ unsigned long long wsum[kScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xFFFFFFFFu, incl, off);
    if (lane >= uint32_t(off)) incl += u;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  unsigned long long base = 0, all = 0;
#pragma unroll
  for (int k = 0; k < kScanThreads / 32; ++k) {
    const unsigned long long s = wsum[k];
    base += uint32_t(k) < wid ? s : 0ull;
    all += s;
  }
  __syncthreads();   // wsum is reused by the next call
  *total = all;
  return base + incl - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(const uint32_t* __restrict__ cnt, size_t n,
                                                                       unsigned long long* __restrict__ tsum) {
  const size_t t0 = size_t(blockIdx.x) * kScanTile;
  unsigned long long s = 0;
  for (int k = 0; k < kScanItems; ++k) {
    const size_t i = t0 + size_t(k) * kScanThreads + threadIdx.x;   // coalesced
    if (i < n) s += cnt[i];
  }
  unsigned long long tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// one CTA: tile sums -> exclusive tile offsets (in place), grand total -> *total
__global__ void __launch_bounds__(kScanThreads) scan_tile_offsets_kernel(unsigned long long* __restrict__ tsum,
                                                                          size_t ntiles,
                                                                          unsigned long long* __restrict__ total) {
  unsigned long long carry = 0;
  for (size_t b = 0; b < ntiles; b += kScanThreads) {
    const size_t i = b + threadIdx.x;
    const unsigned long long v = i < ntiles ? tsum[i] : 0ull;
    unsigned long long tot;
    const unsigned long long ex = block_excl_scan(v, &tot);
    if (i < ntiles) tsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// each thread scans kScanItems consecutive counts of its tile
__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(const uint32_t* __restrict__ cnt, size_t n,
                                                                   const unsigned long long* __restrict__ toff,
                                                                   unsigned long long* __restrict__ offs) {
  const size_t i0 = size_t(blockIdx.x) * kScanTile + size_t(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  unsigned long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = i0 + k < n ? cnt[i0 + k] : 0u;
    s += v[k];
  }
  unsigned long long tot;
  unsigned long long run = toff[blockIdx.x] + block_excl_scan(s, &tot);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (i0 + k < n) offs[i0 + k] = run;
    run += v[k];
  }
}

// Deterministic row-major placement of staged threshold records:
// final index = offset[row * seg_stride + seg] + rank, where rows below split_row are cut into
// segments of seg_cols columns and the rest (the launch's short tail tasks) of seg_cols2.
// Structure-of-arrays output (orow/ocol and uint16 ohalf or int32 ohalf32) or, with
// ocell != nullptr, ap_cell records {row, col, int32 half} (PlotCell, scoring.hpp:33-42).
struct CellRec { uint32_t row, col; int32_t half; };

__global__ void place_kernel(const uint4* __restrict__ stage, unsigned long long nrec,
                             const unsigned long long* __restrict__ offsets, uint32_t seg_stride,
                             uint32_t seg_cols, uint32_t seg_cols2, uint32_t split_row, uint32_t r,
                             uint32_t row_global0, uint32_t* __restrict__ orow, uint32_t* __restrict__ ocol,
                             uint16_t* __restrict__ ohalf, int32_t* __restrict__ ohalf32,
                             CellRec* __restrict__ ocell, unsigned long long cap) {
  for (unsigned long long i = blockIdx.x * 1ull * blockDim.x + threadIdx.x; i < nrec;
       i += 1ull * gridDim.x * blockDim.x) {
    const uint4 rec = stage[i];
    const uint32_t row = rec.x - row_global0;
    const uint32_t seg = (rec.y * r) / (row < split_row ? seg_cols : seg_cols2);
    const unsigned long long pos = offsets[size_t(row) * seg_stride + seg] + rec.w;
    if (pos < cap) {
      if (ocell) {
        ocell[pos] = CellRec{rec.x, rec.y, int32_t(rec.z)};
      } else {
        orow[pos] = rec.x;
        ocol[pos] = rec.y;
        if (ohalf32) ohalf32[pos] = int32_t(rec.z);
        else ohalf[pos] = uint16_t(rec.z);
      }
    }
  }
}

// uint16 half-units -> int32 (ap_plot_dense_i32 on the packed kernels, whose scores fit 16 bits)
__global__ void widen_kernel(const uint16_t* __restrict__ in, size_t n, int32_t* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = int32_t(in[i]);
}

}  // namespace apk
