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
// ycode[c] * 0x10001 followed by `total` zero words (what lanes j != 0 read).
__global__ void ycode_kernel(const uint8_t* __restrict__ y, size_t n, uint32_t r, uint32_t sent,
                             const uint8_t* __restrict__ map, uint8_t* __restrict__ ycode,
                             size_t total, uint32_t* __restrict__ ycol) {
  for (size_t c = blockIdx.x * size_t(blockDim.x) + threadIdx.x; c < total;
       c += size_t(gridDim.x) * blockDim.x) {
    const size_t N = n * r;
    uint8_t v = 0;
    if (c < N) v = (r == 2) ? ((c & 1) ? map[y[c >> 1]] : uint8_t(sent)) : map[y[c]];
    ycode[c] = v;
    if (ycol) {
      ycol[c] = uint32_t(v) * 0x00010001u;
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
                                   uint8_t* __restrict__ ycode, size_t total, uint32_t* __restrict__ ycol) {
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
      ycol[c] = uint32_t(v) * 0x00010001u;
      ycol[total + c] = 0u;
    }
  }
}

// Deterministic row-major placement of staged threshold records:
// final index = offset[row * seg_stride + seg] + rank, where rows below split_row are cut into
// segments of seg_cols columns and the rest (the launch's short tail tasks) of seg_cols2.
__global__ void place_kernel(const uint4* __restrict__ stage, unsigned long long nrec,
                             const unsigned long long* __restrict__ offsets, uint32_t seg_stride,
                             uint32_t seg_cols, uint32_t seg_cols2, uint32_t split_row, uint32_t r,
                             uint32_t row_global0, uint32_t* __restrict__ orow, uint32_t* __restrict__ ocol,
                             uint16_t* __restrict__ ohalf, unsigned long long cap) {
  for (unsigned long long i = blockIdx.x * 1ull * blockDim.x + threadIdx.x; i < nrec;
       i += 1ull * gridDim.x * blockDim.x) {
    const uint4 rec = stage[i];
    const uint32_t row = rec.x - row_global0;
    const uint32_t seg = (rec.y * r) / (row < split_row ? seg_cols : seg_cols2);
    const unsigned long long pos = offsets[size_t(row) * seg_stride + seg] + rec.w;
    if (pos < cap) {
      orow[pos] = rec.x;
      ocol[pos] = rec.y;
      ohalf[pos] = uint16_t(rec.z);
    }
  }
}

}  // namespace apk
