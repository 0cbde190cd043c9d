// ap_kernels.cuh — sm_100a kernels of the alignment-plot engine.
//
// The hot path of the reference:
//   blowup (scoring.cpp:5-17)                       -> fused into the code streams (K1)
//   comb_strip_lanes / sweep<T> (lane_kernel.cpp:28-128)
//   to_bottom_events (lane_kernel.cpp:5-18)
//   window_llcs_from_events (seaweed_scalar.cpp:65-99)
//   llcs_to_half / recover_score (runner.cpp:31-35, scoring.cpp:26-28)
//   PlotGrid fill / apply_threshold (runner.cpp:108, scoring.cpp:30-39)
// all fused into one combing kernel (K2) per launch.
//
// Seaweed representation.  The reference keeps, per lane, the *distance* of a
// seaweed from its start column and saturates it (lane_kernel.cpp:66-77).  We
// keep the seaweed's *start key* instead: key = start_column - kbase, a 16-bit
// unsigned value, two strips packed per 32-bit register (x-windows A and B of
// the same grid-row pair share every y character).  Left-boundary seaweeds
// have key 0 (they start left of everything, seaweed_scalar.cpp:21-22).  The
// cell rule "exchange iff match or start(V) > start(T)"
// (seaweed_scalar.cpp:26-32) becomes, with A = 0x8000 (-32768 as s16) on a
// match and 0 on a mismatch (per 16-bit half):
//     d      = max_s16x2(T + A, V)       // seaweed leaving downwards (VIADDMNMX)
//     V'     = V ^ T ^ d                 // seaweed leaving to the right (LOP3)
// i.e. two ALU instructions for two cells: no increment, no saturation in the
// inner loop.  Keys stay in [0, 0x7BFF] and are rebased (saturating at 0) every
// ~28K columns; a rebased-to-0 seaweed is provably older than any window
// (DESIGN.md §3).
//
// A comes from a per-warp shared-memory table indexed by the y code: the
// x-window characters are fixed for a strip, so table[code][row] holds the
// match words of both strips; one LDS.128 serves four rows.
//
// Mapping.  A warp holds 32/L groups; a group of L lanes combs one strip pair,
// lane j owning R consecutive rows [j*R, j*R+R).  Lane j processes column
// s - j at step s (antidiagonal wavefront across lanes); the seaweed leaving
// the bottom of lane j and the y code move to lane j+1 with one SHFL each.
//
// Extraction without a heap.  For the bottom event at column e with start st
// (countable iff e - st < W), the window count obeys
//     count(K+1) = count(K) + [event e=K+W countable] - [seaweed starting at K
//                  ended inside [K, K+W-1]]
// (DESIGN.md §4), evaluated 32 columns at a time by a segmented warp scan;
// LLCS(K) = W - count(K), reported at K = 0 mod r (seaweed_scalar.cpp:85-96).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apk {

constexpr int kWarpsPerCta = 4;   // warps per CTA the shapes' shared memory and occupancy are sized for
// Warps per CTA of the launches: one-warp CTAs release an SM's resources warp by warp as the
// grid drains (B200: C4 -8.5%, C3 -2.5%, C5 -2% against 4-warp CTAs), except the r = 2 shapes
// with long lanes (RR >= 8: C2 +3% with one-warp CTAs).  Compile-time, so a one-warp CTA's
// shared-memory base is a constant; the host mirrors the rule (launch_wpc in ap_capi.cu).
constexpr int kGenericWpc = 1;
#ifndef AP_R2_LONG_WPC
#define AP_R2_LONG_WPC 4
#endif
__host__ __device__ constexpr int r2_wpc(int rr) { return rr >= 8 ? AP_R2_LONG_WPC : 1; }
constexpr int kChunk = 32;          // steps per extraction batch
#ifndef AP_G_STS64
#define AP_G_STS64 1   // generic kernel: the bottom keys of two steps in one 8-byte ring store
#endif
#ifndef AP_R2_STS64
#define AP_R2_STS64 1   // r = 2 kernel: one 8-byte ring store per step (even ring stride; C2, C4 -1.1%)
#endif
constexpr uint32_t kRebaseAt = 0x7000u;   // fresh keys must stay fp16-finite (<= 0x7BFF)
constexpr uint32_t kRebaseBy = 0x4000u;

struct CombParams {
  const uint8_t* xcode;   // mapped x codes (0xFF = absent from y), local row 0 at xcode[0]
  const uint8_t* ycode;   // effective y codes, N entries + >=128 pad bytes, 16-B aligned
  const uint32_t* ycol;   // generic kernel: code * ycol_mult per effective column (+256 pad), 16-B aligned
  const uint32_t* ycol_zero;  // as many zero words (the column words seen by lanes j != 0)
  uint32_t rows;          // grid rows in this launch
  uint32_t xlen;          // x codes readable from xcode (dual-pair kernel: words of rows past this launch's own)
  uint32_t h, w, r, W, N; // step, window, blowup, blown window, effective y length
  uint32_t sigma;         // table codes (incl. the sentinel code when r = 2)
  uint32_t sent_code;     // code of the $ sentinel (r = 2)
  uint32_t S;             // column segment width (effective columns), multiple of 32
  uint32_t nseg;          // number of column segments
  // pair groups >= g_split are cut into nseg2 segments of S2 columns (short tasks claimed
  // last, so the grid drains on them); g_split = all groups: none
  uint32_t g_split, nseg2, S2;
  uint32_t seg_stride;    // row stride of seg_counts (max(nseg, nseg2))
  uint32_t ring;          // ok-flag ring size (power of two >= W + 64)
  uint32_t cols;          // grid columns
  uint32_t row_global0;   // global grid row of local row 0
  // dense output
  uint16_t* out;          // [rows][cols] half-units (out_kind 0)
  uint8_t* out8;          // [rows][cols] PGM pixels (out_kind 1, io.cpp:136-153 fused)
  uint32_t out_kind;      // 0 = uint16 half-units, 1 = uint8 PGM pixels, 2 = uint8 half-units
  int32_t pgm_threshold;  // cells below it render 0 (when has_pgm_threshold)
  uint32_t has_pgm_threshold;
  // thresholded output
  int32_t t_half;
  uint4* stage;                   // {row, col, int32 half, rank} records
  unsigned long long* cursor;     // staging append cursor
  uint32_t* task_counter;         // AP_DYN_TASKS: tasks handed out after the first static wave (zeroed per launch)
  unsigned long long stage_cap;
  uint32_t* seg_counts;           // [rows][seg_stride] hits per (row, segment)
  // speculative alphabet (ap_capi.cu run_device): the launch was planned for an alphabet of
  // at most sigma_cap codes before y's alphabet size reached the host; every warp checks the
  // device-side size and, if it is larger, flags the launch for a re-run and exits
  const uint32_t* sigma_dev;      // y's alphabet size (written by alphabet_kernel)
  uint32_t sigma_cap;             // 0xFFFFFFFF: not speculative
  uint32_t* abort_flag;
  uint32_t zero;                  // always 0 (HFMA2 addend)
  uint32_t one;                   // always 1 (IMAD forms the compiler must not fold)
  uint32_t minus_one;             // always 0xFFFFFFFF
};

using KernelFn = void (*)(CombParams);

// Task distribution: every warp starts with task (CTA, warp); after that, warps claim the next
// unclaimed task from a per-launch global counter, so warps that run faster (fewer co-resident
// warps, fewer threshold hits, ...) take more tasks and the grid drains evenly (B200: C4 -7%,
// C5 -2%, C2 and C3 -1% against a static stride).
#ifndef AP_DYN_TASKS
#define AP_DYN_TASKS 1
#endif
__device__ __forceinline__ uint64_t next_task(const CombParams& p, uint64_t task, uint64_t wstride, uint32_t lane,
                                              uint64_t ntasks) {
  if constexpr (AP_DYN_TASKS) {
    if (ntasks <= wstride) return ntasks;   // one static wave covers the launch
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(p.task_counter, 1u);
    return uint64_t(__shfl_sync(0xFFFFFFFFu, t, 0)) + wstride;
  } else {
    return task + wstride;
  }
}
// Launch-stub pointers of the instantiated comb kernels (ap_inst_l{8,16,32}.cu).
KernelFn pick_l4(int r, int k, bool dense, bool xm);
KernelFn pick_l8(int r, int k, bool dense, bool xm);
KernelFn pick_l16(int r, int k, bool dense, bool xm);
KernelFn pick_l32(int r, int k, bool dense, bool xm);
// fp16-key variants (table masks only; W + L*K <= kHfMaxSpan): ap_inst_ghf_{a,b}.cu
KernelFn pick_ghf(int l, int r, int k, bool dense);
// The r = 2 specialised kernels (ap_inst_r2.cu): RR real rows per lane.
KernelFn pick_r2(int l, int rr, int k, bool dense, bool hf = false);

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Lane groups.  L lanes comb one strip pair; G = 32 / L groups per warp.  When
// L does not divide 32 the trailing 32 - G*L lanes form an idle "phantom"
// group (no strips, own scratch) so every lane runs the same code.  Shuffles
// are full-width: a group's lane 0 always overrides what it receives, and scans
// only accumulate from lanes of the same group (j >= off).
__host__ __device__ constexpr int groups_per_warp(int L) { return 32 / L; }
__host__ __device__ constexpr int groups_alloc(int L) { return 32 / L + (32 % L ? 1 : 0); }
// bottom-key ring words per group: nb entries rounded up to whole lanes, plus padding so
// the bottom lanes of different groups write different banks; the r = 2 kernel (nb = 64)
// keeps it even so a step's (2c, 2c+1) pair is one 8-byte store
__host__ __device__ constexpr int ring_stride(int L, int nb) {
  return L * ((nb + L - 1) / L) + ((nb == 2 * kChunk && AP_R2_STS64) || (nb == kChunk && AP_G_STS64)
                                      ? 2 - (L * ((nb + L - 1) / L)) % 2 : 1);
}
// ok-flag bytes per group: one u32 per ring slot (byte 0 = strip A, byte 2 =
// strip B, so a slot reads back as the packed pair oA | oB << 16) plus 32 bytes
// of padding so the same slot of different groups falls 8 banks apart.
__host__ __device__ constexpr size_t ok_stride(uint32_t ring) { return size_t(4) * ring + 32; }
// ring slots the extraction needs (extract_body): the W + NB + A starts between
// the oldest unread flag and the end of the clear-ahead window, with the
// clear-ahead offset A = NB (+ (-W) mod CPL when lane runs are CPL-aligned, i.e.
// L divides 32 and NB); a power of two >= 128
__host__ __device__ constexpr uint32_t ring_slots(uint32_t W, int nb, int L) {
  const bool align = 32 % L == 0 && nb % L == 0;
  const uint32_t cpl = uint32_t((nb + L - 1) / L);
  const uint32_t need = W + 2 * uint32_t(nb) + (align ? (cpl - W % cpl) % cpl : 0u);
  uint32_t r = 128;
  while (r < need) r <<= 1;
  return r;
}

template <int L>
__device__ __forceinline__ uint32_t shfl_up1(uint32_t v) {
  if constexpr ((L & (L - 1)) == 0) return __shfl_up_sync(0xFFFFFFFFu, v, 1, L);
  else return __shfl_up_sync(0xFFFFFFFFu, v, 1);
}
template <int L>
__device__ __forceinline__ uint32_t shfl_up_n(uint32_t v, int off) {
  if constexpr ((L & (L - 1)) == 0) return __shfl_up_sync(0xFFFFFFFFu, v, off, L);
  else return __shfl_up_sync(0xFFFFFFFFu, v, off);
}
// value of the group's last lane
template <int L>
__device__ __forceinline__ uint32_t shfl_group_last(uint32_t v, uint32_t g) {
  if constexpr ((L & (L - 1)) == 0) return __shfl_sync(0xFFFFFFFFu, v, L - 1, L);
  else return __shfl_sync(0xFFFFFFFFu, v, (g * L + L - 1) & 31u);
}

// 16-byte shared load at a 32-bit shared-window address
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

#ifndef AP_ABL_LDS
#define AP_ABL_LDS 1   // timing ablation only (wrong results when > 1): one table load per AP_ABL_LDS quads
#endif
#ifndef AP_FMAMIN_RR
#define AP_FMAMIN_RR 4   // r = 2 kernels with RR >= this compute one mismatch min with IMADs (C4: -1.3%)
#endif
#ifndef AP_SUBUNROLL
#define AP_SUBUNROLL 2   // generic kernel: unroll of the 8-step sub loop (4 per chunk; C5 -3%)
#endif
constexpr int kSubUnroll = AP_SUBUNROLL;
#ifndef AP_SUBUNROLL2_RR
#define AP_SUBUNROLL2_RR 4  // r = 2 kernel: shapes with RR <= this unroll all 4 subs of a chunk (C4 -7%; C2 +4%)
#endif
// fp16 key encoding (r = 2 kernels with HF = true): live keys are 0x6400 + k =
// the fp16 value 1024 + k (k < 1024), left-boundary keys 0 (+0.0).  The integer
// order of the patterns is the order of the values, so the integer min/max cells
// are unchanged, and min(v, t) = (v - max(v, t)) + t is exact in fp16 (every
// intermediate is an integer of magnitude < 2048): one mismatch min per row
// moves to the FMA pipe as two 2-operand HADD2s (C2: 6.25 -> 6.06 ms on B200;
// slower than the IMAD form for RR = 4 shapes, so only RR >= 8 use it).  The
// generic kernel with HF = true computes V' = (V - d) + T (two HADD2s) instead
// of the LOP3 for one row of every four (C3 -1.2%, C5 -2%; two rows: slower).
// Keys are rebased every rebase_by columns (W + 2*VB <= kHfMaxSpan, host-checked).
constexpr uint32_t kHfBase = 0x6400u;
constexpr uint32_t kHfRebaseAt = 0x6400u + 0x3C0u;   // fresh keys stay < 0x6400 + 1024
constexpr uint32_t kHfMaxSpan = 0x3C0u - 2 * 32 - 128;   // W + 2*VB bound: rebase step >= 128 columns
#ifndef AP_HF_ROWS
#define AP_HF_ROWS 1   // generic fp16-key kernels: rows of each quad whose V' is formed by two HADD2s
#endif
#ifndef AP_SUBUNROLL_L4
#define AP_SUBUNROLL_L4 2   // generic kernel, L = 4 shapes: unroll of the 8-step sub loop (C3 -0.5% vs 1)
#endif
#ifndef AP_R2_SUBLOAD
#define AP_R2_SUBLOAD 1   // r = 2 kernel, rolled sub loop: each sub prefetches its code words (no per-sub selects)
#endif
#ifndef AP_R2_PRMT
#define AP_R2_PRMT 0   // r = 2 kernel: next code byte by one PRMT instead of SHF + LOP3
#endif
#ifndef AP_R2_IMADSEL
#define AP_R2_IMADSEL 0   // r = 2 kernel: lane-0 key injection as IMAD(shuffled, nz, fresh) instead of SEL
#endif
#ifndef AP_R2_YCOL
#define AP_R2_YCOL 0   // r = 2 kernel, unrolled shapes: u32 column words (code * table stride) instead of code bytes
#endif
// shapes of the r = 2 kernel that take the column-word feed: fully unrolled sub loop and one table array
__host__ __device__ constexpr bool r2_ycol_feed(int rr, int k) {
  return AP_R2_YCOL && rr <= AP_SUBUNROLL2_RR && ((rr / k) % 4 == 0 || (rr / k) < 4);
}
#ifndef AP_R2_MB4
#define AP_R2_MB4 10  // r = 2 kernels with RR <= this are compiled for 4 CTAs per SM (C2: 6.87 -> 6.59 ms)
#endif

// shared-window accesses by 32-bit address (ok-flag slots)
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void lds_v4(uint32_t addr, uint32_t* v) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void lds_v2(uint32_t addr, uint32_t* v) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_zero_v2(uint32_t addr) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %1};" :: "r"(addr), "r"(0u) : "memory");
}
__device__ __forceinline__ void sts_zero_v4(uint32_t addr) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" :: "r"(addr), "r"(0u) : "memory");
}

// hi32(a * b) + c on the FMA pipe
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// a * b + c on the FMA pipe (b opaque to ptxas so it cannot become an IADD)
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// fp16x2 add / subtract (round to nearest: exact on the key encoding below)
__device__ __forceinline__ uint32_t hadd2u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hsub2u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t lop3_xor(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Shared memory bytes per warp: mismatch table (table_words 32-bit words per
// lane per code), the bottom-key ring (nb entries per chunk, padded by one word
// per group so the bottom lanes of different groups hit different banks) and
// the ok-flag rings.
__host__ __device__ inline size_t comb_smem_per_warp(int L, int table_words, uint32_t sigma, uint32_t ring,
                                                     int nb = kChunk) {
  const int Ga = groups_alloc(L);
  const size_t bytes = size_t(4) * 32 * sigma * table_words   // mismatch table (sigma = 0: computed masks)
       + (sigma && L < 8 ? size_t(32 / L) * 64 : 0)            // L < 8: groups 64 B apart (bank halves)
       + ((size_t(Ga) * ring_stride(L, nb) * 4 + 15) & ~size_t(15))   // bottom-key ring per group (padded)
       + size_t(32 / L) * ok_stride(ring)                      // ok flags per group (strip A, strip B)
       + (Ga > 32 / L ? 64 : 0);                               // phantom group: ring mask 0, 64-B scratch
  return (bytes + 15) & ~size_t(15);                           // keep every warp's table 16-B aligned
}

// Window extraction for the NB bottom columns [E0, E0 + NB) held in this
// group's ring (one per step and blown column).  Lane j owns the CPL = NB/L
// consecutive columns E0 + j*CPL + c.  Per column e with bottom key k the
// seaweed is countable iff its span e - start < W (lane_kernel.cpp:79-87 keeps
// exactly those spans); its start then gets an ok flag, and
//   count(K+1) = count(K) + [column K+W countable] - ok[K]
// (the heap of seaweed_scalar.cpp:80-97 replaced by a difference recurrence,
// DESIGN.md §4), evaluated as a segmented scan over the group.  LLCS(K) =
// W - count(K) is reported for K = 0 mod r and converted to half-units
// (runner.cpp:31-35, scoring.cpp:26-28).
//
// Both strips are handled in packed 16-bit halves throughout:
//  * kk = min_u16(k - thr - 1, C) (one VIADDMNMX): countable seaweeds give
//    0..W-1 (= start - (e - W + 1)), the rest wrap to >= 0x8000 and clamp to
//    C = 0x8000 | (W - 1 + A); bit 15 of kk is then "not countable" and
//    (kk + e - W + 1) mod ring is the flag slot -- for non-countable seaweeds
//    the slot of start e + A, a start whose flag nobody has written yet.
//  * Clear-ahead: each chunk zeroes the slots of starts [E0 + A, E0 + A + NB).
//    Those starts cannot have exited yet (A >= NB), so the stray flags of the
//    chunk (all aimed inside this range) are wiped before the slot is used,
//    and no per-seaweed select or branch is needed.  Live slots span
//    W + NB + A starts (ring_slots).
//  * When L divides 32 and NB, slots are offset by delta so that every lane's
//    run of CPL read slots and CPL cleared slots is CPL-aligned: one vector
//    load / store per lane and no per-column wrap masks.
//  * Slot addresses and the running count use IMAD / IMAD.HI on the FMA pipe.
// Packed 32-bit sums are exact whenever every half of the final value is in
// [0, 0xFFFF] (arithmetic is linear mod 2^32), so no per-column bias is needed.
// Extraction phases (extract_body below chains them for one strip pair per group).
// Shared constants:
// phase 1: scatter the ok flags of countable seaweeds (bytes BYTE and BYTE + 2 of a slot:
// strip A and B of the pair); cab[c]: bit 15 / 31 = column countable (strip A / B)
template <int L, int NB, bool CHECK, int BYTE>
__device__ __forceinline__ void extract_scatter(const CombParams& p, const uint32_t* ringB, uint32_t okb,
                                                uint32_t rmask, uint32_t j, int32_t E0, uint32_t nseg_cols,
                                                int32_t kbase, uint32_t* cab) {
  constexpr int CPL = (NB + L - 1) / L;   // columns per lane (the last lane may get fewer real ones)
  constexpr bool ALIGN = 32 % L == 0 && NB % L == 0;   // CPL is a power of two dividing 32
  const uint32_t k18 = p.one << 18;   // opaque: IMAD.HI, not LEA.HI
  const int32_t W = int32_t(p.W);
  const int32_t eb = E0 + int32_t(j) * CPL;
  // delta aligns the read runs (eb - W + delta) and clear runs (E0 + A + delta + j*CPL) to CPL
  const uint32_t delta = ALIGN ? uint32_t(W - E0) & 31u : 0u;
  const uint32_t A = NB + (ALIGN ? uint32_t(-W) & uint32_t(CPL - 1) : 0u);
  const uint32_t clamp2 = (0x8000u | (p.W - 1 + A)) * 0x00010001u;
  const uint32_t rmask2 = rmask * 0x00010001u;
  const uint32_t n0 = (uint32_t(kbase + W - 1 - eb) & 0xFFFFu) * 0x00010001u;          // -(thr+1) at eb
  const uint32_t sb2 = (uint32_t(eb - W + 1 + int32_t(delta)) & rmask) * 0x00010001u;   // slot of start eb-W+1
  const uint32_t xA = okb * 0x00010001u + 0x20000u;   // addrA = imad(addrB, -65536, imad(slot2, 4, xA))
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int32_t e = eb + c;
    const bool real = NB % L == 0 || j * CPL + c < NB;
    const bool valid = real && (!CHECK || (e >= 0 && e < int32_t(nseg_cols)));
    const uint32_t k = real ? ringB[j * CPL + c] : 0u;
    const uint32_t negc = ((0x10000u - uint32_t(c)) & 0xFFFFu) * 0x00010001u;
    const uint32_t nthr = c == 0 ? n0 : __vadd2(n0, negc);
    uint32_t kk = __viaddmin_u16x2(k, nthr, clamp2);
    if (!valid) kk = clamp2;
    const uint32_t pre = kk + sb2 + uint32_t(c) * 0x00010001u;   // halves < 0x10000: no carry
    const uint32_t slot2 = pre & rmask2;
    cab[c] = ~pre & 0x80008000u;
    const uint32_t addrB = madhi(slot2, k18, okb + 2);          // okb + 4 * slotB + 2
    const uint32_t addrA = imad(addrB, 0xFFFF0000u, imad(slot2, 4u, xA));   // okb + 4 * slotA
    sts_u8(addrA + BYTE, 1u);
    sts_u8(addrB + BYTE, 1u);
  }
}

// phase 2: the flag words of starts e - W (both pairs' bytes)
template <int L, int NB, bool CHECK>
__device__ __forceinline__ void extract_flags(const CombParams& p, uint32_t okb, uint32_t rmask, uint32_t j,
                                              int32_t E0, uint32_t nseg_cols, uint32_t* o) {
  constexpr int CPL = (NB + L - 1) / L;
  constexpr bool ALIGN = 32 % L == 0 && NB % L == 0;
  const int32_t W = int32_t(p.W);
  const int32_t eb = E0 + int32_t(j) * CPL;
  const uint32_t delta = ALIGN ? uint32_t(W - E0) & 31u : 0u;
  if constexpr (ALIGN) {
    const uint32_t rb = okb + 4 * (uint32_t(eb - W + int32_t(delta)) & rmask);
    if constexpr (CPL >= 4) {
#pragma unroll
      for (int q = 0; q < CPL / 4; ++q) lds_v4(rb + 16 * q, o + 4 * q);
    } else if constexpr (CPL == 2) {
      lds_v2(rb, o);
    } else {
      o[0] = lds_u32(rb);
    }
    if constexpr (CHECK) {
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (!(eb + c >= 0 && eb + c < int32_t(nseg_cols))) o[c] = 0u;
    }
  } else {
    const uint32_t rsb = uint32_t(eb - W) & rmask;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int32_t e = eb + c;
      const bool real = NB % L == 0 || j * CPL + c < NB;
      const bool valid = real && (!CHECK || (e >= 0 && e < int32_t(nseg_cols)));
      o[c] = 0u;
      if (valid) o[c] = lds_u32(okb + 4 * ((rsb + c) & rmask));
    }
  }
}

// clear ahead: starts [E0 + A, E0 + A + NB), this lane's run of CPL
template <int L, int NB>
__device__ __forceinline__ void extract_clear(const CombParams& p, uint32_t okb, uint32_t rmask, uint32_t j,
                                              int32_t E0) {
  constexpr int CPL = (NB + L - 1) / L;
  constexpr bool ALIGN = 32 % L == 0 && NB % L == 0;
  const int32_t W = int32_t(p.W);
  const uint32_t delta = ALIGN ? uint32_t(W - E0) & 31u : 0u;
  const uint32_t A = NB + (ALIGN ? uint32_t(-W) & uint32_t(CPL - 1) : 0u);
  {
    if constexpr (ALIGN) {
      const uint32_t cb = okb + 4 * (uint32_t(E0 + int32_t(A + delta) + int32_t(j) * CPL) & rmask);
      if constexpr (CPL >= 4) {
#pragma unroll
        for (int q = 0; q < CPL / 4; ++q) sts_zero_v4(cb + 16 * q);
      } else if constexpr (CPL == 2) {
        sts_zero_v2(cb);
      } else {
        sts_u32(cb, 0u);
      }
    } else {
      const uint32_t cb = uint32_t(E0 + int32_t(A) + int32_t(j) * CPL) & rmask;
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (NB % L == 0 || j * CPL + c < NB) sts_u32(okb + 4 * ((cb + c) & rmask), 0u);
    }
  }
}

// phase 3: count deltas (cab = countable bits, o = this pair's flag halves) -> group
// scan -> dense half-units or threshold hits for rows rA, rB
template <int L, int NB, bool DENSE, bool CHECK>
__device__ __forceinline__ void extract_out(const CombParams& p, uint32_t j, uint32_t g, uint32_t lane,
                                            int32_t E0, uint32_t nseg_cols, uint32_t c0, uint32_t* cab,
                                            const uint32_t* o, uint32_t rA, uint32_t rB, bool hasA, bool hasB,
                                            uint32_t& run, uint32_t& hitsA, uint32_t& hitsB) {
  constexpr int CPL = (NB + L - 1) / L;
  const uint32_t rshift = p.r - 1;
  const uint32_t one = p.one;
  const uint32_t k17 = one << 17, k16 = one << 16;   // opaque: IMAD.HI, not LEA.HI
  const int32_t W = int32_t(p.W);
  const int32_t eb = E0 + int32_t(j) * CPL;
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    acc = imad(o[c], 0xFFFFFFFFu, madhi(cab[c], k17, acc));   // acc + countable - ok
    cab[c] = acc;                                            // count delta through column c
  }
  // group scan of the lane totals; count after column c = run + excl + acc_c
  uint32_t incl = acc;
#pragma unroll
  for (int off = 1; off < L; off <<= 1) {
    const uint32_t v = shfl_up_n<L>(incl, off);
    if (j >= uint32_t(off)) incl += v;
  }
  const uint32_t runc = run + incl - acc;
  run = shfl_group_last<L>(run + incl, g);
  const uint32_t kh = (2 * p.W - (rshift ? 2 * p.w : 0u)) * 0x00010001u;   // half = kh - 2 * count
  const int32_t kp0 = eb - W + 1;   // window start of column eb (segment-relative)
  if constexpr (DENSE) {
    // packed halves biased by 0x8000 (r = 2 scores can be negative)
    const uint32_t kb = imad(runc, 0xFFFFFFFEu, kh + 0x80008000u);
    if (!CHECK && p.out_kind != 1) {
      // interior chunk: every column valid; r = 2 reports the columns with c = par (mod 2)
      const uint32_t par = uint32_t(kp0) & rshift;
      const size_t gb = (c0 + uint32_t(kp0) + par) >> rshift;   // output column of the first reported c
      if (p.out_kind == 0) {
        uint16_t* pa = p.out + size_t(rA) * p.cols + gb;
        uint16_t* pb = p.out + size_t(rB) * p.cols + gb;
        if (rshift == 0) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if (NB % L != 0 && j * CPL + c >= NB) continue;
            const uint32_t hb = imad(cab[c], 0xFFFFFFFEu, kb);
            if (hasA) pa[c] = uint16_t(hb - 0x8000u);
            if (hasB) pb[c] = uint16_t(madhi(hb, k16, 0xFFFF8000u));
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            if (NB % L != 0 && j * CPL + c >= NB) continue;
            if ((uint32_t(c) & 1u) != par) continue;
            const uint32_t hb = imad(cab[c], 0xFFFFFFFEu, kb);
            if (hasA) pa[c >> 1] = uint16_t(hb - 0x8000u);
            if (hasB) pb[c >> 1] = uint16_t(madhi(hb, k16, 0xFFFF8000u));
          }
        }
      } else {   // compact: half-units as bytes (w <= 127)
        uint8_t* pa = p.out8 + size_t(rA) * p.cols + gb;
        uint8_t* pb = p.out8 + size_t(rB) * p.cols + gb;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          if (NB % L != 0 && j * CPL + c >= NB) continue;
          if ((uint32_t(c) & rshift) != par) continue;
          const uint32_t hb = imad(cab[c], 0xFFFFFFFEu, kb);
          const uint32_t off = uint32_t(c) >> rshift;
          if (hasA) pa[off] = uint8_t(hb - 0x8000u);
          if (hasB) pb[off] = uint8_t(madhi(hb, k16, 0xFFFF8000u));
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int32_t e = eb + c;
        const bool real = NB % L == 0 || j * CPL + c < NB;
        const bool valid = real && (!CHECK || (e >= 0 && e < int32_t(nseg_cols)));
        const int32_t kp = kp0 + c;
        const bool out_ok = valid && (!CHECK || (kp >= 0 && kp < int32_t(p.S))) && !(uint32_t(kp) & rshift);
        const uint32_t gcol = (c0 + uint32_t(kp)) >> rshift;
        const uint32_t hb = imad(cab[c], 0xFFFFFFFEu, kb);   // (h + 0x8000) per half
        const uint32_t hlo = hb - 0x8000u;                       // low 16 bits: hA
        const uint32_t hhi = madhi(hb, k16, 0xFFFF8000u);        // low 16 bits: hB
        if (p.out_kind == 0) {
          if (out_ok && hasA) p.out[size_t(rA) * p.cols + gcol] = uint16_t(hlo);
          if (out_ok && hasB) p.out[size_t(rB) * p.cols + gcol] = uint16_t(hhi);
        } else if (p.out_kind == 2) {
          if (out_ok && hasA) p.out8[size_t(rA) * p.cols + gcol] = uint8_t(hlo);
          if (out_ok && hasB) p.out8[size_t(rB) * p.cols + gcol] = uint8_t(hhi);
        } else {
          // write_pgm (io.cpp:136-153): pixel = (255*clamp(h,0,2w) + w) / 2w, cut -> 0
          const int32_t hA = int32_t(int16_t(uint16_t(hlo))), hB = int32_t(int16_t(uint16_t(hhi)));
          const int32_t full = 2 * int32_t(p.w);
          const bool cutA = p.has_pgm_threshold && hA < p.pgm_threshold;
          const bool cutB = p.has_pgm_threshold && hB < p.pgm_threshold;
          const int32_t qA = cutA ? 0 : (255 * min(max(hA, 0), full) + full / 2) / full;
          const int32_t qB = cutB ? 0 : (255 * min(max(hB, 0), full) + full / 2) / full;
          if (out_ok && hasA) p.out8[size_t(rA) * p.cols + gcol] = uint8_t(qA);
          if (out_ok && hasB) p.out8[size_t(rB) * p.cols + gcol] = uint8_t(qB);
        }
      }
    }
  } else {
    // (h + 0x8000 - t) per half: bit 15 set iff h >= t (t clamped to +-0x4000 by the host)
    const uint32_t kt = imad(runc, 0xFFFFFFFEu, kh + (0x8000u - uint32_t(p.t_half)) * 0x00010001u);
    uint32_t any = 0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) any |= imad(cab[c], 0xFFFFFFFEu, kt);
    // Row-major ranks: a hit's rank in its (row, segment) = the row's earlier
    // hits (previous chunks, lower lanes of this chunk, lower columns of this lane).
    if (__any_sync(0xFFFFFFFFu, any & 0x80008000u)) {
      uint32_t hmA = 0, hmB = 0;   // threshold hits of this lane's columns (bit c)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int32_t e = eb + c;
        const bool real = NB % L == 0 || j * CPL + c < NB;
        const bool valid = real && (!CHECK || (e >= 0 && e < int32_t(nseg_cols)));
        const int32_t kp = kp0 + c;
        const bool out_ok = valid && (!CHECK || (kp >= 0 && kp < int32_t(p.S))) && !(uint32_t(kp) & rshift);
        const uint32_t ht = imad(cab[c], 0xFFFFFFFEu, kt);
        hmA |= uint32_t(out_ok && hasA && (ht & 0x8000u)) << c;
        hmB |= uint32_t(out_ok && hasB && (ht & 0x80000000u)) << c;
      }
      const uint32_t nA = __popc(hmA), nB = __popc(hmB);
      const uint32_t pk = nA | (nB << 16);
      uint32_t gi = pk;
#pragma unroll
      for (int off = 1; off < L; off <<= 1) {
        const uint32_t v = shfl_up_n<L>(gi, off);
        if (j >= uint32_t(off)) gi += v;
      }
      const uint32_t gex = gi - pk;
      const uint32_t gtot = shfl_group_last<L>(gi, g);
      uint32_t wi = nA + nB;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, wi, off);
        if (lane >= uint32_t(off)) wi += v;
      }
      const uint32_t wtot = __shfl_sync(0xFFFFFFFFu, wi, 31);
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(p.cursor, (unsigned long long)wtot);
      pos = __shfl_sync(0xFFFFFFFFu, pos, 0) + (wi - nA - nB);
      uint32_t rkA = hitsA + (gex & 0xFFFFu), rkB = hitsB + (gex >> 16);
      const uint32_t kb = imad(runc, 0xFFFFFFFEu, kh + 0x80008000u);
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const uint32_t gcol = (c0 + uint32_t(kp0 + c)) >> rshift;
        const uint32_t hb = imad(cab[c], 0xFFFFFFFEu, kb);
        const uint32_t hA = uint32_t(int32_t(hb & 0xFFFFu) - 0x8000), hB = uint32_t(int32_t(hb >> 16) - 0x8000);
        if ((hmA >> c) & 1u) {
          if (pos < p.stage_cap) p.stage[pos] = make_uint4(p.row_global0 + rA, gcol, hA, rkA);
          ++pos;
          ++rkA;
        }
        if ((hmB >> c) & 1u) {
          if (pos < p.stage_cap) p.stage[pos] = make_uint4(p.row_global0 + rB, gcol, hB, rkB);
          ++pos;
          ++rkB;
        }
      }
      hitsA += gtot & 0xFFFFu;
      hitsB += gtot >> 16;
    }
  }
}

template <int L, int NB, bool DENSE, bool CHECK>
__device__ __forceinline__ void extract_body(const CombParams& p, const uint32_t* ringB, uint32_t okb,
                                              uint32_t rmask, uint32_t j, uint32_t g, uint32_t lane,
                                              int32_t E0, uint32_t nseg_cols, int32_t kbase, uint32_t c0,
                                              uint32_t rA, uint32_t rB, bool hasA, bool hasB,
                                              uint32_t& run, uint32_t& hitsA, uint32_t& hitsB) {
  constexpr int CPL = (NB + L - 1) / L;
  uint32_t cab[CPL], o[CPL];
  extract_scatter<L, NB, CHECK, 0>(p, ringB, okb, rmask, j, E0, nseg_cols, kbase, cab);
  __syncwarp();
  extract_flags<L, NB, CHECK>(p, okb, rmask, j, E0, nseg_cols, o);
  extract_clear<L, NB>(p, okb, rmask, j, E0);
  extract_out<L, NB, DENSE, CHECK>(p, j, g, lane, E0, nseg_cols, c0, cab, o, rA, rB, hasA, hasB, run, hitsA,
                                   hitsB);
}

// Chunks whose bottom columns and window starts all lie inside the segment
// (every chunk but the first few and the last) skip the per-column range checks.
template <int L, int NB, bool DENSE>
__device__ __forceinline__ void extract_chunk(const CombParams& p, const uint32_t* ringB, uint32_t okb,
                                              uint32_t rmask,
                                              uint32_t j, uint32_t g, uint32_t lane,
                                              int32_t E0, uint32_t nseg_cols, int32_t kbase, uint32_t c0,
                                              uint32_t rA, uint32_t rB, bool hasA, bool hasB,
                                              uint32_t& run, uint32_t& hitsA, uint32_t& hitsB) {
  const bool interior = E0 >= int32_t(p.W) - 1 &&
                        E0 + NB <= min(int32_t(nseg_cols), int32_t(p.S + p.W) - 1);
  if (interior)
    extract_body<L, NB, DENSE, false>(p, ringB, okb, rmask, j, g, lane, E0, nseg_cols, kbase, c0, rA, rB, hasA, hasB,
                                      run, hitsA, hitsB);
  else
    extract_body<L, NB, DENSE, true>(p, ringB, okb, rmask, j, g, lane, E0, nseg_cols, kbase, c0, rA, rB, hasA, hasB,
                                     run, hitsA, hitsB);
}

// Comb kernel (K2): fused $-interleave, seaweed combing, window extraction
// and output for one (strip-pair group, column segment) task per warp.
//
// Shape: L lanes per strip pair, R rows per lane, split into K bands of R/K
// rows.  Band b of lane j ("virtual band" v = j*K + b) processes column s - v
// at step s, so the K chains of a lane are independent within a step (ILP K);
// band 0 gets the seaweed leaving lane j-1's last band one step earlier via
// SHFL, band b>0 the one its own band b-1 produced one step earlier.  The y
// codes travel the same way, one step ahead, so a step's table rows can be
// loaded as soon as the step starts.
//
// Cell (both strips in 16-bit halves): d = max_s16(T + A, V) (VIADDMNMX),
// V' = V ^ T ^ d (LOP3), with A = 0x8000 (-32768) on a match and 0 otherwise:
// two ALU-pipe ops per cell pair.  Keys stay in [0, 0x7BFF], so T - 32768 < 0
// <= V on a match.
// XM = false (small alphabets): per-group table M[code][row] of the A words,
//   laid out [group][code][quad][lane] (conflict-free LDS.128); the y column
//   word code * 0x10001 gives the table offset by one IMAD.HI.
// XM = true (any alphabet): A computed from the x-code pair registers:
//   A = ~((xpair ^ y * 0x10001) + 0x7FFF7FFF) & 0x80008000 (bit 15 of a half
//   survives iff the codes are equal).
template <int L, int R, int K, bool DENSE, bool XM, bool HF>
__global__ void __launch_bounds__(kGenericWpc * 32, (R <= 16 ? 4 : (R <= 24 ? 3 : 2)) * 4 / kGenericWpc)
comb_kernel(const CombParams p) {
  constexpr int WPC = kGenericWpc;
  constexpr int kHfRows = HF ? AP_HF_ROWS : 0;   // rows of each quad whose V' is formed on the FMA pipe
  // the bottom keys of two steps per 8-byte ring store (long lanes only: the 128-register
  // shapes would spill the held key)
  constexpr bool kSts64 = AP_G_STS64 && R > 16;
  static_assert(32 % L == 0 && L >= 4, "lane groups must tile the warp");
  constexpr int kSU = L < 8 ? AP_SUBUNROLL_L4 : kSubUnroll;
  static_assert(R % (4 * K) == 0, "bands must hold whole LDS.128 quads");
  constexpr int G = 32 / L;
  constexpr int Q = R / 4;        // quads per lane
  constexpr int RB = R / K;       // rows per band
  constexpr int QB = RB / 4;      // quads per band
  constexpr int VB = L * K;       // virtual bands per strip (wavefront depth)
  constexpr uint32_t kTblMul = uint32_t(Q * L * 16) << 16;   // (code * 0x10001) -> code * table stride
  extern __shared__ __align__(16) unsigned char smem[];

  const uint32_t lane = lane_id();
  const uint32_t warp = WPC == 1 ? 0u : threadIdx.x >> 5;
  const uint32_t g = lane / L;
  const uint32_t j = lane % L;
  const size_t per_warp = comb_smem_per_warp(L, R, p.sigma, p.ring);
  unsigned char* wbase = smem + warp * per_warp;
  uint4* tbl = reinterpret_cast<uint4*>(wbase);                       // [G][sigma][Q][L] (+pad)
  // group stride of the table in uint4: with L < 8 a group's LDS.128 covers only
  // 64 B, so consecutive groups are shifted by 64 B to use the other bank half
  const size_t tgs = size_t(p.sigma) * Q * L + (L < 8 && p.sigma ? 4 : 0);
  const size_t tbytes = size_t(G) * tgs * 16;
  constexpr int RSG = ring_stride(L, kChunk);
  uint32_t* ringB = reinterpret_cast<uint32_t*>(wbase + tbytes) + g * RSG;
  const uint32_t okb = uint32_t(__cvta_generic_to_shared(wbase + tbytes)) +
                       ((G * RSG * 4 + 15) & ~15u) + g * uint32_t(ok_stride(p.ring));
  const uint32_t rshift = p.r - 1;

  const uint32_t npairs = (p.rows + 1) / 2;
  const uint32_t ngroups = (npairs + G - 1) / G;
  const uint32_t gsplit = min(p.g_split, ngroups);
  const uint64_t split_tasks = uint64_t(gsplit) * p.nseg;
  const uint64_t ntasks = split_tasks + uint64_t(ngroups - gsplit) * p.nseg2;
  const uint64_t wstride = uint64_t(gridDim.x) * WPC;
  if (p.sigma_cap != 0xFFFFFFFFu && *p.sigma_dev > p.sigma_cap) {   // speculative plan too small
    if (threadIdx.x == 0) *p.abort_flag = 1u;
    return;
  }

  for (uint64_t task = uint64_t(blockIdx.x) * WPC + warp; task < ntasks; task = next_task(p, task, wstride, lane, ntasks)) {
    CombParams pt = p;   // this task's segment width (short tail tasks: S2)
    uint32_t pg, seg;
    if (task < split_tasks) {
      pg = uint32_t(task / p.nseg);
      seg = uint32_t(task % p.nseg);
    } else {
      pg = gsplit + uint32_t((task - split_tasks) / p.nseg2);
      seg = uint32_t((task - split_tasks) % p.nseg2);
      pt.S = p.S2;
    }
    const uint32_t pair = pg * G + g;
    const uint32_t rA = 2 * pair, rB = 2 * pair + 1;
    const bool hasA = rA < p.rows, hasB = rB < p.rows;
    const uint32_t c0 = seg * pt.S;
    const uint32_t nseg_cols = min(pt.S + p.W - 1, p.N - c0);
    const uint32_t nsteps = nseg_cols + VB - 1;
    const uint32_t nch = (nsteps + kChunk - 1) / kChunk;

    // ---- mismatch table / x-code registers (fused $-interleave, scoring.cpp:5-17)
    __syncwarp();
    uint32_t xpair[XM ? R : 1];
    {
      uint32_t xa[R], xb[R];
#pragma unroll
      for (int rho = 0; rho < R; ++rho) {
        const uint32_t i = j * R + rho;
        uint32_t ca = 0x1FFu, cb = 0x1FFu;  // never equals a code (pad rows, missing strips)
        if (i < p.W) {
          if (p.r == 2 && !(i & 1u)) {
            ca = hasA ? p.sent_code : 0x1FFu;
            cb = hasB ? p.sent_code : 0x1FFu;
          } else {
            const uint32_t xi = i >> rshift;
            if (hasA) ca = p.xcode[size_t(rA) * p.h + xi];
            if (hasB) cb = p.xcode[size_t(rB) * p.h + xi];
            if (ca == 0xFFu) ca = 0x1FFu;   // byte absent from y: never matches
            if (cb == 0xFFu) cb = 0x1FFu;
          }
        }
        xa[rho] = ca;
        xb[rho] = cb;
      }
      if constexpr (XM) {
#pragma unroll
        for (int rho = 0; rho < R; ++rho) xpair[rho] = xa[rho] | (xb[rho] << 16);
      } else {
        uint4* tg = tbl + size_t(g) * tgs;
        for (uint32_t a = 0; a < p.sigma; ++a) {
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            uint32_t wv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rho = 4 * q + k;
              wv[k] = (xa[rho] == a ? 0x00008000u : 0u) | (xb[rho] == a ? 0x80000000u : 0u);
            }
            tg[(a * Q + q) * L + j] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
      for (uint32_t k = j; k < p.ring; k += L) sts_u32(okb + 4 * k, 0u);
    }
    __syncwarp();

    // table base of this lane; y column words are byte offsets of a code's quads
    const uint32_t tlb = uint32_t(__cvta_generic_to_shared(tbl + size_t(g) * tgs + j));
    const uint4* yq = reinterpret_cast<const uint4*>((j == 0 ? p.ycol : p.ycol_zero) + c0);
    // lane-select constants: the band-0 inputs are imad(shuffled, nz, own) on the
    // FMA pipe instead of selects (own = fresh key / new column word on lane 0, 0 elsewhere)
    const uint32_t nz = j != 0 ? 1u : 0u;
    const uint32_t finc = j == 0 ? 0x00010001u : 0u;

    uint32_t V[R];
#pragma unroll
    for (int rho = 0; rho < R; ++rho) V[rho] = 0u;     // left-boundary seaweeds: key 0
    uint32_t tb[K];     // seaweed leaving band b at the previous step
    uint32_t tb_prev = 0u;   // bottom key of the previous (even) step, stored with the next one
    uint32_t cd[K];     // y column word of band b at the current step
#pragma unroll
    for (int b = 0; b < K; ++b) { tb[b] = 0u; cd[b] = 0u; }
    int32_t kbase = -int32_t(p.W) - 1 - (HF ? int32_t(kHfBase) : 0);   // key(c) = c - kbase > W for top seaweeds
    uint32_t fresh = j == 0 ? uint32_t(-kbase) * 0x00010001u : 0u;   // key of column s, both halves
    const uint32_t rebase_by = HF ? (kHfRebaseAt - kHfBase - 2 * kChunk - VB - p.W) : kRebaseBy;
    const uint32_t one = p.one;
    const uint32_t tblmul = kTblMul * one;   // opaque: keeps IMAD.HI (FMA pipe), not LEA.HI (ALU)
    uint32_t run = 0u;
    uint32_t hitsA = 0u, hitsB = 0u;

    // group lane 0's y words: a queue of the next 16 columns, refilled 8 at a time
    // (register moves and IMADs only: no byte extraction on the ALU pipe)
    uint4 qa = __ldg(yq), qb = __ldg(yq + 1), qc = __ldg(yq + 2), qd = __ldg(yq + 3);
    cd[0] = qa.x;                                      // column 0 (0 on lanes j != 0)
    uint32_t nsub = 0;

    for (uint32_t ch = 0; ch < nch; ++ch) {
#pragma unroll kSU
      for (int sub = 0; sub < kChunk / 8; ++sub, ++nsub) {
        const uint4 na = __ldg(yq + 2 * nsub + 4), nb = __ldg(yq + 2 * nsub + 5);
        uint32_t* ring_sub = ringB + sub * 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // table quads of this step (codes known since the previous step)
          uint4 nfq[Q];
          if constexpr (!XM) {
#pragma unroll
            for (int b = 0; b < K; ++b)
#pragma unroll
              for (int qq = 0; qq < QB; ++qq)
                nfq[b * QB + qq] = (b * QB + qq) % AP_ABL_LDS == 0
                                       ? lds128(madhi(cd[b], tblmul, tlb) + (b * QB + qq) * L * 16)
                                       : nfq[(b * QB + qq) - (b * QB + qq) % AP_ABL_LDS];
          }
          // seaweeds entering each band
          uint32_t tin[K];
          {
            const uint32_t sh = shfl_up1<L>(tb[K - 1]);
            tin[0] = imad(sh, nz, fresh);
#pragma unroll
            for (int b = 1; b < K; ++b) tin[b] = tb[b - 1];
          }
          fresh = imad(fresh, one, finc);
#pragma unroll
          for (int b = 0; b < K; ++b) {
            uint32_t t = tin[b];
            const uint32_t yrep = cd[b];                 // code * 0x10001
#pragma unroll
            for (int qq = 0; qq < QB; ++qq) {
              uint32_t m[4];
              if constexpr (XM) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  m[k] = ~((xpair[b * RB + 4 * qq + k] ^ yrep) + 0x7FFF7FFFu) & 0x80008000u;
              } else {
                const uint4 w4 = nfq[b * QB + qq];
                m[0] = w4.x; m[1] = w4.y; m[2] = w4.z; m[3] = w4.w;
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                uint32_t& v = V[b * RB + 4 * qq + k];
                const uint32_t d = __viaddmax_s16x2(t, m[k], v);   // max(T + A, V): A = -32768 on a match
                if (k < kHfRows) v = hadd2u(hsub2u(v, d), t);   // fp16 keys: V + T - d, exact
                else v = lop3_xor(v, t, d);
                t = d;
              }
            }
            tb[b] = t;
          }
          if constexpr (kSts64) {
            if (u & 1) {
              if (j == L - 1) *reinterpret_cast<uint2*>(ring_sub + u - 1) = make_uint2(tb_prev, tb[K - 1]);
            } else {
              tb_prev = tb[K - 1];
            }
          } else {
            if (j == L - 1) ring_sub[u] = tb[K - 1];
          }
          // codes of the next step: band b takes band b-1's, band 0 lane j-1's last band's
          {
            const uint32_t ynew = u == 0 ? qa.y : u == 1 ? qa.z : u == 2 ? qa.w : u == 3 ? qb.x :
                                  u == 4 ? qb.y : u == 5 ? qb.z : u == 6 ? qb.w : qc.x;
            const uint32_t sh = shfl_up1<L>(cd[K - 1]);
#pragma unroll
            for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
            cd[0] = imad(sh, nz, ynew);
          }
        }
        qa = qc; qb = qd; qc = na; qd = nb;
      }
      __syncwarp();

      extract_chunk<L, kChunk, DENSE>(pt, ringB, okb, p.ring - 1, j, g, lane,
                                      int32_t(ch * kChunk) - (VB - 1), nseg_cols, kbase, c0, rA, rB,
                                      hasA, hasB, run, hitsA, hitsB);

      // ---- key rebase (saturating at 0): fresh keys stay below 0x7BFF (fp16-finite)
      if (uint32_t(int32_t((ch + 2) * kChunk) - kbase) >= (HF ? kHfRebaseAt : kRebaseAt)) {
        const uint32_t by = rebase_by * 0x00010001u;
        const uint32_t fl = (HF ? kHfBase : 0u) * 0x00010001u + by;   // saturated keys -> the floor
#pragma unroll
        for (int rho = 0; rho < R; ++rho) V[rho] = __vmaxu2(V[rho], fl) - by;
#pragma unroll
        for (int b = 0; b < K; ++b) tb[b] = __vmaxu2(tb[b], fl) - by;
        if (j == 0) fresh -= by;
        kbase += int32_t(rebase_by);
      }
    }
    if constexpr (!DENSE) {
      if (j == 0) {
        if (hasA) p.seg_counts[size_t(rA) * p.seg_stride + seg] = hitsA;
        if (hasB) p.seg_counts[size_t(rB) * p.seg_stride + seg] = hitsB;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Alignment-score kernel (r = 2) specialised on the $-interleave
// (scoring.cpp:5-17).  In the blown strip x'[2i] = y'[2k] = $ and windows start
// at even offsets, so every cell's match status is static except real x real:
//   ($ row, $ col)    always match   -> the two seaweeds swap: zero instructions
//   ($ row, real col) never match    -> d = max(V,T), V' = min(V,T)
//   (real row, $ col) never match    -> same
//   (real row, real col)             -> table mask: VIADDMNMX + LOP3
// (SURVEY.md §7 hard part 8).  A step is one raw column = the blown columns
// 2c ($) and 2c+1 (real); two seaweeds per band move down per step.  The
// table holds only real rows and real codes.  R = 2*RR blown rows per lane,
// K bands of RRB = RR/K real rows; lanes j >= W/R (if any) are idle padding
// whose output is never read (the bottom is lane W/R - 1's last band).
// r = 2 table layout: quads [code][band][quad][lane] (uint4) and the REM =
// RRB % 4 (0..2) leftover words [code][band][lane] (uint32 / uint2), lane =
// g*L + j.  For a fixed (band, quad) the 32 lanes read 32 consecutive 16-B
// slots whatever code each lane holds: conflict-free LDS.128 for every L.
__host__ __device__ constexpr int r2_band_words(int rrb) { return rrb; }

// tq/tr point at this (code, band) block, already offset by the lane.
template <int RRB>
__device__ __forceinline__ void load_band_words(const uint4* tq, const uint32_t* tr, uint32_t* m) {
  constexpr int Q4 = RRB / 4, REM = RRB % 4;
  static_assert(REM <= 2, "band real-row count must be 4q, 4q+1 or 4q+2");
#pragma unroll
  for (int q = 0; q < Q4; ++q) {
    const uint4 v = tq[q * 32];
    m[4 * q] = v.x; m[4 * q + 1] = v.y; m[4 * q + 2] = v.z; m[4 * q + 3] = v.w;
  }
  if constexpr (REM == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(tr);
    m[4 * Q4] = v.x; m[4 * Q4 + 1] = v.y;
  } else if constexpr (REM == 1) {
    m[4 * Q4] = *tr;
  }
}

#ifndef AP_R2_SHORT_WARPS
#define AP_R2_SHORT_WARPS 16   // resident warps per SM the short-lane (RR < 8) r = 2 shapes are compiled for
#endif
__host__ __device__ constexpr int r2_min_blocks(int rr) {
  return rr < 8 ? AP_R2_SHORT_WARPS / r2_wpc(rr) : (rr <= AP_R2_MB4 ? 4 : (rr <= 16 ? 3 : 2)) * 4 / r2_wpc(rr);
}
template <int L, int RR, int K, bool DENSE, bool HF>
__global__ void __launch_bounds__(r2_wpc(RR) * 32, r2_min_blocks(RR))
comb2_kernel(const CombParams p) {
  constexpr int WPC = r2_wpc(RR);
  static_assert(L <= 32 && RR % K == 0, "bad shape");
  constexpr int G = groups_per_warp(L);     // real groups; lanes >= G*L are idle
  constexpr int R = 2 * RR;
  constexpr int RRB = RR / K;
  constexpr int BW = r2_band_words(RRB);
  constexpr int Q4 = RRB / 4, REM = RRB % 4;
  constexpr int NB = 2 * kChunk;   // blown bottom columns per chunk
  constexpr int kSubUnroll2 = RR <= AP_SUBUNROLL2_RR ? kChunk / 8 : 1;
  constexpr bool kFmaMin = RR >= AP_FMAMIN_RR;  // one of the two mismatch mins moves to the FMA pipe
  constexpr bool kSubLoad = AP_R2_SUBLOAD && kSubUnroll2 == 1;   // C2 -0.5%; unrolled shapes: +3.7% (C4)
  constexpr bool kYcol = r2_ycol_feed(RR, K);
  extern __shared__ __align__(16) unsigned char smem[];

  const uint32_t lane = lane_id();
  const uint32_t warp = WPC == 1 ? 0u : threadIdx.x >> 5;
  const uint32_t g = lane / L;
  const uint32_t j = lane % L;
  const size_t per_warp = comb_smem_per_warp(L, K * BW, p.sigma, p.ring, NB);
  unsigned char* wbase = smem + warp * per_warp;
  uint4* tblq = reinterpret_cast<uint4*>(wbase);                       // [sigma][K][Q4][32 lanes]
  uint32_t* tblr = reinterpret_cast<uint32_t*>(tblq + size_t(p.sigma) * K * Q4 * 32);  // [sigma][K][32][REM]
  const size_t tbl_bytes = size_t(4) * 32 * p.sigma * K * BW;
  constexpr int RS = ring_stride(L, NB);
  uint32_t* ringB = reinterpret_cast<uint32_t*>(wbase + tbl_bytes) + g * RS;
  const uint32_t okb = uint32_t(__cvta_generic_to_shared(wbase + tbl_bytes)) +
                       ((groups_alloc(L) * RS * 4 + 15) & ~15u) + g * uint32_t(ok_stride(p.ring));
  // the phantom group (lanes >= G*L) folds every ok slot onto its 64-byte scratch
  const uint32_t okmask = g < uint32_t(G) ? p.ring - 1 : 0u;

  const uint32_t lanes_real = p.W / R;          // host guarantees W % R == 0, lanes_real <= L
  const uint32_t VB = lanes_real * K;           // virtual bands down to the strip bottom
  const uint32_t npairs = (p.rows + 1) / 2;
  const uint32_t ngroups = (npairs + G - 1) / G;
  const uint32_t gsplit = min(p.g_split, ngroups);
  const uint64_t split_tasks = uint64_t(gsplit) * p.nseg;
  const uint64_t ntasks = split_tasks + uint64_t(ngroups - gsplit) * p.nseg2;
  const uint64_t wstride = uint64_t(gridDim.x) * WPC;
  if (p.sigma_cap != 0xFFFFFFFFu && *p.sigma_dev > p.sigma_cap) {   // speculative plan too small
    if (threadIdx.x == 0) *p.abort_flag = 1u;
    return;
  }

  for (uint64_t task = uint64_t(blockIdx.x) * WPC + warp; task < ntasks; task = next_task(p, task, wstride, lane, ntasks)) {
    CombParams pt = p;   // this task's segment width (short tail tasks: S2)
    uint32_t pg, seg;
    if (task < split_tasks) {
      pg = uint32_t(task / p.nseg);
      seg = uint32_t(task % p.nseg);
    } else {
      pg = gsplit + uint32_t((task - split_tasks) / p.nseg2);
      seg = uint32_t((task - split_tasks) % p.nseg2);
      pt.S = p.S2;
    }
    const uint32_t pair = pg * G + g;
    const uint32_t rA = 2 * pair, rB = 2 * pair + 1;
    const bool hasA = g < uint32_t(G) && rA < p.rows, hasB = g < uint32_t(G) && rB < p.rows;
    const uint32_t c0 = seg * pt.S;                        // blown, multiple of 64
    const uint32_t c0r = c0 >> 1;                          // raw, multiple of 32
    const uint32_t nseg_cols = min(pt.S + p.W - 1, p.N - c0);
    const uint32_t nraw = (nseg_cols + 1) >> 1;
    const uint32_t nsteps = nraw + VB - 1;
    const uint32_t nch = (nsteps + kChunk - 1) / kChunk;

    // ---- real-row multiplier table (real rows only, real codes only)
    __syncwarp();
    {
      uint32_t xa[RR], xb[RR];
#pragma unroll
      for (int i = 0; i < RR; ++i) {
        const uint32_t xi = j * RR + i;            // raw offset in the x-window
        uint32_t ca = 0x1FFu, cb = 0x1FFu;
        if (xi < p.w) {
          if (hasA) ca = p.xcode[size_t(rA) * p.h + xi];
          if (hasB) cb = p.xcode[size_t(rB) * p.h + xi];
          if (ca == 0xFFu) ca = 0x1FFu;
          if (cb == 0xFFu) cb = 0x1FFu;
        }
        xa[i] = ca;
        xb[i] = cb;
      }
      for (uint32_t a = 0; a < p.sigma; ++a) {
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const size_t ab = size_t(a) * K + b;
          uint32_t wv[RRB];
#pragma unroll
          for (int i = 0; i < RRB; ++i) {
            const int rr = b * RRB + i;
            wv[i] = (xa[rr] == a ? 0x00008000u : 0u) | (xb[rr] == a ? 0x80000000u : 0u);
          }
#pragma unroll
          for (int q = 0; q < Q4; ++q)
            tblq[(ab * Q4 + q) * 32 + lane] = make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
#pragma unroll
          for (int k = 0; k < REM; ++k) tblr[(ab * 32 + lane) * REM + k] = wv[4 * Q4 + k];
        }
      }
      for (uint32_t k = j; k <= okmask; k += L) sts_u32(okb + 4 * k, 0u);
    }
    __syncwarp();

    const uint4* tq0 = tblq + lane;
    const uint32_t* tr0 = tblr + size_t(lane) * REM;
    const uint32_t* yw = reinterpret_cast<const uint32_t*>(p.ycode + c0r);

    uint32_t V[R];
#pragma unroll
    for (int i = 0; i < R; ++i) V[i] = 0u;
    uint32_t tbD[K], tbR[K], cd[K];
#pragma unroll
    for (int b = 0; b < K; ++b) { tbD[b] = 0u; tbR[b] = 0u; cd[b] = 0u; }
    int32_t kbase = -int32_t(p.W) - 1 - (HF ? int32_t(kHfBase) : 0);
    uint32_t fresh = uint32_t(-kbase) * 0x00010001u;   // key of blown column 2s
#if AP_R2_IMADSEL
    const uint32_t nz2 = j != 0 ? 1u : 0u;
    const uint32_t finc2 = j == 0 ? 0x00020002u : 0u;
    uint32_t freshD0 = j == 0 ? fresh : 0u, freshR0 = j == 0 ? fresh + 0x00010001u : 0u;
#endif
    // rebase step: with the fp16 encoding as large as keeps every seaweed that a
    // later window can count (starts >= the next chunk's E0 - W + 1)
    const uint32_t rebase_by = HF ? (kHfRebaseAt - kHfBase - 2 * kChunk - 2 * VB - p.W) & ~1u : kRebaseBy;
    uint32_t run = 0u, hitsA = 0u, hitsB = 0u;

    // y codes: the unrolled sub loop (small RR) selects its words statically from two uint4
    // per chunk; the rolled one (kSubLoad) reads code words 2s, 2s+1 and 2s+2 (the next
    // step's code) per sub s, prefetched one sub ahead, instead of selecting by sub index
    uint32_t w0n = 0, w1n = 0, w2n = 0, wi = 3;
    uint4 ych = make_uint4(0, 0, 0, 0), ych2 = ych;
    // column-word feed (kYcol): 8 words per sub from a register queue, the next 8 in flight;
    // a band's table address is IMAD(word, 1, lane base)
    const uint4* yq = reinterpret_cast<const uint4*>((j == 0 ? p.ycol : p.ycol_zero) + c0r);
    uint4 qa = make_uint4(0, 0, 0, 0), qb = qa;
    uint32_t nsubq = 0;
    const uint32_t nzy = j != 0 ? 1u : 0u;
    const uint32_t tq32 = uint32_t(__cvta_generic_to_shared(tq0));
    const uint32_t tr32 = uint32_t(__cvta_generic_to_shared(tr0));
    if constexpr (kYcol) {
      qa = __ldg(yq); qb = __ldg(yq + 1);
      cd[0] = qa.x;
    } else if constexpr (kSubLoad) {
      w0n = __ldg(yw); w1n = __ldg(yw + 1); w2n = __ldg(yw + 2);
      if (j == 0) cd[0] = w0n & 0xFFu;
    } else {
      ych = __ldg(reinterpret_cast<const uint4*>(yw));
      ych2 = __ldg(reinterpret_cast<const uint4*>(yw) + 1);
      if (j == 0) cd[0] = ych.x & 0xFFu;
    }

    for (uint32_t ch = 0; ch < nch; ++ch) {
      uint4 nxa = make_uint4(0, 0, 0, 0), nxb = nxa;
      if constexpr (!kSubLoad) {
        nxa = __ldg(reinterpret_cast<const uint4*>(yw) + 2 * ch + 2);
        nxb = __ldg(reinterpret_cast<const uint4*>(yw) + 2 * ch + 3);
      }
#pragma unroll kSubUnroll2
      for (int sub = 0; sub < kChunk / 8; ++sub) {
        uint32_t w0 = 0, w1 = 0, w2 = 0;
        uint4 na = make_uint4(0, 0, 0, 0), nb = na;
        if constexpr (kYcol) {
          na = __ldg(yq + 2 * nsubq + 2);
          nb = __ldg(yq + 2 * nsubq + 3);
          ++nsubq;
        } else if constexpr (kSubLoad) {
          w0 = w0n; w1 = w1n; w2 = w2n;
          w0n = w2n;
          w1n = __ldg(yw + wi);
          w2n = __ldg(yw + wi + 1);
          wi += 2;
        } else {
          w0 = sub == 0 ? ych.x : sub == 1 ? ych.z : sub == 2 ? ych2.x : ych2.z;
          w1 = sub == 0 ? ych.y : sub == 1 ? ych.w : sub == 2 ? ych2.y : ych2.w;
          w2 = sub == 0 ? ych.z : sub == 1 ? ych2.x : sub == 2 ? ych2.z : nxa.x;
        }
        uint32_t* ring_sub = ringB + sub * 16;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t m[K][RRB];
#pragma unroll
          for (int b = 0; b < K; ++b) {
            if constexpr (kYcol) {
              if constexpr (Q4 == 0) {
                const uint32_t a = imad(cd[b], p.one, tr32) + b * (32 * REM * 4);
                if constexpr (REM == 2) lds_v2(a, m[b]);
                else m[b][0] = lds_u32(a);
              } else {
                const uint32_t a = imad(cd[b], p.one, tq32) + b * (Q4 * 512);
#pragma unroll
                for (int q = 0; q < Q4; ++q) lds_v4(a + q * 512, m[b] + 4 * q);
              }
            } else {
              const uint32_t ab = cd[b] * K + b;
              load_band_words<RRB>(tq0 + ab * (Q4 * 32), tr0 + ab * (32 * REM), m[b]);
            }
          }
          uint32_t tinD[K], tinR[K];
          {
            const uint32_t shD = shfl_up1<L>(tbD[K - 1]);
            const uint32_t shR = shfl_up1<L>(tbR[K - 1]);
#if AP_R2_IMADSEL
            tinD[0] = imad(shD, nz2, freshD0);   // lane-0 injection on the FMA pipe (no SEL)
            tinR[0] = imad(shR, nz2, freshR0);
#else
            tinD[0] = j == 0 ? fresh : shD;
            tinR[0] = j == 0 ? fresh + 0x00010001u : shR;
#endif
#pragma unroll
            for (int b = 1; b < K; ++b) { tinD[b] = tbD[b - 1]; tinR[b] = tbR[b - 1]; }
          }
#if AP_R2_IMADSEL
          freshD0 = imad(freshD0, p.one, finc2);
          freshR0 = imad(freshR0, p.one, finc2);
#else
          fresh += 0x00020002u;
#endif
#pragma unroll
          for (int b = 0; b < K; ++b) {
            uint32_t t = tinD[b];                       // blown column 2c: $
#pragma unroll
            for (int i = 0; i < RRB; ++i) {
              uint32_t& vs = V[b * 2 * RRB + 2 * i];     // $ row: match -> swap
              const uint32_t sw = vs;
              vs = t;
              t = sw;
              uint32_t& vr = V[b * 2 * RRB + 2 * i + 1]; // real row: mismatch
              const uint32_t d = __vmaxu2(vr, t);
              vr = __vminu2(vr, t);
              t = d;
            }
            tbD[b] = t;
            t = tinR[b];                                // blown column 2c+1: real char
#pragma unroll
            for (int i = 0; i < RRB; ++i) {
              uint32_t& vs = V[b * 2 * RRB + 2 * i];     // $ row: mismatch
              const uint32_t d0 = __vmaxu2(vs, t);
              if constexpr (HF) {
                vs = hadd2u(hsub2u(vs, d0), t);   // fp16: (vs - max) + t = min, exact
              } else if constexpr (kFmaMin) {
                // min(vs, t) = vs + t - max(vs, t) as two IMADs on the otherwise idle
                // FMA pipe (16-bit halves never carry): unloads the ALU pipe, which
                // this kernel saturates at RR >= 8 (C2: 7.27 -> 6.95 ms on B200)
                uint32_t sum;
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(sum) : "r"(vs), "r"(p.one), "r"(t));
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(vs) : "r"(d0), "r"(p.minus_one), "r"(sum));
              } else {
                vs = __vminu2(vs, t);
              }
              t = d0;
              uint32_t& vr = V[b * 2 * RRB + 2 * i + 1]; // real x real: table
              const uint32_t d1 = __viaddmax_s16x2(t, m[b][i], vr);
              vr = lop3_xor(vr, t, d1);
              t = d1;
            }
            tbR[b] = t;
          }
          if (j == lanes_real - 1) {
            if constexpr (AP_R2_STS64) {
              *reinterpret_cast<uint2*>(ring_sub + 2 * u) = make_uint2(tbD[K - 1], tbR[K - 1]);
            } else {
              ring_sub[2 * u] = tbD[K - 1];
              ring_sub[2 * u + 1] = tbR[K - 1];
            }
          }
          if constexpr (kYcol) {
            const uint32_t ynew = u == 0 ? qa.y : u == 1 ? qa.z : u == 2 ? qa.w : u == 3 ? qb.x :
                                  u == 4 ? qb.y : u == 5 ? qb.z : u == 6 ? qb.w : na.x;
            const uint32_t sh = shfl_up1<L>(cd[K - 1]);
#pragma unroll
            for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
            cd[0] = imad(sh, nzy, ynew);
          } else {
            const uint32_t ww = u < 3 ? w0 : (u < 7 ? w1 : w2);
#if AP_R2_PRMT
            const uint32_t ynew = __byte_perm(ww, 0u, 0x4440u | uint32_t((u + 1) & 3));   // one PRMT
#else
            const uint32_t ynew = (ww >> (8 * ((u + 1) & 3))) & 0xFFu;
#endif
            const uint32_t sh = shfl_up1<L>(cd[K - 1]);
#pragma unroll
            for (int b = K - 1; b > 0; --b) cd[b] = cd[b - 1];
            cd[0] = j == 0 ? ynew : sh;
          }
        }
        if constexpr (kYcol) { qa = na; qb = nb; }
      }
      ych = nxa;
      ych2 = nxb;
      __syncwarp();
      extract_chunk<L, NB, DENSE>(pt, ringB, okb, okmask, j, g, lane,
                                  2 * (int32_t(ch * kChunk) - int32_t(VB - 1)), nseg_cols, kbase, c0, rA,
                                  rB, hasA, hasB, run, hitsA, hitsB);
      if (uint32_t(int32_t((ch + 2) * NB) - kbase) >= (HF ? kHfRebaseAt : kRebaseAt)) {
        const uint32_t by = rebase_by * 0x00010001u;
        const uint32_t fl = (HF ? kHfBase : 0u) * 0x00010001u + by;   // saturated keys -> the floor
#pragma unroll
        for (int i = 0; i < R; ++i) V[i] = __vmaxu2(V[i], fl) - by;
#pragma unroll
        for (int b = 0; b < K; ++b) {
          tbD[b] = __vmaxu2(tbD[b], fl) - by;
          tbR[b] = __vmaxu2(tbR[b], fl) - by;
        }
        fresh -= by;
#if AP_R2_IMADSEL
        if (j == 0) { freshD0 -= by; freshR0 -= by; }
#endif
        kbase += int32_t(rebase_by);
      }
    }
    if constexpr (!DENSE) {
      if (j == 0) {
        if (hasA) p.seg_counts[size_t(rA) * p.seg_stride + seg] = hitsA;
        if (hasB) p.seg_counts[size_t(rB) * p.seg_stride + seg] = hitsB;
      }
    }
  }
}

}  // namespace apk
