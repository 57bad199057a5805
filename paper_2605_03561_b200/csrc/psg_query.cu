// The fused trace query on sm_100a: two passes over the event stream.
//
//   k_bounds       pass 1 — iteration boundaries per trace (itermodel.cpp:111-143):
//                  optimistic mode (default) reads ctx only (4 B/event) and
//                  takes every subtree entry as a boundary; exact mode also
//                  reads each candidate's timestamp and drops same-timestamp
//                  re-entries.  Writes the boundary event indices.
//   k_verify_bounds  after an optimistic pass 1: checks the boundary
//                  timestamps pass 2 recorded (no two equal, gap and
//                  iterations < 2^32 ns); a miss re-runs both passes exactly.
//   k_trace_query  pass 2 — ONE read of ts+ctx (12 B/event) computing
//                    * the window filter + per-(trace, ctx) count/sum/min/max/mean
//                      (ingest.cpp:178-208 + frame.cpp:290-408),
//                    * the time-integrated excl/incl of the window incl. the
//                      carry-in segment (itermodel.cpp:145-183),
//                    * the trace x iteration x node cube incl/excl + gap rows
//                      (itermodel.cpp:242-360), stored with 32-bit cells when
//                      every iteration spans < 2^32 ns,
//                    * exact integer sufficient statistics for the cross-rank and
//                      within-rank diagnostics (diagnostics.cpp:83-158).
//
// Work mapping (both passes): one warp per trace; each lane owns a run of R
// consecutive events of a 32*R-event block step, loaded with 128-bit vector
// loads (the block start is aligned down to 4 events so every run is 16-byte
// aligned).  The per-event logic is plain sequential register code inside a
// lane's run — no shuffles or ballots per event; warp-wide operations happen
// once per block step.  The next block steps are prefetched into L2 with the
// TMA bulk-prefetch (cp.async.bulk.prefetch.L2).  Accumulations go to
// warp-private shared-memory tables with native 32-bit shared atomics (a
// 64-bit value is carried through its two 32-bit halves; 64-bit shared
// atomics would be CAS loops).
//
// Everything on the event stream is integer arithmetic in nanoseconds, which
// is exact and order-free, so the results are bit-identical to the reference
// regardless of thread order.
//
//   k_cross_stats  the cross-rank (iteration, node) Σx, max, Σx² over the
//                  stored cube (diagnostics.cpp:83-158).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <mutex>

#include "psg_internal.h"

namespace psg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned long long kSpan32 = 1ull << 32;
typedef unsigned long long u64;
typedef unsigned __int128 u128;

// Tuning knobs (compile-time; tools/variants.sh builds alternatives for A/B runs).
#ifndef PSG_RM
#define PSG_RM 8
#endif
#ifndef PSG_PIPE_CROSS
#define PSG_PIPE_CROSS 1  // the register pipeline also runs across a chunk flush
#endif
#ifndef PSG_PIPE
#define PSG_PIPE 1  // register software pipeline of block-step loads in k_trace_query
#endif
// k_trace_query CTA shapes (query_params::one_warp, chosen per query on the
// host): one-warp CTAs, 17 resident per SM (96 registers per thread; 17
// carve-outs of ~10.6 KB keep the 196 KB shared-memory configuration, so
// 60 KB of L1 remain for the table reads) for long traces; 16-warp CTAs with
// the tables in shared memory for short ones (warps of a CTA start together:
// fewer instruction-cache misses in the per-trace prologue and epilogue).
#ifndef PSG_B_MINB
#define PSG_B_MINB 1  // k_bounds: resident 256-thread CTAs per SM the registers must allow
#endif
#ifndef PSG_B8_MINB
#define PSG_B8_MINB 8  // k_bounds, optimistic 1-byte-mirror pass: 8 CTAs (64 warps) per SM at 32
                       // registers, no spills (A/B: 0.862 -> 0.797 ms; 6 CTAs at 40: 0.824)
#endif
#ifndef PSG_X_MINB
#define PSG_X_MINB 2  // k_cross_stats: resident 512-thread CTAs per SM the registers must allow
#endif
#ifndef PSG_X_U
#define PSG_X_U 16  // k_cross_stats: 32-bit cell pairs in flight per thread (the batch size)
#endif
#ifndef PSG_WIDE_THREADS
#define PSG_WIDE_THREADS 512  // launch bound of the wide shape (PSG_WMAX warps per CTA)
#endif
#ifndef PSG_WIDE_MINB
#define PSG_WIDE_MINB 1
#endif
#ifndef PSG_ONE_MINB
#define PSG_ONE_MINB 17
#endif
#ifndef PSG_G
#define PSG_G 8
#endif
#ifndef PSG_FLUSH_UNROLL
#define PSG_FLUSH_UNROLL 1
#endif
constexpr int kFlushUnroll = PSG_FLUSH_UNROLL;
#ifndef PSG_COPY_UNROLL
#define PSG_COPY_UNROLL 4  // the flush's block copy (16-byte loads / zeroing / stores)
#endif
constexpr int kCopyUnroll = PSG_COPY_UNROLL;
#ifndef PSG_GEN_ALL
#define PSG_GEN_ALL 1  // general path: specialisations for interior block steps
#endif
#ifndef PSG_GEN_RT
#define PSG_GEN_RT 1  // general path: one copy with the window class at run time (-20 % code, A/B neutral)
#endif

#ifndef PSG_RB
#define PSG_RB 16
#endif
constexpr int RB = PSG_RB;  // events per lane per block step, pass 1 (ctx: RB/8 x 256-bit loads)
constexpr int RM = PSG_RM;  // events per lane per block step, pass 2 (ts: RM/2, ctx: RM/4 x 128-bit)
constexpr int STEP_B = 32 * RB;
constexpr uint32_t GC = PSG_G;  // iterations per chunk of pass 2 (the host passes the same G)
constexpr int STEP_M = 32 * RM;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// TMA bulk prefetch issued by lane 0 only, without a branch (predicated).
__device__ __forceinline__ void prefetch_l2_lane0(const void* p, uint32_t bytes, bool on) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.bulk.prefetch.L2.global [%0], %1;\n\t}" ::"l"(p),
      "r"(bytes), "r"(static_cast<uint32_t>(on))
      : "memory");
}

__device__ __forceinline__ u64 ldg64(const uint64_t* p) {
  return static_cast<u64>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// One block step's events for this lane (RM timestamps + ctx words from r0)
// and, on lane 31, the timestamp after the step.
#ifndef PSG_LD256
#define PSG_LD256 1
#endif
#ifndef PSG_SA
#define PSG_SA 8  // block steps start on multiples of SA events (4 or 8)
#endif
constexpr int SA = PSG_SA, SOFF = SA - 1;
// 32-byte read-only load (one LDG.256: every instruction fills whole 32-byte
// sectors, so no sector is fetched twice when L1 cannot hold it in between)
__device__ __forceinline__ void ldg256(const uint64_t* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}

// 32 ctx-word bytes (two uint4) in one LDG.256; p 32-byte aligned
__device__ __forceinline__ void ldg256x(const uint32_t* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

__device__ __forceinline__ void load_step(const trace_view& tr, u64 r0, u64 s_abs, int lane,
                                          ulonglong2 (&ts)[RM / 2], uint4 (&cx)[RM / 4], u64& nf) {
  if (PSG_LD256) {  // r0 is a multiple of 4 events: 32-byte aligned timestamps
#pragma unroll
    for (int q = 0; q < RM / 4; ++q)
      ldg256(tr.ts + r0 + 4 * q, ts[2 * q].x, ts[2 * q].y, ts[2 * q + 1].x, ts[2 * q + 1].y);
  } else {
    const ulonglong2* tsrc = reinterpret_cast<const ulonglong2*>(tr.ts + r0);
#pragma unroll
    for (int q = 0; q < RM / 2; ++q) ts[q] = __ldg(tsrc + q);
  }
  if (PSG_LD256 && SA == 8 && RM == 8) {  // r0 a multiple of 8 events: 32-byte aligned ctx words
    ldg256x(tr.ctx + r0, cx[0], cx[1]);
  } else {
    const uint4* csrc = reinterpret_cast<const uint4*>(tr.ctx + r0);
#pragma unroll
    for (int q = 0; q < RM / 4; ++q) cx[q] = __ldg(csrc + q);
  }
  if (lane == 31) nf = ldg64(tr.ts + s_abs + 32 * RM);
}

// Interleaved lane layout (pass 2, one-warp CTAs): lane l holds events l, l + 32,
// ..., l + 32 (RM - 1) of a block step, so the 32 lanes of one instruction
// hold 32 CONSECUTIVE events.  Consecutive events of a trace are mostly
// distinct contexts (sequential ids in a call sequence), so their window
// records and cube columns fall in distinct shared-memory banks; with runs of
// RM consecutive events per lane the lanes of an instruction touched contexts
// RM apart, which for an iteration of 67 contexts costs 2-3 wavefronts per
// shared access (measured: conflict-free addressing takes k_trace_query from
// 17.3 to 15.1 ms at configs[1], tools/ab_bench.sh).  Each load instruction
// reads 32 consecutive timestamps (256 B) or ctx words (128 B): whole sectors.
#ifndef PSG_PIPE_UNCOND
#define PSG_PIPE_UNCOND 1  // run layout: always load the next step (no branch)
#endif
// Rotating register pipeline (interleaved layout): as soon as event j of the
// current block step is consumed, its registers receive event j of the next
// step, so the loads of step s + 1 are in flight during step s without a
// second register set or the copy between them.
#define PSG_ROT 1
// the rotating pipeline's source: this lane's events of the step at lp
struct rot_src {
  const unsigned long long* ts;  // tr.ts + lp + lane
  const unsigned int* ctx;       // tr.ctx + lp + lane
};
__device__ __forceinline__ void rot_load(const rot_src& r, int j, u64 (&tv)[RM + 1], uint32_t (&cv)[RM]) {
  tv[j] = __ldg(r.ts + 32 * j);
  cv[j] = __ldg(r.ctx + 32 * j);
}
// lane 31 also loads the event after the step once j = RM - 1 is consumed
__device__ __forceinline__ void rot_tail(const rot_src& r, int lane, u64 (&tv)[RM + 1]) {
  if (lane == 31) tv[RM] = __ldg(r.ts + 32 * RM - 31);
}
__device__ __forceinline__ void load_step_il(const trace_view& tr, u64 s_abs, int lane, u64 (&ts)[RM],
                                             uint32_t (&cx)[RM], u64& nf) {
  const unsigned long long* tp = reinterpret_cast<const unsigned long long*>(tr.ts + s_abs) + lane;
  const unsigned int* cp = reinterpret_cast<const unsigned int*>(tr.ctx + s_abs) + lane;
#pragma unroll
  for (int j = 0; j < RM; ++j) ts[j] = __ldg(tp + 32 * j);
#pragma unroll
  for (int j = 0; j < RM; ++j) cx[j] = __ldg(cp + 32 * j);
  if (lane == 31) nf = ldg64(tr.ts + s_abs + 32 * RM);
}

// Timestamp of the event after (lane, j) in the interleaved layout: lane + 1's
// event j, lane 0's event j + 1 for lane 31, and the step's successor (tv[RM]
// on lane 31) for the last one.  Warp-uniform call (a shuffle).
__device__ __forceinline__ u64 next_ts_il(const u64 (&tv)[RM + 1], int j, int lane) {
  const u64 src = (lane == 0 && j + 1 < RM) ? tv[j + 1] : tv[j];
  const u64 x = __shfl_sync(FULL, src, (lane + 1) & 31);
  return (lane == 31 && j == RM - 1) ? tv[RM] : x;
}
__device__ __forceinline__ uint32_t next_lo_il(const u64 (&tv)[RM + 1], int j, int lane) {
  const uint32_t src = static_cast<uint32_t>((lane == 0 && j + 1 < RM) ? tv[j + 1] : tv[j]);
  const uint32_t x = __shfl_sync(FULL, src, (lane + 1) & 31);
  return (lane == 31 && j == RM - 1) ? static_cast<uint32_t>(tv[RM]) : x;
}

// 64-bit add into shared memory through two 32-bit words (lo, hi) with
// native 32-bit atomics: the carry of the low word is added to the high word.
__device__ __forceinline__ void sadd64(uint32_t* lo, uint32_t* hi, u64 v) {
  const uint32_t l = static_cast<uint32_t>(v);
  const uint32_t old = atomicAdd(lo, l);
  const uint32_t h = static_cast<uint32_t>(v >> 32) + (old + l < old ? 1u : 0u);
  if (h) atomicAdd(hi, h);
}

__device__ __forceinline__ double u128_to_double(u128 v) {
  return static_cast<double>(static_cast<u64>(v >> 64)) * 18446744073709551616.0 +
         static_cast<double>(static_cast<u64>(v));
}

// Exclusive prefix of n u64 values (src) into dst[0..n] by one warp.
__device__ __forceinline__ void warp_prefix(const u64* src, u64* dst, uint32_t n, int lane) {
  u64 carry = 0;
  for (uint32_t b = 0; b < n; b += 32) {
    const uint32_t j = b + lane;
    u64 v = j < n ? src[j] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u64 y = __shfl_up_sync(FULL, v, d);
      if (lane >= d) v += y;
    }
    if (j < n) dst[j + 1] = carry + v;
    carry += __shfl_sync(FULL, v, 31);
  }
  if (lane == 0) dst[0] = 0;
  __syncwarp();
}

}  // namespace

// ===========================================================================
// Pass 1: boundaries.  A boundary is an event entering the anchor subtree
// (contains[ctx] && !contains[previous ctx]) whose timestamp is strictly later
// than the previous candidate's (= the previous boundary's: timestamps are
// non-decreasing, so among candidates sharing a timestamp only the first is
// kept).  The number of iterations drops a zero-length last interval
// (boundary at t_end).  Boundary event indices are relative to the trace's
// first event.
//
// EXACT = false is the optimistic pass: it reads only ctx words (4 B/event)
// and takes every candidate as a boundary, with no timestamp loads (each one
// costs a whole 128-byte line from HBM) except the last candidate's.  It is
// exact unless two candidates share a timestamp; pass 2 reads every
// boundary's timestamp from its own stream, flags that case, and the host
// re-runs both passes with EXACT = true.
// C8: the ctx words come from the narrow mirror (1 B/event): a lane owns a run
// of 32 events (one 32-byte load), block steps of 1024 events start on
// multiples of 32 events.  Otherwise a lane owns RB events of u32 ctx words.
template <bool C8> struct bounds_geom {
  static constexpr int R = C8 ? 32 : RB;        // events per lane per block step
  static constexpr int STEP = 32 * R;
  static constexpr u64 ALIGN = C8 ? 31 : 7;     // block steps start on multiples of ALIGN + 1
  static constexpr int NV = C8 ? 2 : RB / 4;    // uint4 registers per lane per block step
};

// lanes' bits [lo, hi) of a 32-bit run mask (0 <= lo, hi <= 32)
__device__ __forceinline__ uint32_t run_mask(int lo, int hi) {
  const uint32_t h = hi >= 32 ? FULL : ((1u << hi) - 1u);
  const uint32_t l = lo >= 32 ? FULL : ((1u << lo) - 1u);
  return h & ~l;
}

template <bool SMALL, bool EXACT, bool C8>  // SMALL: <= 128 contexts, membership bits live in registers
__global__ void __launch_bounds__(256, (C8 && !EXACT) ? PSG_B8_MINB : PSG_B_MINB) k_bounds(bound_params p) {
  typedef bounds_geom<C8> GM;
  constexpr int RR = GM::R, STEP = GM::STEP, NV = GM::NV;
  extern __shared__ uint32_t s_bits[];
  for (uint32_t i = threadIdx.x; i < p.words; i += blockDim.x) s_bits[i] = p.contains[i];
  auto word = [&](uint32_t w) -> u64 { return w < p.words ? static_cast<u64>(p.contains[w]) : 0ull; };
  const u64 bits_lo = SMALL ? (word(0) | (word(1) << 32)) : 0ull;
  const u64 bits_hi = SMALL ? (word(2) | (word(3) << 32)) : 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= p.tr.n) return;
  const u64 b = p.tr.off[t], e = p.tr.off[t + 1];
  const u64 cap = p.cap_off[t + 1] - p.cap_off[t];
  const uint32_t lo4 = p.sub_lo * 0x01010101u, sz4 = p.sub_size * 0x01010101u;
  const bool sub_all = p.sub_size >= 256;
  const uint32_t c7lo = (128u - p.sub_lo) * 0x01010101u;                // ctx7: bytes >= lo
  const uint32_t c7hi = (128u - (p.sub_lo + p.sub_size)) * 0x01010101u;  // ctx7: bytes >= hi
#define BTS(i) ldg64(p.tr.ts + (i))
  uint32_t* out = p.bidx + p.cap_off[t];
  uint64_t* out_ts = p.bts + p.cap_off[t];
  uint32_t prev_in = 0;  // containment of the event before the block step
  bool have_c = false;   // a candidate has been seen ...
  u64 last_c = 0;        // ... with this timestamp
  u64 nb = 0, last_b = 0;
  // software pipeline: the next block step's ctx words are loaded into
  // registers while this one is processed (the arrays carry one block step of
  // slack past the last event).  Every load is one 32-byte aligned LDG.256
  // (whole sectors per instruction).
  static_assert(RB % 8 == 0, "RB must be a multiple of 8");
  uint4 nxt[NV];
  auto load = [&](u64 r) {
    if (C8) {
      ldg256x(reinterpret_cast<const uint32_t*>(p.ctx8 + r), nxt[0], nxt[1]);
    } else {
#pragma unroll
      for (int q = 0; q < NV / 2; ++q) ldg256x(p.tr.ctx + r + 8 * q, nxt[2 * q], nxt[2 * q + 1]);
    }
  };
  load((b & ~GM::ALIGN) + static_cast<u64>(lane) * RR);
  for (u64 s = b & ~GM::ALIGN; s < e; s += STEP) {
    const u64 r0 = s + static_cast<u64>(lane) * RR;
#ifndef PSG_NO_BOUNDS_PREFETCH
#ifndef PSG_B_PF_DIST
#define PSG_B_PF_DIST 0  // block steps of L2 prefetch run-ahead in pass 1 (0: none;
                         // with the 256-bit loads it no longer pays: 3.07 vs 3.04 ms)
#endif
    if (!C8 && PSG_B_PF_DIST > 0 && lane == 0 && s + (PSG_B_PF_DIST + 1) * STEP <= e)
      prefetch_l2(p.tr.ctx + s + PSG_B_PF_DIST * STEP, 4 * STEP);
#endif
#ifndef PSG_B8_PF_DIST
#define PSG_B8_PF_DIST 0  // C8: block steps of TMA L2 prefetch run-ahead (measured: 2, 3, 6 all slower;
                          // 1.33 vs 1.23 ms at configs[1])
#endif
    if (C8 && PSG_B8_PF_DIST > 0)
      prefetch_l2_lane0(p.ctx8 + s + PSG_B8_PF_DIST * STEP, STEP,
                        lane == 0 && s + (PSG_B8_PF_DIST + 1) * STEP <= e);
    uint32_t w[4 * NV];  // this step's ctx words (C8: 4 ctx bytes per word)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      w[4 * q] = nxt[q].x;
      w[4 * q + 1] = nxt[q].y;
      w[4 * q + 2] = nxt[q].z;
      w[4 * q + 3] = nxt[q].w;
    }
    // events of this trace in the lane's run: local indices [lo, hi) of [0, RR)
    // (interior block steps, warp-uniform: all of them)
    uint32_t real = FULL;
    if (s < b || s + STEP > e) {
      const int64_t lo64 = static_cast<int64_t>(b) - static_cast<int64_t>(r0);
      const int64_t hi64 = static_cast<int64_t>(e) - static_cast<int64_t>(r0);
      const int lo = lo64 < 0 ? 0 : static_cast<int>(lo64 > RR ? RR : lo64);
      const int hi = hi64 < 0 ? 0 : static_cast<int>(hi64 > RR ? RR : hi64);
      real = run_mask(lo, hi);
    }
    uint32_t inm = 0;
    if (C8 && p.ctx7) {
      // every preorder byte x < 128 (the top bit is free): x + (128 - lo) has
      // its top bit set iff x >= lo, x + (128 - hi) iff x >= hi, and neither
      // sum carries into the next byte (bytes past the trace may carry, but
      // only into later bytes, which are masked too) -- three ops per four
      // events.  Two words' top bits, interleaved by a shift, fold into eight
      // in-order bits with one high multiply (every partial product lands on
      // its own bit: no carries).
#pragma unroll
      for (int q = 0; q < RR / 8; ++q) {
        const uint32_t x0 = w[2 * q], x1 = w[2 * q + 1];
        const uint32_t m0 = (x0 + c7lo) & ~(x0 + c7hi) & 0x80808080u;
        const uint32_t m1 = (x1 + c7lo) & ~(x1 + c7hi) & 0x80808080u;
        inm |= (__umulhi((m0 >> 4) | m1, 0x20408100u) & 0xFFu) << (8 * q);
      }
    } else if (C8) {
      // preorder bytes: in the subtree iff (b - lo) mod 256 < size, four
      // events per SIMD compare; the four 0xff/0 bytes fold into a nibble
      // (bit k of byte k, summed into the top byte by one multiply)
#pragma unroll
      for (int q = 0; q < RR / 4; ++q) {
        const uint32_t m = sub_all ? FULL : __vcmpltu4(__vsub4(w[q], lo4), sz4);
        inm |= (((m & 0x08040201u) * 0x01010101u) >> 24) << (4 * q);
      }
    } else {
#pragma unroll
      for (int j = 0; j < RR; ++j) {
        const uint32_t c = w[j];
        uint32_t in;
        if (SMALL)  // ctx < 128 on real events
          in = static_cast<uint32_t>((c & 64 ? bits_hi : bits_lo) >> (c & 63)) & 1u;
        else
          in = (s_bits[min(c, p.words * 32 - 1) >> 5] >> (c & 31)) & 1u;
        inm |= in << j;
      }
    }
    inm &= real;
    // the next block step's words load into the registers this one's just
    // left (no copy between register sets; in flight during the rest)
    if (s + STEP < e) load(r0 + STEP);
    uint32_t up = __shfl_up_sync(FULL, inm >> (RR - 1), 1);
    if (lane == 0) up = prev_in;
    const uint32_t candm = inm & ~((inm << 1) | (up & 1u));
    prev_in = __shfl_sync(FULL, (inm >> (RR - 1)) & 1u, 31);
    const unsigned any = __ballot_sync(FULL, candm != 0);
    if (!any) continue;
    if (!EXACT) {  // every candidate is a boundary (verified by pass 2)
      const uint32_t nbl = __popc(candm);
      uint32_t inc = nbl;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, d);
        if (lane >= d) inc += y;
      }
      u64 kk = nb + inc - nbl;
      for (uint32_t m = candm; m; m &= m - 1, ++kk)
        if (kk < cap) out[kk] = static_cast<uint32_t>(r0 + (__ffs(m) - 1) - b);
      nb += __shfl_sync(FULL, inc, 31);
      continue;
    }
    // timestamp of this lane's last candidate; the previous candidate before
    // this lane's first one comes from the nearest lower lane with candidates
    u64 my_last = 0;
    if (candm) my_last = BTS(r0 + (31 - __clz(candm)));
    const unsigned lower = any & lanemask_lt();
    u64 prv = __shfl_sync(FULL, my_last, lower ? 31 - __clz(lower) : lane);
    bool has_prv = lower != 0 || have_c;
    if (!lower) prv = last_c;
    uint32_t bm = 0, nbl = 0;
    u64 lb = 0;
    for (uint32_t m = candm; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const u64 tj = (m & (m - 1)) ? BTS(r0 + j) : my_last;
      if (!has_prv || prv < tj) {
        bm |= 1u << j;
        ++nbl;
        lb = tj;
      }
      prv = tj;
      has_prv = true;
    }
    uint32_t inc = nbl;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, d);
      if (lane >= d) inc += y;
    }
    const uint32_t tot = __shfl_sync(FULL, inc, 31);
    u64 kk = nb + inc - nbl;
    for (uint32_t m = bm; m; m &= m - 1, ++kk)
      if (kk < cap) {
        const int j = __ffs(m) - 1;
        out[kk] = static_cast<uint32_t>(r0 + j - b);
        out_ts[kk] = BTS(r0 + j);
      }
    nb += tot;
    last_c = __shfl_sync(FULL, my_last, 31 - __clz(any));
    have_c = true;
    const unsigned bl = __ballot_sync(FULL, nbl != 0);
    if (bl) last_b = __shfl_sync(FULL, lb, 31 - __clz(bl));
  }
  if (!EXACT) {
    __syncwarp();  // the other lanes' boundary indices are visible to lane 0
    if (lane == 0 && nb > 0 && nb <= cap) last_b = ldg64(p.tr.ts + b + out[nb - 1]);
  }
  if (lane == 0) {
    uint32_t it = static_cast<uint32_t>(nb);
    if (nb > 0 && last_b >= p.tr.t_end[t]) it -= 1;  // empty last interval dropped
    if (nb > cap) {  // the query re-runs with larger regions; until then every
      atomicAdd(p.overflow, 1ull);  // reader stays inside this trace's region
      nb = cap;
      it = static_cast<uint32_t>(cap);
    }
    p.n_bounds[t] = static_cast<uint32_t>(nb);
    p.iter_count[t] = it;
  }
}
#undef BTS

void launch_bounds(const bound_params& p, bool exact, cudaStream_t s) {
  if (p.tr.n == 0) return;
  const unsigned g = (p.tr.n + 7) / 8, sm = 4u * p.words;
  if (p.ctx8) {  // membership from the preorder bytes: no bit tables
    if (exact)
      k_bounds<true, true, true><<<g, 256, sm, s>>>(p);
    else
      k_bounds<true, false, true><<<g, 256, sm, s>>>(p);
  } else if (p.words <= 4) {
    if (exact)
      k_bounds<true, true, false><<<g, 256, sm, s>>>(p);
    else
      k_bounds<true, false, false><<<g, 256, sm, s>>>(p);
  } else {
    if (exact)
      k_bounds<false, true, false><<<g, 256, sm, s>>>(p);
    else
      k_bounds<false, false, false><<<g, 256, sm, s>>>(p);
  }
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// Verdict on an optimistic pass 1 after pass 2 recorded every boundary's
// timestamp: bit 0 = two boundaries on one timestamp (the exact pass drops the
// second, itermodel.cpp:121-130), bit 1 = the gap or a stored iteration spans
// >= 2^32 ns (32-bit cells could have wrapped).  One warp per trace.
__global__ void k_verify_bounds(trace_view tr, const uint64_t* cap_off, const uint64_t* bts,
                                const uint32_t* n_bounds, const uint32_t* iter_count,
                                unsigned long long* verify) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= tr.n) return;
  const uint32_t it = iter_count[t], nbd = n_bounds[t];
  if (it == 0) return;  // skipped trace: no cube rows
  const uint64_t* bt = bts + cap_off[t];
  const u64 first = ldg64(tr.ts + tr.off[t]), tend = tr.t_end[t];
  bool dup = false, wide = false;
  // four rows of 32 boundaries per round: twelve independent loads in flight
  // per lane (the kernel is latency-bound: one short trace region per warp)
  for (uint32_t j0 = lane; j0 < nbd; j0 += 128) {
    u64 tj[4], pv[4], nx[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = j0 + 32 * q;
      tj[q] = j < nbd ? ldg64(bt + j) : 0;
      pv[q] = (j < nbd && j > 0) ? ldg64(bt + j - 1) : first;
      nx[q] = j + 1 < nbd ? ldg64(bt + j + 1) : tend;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = j0 + 32 * q;
      if (j >= nbd) continue;
      if (j > 0) dup |= tj[q] == pv[q];
      else wide |= tj[q] - pv[q] >= kSpan32;  // the gap row [first, b_0)
      if (j < it) wide |= nx[q] - tj[q] >= kSpan32;
    }
  }
  const unsigned v = (__ballot_sync(FULL, dup) ? 1u : 0u) | (__ballot_sync(FULL, wide) ? 2u : 0u);
  if (v && lane == 0) atomicOr(verify, static_cast<unsigned long long>(v));
}

void launch_verify_bounds(const trace_view& tr, const uint64_t* cap_off, const uint64_t* bts,
                          const uint32_t* n_bounds, const uint32_t* iter_count,
                          unsigned long long* verify, cudaStream_t s) {
  if (tr.n == 0) return;
  k_verify_bounds<<<(tr.n + 7) / 8, 256, 0, s>>>(tr, cap_off, bts, n_bounds, iter_count, verify);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// Pass 2: the fused query.  A CTA owns `warps` consecutive traces, one warp
// each, and advances in chunks of G iterations.  Phase 1: every warp consumes
// events until its trace has passed the end of chunk c (it may run ahead into
// chunk c+1: the cube rows form a ring of 2G iterations plus the gap row).
// Phase 2: each warp rolls the chunk's rows up to inclusive time and stores
// them (coalesced along the node axis); with statistics on, the CTA then
// folds its traces into the within-rank sums and the cross-rank (iteration,
// node) accumulators.  Without statistics the warps never synchronise.
//
// Overflow guards for the 32-bit reductions.  A cube cell sums disjoint
// segments of one iteration, so it cannot exceed the iteration's time span;
// a chunk whose iterations all span < 2^32 ns (4.29 s) accumulates with
// 32-bit REDs into the low words, otherwise with carried 64-bit adds.  The
// window sums of a block step cannot exceed the block's time span, so the
// 32-bit pending sums are folded into 64-bit accumulators before the spans
// added since the last fold can reach 2^32; a block spanning >= 2^32 ns (or
// holding the trace's last event, whose segment runs to t1) takes the 64-bit
// path.
namespace {


enum : int { WIN_NONE = 0, WIN_FULL = 1, WIN_PART = 2, WIN_WIDE = 3 };

struct warp_tables {
  bool il;       // the records' slot map (wt_word): interleaved or run lane layout
  uint32_t* wt;  // n_ctx records of WT_STRIDE words (psg_internal.h)
  unsigned long long *gminb, *gmaxb;  // the trace's global w_min / w_max rows (durations >= 2^32)
  u64* carry;
  __device__ __forceinline__ u64 acc(uint32_t c) const {
    const uint32_t* r = wt + wt_word(c, il) + WT_ACC;
    return static_cast<u64>(r[0]) | (static_cast<u64>(r[1]) << 32);
  }
  __device__ __forceinline__ void set_acc(uint32_t c, u64 v) const {
    uint32_t* r = wt + wt_word(c, il) + WT_ACC;
    r[0] = static_cast<uint32_t>(v);
    r[1] = static_cast<uint32_t>(v >> 32);
  }
};

// One window row of duration d for ctx c (frame::group_aggregate's
// count/sum/min/max fold, order-free in integers).
__device__ __forceinline__ void win_row32(const warp_tables& T, uint32_t c, uint32_t d) {
  uint32_t* r = T.wt + wt_word(c, T.il);
  atomicAdd(r + WT_CNT, 1u);
  atomicAdd(r + WT_LO, d);
  atomicMin(r + WT_MIN, d);
  atomicMax(r + WT_MAX, d);
}

__device__ __forceinline__ void win_row64(const warp_tables& T, uint32_t c, u64 d) {
  uint32_t* r = T.wt + wt_word(c, T.il);
  atomicAdd(r + WT_CNT, 1u);
  sadd64(r + WT_ACC, r + WT_ACC + 1, d);
  if (d >> 32) {
    atomicAdd(r + WT_NBIG, 1u);
    atomicMin(T.gminb + c, d);
    atomicMax(T.gmaxb + c, d);
  } else {
    atomicMin(r + WT_MIN, static_cast<uint32_t>(d));
    atomicMax(r + WT_MAX, static_cast<uint32_t>(d));
  }
}

__device__ __forceinline__ void carry_in(const warp_tables& T, uint32_t c, u64 ts, u64 end, u64 t0) {
  T.carry[0] = ts;
  T.carry[1] = end > t0 ? end - t0 : 0;
  T.carry[2] = (1ull << 32) | c;
}

// x^2 accumulated into a 128-bit (hi, lo) pair; one IMAD.WIDE when x < 2^32.
// a * b + c in one IMAD.WIDE.U32 (64-bit addend)
__device__ __forceinline__ u64 mad_wide(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

__device__ __forceinline__ void acc_sq(u64& lo, u64& hi, u64 x) {
  if ((x >> 32) == 0) {
    const u64 q = static_cast<u64>(static_cast<uint32_t>(x)) * static_cast<uint32_t>(x);
    lo += q;
    hi += lo < q ? 1ull : 0ull;
  } else {
    const u128 q = static_cast<u128>(x) * x;
    const u64 ql = static_cast<u64>(q);
    lo += ql;
    hi += static_cast<u64>(q >> 64) + (lo < ql ? 1ull : 0ull);
  }
}

// Boundary windows hold event indices relative to the trace plus SOFF (the block
// step start is aligned down by at most SOFF events), so all index arithmetic is
// unsigned 32-bit (traces have < 2^32 - 4096 events).  Local index of a
// boundary in the block step starting at base3 (clamped past the step).
__device__ __forceinline__ int local_of(uint32_t bw3, uint32_t base3) {
  const uint32_t v = bw3 - base3;
  return v > static_cast<uint32_t>(STEP_M) ? STEP_M + 1 : static_cast<int>(v);
}

struct run_state {
  int k;          // iteration of the current event (-1: before the first boundary)
  uint32_t cnt;   // boundaries of the window at or before the current event
  int nxt;        // local index of the next boundary
  bool cube_ok;   // k is a stored iteration (or the gap of a kept trace)
  uint32_t slot;  // ring slot of k
  uint32_t rowb;  // slot * nnp
};

struct run_ctx {
  const int32_t* s_sub_pre;
  const uint32_t* bwin;
  uint32_t *rlo, *rhi;
  uint32_t base3;  // block step start relative to the trace, + SOFF
  u64 tend, t0, t1w;
  uint32_t R2, nnp;  // ring size, cube row stride
  int iters;  // iterations stored for this trace; -1 for a skipped trace (no gap row either)
  int lb, lo, hi, last_li;
  bool root_only;
  uint64_t* bts_out;  // optimistic pass 1: boundary timestamps are recorded here (k < nbd)
  uint32_t nbd;
};

// ALL: every event of the block step is valid and none is the trace's last
// (the common interior step): no per-event range or end checks.
template <bool WIN, bool CUBE, int WM, bool CWIDE, bool ALL>
__device__ __forceinline__ void run_events(const u64 (&tv)[RM + 1], const uint32_t (&cv)[RM],
                                           const run_ctx& R, run_state& st, const warp_tables& T,
                                           int wm_rt = 0) {
  const int wmx = WM >= 0 ? WM : wm_rt;  // WM < 0: the window class is a (warp-uniform) runtime value
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    const int li = R.lb + j;
    const bool valid =
        ALL || static_cast<unsigned>(li - R.lo) < static_cast<unsigned>(R.hi - R.lo);
    const u64 tsj = tv[j], nts = tv[j + 1];
    const uint32_t cj = valid ? cv[j] : 0u;
    if (CUBE) {
      if (li >= st.nxt) {  // boundaries are distinct events: at most one per event
        ++st.k;
        ++st.cnt;
        if (R.bts_out && static_cast<uint32_t>(st.k) < R.nbd) R.bts_out[st.k] = tsj;
        st.nxt = st.cnt <= R.R2 ? local_of(R.bwin[st.cnt], R.base3) : INT_MAX;
        st.slot = st.k < 0 ? R.R2 : (static_cast<uint32_t>(st.k) & (R.R2 - 1));
        st.rowb = st.slot * R.nnp;
        st.cube_ok = st.k < R.iters;
      }
      const int pp = R.s_sub_pre[cj];
      if (valid && pp >= 0 && st.cube_ok) {
        const uint32_t idx = st.rowb + pp;
        if (CWIDE) {
          const u64 dc = ((!ALL && li == R.last_li) ? R.tend : nts) - tsj;
          sadd64(R.rlo + idx, R.rhi + idx, dc);
        } else {  // the iteration spans < 2^32 ns: 32-bit differences are exact
          const uint32_t dc = static_cast<uint32_t>((!ALL && li == R.last_li) ? R.tend : nts) -
                              static_cast<uint32_t>(tsj);
          atomicAdd(R.rlo + idx, dc);
        }
      }
    }
    if (WIN && wmx == WIN_FULL) {  // the block spans < 2^32 ns
      if (valid) win_row32(T, cj, static_cast<uint32_t>(nts) - static_cast<uint32_t>(tsj));
    } else if (WIN && wmx == WIN_PART) {  // no trace end in this block step
      if (valid) {
        if (tsj >= R.t0) {
          if (tsj < R.t1w)
            win_row32(T, cj, static_cast<uint32_t>(min(nts, R.t1w)) - static_cast<uint32_t>(tsj));
        } else if (nts >= R.t0) {  // the carry-in event (store.cpp:667-670): unique
          carry_in(T, cj, tsj, min(nts, R.t1w), R.t0);
        }
      }
    } else if (WIN && wmx == WIN_WIDE) {
      if (valid) {
        const bool last = li == R.last_li;
        const u64 e2 = last ? R.t1w : min(nts, R.t1w);
        if (tsj >= R.t0) {
          if (tsj < R.t1w) win_row64(T, cj, e2 - tsj);
        } else if (last || nts >= R.t0) {
          carry_in(T, cj, tsj, e2, R.t0);
        }
      }
    }
  }
}

// The general path in the interleaved layout: lane event j is li = lane + 32 j
// of the block step; its successor comes from the neighbouring lane.  Between
// two of a lane's events lie 32 events, so several boundaries may be crossed
// (each recorded by the lane owning its event).
template <bool WIN, bool CUBE, int WM, bool CWIDE, bool ALL>
__device__ __forceinline__ void run_events_il(u64 (&tv)[RM + 1], uint32_t (&cv)[RM], int lane,
                                              const run_ctx& R, run_state& st,
                                              const warp_tables& T, const rot_src& rs, int wm_rt = 0) {
  const int wmx = WM >= 0 ? WM : wm_rt;  // WM < 0: the window class is a (warp-uniform) runtime value
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    const int li = lane + 32 * j;
    const bool valid =
        ALL || static_cast<unsigned>(li - R.lo) < static_cast<unsigned>(R.hi - R.lo);
    const u64 tsj = tv[j];
    const u64 nts = next_ts_il(tv, j, lane);
    const uint32_t cj = valid ? cv[j] : 0u;
    if (CUBE) {
      if (li >= st.nxt) {
        do {
          ++st.k;
          ++st.cnt;
          if (li == st.nxt && R.bts_out && static_cast<uint32_t>(st.k) < R.nbd) R.bts_out[st.k] = tsj;
          st.nxt = st.cnt <= R.R2 ? local_of(R.bwin[st.cnt], R.base3) : INT_MAX;
        } while (li >= st.nxt);
        st.slot = st.k < 0 ? R.R2 : (static_cast<uint32_t>(st.k) & (R.R2 - 1));
        st.rowb = st.slot * R.nnp;
        st.cube_ok = st.k < R.iters;
      }
      const int pp = R.s_sub_pre[cj];
      if (valid && pp >= 0 && st.cube_ok) {
        const uint32_t idx = st.rowb + pp;
        if (CWIDE) {
          const u64 dc = ((!ALL && li == R.last_li) ? R.tend : nts) - tsj;
          sadd64(R.rlo + idx, R.rhi + idx, dc);
        } else {
          const uint32_t dc = static_cast<uint32_t>((!ALL && li == R.last_li) ? R.tend : nts) -
                              static_cast<uint32_t>(tsj);
          atomicAdd(R.rlo + idx, dc);
        }
      }
    }
    if (WIN && wmx == WIN_FULL) {
      if (valid) win_row32(T, cj, static_cast<uint32_t>(nts) - static_cast<uint32_t>(tsj));
    } else if (WIN && wmx == WIN_PART) {
      if (valid) {
        if (tsj >= R.t0) {
          if (tsj < R.t1w)
            win_row32(T, cj, static_cast<uint32_t>(min(nts, R.t1w)) - static_cast<uint32_t>(tsj));
        } else if (nts >= R.t0) {
          carry_in(T, cj, tsj, min(nts, R.t1w), R.t0);
        }
      }
    } else if (WIN && wmx == WIN_WIDE) {
      if (valid) {
        const bool last = li == R.last_li;
        const u64 e2 = last ? R.t1w : min(nts, R.t1w);
        if (tsj >= R.t0) {
          if (tsj < R.t1w) win_row64(T, cj, e2 - tsj);
        } else if (last || nts >= R.t0) {
          carry_in(T, cj, tsj, e2, R.t0);
        }
      }
    }
    if (PSG_ROT) rot_load(rs, j, tv, cv);
  }
  if (PSG_ROT) rot_tail(rs, lane, tv);
}

template <bool WIN, bool CUBE, bool CWIDE>
__device__ __forceinline__ void run_block_il(int wm, u64 (&tv)[RM + 1], uint32_t (&cv)[RM], int lane,
                                             const run_ctx& R, run_state& st,
                                             const warp_tables& T, const rot_src& rs) {
  const bool all = R.lo == 0 && R.hi == STEP_M && R.last_li < 0;  // warp-uniform
  if (PSG_GEN_RT) {  // one copy of the general path (less code in the step loop)
    run_events_il<WIN, CUBE, -1, CWIDE, false>(tv, cv, lane, R, st, T, rs, wm);
    return;
  }
  if (PSG_GEN_ALL && !CWIDE && all && wm == WIN_FULL)
    run_events_il<WIN, CUBE, WIN_FULL, false, true>(tv, cv, lane, R, st, T, rs);
  else if (PSG_GEN_ALL && !CWIDE && all && wm == WIN_NONE)
    run_events_il<WIN, CUBE, WIN_NONE, false, true>(tv, cv, lane, R, st, T, rs);
  else if (wm == WIN_FULL)
    run_events_il<WIN, CUBE, WIN_FULL, CWIDE, false>(tv, cv, lane, R, st, T, rs);
  else if (wm == WIN_PART)
    run_events_il<WIN, CUBE, WIN_PART, CWIDE, false>(tv, cv, lane, R, st, T, rs);
  else if (wm == WIN_WIDE)
    run_events_il<WIN, CUBE, WIN_WIDE, CWIDE, false>(tv, cv, lane, R, st, T, rs);
  else
    run_events_il<WIN, CUBE, WIN_NONE, CWIDE, false>(tv, cv, lane, R, st, T, rs);
}

template <bool WIN, bool CUBE, bool CWIDE>
__device__ __forceinline__ void run_block(int wm, const u64 (&tv)[RM + 1], const uint32_t (&cv)[RM],
                                          const run_ctx& R, run_state& st, const warp_tables& T) {
  if (PSG_GEN_RT) {  // one copy of the general path (less code in the step loop)
    run_events<WIN, CUBE, -1, CWIDE, false>(tv, cv, R, st, T, wm);
    return;
  }
  const bool all = R.lo == 0 && R.hi == STEP_M && R.last_li < 0;  // warp-uniform
  if (!CWIDE && all && wm == WIN_FULL)
    run_events<WIN, CUBE, WIN_FULL, false, true>(tv, cv, R, st, T);
  else if (!CWIDE && all && wm == WIN_NONE)
    run_events<WIN, CUBE, WIN_NONE, false, true>(tv, cv, R, st, T);
  else if (wm == WIN_FULL)
    run_events<WIN, CUBE, WIN_FULL, CWIDE, false>(tv, cv, R, st, T);
  else if (wm == WIN_PART)
    run_events<WIN, CUBE, WIN_PART, CWIDE, false>(tv, cv, R, st, T);
  else if (wm == WIN_WIDE)
    run_events<WIN, CUBE, WIN_WIDE, CWIDE, false>(tv, cv, R, st, T);
  else
    run_events<WIN, CUBE, WIN_NONE, CWIDE, false>(tv, cv, R, st, T);
}

__device__ __forceinline__ u64 cell64(const uint32_t* lo, const uint32_t* hi, uint32_t i) {
  return static_cast<u64>(lo[i]) | (hi ? static_cast<u64>(hi[i]) << 32 : 0ull);
}

// One cube cell into HBM storage (32-bit cells when the query's iterations all
// span < 2^32 ns, else 64-bit); idx counts storage cells (rows of stride nnp).
__device__ __forceinline__ void store_cell(const query_params& p, u64 idx, u64 v) {
  if (p.cube32)
    reinterpret_cast<uint32_t*>(p.cube_incl)[idx] = static_cast<uint32_t>(v);
  else
    p.cube_incl[idx] = v;
}

// Exclusive prefix, in subtree preorder, over a node-indexed (lo, hi) word row
// into dst[0..n] (generic roll-up: incl(node) = dst[pre + size] - dst[pre]).
__device__ __forceinline__ void warp_prefix_row(const uint32_t* lo, const uint32_t* hi,
                                                const int4* node, u64* dst, uint32_t n, int lane) {
  u64 carry = 0;
  for (uint32_t b = 0; b < n; b += 32) {
    const uint32_t j = b + lane;
    u64 v = j < n ? cell64(lo, hi, static_cast<uint32_t>(node[j].w)) : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u64 y = __shfl_up_sync(FULL, v, d);
      if (lane >= d) v += y;
    }
    if (j < n) dst[j + 1] = carry + v;
    carry += __shfl_sync(FULL, v, 31);
  }
  if (lane == 0) dst[0] = 0;
  __syncwarp();
}

// Interior block step, fast path: every event of the step is valid and none
// is the trace's last, the chunk is narrow (cells and block spans fit 32
// bits), the window class is FULL or NONE, and the lane's run holds at most
// one iteration boundary (local index bpos; RM when none).  Per event: one
// window-record address, one load of the ctx's cube column offset, one cube
// RED into the row selected by bpos (contexts outside the anchor subtree land
// in the rows' pad column) and, inside the window, the four window REDs; no
// branches.
template <int WM>
__device__ __forceinline__ void run_fast(const u64 (&tv)[RM + 1], const uint32_t (&cv)[RM],
                                         uint8_t* sm, uint32_t wt_off, int bpos,
                                         uint32_t rb_before, uint32_t rb_after,
                                         const uint32_t (&ppo)[RM]) {
  uint32_t d[RM];
#pragma unroll
  for (int j = 0; j < RM; ++j) d[j] = static_cast<uint32_t>(tv[j + 1]) - static_cast<uint32_t>(tv[j]);
  // the window reductions first (they need no column offset): the column
  // loads' latency is hidden behind them
  if (WM == WIN_FULL) {
#pragma unroll
    for (int j = 0; j < RM; ++j) {
      uint32_t* r = reinterpret_cast<uint32_t*>(sm + wt_off + 4u * wt_word_l<false>(cv[j]));
      atomicAdd(r + WT_CNT, 1u);
      atomicAdd(r + WT_LO, d[j]);
      atomicMin(r + WT_MIN, d[j]);
      atomicMax(r + WT_MAX, d[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    const uint32_t rb = j >= bpos ? rb_after : rb_before;
    atomicAdd(reinterpret_cast<uint32_t*>(sm + rb + ppo[j]), d[j]);
  }
}

// Interior block step, fast path in the interleaved layout: every event of the
// step is valid and none is the trace's last, the chunk is narrow, the window
// class is FULL or NONE, and each group of 32 consecutive events (one j)
// holds at most one iteration boundary.  fa / fb carry, per group, its
// boundary's lane + 1 in 6-bit fields (0: none; groups 0-4 in fa, 5-7 in fb)
// and ra is the ring row of the iteration before the step (>= 0): lanes below
// the group's boundary add into row ra, the others into the next ring row
// (uniform per group).  Contexts outside the anchor subtree add into the
// rows' pad column (no branch).
template <int WM, bool GT>
__device__ __forceinline__ void run_fast_il(u64 (&tv)[RM + 1], uint32_t (&cv)[RM], int lane,
                                            uint8_t* sm, uint32_t wt_off, const uint32_t* ppo_g,
                                            uint32_t fa, uint32_t fb, uint32_t ra, uint32_t rows_off,
                                            uint32_t rows_end, uint32_t row_bytes, const rot_src& rs) {
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    const uint32_t field = j < 5 ? (fa >> (6 * j)) & 63u : (fb >> (6 * (j - 5))) & 63u;
    const uint32_t bj = (field - 1u) & 63u;  // the boundary's lane; 63: none
    uint32_t rn = ra + row_bytes;  // the next iteration's ring row
    rn = rn == rows_end ? rows_off : rn;
    const uint32_t d = next_lo_il(tv, j, lane) - static_cast<uint32_t>(tv[j]);
    uint32_t* r = reinterpret_cast<uint32_t*>(sm + wt_off + 4u * wt_word_l<true>(cv[j]));
    if (WM == WIN_FULL) {
      atomicAdd(r + WT_CNT, 1u);
      atomicAdd(r + WT_LO, d);
      atomicMin(r + WT_MIN, d);
      atomicMax(r + WT_MAX, d);
    }
    const uint32_t ppo = GT ? __ldg(ppo_g + cv[j]) : r[WT_PPO];
    const uint32_t rb = static_cast<uint32_t>(lane) >= bj ? rn : ra;
    atomicAdd(reinterpret_cast<uint32_t*>(sm + rb + ppo), d);
    ra = field ? rn : ra;
    if (PSG_ROT) rot_load(rs, j, tv, cv);
  }
  if (PSG_ROT) rot_tail(rs, lane, tv);
}

// Flush of a full narrow chunk (G rows, every cell < 2^32) when the anchor is
// the only internal node.  A leaf's inclusive time IS its exclusive time, and
// the chunk's G ring rows (stride nnp) are byte for byte the cube block of its
// G iterations (same stride; the pad columns are zeroed), so:
//  1. a lane owns leaves across the rows: row sums and the within-rank Σx, Σx²
//     in registers (G squares in 64 bits while its cells are < 2^30, else
//     redone in 128 bits);
//  2. the anchor's inclusive time (row total, one REDUX per row) replaces its
//     exclusive time in the block (that one goes to the compact excl cube);
//  3. the block is copied to the cube with 16-byte stores, then zeroed.
template <bool STATS>
__device__ __forceinline__ void flush_fast(const query_params& p, uint32_t* rows, uint32_t nn,
                                           uint32_t nnp, u64 ob, u64 xbase, u64* wsx, u64* wsqlo,
                                           u64* wsqhi, int lane) {
  constexpr uint32_t G = GC;
  const uint4* src = reinterpret_cast<const uint4*>(rows);
  const uint32_t nq = G * nnp / 4;
  uint32_t rs[GC];
#pragma unroll
  for (uint32_t r = 0; r < G; ++r) rs[r] = 0u;
  const uint32_t ax = lane < static_cast<int>(G) ? rows[lane * nnp] : 0u;  // the anchor's excl
  // leaves 1..nn-1: whole groups of 32 columns one column per lane; a tail
  // of at most 32/G columns (65 leaves = 2 groups + 1 in the iterative
  // scenarios) one cell per lane instead, so the warp does not run a G-row
  // pass for a handful of active lanes
  constexpr uint32_t TW = 32 / GC;  // tail columns per pass
  const uint32_t nl = nn - 1, tail = nl & 31u;
  const uint32_t n_cols = (tail != 0 && tail <= TW) ? nn - tail : nn;
#pragma unroll kFlushUnroll  // two columns per lane at once (latency of the row chains)
  for (uint32_t n = 1 + lane; n < n_cols; n += 32) {
    u64 sq = 0, sqh = 0;
    uint32_t sx32 = 0, orv = 0;
#pragma unroll
    for (uint32_t r = 0; r < G; ++r) {
      const uint32_t ex = rows[r * nnp + n];
      rs[r] += ex;
      if (STATS) {
        sx32 += ex;  // exact while every cell < 2^29 (G = 8)
        sq = mad_wide(ex, ex, sq);  // G squares fit 64 bits while every cell < 2^30
        orv |= ex;
      }
    }
    static_assert(GC <= 8, "32-bit sums of G cells < 2^29");
    if (STATS) {
      u64 sx = sx32;
      if (orv >> 29) {  // a cell >= 2^29: redo the sum in 64 bits and the squares in 128
        sq = 0;
        sx = 0;
#pragma unroll
        for (uint32_t r = 0; r < G; ++r) {
          const uint32_t ex = rows[r * nnp + n];
          sx += ex;
          acc_sq(sq, sqh, ex);
        }
      }
      wsx[n] += sx;
      const u64 l2 = wsqlo[n] + sq;
      wsqhi[n] += sqh + (l2 < sq ? 1ull : 0ull);
      wsqlo[n] = l2;
    }
  }
  uint32_t trs = 0;  // tail cells of row lane % G
  if (n_cols < nn) {
    const uint32_t n = n_cols + static_cast<uint32_t>(lane) / G, r = static_cast<uint32_t>(lane) % G;
    const u64 ex = n < nn ? rows[r * nnp + n] : 0u;
    trs = static_cast<uint32_t>(ex);
    if (STATS) {  // the G lanes of a column (aligned group): its within-rank sums
      u64 sx = ex, sq = ex * ex, sqh = 0;
      if (!__any_sync(FULL, (ex >> 30) != 0)) {
#pragma unroll
        for (int d = 1; d < static_cast<int>(G); d <<= 1) {
          sx += __shfl_xor_sync(FULL, sx, d);
          sq += __shfl_xor_sync(FULL, sq, d);
        }
      } else {
#pragma unroll
        for (int d = 1; d < static_cast<int>(G); d <<= 1) {
          sx += __shfl_xor_sync(FULL, sx, d);
          const u64 ol = __shfl_xor_sync(FULL, sq, d), oh = __shfl_xor_sync(FULL, sqh, d);
          sq += ol;
          sqh += oh + (sq < ol ? 1ull : 0ull);
        }
      }
      if (r == 0 && n < nn) {
        wsx[n] += sx;
        const u64 l2 = wsqlo[n] + sq;
        wsqhi[n] += sqh + (l2 < sq ? 1ull : 0ull);
        wsqlo[n] = l2;
      }
    }
#pragma unroll
    for (int d = G; d < 32; d <<= 1) trs += __shfl_xor_sync(FULL, trs, d);  // row lane % G
  }
#pragma unroll
  for (uint32_t r = 0; r < G; ++r) rs[r] = __reduce_add_sync(FULL, rs[r]);  // leaves, < 2^32
  uint32_t mine = rs[0];
#pragma unroll
  for (uint32_t r = 1; r < G; ++r)
    if (static_cast<uint32_t>(lane) == r) mine = rs[r];
  mine += ax + trs;  // lane r < G: the anchor's inclusive time in row r
  if (lane < static_cast<int>(G)) {
    rows[lane * nnp] = mine;
    rows[lane * nnp + nn] = 0u;  // pad column
    if (p.store_cube) p.cube_xint[xbase + lane] = ax;  // m == 1
  }
  if (STATS) {  // the anchor's within-rank sums: lanes r < G hold its G cells
    u64 sx = lane < static_cast<int>(G) ? mine : 0u;
    u64 sq = sx * sx, sqh = 0;
    if (!__any_sync(FULL, (sx >> 30) != 0)) {
#pragma unroll
      for (int d = 1; d < static_cast<int>(G); d <<= 1) {
        sx += __shfl_xor_sync(FULL, sx, d);
        sq += __shfl_xor_sync(FULL, sq, d);
      }
    } else {  // a row total >= 2^30: 128-bit squares
      sq = 0;
      acc_sq(sq, sqh, sx);
#pragma unroll
      for (int d = 1; d < static_cast<int>(G); d <<= 1) {
        sx += __shfl_xor_sync(FULL, sx, d);
        const u64 ol = __shfl_xor_sync(FULL, sq, d), oh = __shfl_xor_sync(FULL, sqh, d);
        sq += ol;
        sqh += oh + (sq < ol ? 1ull : 0ull);
      }
    }
    if (lane == 0) {
      wsx[0] += sx;
      const u64 l2 = wsqlo[0] + sq;
      wsqhi[0] += sqh + (l2 < sq ? 1ull : 0ull);
      wsqlo[0] = l2;
    }
  }
  __syncwarp();
  // the block: G * nnp cells, a multiple of 4; 16-byte aligned on both sides
  // (ring rows from a 16-byte boundary, trace blocks padded to 4 cells, kb * nnp
  // a multiple of 8)
  // each lane zeroes the 16 bytes it has just read
  uint4* z = reinterpret_cast<uint4*>(rows);
  if (p.cube32) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(p.cube_incl) + ob);
#pragma unroll kCopyUnroll
    for (uint32_t i = lane; i < nq; i += 32) {
      const uint4 v = src[i];
      z[i] = make_uint4(0u, 0u, 0u, 0u);
      dst[i] = v;
    }
  } else {
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(p.cube_incl + ob);
#pragma unroll kCopyUnroll
    for (uint32_t i = lane; i < nq; i += 32) {
      const uint4 v = src[i];
      z[i] = make_uint4(0u, 0u, 0u, 0u);
      dst[2 * i] = make_ulonglong2(v.x, v.y);
      dst[2 * i + 1] = make_ulonglong2(v.z, v.w);
    }
  }
  __syncwarp();
}

// First chunk c in [0, n_chunks] whose start event is at or after e: chunk 0
// starts at event 0, chunk c at boundary c * G (bt, strictly increasing), and
// chunk n_chunks "starts" at n_t.  Two rounds of 32 sampled loads for up to
// 1024 chunks (warp-uniform result).
__device__ __forceinline__ uint32_t first_chunk_at(const uint32_t* bt, uint32_t n_chunks, u64 n_t, u64 e,
                                                   int lane) {
  if (e == 0) return 0;
  if (e >= n_t) return n_chunks;
  uint32_t lo = 1, hi = n_chunks;  // the answer lies in [lo, hi]; chunk hi starts at or after e
  while (hi > lo) {
    const uint32_t S = (hi - lo + 31) / 32;
    const uint32_t c = lo + static_cast<uint32_t>(lane) * S;
    const bool ge = c < hi && static_cast<u64>(__ldg(bt + static_cast<size_t>(c) * GC)) >= e;
    const unsigned m = __ballot_sync(FULL, ge);
    if (m) {
      const uint32_t f = static_cast<uint32_t>(__ffs(m)) - 1u;
      if (f == 0) return lo;
      hi = lo + f * S;
      lo = lo + (f - 1) * S + 1;
    } else {
      lo = lo + ((hi - lo + S - 1) / S - 1) * S + 1;
    }
  }
  return lo;
}

// EXACT: pass 1 ran in the exact mode (p.exact_bounds): boundary timestamps
// are known and chunks may need 64-bit cells.  The optimistic instantiation
// runs 32-bit throughout and carries none of the 64-bit cell code (a third
// smaller, which the instruction cache notices).
// ONE: one warp per CTA (else up to 16).
// (the optimistic cube-only one-warp instantiation spills at 96 registers: 16 CTAs per SM, 128)
// GT: the cube's column offsets come from a global per-ctx table (p.ppo_g)
// instead of the per-warp window records (cube-only queries over calling-
// context trees too large for the records; the window then takes the sparse
// path, psg_sparse.cu).
template <bool WIN, bool CUBE, bool EXACT, bool ONE, bool GT = false>
__global__ void __launch_bounds__(ONE ? 32 : PSG_WIDE_THREADS, ONE ? ((!WIN && !EXACT) ? 16 : PSG_ONE_MINB) : PSG_WIDE_MINB)
    k_trace_query(query_params p) {
  static_assert(!GT || (!WIN && ONE), "global column tables: cube-only, one-warp CTAs");
  // lane layout: interleaved for one-warp CTAs (long traces; bank-conflict
  // free shared accesses), runs of RM events for wide CTAs (short traces: the
  // interleaved layout measured 19 % slower there, C5 at 100k traces)
  constexpr bool IL = ONE;
  extern __shared__ __align__(16) uint8_t smem[];
  // one-warp CTAs: the trace index and everything derived from it are
  // uniform across the CTA, so they live in uniform registers
  const int lane = ONE ? static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x & 31);
  const int warp = ONE ? 0 : static_cast<int>(threadIdx.x >> 5);
  const uint32_t CT = ONE ? 32u : blockDim.x;  // threads per CTA
  const uint32_t W = p.warps, n_ctx = p.n_ctx, nn = p.nn;
  constexpr uint32_t G = GC, R2 = 2 * GC;  // p.G == GC (same PSG_G on both sides)
  const bool root_only = p.root_only != 0;

  // one-warp CTAs read the tables straight from global memory (L1-cached: the
  // fast path never reads them, and the carve-out stays small); wider CTAs
  // share one copy in shared memory
  int4* t_node = reinterpret_cast<int4*>(smem);
  int32_t* t_sub_pre = reinterpret_cast<int32_t*>(t_node + nn);
  int32_t* t_cct_pre = t_sub_pre + n_ctx;
  int32_t* t_cct_size = t_cct_pre + n_ctx;
  const int4* s_node = ONE ? p.node_tab : t_node;
  const int32_t* s_sub_pre = ONE ? p.sub_pre : t_sub_pre;
  const int32_t* s_cct_pre = ONE ? p.cct_pre : t_cct_pre;
  const int32_t* s_cct_size = ONE ? p.cct_size : t_cct_size;

  const warp_smem_layout& L = p.L;
  const uint32_t nnp = L.nnp;
  const uint32_t wb_off = p.cta_bytes + static_cast<uint32_t>(warp) * L.bytes;
  uint8_t* wb = smem + wb_off;
  uint32_t* rlo = reinterpret_cast<uint32_t*>(wb + L.off_rlo);
  uint32_t* rhi = reinterpret_cast<uint32_t*>(wb + L.off_rhi);
  u64* pref = reinterpret_cast<u64*>(wb + L.off_pref);
  uint32_t* bwin = reinterpret_cast<uint32_t*>(wb + L.off_bwin);
  u64* bts = reinterpret_cast<u64*>(wb + L.off_bts);
  u64* wsx = reinterpret_cast<u64*>(wb + L.off_wsx);
  u64* wsqlo = reinterpret_cast<u64*>(wb + L.off_wsqlo);
  u64* wsqhi = reinterpret_cast<u64*>(wb + L.off_wsqhi);
  warp_tables T;
  T.il = IL;
  T.wt = reinterpret_cast<uint32_t*>(wb + L.off_wtab);
  T.carry = reinterpret_cast<u64*>(wb + L.off_carry);
  // byte offsets from smem for the fast path
  const uint32_t wt_off = wb_off + L.off_wtab;
  const uint32_t rows_off = wb_off + L.off_rlo;
  const uint32_t row_bytes = 4u * nnp;

  if (!ONE)
    for (uint32_t i = threadIdx.x; i < n_ctx; i += CT) {
      t_sub_pre[i] = CUBE ? p.sub_pre[i] : -1;
      t_cct_pre[i] = WIN ? p.cct_pre[i] : 0;
      t_cct_size[i] = WIN ? p.cct_size[i] : 0;
    }
  if (CUBE) {
    if (!ONE)
      for (uint32_t i = threadIdx.x; i < nn; i += CT) t_node[i] = p.node_tab[i];
    for (uint32_t j = lane; j < (R2 + 1) * nnp; j += 32) rlo[j] = 0;
    if (p.exact_bounds)
      for (uint32_t j = lane; j < (R2 + 1) * nnp; j += 32) rhi[j] = 0;
    for (uint32_t j = lane; j < nn; j += 32) wsx[j] = wsqlo[j] = wsqhi[j] = 0;
  }
  for (uint32_t c = lane; c < (GT ? 0u : n_ctx); c += 32) {
    uint32_t* r = T.wt + wt_word(c, IL);
    r[WT_CNT] = r[WT_LO] = r[WT_MAX] = r[WT_NBIG] = 0u;
    r[WT_MIN] = 0xFFFFFFFFu;
    const int32_t sp = CUBE ? p.sub_pre[c] : -1;
    // contexts outside the anchor subtree: the rows' pad column nn
    r[WT_PPO] = 4u * (sp >= 0 ? static_cast<uint32_t>(sp) : nn);
    T.set_acc(c, 0ull);
  }
  if (lane == 0) T.carry[0] = T.carry[1] = T.carry[2] = 0;

  uint32_t t = p.t_base + blockIdx.x * W + warp;
  bool active = t < p.t_stop;
  u64 ue0 = 0, ue1 = ~0ull;  // this unit's event range (relative; snapped to chunk starts below)
  bool split = false;
  if (p.units) {
    const uint32_t ui = blockIdx.x * W + warp;
    active = ui < p.n_units;
    const uint4 u = active ? p.units[ui] : make_uint4(0u, 0u, 0u, 0u);
    t = u.x;
    ue0 = u.y;
    ue1 = u.z;
    split = u.w != 0;
  }
  // K from the device status block (no host round trip between the passes)
  const uint32_t Kq = p.qs ? qs_K(p.qs) : p.K;
  if (WIN && active) {
    T.gminb = reinterpret_cast<unsigned long long*>(p.w_min) + static_cast<size_t>(t) * n_ctx;
    T.gmaxb = reinterpret_cast<unsigned long long*>(p.w_max) + static_cast<size_t>(t) * n_ctx;
    if (!split)  // split traces: k_split_init prepared the rows
      for (uint32_t c = lane; c < n_ctx; c += 32) {
        T.gminb[c] = ~0ull;
        T.gmaxb[c] = 0ull;
      }
  }
  uint32_t iters = (CUBE && active) ? p.iter_count[t] : 0;
  const uint32_t tp = iters > 0 ? p.tpos[t] : 0;
  const u64 bo = iters > 0 ? p.block_off[t] : 0;
  const u64 ib = iters > 0 ? p.iter_off[t] : 0;  // iterations stored before this trace
  if (p.cap_miss && iters > 0) {
    // speculative capacities (sized by an earlier query): a trace whose block
    // does not fit flags the query, which re-runs with exact sizes
    const bool over_c = bo + ((static_cast<u64>(iters) * nnp + 3) & ~3ull) > p.cube_cap;
    const bool over_x = p.store_cube && (ib + iters) * p.m > p.xint_cap;
    if (over_c || over_x) {
      if (lane == 0) atomicOr(p.cap_miss, over_c ? 1ull : 2ull);
      active = false;
      iters = 0;
    }
  }
  const u64 b = active ? p.tr.off[t] : 0, e = active ? p.tr.off[t + 1] : 0;
  const u64 n_t = e - b;
  const u64 tend = active ? p.tr.t_end[t] : 0;
  const uint32_t nbd = (CUBE && active) ? p.n_bounds[t] : 0;
  const bool kept = iters > 0;
  const u64 region = (CUBE && active) ? p.cap_off[t] : 0;
  const uint32_t* bt = p.bidx + region;
  const uint64_t* btt = p.bts + region;
  // this lane's entry of the boundary windows of the next chunk (index and
  // timestamp) and of the one after (index): the timestamp load depends on
  // the index, so indices run one chunk further ahead
  // a split trace's unit: chunks [c_lo, c_hi), events [pos0, end) (kept
  // traces: the unit's nominal event range snapped to chunk starts; others:
  // the range itself)
  uint32_t c_lo = 0, c_stop = (iters + G - 1) / G;  // chunks [c_lo, c_stop)
  uint32_t pos0 = 0, end = static_cast<uint32_t>(n_t);  // relative event indices are 32-bit (finish_load)
  if (split) {
    if (CUBE && kept) {
      const uint32_t n_chunks = (iters + G - 1) / G;
      c_lo = first_chunk_at(bt, n_chunks, n_t, ue0, lane);
      const uint32_t c_hi = first_chunk_at(bt, n_chunks, n_t, ue1, lane);
      pos0 = c_lo == 0 ? 0u : __ldg(bt + c_lo * G);
      end = c_hi >= n_chunks ? static_cast<uint32_t>(n_t) : __ldg(bt + c_hi * G);
      c_stop = c_hi;
      if (c_lo >= c_hi) active = false;  // no chunk starts in this unit's range
    } else {
      pos0 = static_cast<uint32_t>(min(ue0, n_t));
      end = static_cast<uint32_t>(min(ue1, n_t));
      if (pos0 >= end) active = false;
    }
    if (!active) return;  // nothing to do; no CTA barrier follows (one-warp CTAs)
  }
  const uint32_t kb0 = c_lo * G;
  uint32_t nx_idx = static_cast<uint32_t>(n_t), nn_idx = static_cast<uint32_t>(n_t);
  u64 nx_ts = tend;
  // Boundary timestamps come from pass 1 in its exact mode.  After the
  // optimistic pass 1 there are none: every chunk runs with 32-bit cells
  // (exact while iterations span < 2^32 ns), each boundary's timestamp is
  // written out as its event is processed, and k_verify_bounds checks the
  // optimistic assumptions afterwards.
  constexpr bool optimistic = !EXACT;  // == !p.exact_bounds (launch_variant)
  uint64_t* bts_out = optimistic ? p.bts + region : nullptr;
  if (CUBE && kept && lane <= static_cast<int>(2 * G)) {
    const bool have = kb0 + static_cast<uint32_t>(lane) < nbd;
    nx_idx = have ? __ldg(bt + kb0 + lane) : static_cast<uint32_t>(n_t);
    nx_ts = (have && !optimistic) ? ldg64(btt + kb0 + lane) : tend;
    const bool have2 = kb0 + static_cast<uint32_t>(lane) + G < nbd;
    nn_idx = have2 ? __ldg(bt + kb0 + G + lane) : static_cast<uint32_t>(n_t);
  }
  const u64 t0 = p.t0, t1w = (p.clamp_tend && tend < p.t1) ? tend : p.t1;
  uint32_t pos = pos0;  // next unprocessed event, relative to b
  // block steps start on multiples of SA events of the whole stream: relative
  // to the aligned trace base b0 = b - d0 every step position is 32-bit
  const u64 b0 = b & ~static_cast<u64>(SOFF);
  const uint32_t d0 = static_cast<uint32_t>(b - b0), n32 = static_cast<uint32_t>(n_t);
  const uint64_t* ts_b0 = p.tr.ts + b0;
  const uint32_t* cx_b0 = p.tr.ctx + b0;
  const unsigned long long* ts_lane = reinterpret_cast<const unsigned long long*>(ts_b0) + lane;
  const unsigned int* cx_lane = reinterpret_cast<const unsigned int*>(cx_b0) + lane;
  uint32_t pf_rel = 0xFFFFFFFFu;  // step (relative to b0) whose events sit in tv / cv (interleaved layout)
  u64 wspan = 0;  // time span added to the 32-bit pending window sums since the last fold
  uint32_t mybw = 0xFFFFFFFFu;  // lane j <= 2G: relative event index of boundary kb + j

  // ring row of iteration k (byte offset from smem): the gap row for k < 0
  auto row_of = [&](int k) -> uint32_t {
    return rows_off + (k < 0 ? R2 : (static_cast<uint32_t>(k) & (R2 - 1))) * row_bytes;
  };

  run_ctx R;
  R.s_sub_pre = s_sub_pre;
  R.bwin = bwin;
  R.rlo = rlo;
  R.rhi = rhi;
  R.tend = tend;
  R.t0 = t0;
  R.t1w = t1w;
  R.R2 = R2;
  R.iters = kept ? static_cast<int>(iters) : -1;
  R.nnp = nnp;
  R.root_only = root_only;
  R.lb = lane * RM;
  R.bts_out = kept ? bts_out : nullptr;
  R.nbd = nbd;
  __syncthreads();
  // register pipelines of the two lane layouts: the interleaved one (one-warp
  // CTAs) rotates the step registers (tv / cv hold the step loaded ahead); the
  // run layout (wide CTAs) loads the next step into a second register set
  u64 tv[RM + 1];
  uint32_t cv[RM];
  u64 pf_pos = ~0ull;  // block start whose events sit in the pipeline registers
  ulonglong2 pts[RM / 2];
  uint4 pcx[RM / 4];
  u64 pnf = 0;

  for (uint32_t c = c_lo;; ++c) {
    const uint32_t kb = c * G;
    uint32_t E1 = end, E2 = end;
    bool cwide = false;
    if (CUBE && kept) {
      // boundary window of this chunk (prefetched during the previous one)
      if (lane <= static_cast<int>(R2)) {
        bwin[lane] = nx_idx + SOFF;  // stored + SOFF, see local_of
        bts[lane] = nx_ts;
      }
      mybw = lane <= static_cast<int>(R2) ? nx_idx : 0xFFFFFFFFu;
      // prefetch the next chunk's window: its loads overlap this chunk's events
      const u64 k = static_cast<u64>(kb + G) + lane;
      const bool have = lane <= static_cast<int>(R2) && k < nbd;
      nx_idx = nn_idx;
      nx_ts = (have && !optimistic) ? ldg64(btt + k) : tend;
      const bool have2 = lane <= static_cast<int>(R2) && k + G < nbd;
      nn_idx = have2 ? __ldg(bt + k + G) : static_cast<uint32_t>(n_t);
      __syncwarp();
      E1 = min(bwin[G] - SOFF, end);
      E2 = min(bwin[R2] - SOFF, end);
      // iteration spans of the ring (and the gap in chunk 0) decide 32- vs
      // 64-bit cells (exact mode; the optimistic mode runs 32-bit throughout)
      if (EXACT) {
        bool w = lane < static_cast<int>(R2) && bts[lane + 1] - bts[lane] >= kSpan32;
        if (c == 0 && lane == 0 && n_t) w = w || bts[0] - ldg64(p.tr.ts + b) >= kSpan32;
        cwide = __any_sync(FULL, w);
      }
    } else if (CUBE && active) {
      // skipped trace: only the window runs; iterations are not stored
      if (lane <= static_cast<int>(R2)) bwin[lane] = static_cast<uint32_t>(n_t) + SOFF;
      mybw = lane <= static_cast<int>(R2) ? static_cast<uint32_t>(n_t) : 0xFFFFFFFFu;
      __syncwarp();
    }

    // ---- phase 1: consume events [pos, E1), possibly running ahead to E2 ----
    while (pos < E1) {
      // step start sr (relative to b0); its base relative to b is sr - d0
      // >= -SOFF, kept as base3 = base + SOFF >= 0 so all of it is unsigned
      const uint32_t sr = (pos + d0) & ~static_cast<uint32_t>(SOFF);
      const uint32_t base3 = sr - d0 + SOFF;
      const uint32_t lim = min(base3 - SOFF + STEP_M, E2);
      const u64 s_abs = b0 + sr;
      R.base3 = base3;
      R.lo = static_cast<int>(pos + SOFF - base3);
      R.hi = static_cast<int>(lim + SOFF - base3);
      const uint32_t lr = n32 + SOFF - 1 - base3;  // the trace's last event, local index
      R.last_li = lr < static_cast<uint32_t>(STEP_M) ? static_cast<int>(lr) : -1;
      const u64 r0 = s_abs + static_cast<u64>(R.lb);
#ifndef PSG_Q_PF_DIST
#define PSG_Q_PF_DIST 3  // block steps of L2 prefetch run-ahead (0: none; 0 costs +18 %)
#endif
      if (PSG_Q_PF_DIST > 0) {
        const bool pf = lane == 0 && static_cast<u64>(sr) + (PSG_Q_PF_DIST + 1) * STEP_M <= static_cast<u64>(n32) + d0;
        prefetch_l2_lane0(ts_b0 + sr + PSG_Q_PF_DIST * STEP_M, 8 * STEP_M, pf);
        prefetch_l2_lane0(cx_b0 + sr + PSG_Q_PF_DIST * STEP_M, 4 * STEP_M, pf);
      }
      rot_src rs{};
      if constexpr (IL) {
      {
        // step positions relative to the aligned trace base b0 (32-bit), on
        // per-trace lane base pointers: no 64-bit address arithmetic per step
        if (pf_rel != sr) {  // first step (or the pipeline did not run ahead): load now
          u64 nf = 0;
          u64 t8[RM];
          load_step_il(p.tr, s_abs, lane, t8, cv, nf);
#pragma unroll
          for (int q = 0; q < RM; ++q) tv[q] = t8[q];
          tv[RM] = nf;
        }
        const bool more = lim < n32 && (PSG_PIPE_CROSS || lim < E1);
        const uint32_t nxt = (lim + d0) & ~static_cast<uint32_t>(SOFF);
        const uint32_t lp = more ? nxt : sr;
        pf_rel = more ? nxt : 0xFFFFFFFFu;
        rs.ts = ts_lane + lp;
        rs.ctx = cx_lane + lp;
      }
      } else {
      // software pipeline: this block step's events were loaded into registers
      // while the previous one was processed; load the next one now
      if (pf_pos != s_abs) {
        load_step(p.tr, r0, s_abs, lane, pts, pcx, pnf);
      }
#pragma unroll
      for (int q = 0; q < RM / 2; ++q) {
        tv[2 * q] = pts[q].x;
        tv[2 * q + 1] = pts[q].y;
      }
#pragma unroll
      for (int q = 0; q < RM / 4; ++q) {
        cv[4 * q] = pcx[q].x;
        cv[4 * q + 1] = pcx[q].y;
        cv[4 * q + 2] = pcx[q].z;
        cv[4 * q + 3] = pcx[q].w;
      }
      {
        u64 nf = __shfl_down_sync(FULL, tv[0], 1);
        if (lane == 31) nf = pnf;
        tv[RM] = nf;
      }
      if (PSG_PIPE_UNCOND) {
        // always load (this step again past the trace end: no branch, so the
        // loaded registers need no copies to join the paths)
        const bool more = lim < n32 && (PSG_PIPE_CROSS || lim < E1);
        const u64 nxt = b0 + ((lim + d0) & ~static_cast<uint32_t>(SOFF));
        const u64 lp = more ? nxt : s_abs;
        pf_pos = more ? nxt : ~0ull;
        load_step(p.tr, lp + static_cast<u64>(R.lb), lp, lane, pts, pcx, pnf);
      } else if (lim < n32 && (PSG_PIPE_CROSS || lim < E1)) {
        pf_pos = b0 + ((lim + d0) & ~static_cast<uint32_t>(SOFF));
        load_step(p.tr, pf_pos + static_cast<u64>(R.lb), pf_pos, lane, pts, pcx, pnf);
      } else {
        pf_pos = ~0ull;
      }
      }
      const bool all = R.lo == 0 && R.hi == STEP_M && R.last_li < 0;  // warp-uniform

      // window class of this block step (warp-uniform)
      int wm = WIN_NONE;
      if (WIN) {
        u64 first, after;
        if (all) {
          first = __shfl_sync(FULL, tv[0], 0);
          after = __shfl_sync(FULL, tv[RM], 31);
        } else if (IL) {
          // event i sits in lane i % 32, register i / 32; lo <= SOFF < 32
          u64 a = tv[0];
          {
            const int hx = R.hi >> 5;
#pragma unroll
            for (int q = 1; q < RM; ++q)
              if (hx == q) a = tv[q];
          }
          first = __shfl_sync(FULL, tv[0], R.lo);
          after = R.hi >= STEP_M ? __shfl_sync(FULL, tv[RM], 31) : __shfl_sync(FULL, a, R.hi & 31);
        } else {
          u64 f = tv[0];  // lo <= SOFF < RM: lane 0 owns the first valid event
#pragma unroll
          for (int q = 1; q < SA; ++q)
            if (R.lo == q) f = tv[q];
          // first valid event and the successor of the last valid one (index hi)
          u64 a;
          {  // warp-uniform index; constant register indices
            const int hx = R.hi & (RM - 1);
            a = tv[0];
#pragma unroll
            for (int q = 1; q < RM; ++q)
              if (hx == q) a = tv[q];
          }
          first = __shfl_sync(FULL, f, 0);
          after = R.hi >= STEP_M ? __shfl_sync(FULL, tv[RM], 31) : __shfl_sync(FULL, a, R.hi / RM);
        }
        const bool has_end = R.last_li >= 0 && R.last_li < R.hi;
        if ((first >= t1w && first >= t0) || (!has_end && after < t0)) {
          wm = WIN_NONE;
        } else if (has_end || after - first >= kSpan32) {
          wm = WIN_WIDE;
        } else {
          const u64 span = after - first;
          if (wspan + span >= kSpan32) {  // fold the pending 32-bit sums
            __syncwarp();
            for (uint32_t x = lane; x < n_ctx; x += 32) {
              uint32_t* r = T.wt + wt_word(x, IL);
              T.set_acc(x, T.acc(x) + r[WT_LO]);
              r[WT_LO] = 0;
            }
            __syncwarp();
            wspan = 0;
          }
          wspan += span;
          wm = (first >= t0 && after < t1w) ? WIN_FULL : WIN_PART;
        }
      }

      bool done = false;
      if constexpr (IL) {
      if (CUBE && kept && all && !cwide && (wm == WIN_FULL || wm == WIN_NONE)) {
        // boundaries of this block step: lane j <= 2G holds boundary kb + j;
        // fast path: at most one per group of 32 events, and every iteration
        // of the step is stored
        const uint32_t base32 = base3 - SOFF;  // >= 0 here (lo == 0)
        const uint32_t rel = mybw - base32;
        const bool inb = mybw >= base32 && rel < static_cast<uint32_t>(STEP_M);
        const uint32_t g = rel >> 5;
        const uint32_t H = __reduce_or_sync(FULL, inb ? 1u << g : 0u);
        const unsigned inm = __ballot_sync(FULL, inb);
        const uint32_t nb0 = __popc(__ballot_sync(FULL, mybw < base32));
        const int k0 = static_cast<int>(kb) - 1 + static_cast<int>(nb0);
        if (__popc(H) == __popc(inm) && kb + nb0 + __popc(inm) <= iters && k0 >= 0) {
          const uint32_t f = (rel & 31u) + 1u;
          const uint32_t fa = __reduce_or_sync(FULL, (inb && g < 5) ? f << (6 * g) : 0u);
          const uint32_t fb = __reduce_or_sync(FULL, (inb && g >= 5) ? f << (6 * (g - 5)) : 0u);
          // the boundaries' timestamps (optimistic pass 1): loaded now by the
          // lanes holding them, stored after the step's reductions
          const bool rec = bts_out && inb && kb + static_cast<uint32_t>(lane) < nbd;
          const u64 bval = rec ? ldg64(p.tr.ts + b + mybw) : 0ull;
          const uint32_t ra = rows_off + (static_cast<uint32_t>(k0) & (R2 - 1)) * row_bytes;
          const uint32_t rows_end = rows_off + R2 * row_bytes;
          if (wm == WIN_FULL)
            run_fast_il<WIN_FULL, GT>(tv, cv, lane, smem, wt_off, p.ppo_g, fa, fb, ra, rows_off, rows_end,
                                      row_bytes, rs);
          else
            run_fast_il<WIN_NONE, GT>(tv, cv, lane, smem, wt_off, p.ppo_g, fa, fb, ra, rows_off, rows_end,
                                      row_bytes, rs);
          if (rec) bts_out[kb + lane] = bval;
          done = true;
        }
      }
      } else {
      if (CUBE && kept && all && !cwide && (wm == WIN_FULL || wm == WIN_NONE)) {
        // boundaries of this block step: lane j <= 2G holds boundary kb + j;
        // H marks the lanes whose run holds one (fast path: at most one per
        // run, and every iteration of the step is stored)
        const uint32_t base32 = base3 - SOFF;  // >= 0 here (lo == 0)
        const uint32_t rel = mybw - base32;
        const bool inb = mybw >= base32 && rel < static_cast<uint32_t>(STEP_M);
        const uint32_t H = __reduce_or_sync(FULL, inb ? 1u << (rel / RM) : 0u);
        const unsigned inm = __ballot_sync(FULL, inb);
        const uint32_t nb0 = __popc(__ballot_sync(FULL, mybw < base32));
        if (__popc(H) == __popc(inm) && kb + nb0 + __popc(inm) <= iters) {
          const uint32_t jb = nb0 + __popc(H & lanemask_lt());  // first boundary at/after the run
          const uint32_t bw = __shfl_sync(FULL, mybw, static_cast<int>(jb & 31));
          const int bpos = ((H >> lane) & 1u) ? static_cast<int>(bw - base32) - R.lb : RM;
          const int k0 = static_cast<int>(kb) - 1 + static_cast<int>(jb);
          const uint32_t rb0 = row_of(k0), rb1 = row_of(k0 + 1);
          // the boundary's timestamp (optimistic pass 1): loaded now, stored
          // after the step's reductions so its latency is hidden behind them
          const bool rec = bts_out && bpos < RM && static_cast<uint32_t>(k0 + 1) < nbd;
          const u64 bval = rec ? ldg64(p.tr.ts + b + bw) : 0ull;
          // column offsets of the step's events (loading them earlier, before
          // the window classification, measured slower: register pressure)
          uint32_t ppo[RM];
#pragma unroll
          for (int j = 0; j < RM; ++j)
            ppo[j] = GT ? __ldg(p.ppo_g + cv[j])
                        : *reinterpret_cast<const uint32_t*>(smem + wt_off + 4u * (wt_word_l<false>(cv[j]) + WT_PPO));
          if (wm == WIN_FULL)
            run_fast<WIN_FULL>(tv, cv, smem, wt_off, bpos, rb0, rb1, ppo);
          else
            run_fast<WIN_NONE>(tv, cv, smem, wt_off, bpos, rb0, rb1, ppo);
          if (rec) bts_out[k0 + 1] = bval;
          done = true;
        }
      }
      }
      if (!done) {
        run_state st;
        st.k = -1;
        st.cnt = 0;
        st.nxt = INT_MAX;
        st.cube_ok = false;
        st.slot = R2;
        st.rowb = R2 * nnp;
        if (CUBE) {
          // iteration of this lane's first event: boundaries of the window at or before it
          uint32_t cnt = 0;
          const uint32_t lp3 = R.base3 + static_cast<uint32_t>(IL ? lane : R.lb);
          for (uint32_t j = 0; j <= R2; ++j) cnt += bwin[j] <= lp3 ? 1u : 0u;
          st.cnt = cnt;
          // a boundary on the lane's first event is counted here, not crossed
          // in run_events: record its timestamp (optimistic pass 1)
          if (R.bts_out && cnt > 0 && bwin[cnt - 1] == lp3 && kb - 1 + cnt < nbd)
            R.bts_out[kb - 1 + cnt] = tv[0];
          st.k = static_cast<int>(kb) - 1 + static_cast<int>(cnt);
          st.nxt = cnt <= R2 ? local_of(bwin[cnt], R.base3) : INT_MAX;
          st.slot = st.k < 0 ? R2 : (static_cast<uint32_t>(st.k) & (R2 - 1));
          st.rowb = st.slot * nnp;
          st.cube_ok = st.k < R.iters;
        }
        if constexpr (IL) {
        if (cwide)
          run_block_il<WIN, CUBE, true>(wm, tv, cv, lane, R, st, T, rs);
        else
          run_block_il<WIN, CUBE, false>(wm, tv, cv, lane, R, st, T, rs);
        } else {
        if (cwide)
          run_block<WIN, CUBE, true>(wm, tv, cv, R, st, T);
        else
          run_block<WIN, CUBE, false>(wm, tv, cv, R, st, T);
        }
      }
      pos = lim;
    }
    __syncwarp();

    // ---- phase 2: inclusive roll-up, cube stores (node-contiguous), within-rank sums ----
    const uint32_t k_lo = kb;
    const uint32_t k_hi = min(kb + G, iters);
    const uint32_t n_iter_rows = k_hi > k_lo ? k_hi - k_lo : 0;
    const uint32_t kcap = (CUBE && p.do_stats && kb < Kq) ? min(n_iter_rows, Kq - kb) : 0;
    if (CUBE && kept) {
      const uint32_t s0 = kb & (R2 - 1);  // the chunk's rows are slots [s0, s0 + G)
      uint32_t* rhw = cwide ? rhi : nullptr;  // high words (all zero in narrow chunks)
      const u64 ob = bo + static_cast<u64>(kb) * nnp;  // storage cell of the chunk's first row
      if (root_only && !cwide && n_iter_rows == G && (kcap == 0 || kcap == G)) {
        if (kcap)
          flush_fast<true>(p, rlo + s0 * nnp, nn, nnp, ob, ib + kb, wsx, wsqlo, wsqhi, lane);
        else
          flush_fast<false>(p, rlo + s0 * nnp, nn, nnp, ob, ib + kb, wsx, wsqlo, wsqhi, lane);
      } else if (root_only && !cwide) {
        // narrow partial chunk (the trace's last): the same straight copies, row by row
        uint32_t rs[GC];
#pragma unroll
        for (uint32_t r = 0; r < GC; ++r)
          rs[r] = (lane == 0 && r < n_iter_rows) ? rlo[(s0 + r) * nnp] : 0u;  // anchor's own excl
        for (uint32_t n = 1 + lane; n < nn; n += 32) {
          u64 sx = 0, sq = 0, sqh = 0;
#pragma unroll
          for (uint32_t r = 0; r < GC; ++r) {
            if (r < n_iter_rows) {
              const uint32_t idx = (s0 + r) * nnp + n;
              const uint32_t ex = rlo[idx];
              rs[r] += ex;
              store_cell(p, ob + r * nnp + n, ex);
              rlo[idx] = 0;
              if (r < kcap) {
                sx += ex;
                acc_sq(sq, sqh, ex);
              }
            }
          }
          if (kcap) {
            wsx[n] += sx;
            const u64 l2 = wsqlo[n] + sq;
            wsqhi[n] += sqh + (l2 < sq ? 1ull : 0ull);
            wsqlo[n] = l2;
          }
        }
#pragma unroll
        for (uint32_t r = 0; r < GC; ++r) rs[r] = __reduce_add_sync(FULL, rs[r]);
        // the anchor's cells: lane r writes row r; lane 0 folds the within sums
        uint32_t mine = rs[0];
#pragma unroll
        for (uint32_t r = 1; r < GC; ++r)
          if (static_cast<uint32_t>(lane) == r) mine = rs[r];
        if (static_cast<uint32_t>(lane) < n_iter_rows) {
          const uint32_t idx = (s0 + lane) * nnp;
          store_cell(p, ob + static_cast<u64>(lane) * nnp, mine);
          if (p.store_cube) p.cube_xint[ib + kb + lane] = rlo[idx];  // m == 1
          rlo[idx] = 0;
        }
        if (kcap && lane == 0) {
          u64 sx = 0, sq = 0, sqh = 0;
#pragma unroll
          for (uint32_t r = 0; r < GC; ++r)
            if (r < kcap) {
              sx += rs[r];
              acc_sq(sq, sqh, rs[r]);
            }
          wsx[0] += sx;
          const u64 l2 = wsqlo[0] + sq;
          wsqhi[0] += sqh + (l2 < sq ? 1ull : 0ull);
          wsqlo[0] = l2;
        }
      } else {
        for (uint32_t r = 0; r < n_iter_rows; ++r) {
          const uint32_t slot = s0 + r;
          warp_prefix_row(rlo + slot * nnp, rhw ? rhw + slot * nnp : nullptr, s_node, pref, nn, lane);
          for (uint32_t n = lane; n < nn; n += 32) {
            const int4 nd = s_node[n];
            const u64 ex = cell64(rlo, rhw, slot * nnp + n);
            const u64 in = nd.z ? pref[nd.x + nd.y] - pref[nd.x] : ex;
            store_cell(p, ob + static_cast<u64>(r) * nnp + n, in);
            if (nd.z && p.store_cube) p.cube_xint[(ib + kb + r) * p.m + (nd.z - 1)] = ex;
            if (r < kcap) {
              wsx[n] += in;
              u64 ql = 0, qh = 0;
              acc_sq(ql, qh, in);
              const u64 l2 = wsqlo[n] + ql;
              wsqhi[n] += qh + (l2 < ql ? 1ull : 0ull);
              wsqlo[n] = l2;
            }
          }
          __syncwarp();
          for (uint32_t n = lane; n < nn; n += 32) {
            rlo[slot * nnp + n] = 0;
            if (rhw) rhw[slot * nnp + n] = 0;
          }
          __syncwarp();
        }
      }
      if (c == 0) {  // the gap row [first_ts, b_0) (itermodel.cpp:331-338)
        __syncwarp();
        warp_prefix_row(rlo + R2 * nnp, rhw ? rhw + R2 * nnp : nullptr, s_node, pref, nn, lane);
        for (uint32_t n = lane; n < nn; n += 32) {
          const int4 nd = s_node[n];
          const u64 ex = cell64(rlo, rhw, R2 * nnp + n);
          const u64 in = !nd.z ? ex : pref[nd.x + nd.y] - pref[nd.x];
          p.gap_excl[static_cast<size_t>(tp) * nn + n] = ex;
          p.gap_incl[static_cast<size_t>(tp) * nn + n] = in;
        }
        __syncwarp();
        for (uint32_t n = lane; n < nn; n += 32) {
          rlo[R2 * nnp + n] = 0;
          if (rhw) rhw[R2 * nnp + n] = 0;
        }
      }
      __syncwarp();
    }
    if (pos >= end && c + 1 >= c_stop) break;
  }

  if (!active) return;
  if (WIN) {
    // exclusive ns incl. the carry-in segment, in CCT preorder, then the
    // inclusive roll-up: every subtree is a contiguous preorder range
    __syncwarp();
    u64* tmp = reinterpret_cast<u64*>(wb + L.off_scan);
    u64* scan = tmp + (n_ctx + 1);
    const bool c_has = (T.carry[2] >> 32) != 0;
    const uint32_t c_ctx = static_cast<uint32_t>(T.carry[2]);
    const u64 c_d = T.carry[1];
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      const u64 sum = T.acc(c) + T.wt[wt_word(c, IL) + WT_LO];
      tmp[s_cct_pre[c]] = sum + ((c_has && c == c_ctx) ? c_d : 0ull);
    }
    __syncwarp();
    warp_prefix(tmp, scan, n_ctx, lane);
    __threadfence();  // the big min/max atomics of all lanes, before the read-back
    __syncwarp();
    const size_t base = static_cast<size_t>(t) * n_ctx;
    if (split) {
      // one unit of a split trace: merge into the rows k_split_init prepared
      // (the min / max of durations >= 2^32 are already in them)
      for (uint32_t c = lane; c < n_ctx; c += 32) {
        const uint32_t* r = T.wt + wt_word(c, IL);
        const int pr = s_cct_pre[c], sz = s_cct_size[c];
        const u64 cnt = r[WT_CNT], nbig = r[WT_NBIG];
        unsigned long long* wc = reinterpret_cast<unsigned long long*>(p.w_cnt) + base + c;
        if (cnt) {
          atomicAdd(wc, cnt);
          atomicAdd(reinterpret_cast<unsigned long long*>(p.w_sum) + base + c, T.acc(c) + r[WT_LO]);
        }
        if (cnt > nbig) {
          atomicMin(reinterpret_cast<unsigned long long*>(p.w_min) + base + c, static_cast<u64>(r[WT_MIN]));
          atomicMax(reinterpret_cast<unsigned long long*>(p.w_max) + base + c, static_cast<u64>(r[WT_MAX]));
        }
        const u64 ex = scan[pr + 1] - scan[pr], in = scan[pr + sz] - scan[pr];
        if (ex) atomicAdd(reinterpret_cast<unsigned long long*>(p.w_excl) + base + c, ex);
        if (in) atomicAdd(reinterpret_cast<unsigned long long*>(p.w_incl) + base + c, in);
      }
      if (lane == 0 && c_has) {  // the carry-in event lies in exactly one unit
        p.c_has[t] = 1;
        p.c_ts[t] = T.carry[0];
        p.c_ctx[t] = c_ctx;
      }
    }
    for (uint32_t c = lane; c < (split ? 0u : n_ctx); c += 32) {
      const uint32_t* r = T.wt + wt_word(c, IL);
      const int pr = s_cct_pre[c], sz = s_cct_size[c];
      const u64 cnt = r[WT_CNT], nbig = r[WT_NBIG];
      const u64 sum = T.acc(c) + r[WT_LO];
      const u64 minb = nbig ? __ldcg(T.gminb + c) : 0ull, maxb = nbig ? __ldcg(T.gmaxb + c) : 0ull;
      p.w_cnt[base + c] = cnt;
      p.w_sum[base + c] = sum;
      p.w_min[base + c] = cnt == 0 ? 0ull : (cnt > nbig ? static_cast<u64>(r[WT_MIN]) : minb);
      p.w_max[base + c] = nbig ? maxb : static_cast<u64>(r[WT_MAX]);
      p.w_mean[base + c] = cnt ? static_cast<double>(sum) / static_cast<double>(cnt) : 0.0;
      p.w_excl[base + c] = scan[pr + 1] - scan[pr];
      p.w_incl[base + c] = scan[pr + sz] - scan[pr];
    }
    if (lane == 0 && !split) {
      p.c_has[t] = c_has ? 1 : 0;
      p.c_ts[t] = c_has ? T.carry[0] : 0;
      p.c_ctx[t] = c_has ? c_ctx : 0;
    }
  }
  if (CUBE && p.do_stats && kept && Kq > 0 && split) {
    // a unit's within-rank sums into the trace's accumulators (128-bit Σx²:
    // the low word's carry goes to the high word)
    unsigned long long* a = p.wacc + static_cast<size_t>(tp) * nn * 3;
    for (uint32_t n = lane; n < nn; n += 32) {
      if (wsx[n]) atomicAdd(a + 3 * n, wsx[n]);
      const u64 ql = wsqlo[n];
      u64 qh = wsqhi[n];
      if (ql) {
        const u64 old = atomicAdd(a + 3 * n + 1, ql);
        qh += old + ql < old ? 1ull : 0ull;
      }
      if (qh) atomicAdd(a + 3 * n + 2, qh);
    }
  } else if (CUBE && p.do_stats && kept && Kq > 0) {
    for (uint32_t n = lane; n < nn; n += 32) {
      const u64 sx = wsx[n];
      const u128 sq = (static_cast<u128>(wsqhi[n]) << 64) | wsqlo[n];
      const u128 num = static_cast<u128>(Kq) * sq - static_cast<u128>(sx) * sx;
      const bool ok = sx > 0;
      p.within_cv[static_cast<size_t>(tp) * nn + n] =
          ok ? 100.0 * sqrt(u128_to_double(num)) / static_cast<double>(sx) : 0.0;
      p.within_ok[static_cast<size_t>(tp) * nn + n] = ok ? 1 : 0;
    }
  }
}

template <bool WIN, bool CUBE, bool EXACT, bool ONE, bool GT = false>
void launch_shape(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  // the dynamic shared-memory opt-in is a per-device function attribute: track
  // it per device (one process may drive several GPUs) under a lock
  static std::mutex mu;
  static int configured_bytes[64] = {};
  int dev = 0;
  PSG_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 64 || static_cast<int>(smem_bytes) > configured_bytes[dev]) {
      PSG_CUDA(cudaFuncSetAttribute(k_trace_query<WIN, CUBE, EXACT, ONE, GT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem_bytes)));
      if (dev < 64) configured_bytes[dev] = static_cast<int>(smem_bytes);
    }
  }
  const unsigned blocks = p.units ? (p.n_units + p.warps - 1) / p.warps
                                  : (p.t_stop - p.t_base + p.warps - 1) / p.warps;
  k_trace_query<WIN, CUBE, EXACT, ONE, GT><<<blocks, p.warps * 32, smem_bytes, s>>>(p);
}

template <bool WIN, bool CUBE, bool EXACT>
void launch_variant(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  if (p.one_warp) {
    if (p.warps != 1) fail(PS_E_INTERNAL, "one-warp CTA shape with warps != 1");
    launch_shape<WIN, CUBE, EXACT, true>(p, smem_bytes, s);
  } else {
    if (p.warps * 32 > PSG_WIDE_THREADS) fail(PS_E_INTERNAL, "more warps per CTA than the launch bound");
    launch_shape<WIN, CUBE, EXACT, false>(p, smem_bytes, s);
  }
}

template <bool WIN, bool CUBE, bool EXACT, bool GT>
uint32_t one_warp_occupancy(uint32_t smem_bytes) {
  int per_sm = 0;
  PSG_CUDA(cudaFuncSetAttribute(k_trace_query<WIN, CUBE, EXACT, true, GT>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes)));
  PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trace_query<WIN, CUBE, EXACT, true, GT>, 32,
                                                         smem_bytes));
  return static_cast<uint32_t>(per_sm);
}

}  // namespace

uint32_t trace_query_one_warp_per_sm(bool win, bool cube, bool exact, bool gt, uint32_t smem_bytes) {
  if (gt) return exact ? one_warp_occupancy<false, true, true, true>(smem_bytes)
                       : one_warp_occupancy<false, true, false, true>(smem_bytes);
  if (win && cube) return exact ? one_warp_occupancy<true, true, true, false>(smem_bytes)
                                : one_warp_occupancy<true, true, false, false>(smem_bytes);
  if (win) return one_warp_occupancy<true, false, false, false>(smem_bytes);
  return exact ? one_warp_occupancy<false, true, true, false>(smem_bytes)
               : one_warp_occupancy<false, true, false, false>(smem_bytes);
}

void launch_trace_query(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  if (p.t_stop <= p.t_base || p.t_stop > p.tr.n) {
    if (p.t_stop > p.tr.n) fail(PS_E_INTERNAL, "trace range past the loaded traces");
    return;
  }
  if (p.G != GC) fail(PS_E_INTERNAL, "chunk size mismatch between host and kernel (PSG_G)");
  const bool exact = p.do_cube && p.exact_bounds;
  if (p.ppo_g) {  // cube only, global column table (large calling-context trees)
    if (p.do_window || !p.do_cube || !p.one_warp || p.warps != 1)
      fail(PS_E_INTERNAL, "global column tables need a cube-only query on one-warp CTAs");
    exact ? launch_shape<false, true, true, true, true>(p, smem_bytes, s)
          : launch_shape<false, true, false, true, true>(p, smem_bytes, s);
  } else if (p.do_window && p.do_cube)
    exact ? launch_variant<true, true, true>(p, smem_bytes, s) : launch_variant<true, true, false>(p, smem_bytes, s);
  else if (p.do_window)
    launch_variant<true, false, false>(p, smem_bytes, s);
  else
    exact ? launch_variant<false, true, true>(p, smem_bytes, s) : launch_variant<false, true, false>(p, smem_bytes, s);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ---- split traces (work units) ----------------------------------------------
// One warp per split trace: its global window rows start empty (min at ~0 for
// the atomicMin merges), its carry-in absent, its within-rank accumulators 0.
__global__ void k_split_init(query_params p, const uint32_t* split, uint32_t n_split) {
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_split) return;
  const uint32_t t = split[i];
  if (p.do_window) {
    const size_t base = static_cast<size_t>(t) * p.n_ctx;
    for (uint32_t c = lane; c < p.n_ctx; c += 32) {
      p.w_cnt[base + c] = p.w_sum[base + c] = p.w_max[base + c] = 0;
      p.w_excl[base + c] = p.w_incl[base + c] = 0;
      p.w_min[base + c] = ~0ull;
    }
    if (lane == 0) {
      p.c_has[t] = 0;
      p.c_ts[t] = 0;
      p.c_ctx[t] = 0;
    }
  }
  if (p.do_cube && p.do_stats && p.wacc && p.iter_count[t] > 0) {
    unsigned long long* a = p.wacc + static_cast<size_t>(p.tpos[t]) * p.nn * 3;
    for (uint32_t j = lane; j < 3 * p.nn; j += 32) a[j] = 0;
  }
}

// After pass 2: a split trace's window mean and empty-group min, and its
// within-rank CVs from the merged sums (the same formula as pass 2's epilogue).
__global__ void k_split_finish(query_params p, const uint32_t* split, uint32_t n_split) {
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n_split) return;
  const uint32_t t = split[i];
  if (p.do_window) {
    const size_t base = static_cast<size_t>(t) * p.n_ctx;
    for (uint32_t c = lane; c < p.n_ctx; c += 32) {
      const u64 cnt = p.w_cnt[base + c];
      if (cnt == 0) p.w_min[base + c] = 0;
      p.w_mean[base + c] = cnt ? static_cast<double>(p.w_sum[base + c]) / static_cast<double>(cnt) : 0.0;
    }
  }
  const uint32_t Kq = p.qs ? qs_K(p.qs) : p.K;
  if (p.do_cube && p.do_stats && p.wacc && p.iter_count[t] > 0 && Kq > 0) {
    const uint32_t tp = p.tpos[t];
    const unsigned long long* a = p.wacc + static_cast<size_t>(tp) * p.nn * 3;
    for (uint32_t n = lane; n < p.nn; n += 32) {
      const u64 sx = a[3 * n];
      const u128 sq = (static_cast<u128>(a[3 * n + 2]) << 64) | a[3 * n + 1];
      const u128 num = static_cast<u128>(Kq) * sq - static_cast<u128>(sx) * sx;
      const bool ok = sx > 0;
      p.within_cv[static_cast<size_t>(tp) * p.nn + n] =
          ok ? 100.0 * sqrt(u128_to_double(num)) / static_cast<double>(sx) : 0.0;
      p.within_ok[static_cast<size_t>(tp) * p.nn + n] = ok ? 1 : 0;
    }
  }
}

void launch_split_init(const query_params& p, const uint32_t* split, uint32_t n_split, cudaStream_t s) {
  if (!n_split) return;
  k_split_init<<<(n_split + 7) / 8, 256, 0, s>>>(p, split, n_split);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

void launch_split_finish(const query_params& p, const uint32_t* split, uint32_t n_split, uint32_t,
                         cudaStream_t s) {
  if (!n_split) return;
  k_split_finish<<<(n_split + 7) / 8, 256, 0, s>>>(p, split, n_split);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// Cross-rank (iteration, node) statistics over the stored inclusive cube: the
// sufficient statistics of node_matrix / savings_report / iteration_cv_report
// (diagnostics.cpp:83-158) — per cell Σx, max x and Σx² over the kept traces,
// for k < K (the ordinal intersection).  Grid = (k tiles) x (trace tiles): a
// thread owns two adjacent cells (k, 2q), (k, 2q + 1) of its tile (rows have
// an even stride nnp, so the pair is one 8- or 16-byte load) and streams them
// over the tile's traces (a trace's tile is kt rows of nnp contiguous cells,
// so the loads coalesce); the global atomics happen once per cell per tile.
template <typename CELL> struct cell_pair;
template <> struct cell_pair<uint32_t> {
  __device__ static void get(const uint32_t* p, uint32_t& a, uint32_t& b) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    a = v.x;
    b = v.y;
  }
};
template <> struct cell_pair<unsigned long long> {
  __device__ static void get(const unsigned long long* p, unsigned long long& a,
                             unsigned long long& b) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    a = v.x;
    b = v.y;
  }
};

struct cell_acc {
  u64 sum = 0, mx = 0, ql = 0, qh = 0;
  __device__ __forceinline__ void add32(u64 v) {  // squares on the 32-bit fast path
    sum += v;
    mx = max(mx, v);
    const u64 q = static_cast<u64>(static_cast<uint32_t>(v)) * static_cast<uint32_t>(v);
    ql += q;
    qh += ql < q ? 1ull : 0ull;
  }
  // a batch's sum, maximum and (non-overflowing) sum of squares
  __device__ __forceinline__ void add_batch(u64 s, uint32_t m, u64 q) {
    sum += s;
    mx = max(mx, static_cast<u64>(m));
    ql += q;
    qh += ql < q ? 1ull : 0ull;
  }
};

template <typename CELL>
__global__ void __launch_bounds__(512, PSG_X_MINB) k_cross_stats(const CELL* __restrict__ incl,
                                                        const uint64_t* __restrict__ kept_bo,
                                                        uint32_t n_kept, uint32_t nn, uint32_t nnp,
                                                        uint32_t K, uint32_t kt, uint32_t per_tile,
                                                        unsigned long long* x_sum,
                                                        unsigned long long* x_max,
                                                        unsigned long long* x_sq,
                                                        const unsigned long long* qs,
                                                        const uint32_t* tpos, uint32_t ta,
                                                        uint32_t tb, uint32_t n_tr) {
  // The tile's trace block offsets are staged in shared memory in batches and
  // read as broadcasts; U independent pair loads are in flight per thread.
  constexpr int U = sizeof(CELL) == 4 ? PSG_X_U : 8;
  constexpr uint32_t TB = 512;
  __shared__ u64 s_bo[TB];
  // K (the accumulator plane's stride) and n_kept are capacities when the
  // status block is given: the actual values come from it
  const size_t plane = static_cast<size_t>(K) * nn;
  if (qs) {
    if (qs[QS_CAP_MISS]) return;  // the query re-runs
    K = min(K, qs_K(qs));
    n_kept = min(n_kept, static_cast<uint32_t>(qs[QS_KEPT]));
  }
  const uint32_t k0 = blockIdx.x * kt;
  if (k0 >= K) return;
  const uint32_t kc = min(kt, K - k0);
  // a part: the kept traces among loaded traces [ta, tb)
  const uint32_t ka = tpos ? (ta < n_tr ? tpos[ta] : n_kept) : 0u;
  const uint32_t kb = tpos ? (tb < n_tr ? tpos[tb] : n_kept) : n_kept;
  const uint32_t t_lo = ka + blockIdx.y * per_tile, t_hi = min(kb, t_lo + per_tile);
  const uint32_t hp = nnp / 2;  // pairs per row
  const uint32_t npairs = kc * hp;
  for (uint32_t pr0 = 0; pr0 < npairs; pr0 += blockDim.x) {
    const uint32_t pr = pr0 + threadIdx.x;
    const bool mine = pr < npairs;
    const uint32_t kk = mine ? pr / hp : 0, n0 = mine ? 2 * (pr - kk * hp) : 0;
    const u64 off = static_cast<u64>(k0 + kk) * nnp + n0;  // storage cell within the trace block
    cell_acc A, B;
    bool wide = false;
    for (uint32_t tb = t_lo; tb < t_hi; tb += TB) {
      const uint32_t nb = min(TB, t_hi - tb);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) s_bo[i] = kept_bo[tb + i];
      __syncthreads();
      if (!mine) continue;
      uint32_t i = 0;
      for (; i + U <= nb; i += U) {
        CELL a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cell_pair<CELL>::get(incl + s_bo[i + u] + off, a[u], b[u]);
        if (sizeof(CELL) == 4) {
          // 32-bit cells: the batch's maxima first; below 2^30 the U squares
          // fit 64 bits, so the 128-bit accumulators are touched once per
          // batch instead of once per cell (2^30 ns = 1.07 s: the anchor's
          // inclusive cells, ~2^28 here, stay on this path with the leaves,
          // so warps do not diverge over the anchor column)
          uint32_t ma = 0, mb = 0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            ma = max(ma, static_cast<uint32_t>(a[u]));
            mb = max(mb, static_cast<uint32_t>(b[u]));
          }
          static_assert(U <= 16, "U squares of values < 2^30 must fit 64 bits");
          if (((ma | mb) >> 30) == 0) {
            u64 sa = 0, sb = 0, qa = 0, qb = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t x = static_cast<uint32_t>(a[u]), y = static_cast<uint32_t>(b[u]);
              sa += x;
              sb += y;
              qa = mad_wide(x, x, qa);
              qb = mad_wide(y, y, qb);
            }
            A.add_batch(sa, ma, qa);
            B.add_batch(sb, mb, qb);
            continue;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          A.add32(a[u]);
          B.add32(b[u]);
        }
      }
      for (; i < nb; ++i) {
        CELL a, b;
        cell_pair<CELL>::get(incl + s_bo[i] + off, a, b);
        A.add32(a);
        B.add32(b);
      }
    }
    if (!mine || t_hi <= t_lo) continue;
    // a value >= 2^32 (64-bit cells only): exact 128-bit squares for that cell
    wide = (A.mx >> 32) || (B.mx >> 32);
    if (wide) {
      A.ql = A.qh = B.ql = B.qh = 0;
      for (uint32_t t = t_lo; t < t_hi; ++t) {
        CELL a, b;
        cell_pair<CELL>::get(incl + ldg64(kept_bo + t) + off, a, b);
        acc_sq(A.ql, A.qh, a);
        acc_sq(B.ql, B.qh, b);
      }
    }
    const u64 mask43 = (1ull << 43) - 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const cell_acc& C = h ? B : A;
      if (n0 + h >= nn) continue;  // pad column
      const size_t ci = static_cast<size_t>(k0 + kk) * nn + n0 + h;
      atomicAdd(x_sum + ci, C.sum);
      atomicMax(x_max + ci, C.mx);
      atomicAdd(x_sq + ci, C.ql & mask43);
      atomicAdd(x_sq + plane + ci, ((C.ql >> 43) | (C.qh << 21)) & mask43);
      const u64 top = C.qh >> 22;
      if (top) atomicAdd(x_sq + 2 * plane + ci, top);
    }
  }
}

void launch_cross_stats(const void* incl, bool cube32, const uint64_t* kept_bo, uint32_t n_kept,
                        uint32_t nn, uint32_t nnp, uint32_t K, unsigned long long* x_sum,
                        unsigned long long* x_max, unsigned long long* x_sq,
                        const unsigned long long* qs, cudaStream_t s, const cross_part& part) {
  if (part.tpos) n_kept = part.tb - part.ta;  // the part's traces bound its kept ones
  if (n_kept == 0 || K == 0 || nn == 0) return;
  const uint32_t th = part.threads;
  const uint32_t kt = nnp >= 2 * th ? 1u : 2 * th / nnp;  // ~th pairs per CTA
  const uint32_t gx = (K + kt - 1) / kt;  // iteration tiles
  // trace ranges: the CTA count fills whole waves of the resident slots as
  // closely as possible (a last wave of a few CTAs would leave the GPU idle
  // for a whole CTA duration)
  int dev = 0, sms = 148, per_sm = 2;
  PSG_CUDA(cudaGetDevice(&dev));
  PSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (cube32)
    PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cross_stats<uint32_t>, th, 0));
  else
    PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cross_stats<unsigned long long>, th, 0));
  const uint32_t slots = static_cast<uint32_t>(std::max(1, sms * std::max(1, per_sm)));
  const uint32_t gy_cap = std::max(1u, (n_kept + 63) / 64);  // >= 64 traces per CTA
  uint32_t gy = 1, per_tile = n_kept;
  double best = -1.0;
  for (uint32_t w = 2; w <= 8; ++w) {
    uint32_t g = std::min(gy_cap, std::max(1u, w * slots / gx));
    const uint32_t pt = (n_kept + g - 1) / g;
    g = (n_kept + pt - 1) / pt;
    const double ctas = static_cast<double>(gx) * g;
    const double eff = ctas / (std::ceil(ctas / slots) * slots);
    if (eff > best + 0.01) {
      best = eff;
      gy = g;
      per_tile = pt;
    }
  }
  const uint32_t nk_arg = part.tpos ? 0xFFFFFFFFu : n_kept;  // parts: the kept total comes from qs
  if (cube32)
    k_cross_stats<uint32_t><<<dim3(gx, gy), th, 0, s>>>(static_cast<const uint32_t*>(incl), kept_bo,
                                                        nk_arg, nn, nnp, K, kt, per_tile, x_sum,
                                                        x_max, x_sq, qs, part.tpos, part.ta, part.tb,
                                                        part.n);
  else
    k_cross_stats<unsigned long long><<<dim3(gx, gy), th, 0, s>>>(
        static_cast<const unsigned long long*>(incl), kept_bo, nk_arg, nn, nnp, K, kt, per_tile,
        x_sum, x_max, x_sq, qs, part.tpos, part.ta, part.tb, part.n);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
