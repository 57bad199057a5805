// The fused trace query on sm_100a: two passes over the event stream.
//
//   k_bounds       pass 1 — iteration boundaries per trace (itermodel.cpp:111-143):
//                  reads ctx only (4 B/event) plus the timestamp of each
//                  boundary candidate, writes the boundary event indices.
//   k_trace_query  pass 2 — ONE read of ts+ctx (12 B/event) computing
//                    * the window filter + per-(trace, ctx) count/sum/min/max/mean
//                      (ingest.cpp:178-208 + frame.cpp:290-408),
//                    * the time-integrated excl/incl of the window incl. the
//                      carry-in segment (itermodel.cpp:145-183),
//                    * the trace x iteration x node cube incl/excl + gap rows
//                      (itermodel.cpp:242-360),
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
#include <climits>
#include <cstdint>

#include "psg_internal.h"

namespace psg {

namespace {

constexpr unsigned FULL = 0xffffffffu;
typedef unsigned long long u64;
typedef unsigned __int128 u128;

constexpr int RB = 16;  // events per lane per block step, pass 1 (ctx: 4 x 128-bit loads)
constexpr int RM = 8;   // events per lane per block step, pass 2 (ts: 4, ctx: 2 x 128-bit loads)
constexpr int STEP_B = 32 * RB;
constexpr int STEP_M = 32 * RM;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ u64 ldg64(const uint64_t* p) {
  return static_cast<u64>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
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
__global__ void __launch_bounds__(256) k_bounds(bound_params p) {
  extern __shared__ uint32_t s_bits[];
  for (uint32_t i = threadIdx.x; i < p.words; i += blockDim.x) s_bits[i] = p.contains[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= p.tr.n) return;
  const u64 b = p.tr.off[t], e = p.tr.off[t + 1];
  const u64 cap = p.cap_off[t + 1] - p.cap_off[t];
  uint32_t* out = p.bidx + p.cap_off[t];
  uint32_t prev_in = 0;  // containment of the event before the block step
  bool have_c = false;   // a candidate has been seen ...
  u64 last_c = 0;        // ... with this timestamp
  u64 nb = 0, last_b = 0;
  for (u64 s = b & ~3ull; s < e; s += STEP_B) {
    const u64 r0 = s + static_cast<u64>(lane) * RB;
    if (lane == 0 && s + 3 * STEP_B <= e)
      prefetch_l2(p.tr.ctx + s + 2 * STEP_B, 4 * STEP_B);
    uint32_t cx[RB];
    const uint4* src = reinterpret_cast<const uint4*>(p.tr.ctx + r0);
#pragma unroll
    for (int q = 0; q < RB / 4; ++q) {
      const uint4 v = __ldg(src + q);
      cx[4 * q] = v.x;
      cx[4 * q + 1] = v.y;
      cx[4 * q + 2] = v.z;
      cx[4 * q + 3] = v.w;
    }
    uint32_t inm = 0;
#pragma unroll
    for (int j = 0; j < RB; ++j) {
      const u64 i = r0 + j;
      const bool real = i >= b && i < e;
      const uint32_t c = real ? cx[j] : 0u;
      const uint32_t in = real ? ((s_bits[c >> 5] >> (c & 31)) & 1u) : 0u;
      inm |= in << j;
    }
    uint32_t up = __shfl_up_sync(FULL, inm >> (RB - 1), 1);
    if (lane == 0) up = prev_in;
    const uint32_t candm = inm & ~((inm << 1) | (up & 1u));
    prev_in = __shfl_sync(FULL, (inm >> (RB - 1)) & 1u, 31);
    const unsigned any = __ballot_sync(FULL, candm != 0);
    if (!any) continue;
    // timestamp of this lane's last candidate; the previous candidate before
    // this lane's first one comes from the nearest lower lane with candidates
    u64 my_last = 0;
    if (candm) my_last = ldg64(p.tr.ts + r0 + (31 - __clz(candm)));
    const unsigned lower = any & lanemask_lt();
    u64 prv = __shfl_sync(FULL, my_last, lower ? 31 - __clz(lower) : lane);
    bool has_prv = lower != 0 || have_c;
    if (!lower) prv = last_c;
    uint32_t bm = 0, nbl = 0;
    u64 lb = 0;
    for (uint32_t m = candm; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const u64 tj = (m & (m - 1)) ? ldg64(p.tr.ts + r0 + j) : my_last;
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
      if (kk < cap) out[kk] = static_cast<uint32_t>(r0 + (__ffs(m) - 1) - b);
    nb += tot;
    last_c = __shfl_sync(FULL, my_last, 31 - __clz(any));
    have_c = true;
    const unsigned bl = __ballot_sync(FULL, nbl != 0);
    if (bl) last_b = __shfl_sync(FULL, lb, 31 - __clz(bl));
  }
  if (lane == 0) {
    uint32_t it = static_cast<uint32_t>(nb);
    if (nb > 0 && last_b >= p.tr.t_end[t]) it -= 1;  // empty last interval dropped
    p.n_bounds[t] = static_cast<uint32_t>(nb);
    p.iter_count[t] = it;
    if (nb > cap) atomicAdd(p.overflow, 1ull);
  }
}

void launch_bounds(const bound_params& p, cudaStream_t s) {
  if (p.tr.n == 0) return;
  k_bounds<<<(p.tr.n + 7) / 8, 256, 4u * p.words, s>>>(p);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// Pass 2: the fused query.  A CTA owns `warps` consecutive traces, one warp
// each, and advances in chunks of G iterations.  Phase 1: every warp consumes
// events until its trace has passed the end of chunk c (it may run ahead into
// chunk c+1: the cube rows form a ring of 2G iterations plus the gap row).
// Phase 2: each warp rolls the chunk's rows up to inclusive time, stores them
// (coalesced along the node axis) and folds them into its within-rank sums;
// with statistics on, the CTA then folds its traces into the cross-rank
// (iteration, node) accumulators.  Without statistics the warps never
// synchronise with each other.
namespace {

enum : int { WIN_NONE = 0, WIN_FULL = 1, WIN_PART = 2 };

struct warp_tables {
  uint32_t *wcnt, *wslo, *wshi, *wmin, *wmax, *wnbig;
  u64 *wminb, *wmaxb;
  u64* carry;
};

// One window row of duration d for ctx c (frame::group_aggregate's
// count/sum/min/max fold, order-free in integers).
__device__ __forceinline__ void win_row(const warp_tables& T, uint32_t c, u64 d) {
  atomicAdd(T.wcnt + c, 1u);
  sadd64(T.wslo + c, T.wshi + c, d);
  if (d >> 32) {
    atomicAdd(T.wnbig + c, 1u);
    atomicMin(reinterpret_cast<unsigned long long*>(T.wminb + c), d);
    atomicMax(reinterpret_cast<unsigned long long*>(T.wmaxb + c), d);
  } else {
    atomicMin(T.wmin + c, static_cast<uint32_t>(d));
    atomicMax(T.wmax + c, static_cast<uint32_t>(d));
  }
}

struct run_state {
  int k;            // iteration of the current event (-1: before the first boundary)
  uint32_t cnt;     // boundaries of the window at or before the current event
  int nxt;          // local index of the next boundary
  bool cube_ok;     // k is a stored iteration (or the gap of a kept trace)
  uint32_t* rb;     // cube row of k (32-bit words)
  u64* rt;          // row total of k
  u64 racc;         // this lane's pending contribution to *rt
};

// Boundary event index (relative to the trace) as a local index of the block
// step starting at `base` (clamped past the step).
__device__ __forceinline__ int local_of(uint32_t bw, int64_t base) {
  const int64_t v = static_cast<int64_t>(bw) - base;
  return v > STEP_M ? STEP_M + 1 : static_cast<int>(v);
}

template <bool WIN, bool CUBE, int WM>
__device__ __forceinline__ void run_events(const u64 (&tv)[RM + 1], const uint32_t (&cv)[RM],
                                           int lb, int lo, int hi, int last_li, u64 tend, u64 t0,
                                           u64 t1w, const int32_t* s_sub_pre,
                                           const uint32_t* bwin, int64_t base, uint32_t R2,
                                           uint32_t iters, u64* rows, u64* rtot, uint32_t nn,
                                           bool root_only, run_state& st, const warp_tables& T) {
#pragma unroll
  for (int j = 0; j < RM; ++j) {
    const int li = lb + j;
    const bool valid = static_cast<unsigned>(li - lo) < static_cast<unsigned>(hi - lo);
    const u64 tsj = tv[j], nts = tv[j + 1];
    const uint32_t cj = valid ? cv[j] : 0u;
    const bool last = li == last_li;
    if (CUBE) {
      if (li >= st.nxt) {  // boundaries are distinct events: at most one per event
        if (root_only && st.racc) {
          sadd64(reinterpret_cast<uint32_t*>(st.rt), reinterpret_cast<uint32_t*>(st.rt) + 1,
                 st.racc);
          st.racc = 0;
        }
        ++st.k;
        ++st.cnt;
        st.nxt = st.cnt <= R2 ? local_of(bwin[st.cnt], base) : INT_MAX;
        const uint32_t slot = st.k < 0 ? R2 : (static_cast<uint32_t>(st.k) & (R2 - 1));
        st.cube_ok = st.k < static_cast<int>(iters);
        st.rb = reinterpret_cast<uint32_t*>(rows + slot * nn);
        st.rt = rtot + slot;
      }
      const int pp = s_sub_pre[cj];
      if (valid && pp >= 0 && st.cube_ok) {
        const u64 dc = (last ? tend : nts) - tsj;
        sadd64(st.rb + 2 * pp, st.rb + 2 * pp + 1, dc);
        if (root_only) st.racc += dc;
      }
    }
    if (WIN && WM == WIN_FULL) {
      if (valid) win_row(T, cj, nts - tsj);
    } else if (WIN && WM == WIN_PART) {
      if (valid) {
        if (tsj >= t0) {
          if (tsj < t1w) win_row(T, cj, (last ? t1w : min(nts, t1w)) - tsj);
        } else if (last || nts >= t0) {  // the carry-in event (store.cpp:667-670): unique
          const u64 e2 = last ? t1w : min(nts, t1w);
          T.carry[0] = tsj;
          T.carry[1] = e2 > t0 ? e2 - t0 : 0;
          T.carry[2] = (1ull << 32) | cj;
        }
      }
    }
  }
}

template <bool WIN, bool CUBE>
__global__ void __launch_bounds__(512, 1) k_trace_query(query_params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t W = p.warps, n_ctx = p.n_ctx, nn = p.nn, G = p.G, R2 = 2 * G;
  const bool root_only = p.root_only != 0;

  int4* s_node = reinterpret_cast<int4*>(smem);
  int32_t* s_sub_pre = reinterpret_cast<int32_t*>(s_node + nn);
  int32_t* s_cct_pre = s_sub_pre + n_ctx;
  int32_t* s_cct_size = s_cct_pre + n_ctx;
  uint32_t* s_kept = reinterpret_cast<uint32_t*>(s_cct_size + n_ctx);

  warp_smem_layout L;
  L.init(n_ctx, nn, G);
  const uint32_t tbl = cta_table_bytes(n_ctx, nn, W);
  auto wbase = [&](uint32_t w) { return smem + tbl + static_cast<size_t>(w) * L.bytes; };
  uint8_t* wb = wbase(warp);
  u64* rows = reinterpret_cast<u64*>(wb + L.off_rows);
  u64* rtot = reinterpret_cast<u64*>(wb + L.off_rtot);
  u64* pref = reinterpret_cast<u64*>(wb + L.off_pref);
  u64* inrow = reinterpret_cast<u64*>(wb + L.off_inrow);
  uint32_t* bwin = reinterpret_cast<uint32_t*>(wb + L.off_bwin);
  u64* wsx = reinterpret_cast<u64*>(wb + L.off_wsx);
  u64* wsqlo = reinterpret_cast<u64*>(wb + L.off_wsqlo);
  u64* wsqhi = reinterpret_cast<u64*>(wb + L.off_wsqhi);
  warp_tables T;
  T.wcnt = reinterpret_cast<uint32_t*>(wb + L.off_wcnt);
  T.wslo = reinterpret_cast<uint32_t*>(wb + L.off_wslo);
  T.wshi = reinterpret_cast<uint32_t*>(wb + L.off_wshi);
  T.wmin = reinterpret_cast<uint32_t*>(wb + L.off_wmin);
  T.wmax = reinterpret_cast<uint32_t*>(wb + L.off_wmax);
  T.wnbig = reinterpret_cast<uint32_t*>(wb + L.off_wnbig);
  T.wminb = reinterpret_cast<u64*>(wb + L.off_wminb);
  T.wmaxb = reinterpret_cast<u64*>(wb + L.off_wmaxb);
  T.carry = reinterpret_cast<u64*>(wb + L.off_carry);

  for (uint32_t i = threadIdx.x; i < n_ctx; i += blockDim.x) {
    s_sub_pre[i] = CUBE ? p.sub_pre[i] : -1;
    s_cct_pre[i] = WIN ? p.cct_pre[i] : 0;
    s_cct_size[i] = WIN ? p.cct_size[i] : 0;
  }
  if (CUBE)
    for (uint32_t i = threadIdx.x; i < nn; i += blockDim.x) s_node[i] = p.node_tab[i];
  if (CUBE) {
    for (uint32_t j = lane; j < (R2 + 1) * nn; j += 32) rows[j] = 0;
    for (uint32_t j = lane; j <= R2; j += 32) rtot[j] = 0;
    for (uint32_t j = lane; j < nn; j += 32) wsx[j] = wsqlo[j] = wsqhi[j] = 0;
  }
  if (WIN) {
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      T.wcnt[c] = T.wslo[c] = T.wshi[c] = T.wmax[c] = T.wnbig[c] = 0u;
      T.wmin[c] = 0xFFFFFFFFu;
      T.wminb[c] = ~0ull;
      T.wmaxb[c] = 0ull;
    }
  }
  if (lane == 0) T.carry[0] = T.carry[1] = T.carry[2] = 0;

  const uint32_t t = blockIdx.x * W + warp;
  const bool active = t < p.tr.n;
  const u64 b = active ? p.tr.off[t] : 0, e = active ? p.tr.off[t + 1] : 0;
  const u64 n_t = e - b;
  const u64 tend = active ? p.tr.t_end[t] : 0;
  const uint32_t iters = (CUBE && active) ? p.iter_count[t] : 0;
  const uint32_t nbd = (CUBE && active) ? p.n_bounds[t] : 0;
  const bool kept = iters > 0;
  const uint32_t tp = kept ? p.tpos[t] : 0;
  const u64 bo = kept ? p.block_off[t] : 0;
  const uint32_t* bt = p.bidx + ((CUBE && active) ? p.cap_off[t] : 0);
  const u64 t0 = p.t0, t1w = (p.clamp_tend && tend < p.t1) ? tend : p.t1;
  if (lane == 0) s_kept[warp] = kept ? 1u : 0u;
  u64 pos = 0;  // next unprocessed event, relative to b
  __syncthreads();

  for (uint32_t c = 0;; ++c) {
    const uint32_t kb = c * G;
    u64 E1 = n_t, E2 = n_t;
    if (CUBE) {
      if (lane <= static_cast<int>(R2)) {
        const u64 k = static_cast<u64>(kb) + lane;
        bwin[lane] = k < nbd ? __ldg(bt + k) : static_cast<uint32_t>(n_t);
      }
      __syncwarp();
      E1 = bwin[G];
      E2 = bwin[R2];
    }

    // ---- phase 1: consume events [pos, E1), possibly running ahead to E2 ----
    while (pos < E1) {
      const u64 s_abs = (b + pos) & ~3ull;
      const int64_t base = static_cast<int64_t>(s_abs) - static_cast<int64_t>(b);  // >= -3
      const u64 lim = min(static_cast<u64>(base + STEP_M), E2);
      const int lo = static_cast<int>(static_cast<int64_t>(pos) - base);
      const int hi = static_cast<int>(static_cast<int64_t>(lim) - base);
      const int64_t lr = static_cast<int64_t>(n_t) - 1 - base;
      const int last_li = lr < STEP_M ? static_cast<int>(lr) : -1;
      const int lb = lane * RM;
      const u64 r0 = s_abs + static_cast<u64>(lb);
      if (lane == 0 && s_abs + 3 * STEP_M <= e) {
        prefetch_l2(p.tr.ts + s_abs + 2 * STEP_M, 8 * STEP_M);
        prefetch_l2(p.tr.ctx + s_abs + 2 * STEP_M, 4 * STEP_M);
      }
      u64 tv[RM + 1];
      uint32_t cv[RM];
      {
        const ulonglong2* tsrc = reinterpret_cast<const ulonglong2*>(p.tr.ts + r0);
#pragma unroll
        for (int q = 0; q < RM / 2; ++q) {
          const ulonglong2 v = __ldg(tsrc + q);
          tv[2 * q] = v.x;
          tv[2 * q + 1] = v.y;
        }
        const uint4* csrc = reinterpret_cast<const uint4*>(p.tr.ctx + r0);
#pragma unroll
        for (int q = 0; q < RM / 4; ++q) {
          const uint4 v = __ldg(csrc + q);
          cv[4 * q] = v.x;
          cv[4 * q + 1] = v.y;
          cv[4 * q + 2] = v.z;
          cv[4 * q + 3] = v.w;
        }
      }
      u64 nf = __shfl_down_sync(FULL, tv[0], 1);
      if (lane == 31) nf = ldg64(p.tr.ts + s_abs + STEP_M);
      tv[RM] = nf;

      // window mode of this block step (warp-uniform)
      int wm = WIN_NONE;
      if (WIN) {
        u64 f = tv[0];
        if (lo >= 1) f = tv[1];
        if (lo >= 2) f = tv[2];
        if (lo >= 3) f = tv[3];
        const u64 first = __shfl_sync(FULL, f, 0);                // first valid event
        const u64 after = __shfl_sync(FULL, tv[RM], (hi - 1) >> 3);  // ts after the last valid one
        const bool has_end = last_li >= 0 && last_li < hi;
        // "after" bounds the successor timestamp of every valid event
        if ((first >= t1w && first >= t0) || (!has_end && after < t0))
          wm = WIN_NONE;
        else if (!has_end && first >= t0 && after < t1w)
          wm = WIN_FULL;
        else
          wm = WIN_PART;
      }

      run_state st;
      st.racc = 0;
      st.k = -1;
      st.cnt = 0;
      st.nxt = INT_MAX;
      st.cube_ok = false;
      st.rb = nullptr;
      st.rt = nullptr;
      if (CUBE) {
        // iteration of this lane's first event: boundaries of the window at or before it
        uint32_t cnt = 0;
        for (uint32_t j = 0; j <= R2; ++j) cnt += lb >= local_of(bwin[j], base) ? 1u : 0u;
        st.cnt = cnt;
        st.k = static_cast<int>(kb) - 1 + static_cast<int>(cnt);
        st.nxt = cnt <= R2 ? local_of(bwin[cnt], base) : INT_MAX;
        const uint32_t slot = st.k < 0 ? R2 : (static_cast<uint32_t>(st.k) & (R2 - 1));
        st.cube_ok = st.k < static_cast<int>(iters);
        st.rb = reinterpret_cast<uint32_t*>(rows + slot * nn);
        st.rt = rtot + slot;
      }
      if (wm == WIN_FULL)
        run_events<WIN, CUBE, WIN_FULL>(tv, cv, lb, lo, hi, last_li, tend, t0, t1w, s_sub_pre, bwin,
                                        base, R2, iters, rows, rtot, nn, root_only, st, T);
      else if (wm == WIN_PART)
        run_events<WIN, CUBE, WIN_PART>(tv, cv, lb, lo, hi, last_li, tend, t0, t1w, s_sub_pre, bwin,
                                        base, R2, iters, rows, rtot, nn, root_only, st, T);
      else
        run_events<WIN, CUBE, WIN_NONE>(tv, cv, lb, lo, hi, last_li, tend, t0, t1w, s_sub_pre, bwin,
                                        base, R2, iters, rows, rtot, nn, root_only, st, T);
      if (CUBE && root_only && st.racc)
        sadd64(reinterpret_cast<uint32_t*>(st.rt), reinterpret_cast<uint32_t*>(st.rt) + 1, st.racc);
      pos = lim;
    }
    __syncwarp();

    // ---- phase 2a: inclusive roll-up, cube stores, within-rank sums ----
    const uint32_t k_lo = kb;
    const uint32_t k_hi = min(kb + G, iters);
    const uint32_t n_iter_rows = k_hi > k_lo ? k_hi - k_lo : 0;
    if (CUBE && kept) {
      const uint32_t s0 = k_lo & (R2 - 1);  // the chunk's rows are slots [s0, s0 + G)
      const bool stats = p.do_stats && k_lo < p.K;
      const uint32_t kcap = stats ? min(n_iter_rows, p.K - k_lo) : 0;
      const u64 ob = bo + static_cast<u64>(k_lo) * nn;
      const uint32_t n_rows = n_iter_rows + (c == 0 ? 1u : 0u);  // + the gap row
      for (uint32_t r = 0; r < n_rows; ++r) {
        const bool gap = r >= n_iter_rows;
        const uint32_t slot = gap ? R2 : s0 + r;
        u64* row = rows + slot * nn;
        if (!root_only) warp_prefix(row, pref, nn, lane);  // generic roll-up over preorder ranges
        const u64 tot = rtot[slot];
        for (uint32_t n = lane; n < nn; n += 32) {
          const int4 nd = s_node[n];
          const u64 ex = row[nd.x];
          const u64 in = !nd.z ? ex : (root_only ? tot : pref[nd.x + nd.y] - pref[nd.x]);
          if (gap) {
            p.gap_excl[static_cast<size_t>(tp) * nn + n] = ex;
            p.gap_incl[static_cast<size_t>(tp) * nn + n] = in;
          } else {
            if (p.store_cube) {
              p.cube_excl[ob + static_cast<u64>(r) * nn + n] = ex;
              p.cube_incl[ob + static_cast<u64>(r) * nn + n] = in;
            }
          }
          if (!gap && r < kcap) {
            // within-rank sums (iteration_cv_report) and the value for the
            // CTA's cross-rank fold, kept (node-indexed) until phase 2b reads it
            inrow[n] = in;
            wsx[n] += in;
            const u128 sq = static_cast<u128>(in) * in;
            const u64 lo2 = wsqlo[n] + static_cast<u64>(sq);
            wsqhi[n] += static_cast<u64>(sq >> 64) + (lo2 < wsqlo[n] ? 1ull : 0ull);
            wsqlo[n] = lo2;
          }
        }
        __syncwarp();
        // slots [0, kcap) keep their inclusive values for phase 2b (indexed by
        // node); everything else is released for chunk c + 2 right away
        if (!gap && r < kcap) {
          for (uint32_t n = lane; n < nn; n += 32) row[n] = inrow[n];
        } else {
          for (uint32_t n = lane; n < nn; n += 32) row[n] = 0;
        }
        __syncwarp();
        if (lane == 0) rtot[slot] = 0;
      }
    }

    // ---- phase 2b: cross-rank statistics over k < K (diagnostics.cpp:83-158) ----
    if (CUBE && p.do_stats) {
      __syncthreads();
      if (kb < p.K) {
        const uint32_t kcap = min(G, p.K - kb);
        const uint32_t s0 = kb & (R2 - 1);
        for (uint32_t cell = threadIdx.x; cell < kcap * nn; cell += blockDim.x) {
          const uint32_t off = (s0 * nn + cell) * 8u + L.off_rows;  // rows are node-indexed now
          u64 sum = 0, mx = 0, sqlo = 0, sqhi = 0;
          bool any = false;
          for (uint32_t w = 0; w < W; ++w) {
            if (!s_kept[w]) continue;
            u64* vp = reinterpret_cast<u64*>(wbase(w) + off);
            const u64 v = *vp;
            *vp = 0;
            sum += v;
            mx = max(mx, v);
            const u128 sq = static_cast<u128>(v) * v;
            const u64 l2 = sqlo + static_cast<u64>(sq);
            sqhi += static_cast<u64>(sq >> 64) + (l2 < sqlo ? 1ull : 0ull);
            sqlo = l2;
            any = true;
          }
          if (any) {
            const uint32_t s = cell / nn, n = cell - s * nn;
            const size_t ci = static_cast<size_t>(kb + s) * nn + n;
            const size_t plane = static_cast<size_t>(p.K) * nn;
            const u64 mask43 = (1ull << 43) - 1;
            atomicAdd(p.x_sum + ci, sum);
            atomicMax(p.x_max + ci, mx);
            atomicAdd(p.x_sq + ci, sqlo & mask43);
            atomicAdd(p.x_sq + plane + ci, ((sqlo >> 43) | (sqhi << 21)) & mask43);
            const u64 top = sqhi >> 22;
            if (top) atomicAdd(p.x_sq + 2 * plane + ci, top);
          }
        }
      }
    }
    const bool done = pos >= n_t && static_cast<u64>(kb) + G >= iters;
    if (CUBE && p.do_stats) {
      if (__syncthreads_and(done ? 1 : 0)) break;
    } else if (done) {
      break;
    }
  }

  if (!active) return;
  if (WIN) {
    // exclusive ns incl. the carry-in segment, in CCT preorder, then the
    // inclusive roll-up: every subtree is a contiguous preorder range
    u64* tmp = reinterpret_cast<u64*>(wb + L.off_scan);
    u64* scan = tmp + (n_ctx + 1);
    const bool c_has = (T.carry[2] >> 32) != 0;
    const uint32_t c_ctx = static_cast<uint32_t>(T.carry[2]);
    const u64 c_d = T.carry[1];
    __syncwarp();
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      const u64 sum = (static_cast<u64>(T.wshi[c]) << 32) | T.wslo[c];
      tmp[s_cct_pre[c]] = sum + ((c_has && c == c_ctx) ? c_d : 0ull);
    }
    __syncwarp();
    warp_prefix(tmp, scan, n_ctx, lane);
    const size_t base = static_cast<size_t>(t) * n_ctx;
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      const int pr = s_cct_pre[c], sz = s_cct_size[c];
      const u64 cnt = T.wcnt[c], nbig = T.wnbig[c];
      const u64 sum = (static_cast<u64>(T.wshi[c]) << 32) | T.wslo[c];
      p.w_cnt[base + c] = cnt;
      p.w_sum[base + c] = sum;
      p.w_min[base + c] = cnt == 0 ? 0ull : (cnt > nbig ? static_cast<u64>(T.wmin[c]) : T.wminb[c]);
      p.w_max[base + c] = nbig ? T.wmaxb[c] : static_cast<u64>(T.wmax[c]);
      p.w_mean[base + c] = cnt ? static_cast<double>(sum) / static_cast<double>(cnt) : 0.0;
      p.w_excl[base + c] = scan[pr + 1] - scan[pr];
      p.w_incl[base + c] = scan[pr + sz] - scan[pr];
    }
    if (lane == 0) {
      p.c_has[t] = c_has ? 1 : 0;
      p.c_ts[t] = c_has ? T.carry[0] : 0;
      p.c_ctx[t] = c_has ? c_ctx : 0;
    }
  }
  if (CUBE && p.do_stats && kept && p.K > 0) {
    for (uint32_t n = lane; n < nn; n += 32) {
      const u64 sx = wsx[n];
      const u128 sq = (static_cast<u128>(wsqhi[n]) << 64) | wsqlo[n];
      const u128 num = static_cast<u128>(p.K) * sq - static_cast<u128>(sx) * sx;
      const bool ok = sx > 0;
      p.within_cv[static_cast<size_t>(tp) * nn + n] =
          ok ? 100.0 * sqrt(u128_to_double(num)) / static_cast<double>(sx) : 0.0;
      p.within_ok[static_cast<size_t>(tp) * nn + n] = ok ? 1 : 0;
    }
  }
}

template <bool WIN, bool CUBE>
void launch_variant(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  static int configured_bytes = 0;
  if (static_cast<int>(smem_bytes) > configured_bytes) {
    PSG_CUDA(cudaFuncSetAttribute(k_trace_query<WIN, CUBE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_bytes)));
    configured_bytes = static_cast<int>(smem_bytes);
  }
  const unsigned blocks = (p.tr.n + p.warps - 1) / p.warps;
  k_trace_query<WIN, CUBE><<<blocks, p.warps * 32, smem_bytes, s>>>(p);
}

}  // namespace

void launch_trace_query(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  if (p.tr.n == 0) return;
  if (p.do_window && p.do_cube)
    launch_variant<true, true>(p, smem_bytes, s);
  else if (p.do_window)
    launch_variant<true, false>(p, smem_bytes, s);
  else
    launch_variant<false, true>(p, smem_bytes, s);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
