// Hand-written sm_100a kernels of the perfslice trace query path.
//
//   K1 k_aos_to_soa      trace.db 12-byte AoS -> SoA ts/ctx      (store.cpp:573-580, 678-692)
//   K1v k_validate       format invariants of the loaded events   (store.cpp:743-761)
//   K0 k_gen_*           device replay of synthgen's iterative scenario (synthgen.cpp:146-246)
//   K4a k_iter_count     boundary detection -> iterations per trace (itermodel.cpp:111-143)
//   K3+K4+K5+K6a k_trace_query  ONE pass over every event: window filter + per-(trace,ctx)
//                        count/sum/min/max/mean + time integration (ingest.cpp:178-208,
//                        frame.cpp:290-408, itermodel.cpp:145-183), iteration boundaries and
//                        the trace x iteration x node cube (itermodel.cpp:242-360), and the
//                        cross-rank / within-rank sufficient statistics (diagnostics.cpp:83-158)
//   K6b k_within_reduce / k_stats_finalize   savings + CV rows
//   K2 k_window_bounds / k_window_copy       ingest_traces rows + carry-ins
//   K7 k_site_acc / k_pick_worst / k_node_acc / k_node_stats   balance ratio, node means,
//                        z-score, top-k (workflows.cpp:42-62, 442-539; diagnostics.cpp:10-19, 378-403)
//   K8 k_topology        rack/chassis localisation (topology.cpp:54-92)
//
// Everything on the event stream is integer arithmetic in int64 nanoseconds,
// which is exact and order-free, so the GPU reproduces the reference's integer
// outputs bit for bit regardless of thread order.  Floating-point outputs are
// derived from exact integer sufficient statistics at the end.
#include <cub/cub.cuh>

#include <atomic>
#include <climits>
#include <cstdint>

#include "psg_internal.h"

namespace psg {

namespace {
std::atomic<unsigned long long> g_launches{0};
}  // namespace

void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
unsigned long long kernel_launches() { return g_launches.load(std::memory_order_relaxed); }

namespace {

constexpr unsigned FULL = 0xffffffffu;
typedef unsigned long long u64;
typedef unsigned __int128 u128;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ unsigned lanemask_le() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}
__device__ __forceinline__ u64 ldg_u64(const uint64_t* p) {
  return static_cast<u64>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}
__device__ __forceinline__ double u128_to_double(u128 v) {
  return static_cast<double>(static_cast<u64>(v >> 64)) * 18446744073709551616.0 +
         static_cast<double>(static_cast<u64>(v));
}

// ---------------------------------------------------------------------------
// Iteration-boundary scan state (itermodel.cpp:111-143).  `inside` is the
// containment of the previous event; a boundary is a candidate (entering the
// anchor subtree) whose timestamp is strictly greater than the last accepted
// boundary, which for sorted timestamps is the same as "no earlier candidate
// at the same timestamp".
struct bstate {
  int k;         // iteration index of the last processed event (-1: gap)
  int inside;    // containment of the last processed event
  int has_lct;   // a candidate has been seen
  u64 lct;       // timestamp of the last candidate
};

__device__ __forceinline__ int boundary_step(const bstate& st, bool valid, bool in_sub, u64 ts,
                                             int lane, unsigned& cmask, unsigned& bmask) {
  int prev_in = __shfl_up_sync(FULL, (int)in_sub, 1);
  if (lane == 0) prev_in = st.inside;
  bool cand = valid && in_sub && !prev_in;
  cmask = __ballot_sync(FULL, cand);
  unsigned lower = cmask & lanemask_lt();
  int src = lower ? 31 - __clz(lower) : lane;
  u64 pts = __shfl_sync(FULL, ts, src);
  bool have = lower != 0 || st.has_lct;
  if (lower == 0) pts = st.lct;
  bool bnd = cand && (!have || pts < ts);
  bmask = __ballot_sync(FULL, bnd);
  return st.k + __popc(bmask & lanemask_le());
}

__device__ __forceinline__ void boundary_advance(bstate& st, int nproc, bool in_sub, unsigned cmask,
                                                 u64 ts, int ki) {
  if (nproc <= 0) return;
  int last = nproc - 1;
  st.inside = __shfl_sync(FULL, (int)in_sub, last);
  st.k = __shfl_sync(FULL, ki, last);
  unsigned pc = cmask & (nproc >= 32 ? FULL : ((1u << nproc) - 1u));
  if (pc) {
    st.lct = __shfl_sync(FULL, ts, 31 - __clz(pc));
    st.has_lct = 1;
  }
}

// Warp-private non-atomic accumulation keyed by a small integer.  The fast
// path is conflict-free (one lane per key, detected with a byte tag table);
// duplicates fall back to __match_any_sync plus a shuffle fold so that one
// leader lane writes each key.  All lanes of the warp must call it.
template <int NV>
__device__ __forceinline__ void warp_keyed_update(uint8_t* tag, unsigned key, bool flag, int lane,
                                                 u64 v, u64* sum, u64* cnt, u64* mn, u64* mx) {
  if (!__any_sync(FULL, flag)) return;
  if (flag) tag[key] = static_cast<uint8_t>(lane);
  __syncwarp();
  bool conf = flag && tag[key] != static_cast<uint8_t>(lane);
  if (!__any_sync(FULL, conf)) {
    if (flag) {
      sum[key] += v;
      if (NV > 1) {
        cnt[key] += 1;
        mn[key] = min(mn[key], v);
        mx[key] = max(mx[key], v);
      }
    }
  } else {
    unsigned k2 = flag ? key : (0x80000000u | static_cast<unsigned>(lane));
    unsigned peers = __match_any_sync(FULL, k2);
    unsigned others = peers & ~(1u << lane);
    unsigned rounds = __reduce_max_sync(FULL, static_cast<unsigned>(__popc(others)));
    u64 s = v, lo = v, hi = v, c = 1;
    for (unsigned r = 0; r < rounds; ++r) {
      int src = others ? __ffs(others) - 1 : lane;
      u64 x = __shfl_sync(FULL, v, src);
      if (others) {
        s += x;
        lo = min(lo, x);
        hi = max(hi, x);
        c += 1;
        others &= others - 1;
      }
    }
    if (flag && lane == __ffs(peers) - 1) {
      sum[key] += s;
      if (NV > 1) {
        cnt[key] += c;
        mn[key] = min(mn[key], lo);
        mx[key] = max(mx[key], hi);
      }
    }
  }
  __syncwarp();
}

// Warp inclusive scan of u64 over `n` values at src (any order), written as an
// exclusive-prefix array dst[0..n] (dst[0] = 0).
__device__ __forceinline__ void warp_prefix(const u64* src, u64* dst, uint32_t n, int lane) {
  u64 carry = 0;
  for (uint32_t b = 0; b < n; b += 32) {
    uint32_t j = b + lane;
    u64 v = j < n ? src[j] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u64 y = __shfl_up_sync(FULL, v, d);
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
// K1: AoS -> SoA.  Events are 12 bytes; 4 events = 48 bytes = three 128-bit
// loads, written as two 128-bit ts stores and one 128-bit ctx store.
__global__ void k_aos_to_soa(const uint4* __restrict__ body, uint64_t n_events,
                             uint64_t* __restrict__ ts, uint32_t* __restrict__ ctx) {
  uint64_t groups = n_events / 4;
  uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
       g += stride) {
    uint4 a = __ldg(body + 3 * g), b = __ldg(body + 3 * g + 1), c = __ldg(body + 3 * g + 2);
    // words: a.x a.y | a.z | a.w b.x | b.y | b.z b.w | c.x | c.y c.z | c.w
    ulonglong2 t01, t23;
    t01.x = (static_cast<u64>(a.y) << 32) | a.x;
    t01.y = (static_cast<u64>(b.x) << 32) | a.w;
    t23.x = (static_cast<u64>(b.w) << 32) | b.z;
    t23.y = (static_cast<u64>(c.z) << 32) | c.y;
    uint4 cx = make_uint4(a.z, b.y, c.x, c.w);
    reinterpret_cast<ulonglong2*>(ts)[2 * g] = t01;
    reinterpret_cast<ulonglong2*>(ts)[2 * g + 1] = t23;
    reinterpret_cast<uint4*>(ctx)[g] = cx;
  }
  // tail (< 4 events)
  if (blockIdx.x == 0 && threadIdx.x < n_events - groups * 4) {
    uint64_t e = groups * 4 + threadIdx.x;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(body) + 3 * e;
    ts[e] = (static_cast<u64>(w[1]) << 32) | w[0];
    ctx[e] = w[2];
  }
}

void launch_aos_to_soa(const uint8_t* body, uint64_t n_events, uint64_t* ts, uint32_t* ctx,
                       cudaStream_t s) {
  if (n_events == 0) return;
  uint64_t groups = (n_events + 3) / 4;
  unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((groups + 255) / 256, 148ull * 16));
  k_aos_to_soa<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(body), n_events, ts, ctx);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// K1 inverse (trace.db body export): SoA -> packed 12-byte AoS.
__global__ void k_soa_to_aos(const uint64_t* __restrict__ ts, const uint32_t* __restrict__ ctx,
                             uint64_t n_events, uint4* __restrict__ body) {
  uint64_t groups = n_events / 4;
  uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
       g += stride) {
    ulonglong2 t01 = reinterpret_cast<const ulonglong2*>(ts)[2 * g];
    ulonglong2 t23 = reinterpret_cast<const ulonglong2*>(ts)[2 * g + 1];
    uint4 cx = reinterpret_cast<const uint4*>(ctx)[g];
    body[3 * g] = make_uint4(static_cast<uint32_t>(t01.x), static_cast<uint32_t>(t01.x >> 32), cx.x,
                             static_cast<uint32_t>(t01.y));
    body[3 * g + 1] = make_uint4(static_cast<uint32_t>(t01.y >> 32), cx.y,
                                 static_cast<uint32_t>(t23.x), static_cast<uint32_t>(t23.x >> 32));
    body[3 * g + 2] = make_uint4(cx.z, static_cast<uint32_t>(t23.y),
                                 static_cast<uint32_t>(t23.y >> 32), cx.w);
  }
  if (blockIdx.x == 0 && threadIdx.x < n_events - groups * 4) {
    uint64_t e = groups * 4 + threadIdx.x;
    uint32_t* w = reinterpret_cast<uint32_t*>(body) + 3 * e;
    w[0] = static_cast<uint32_t>(ts[e]);
    w[1] = static_cast<uint32_t>(ts[e] >> 32);
    w[2] = ctx[e];
  }
}

void launch_soa_to_aos(const uint64_t* ts, const uint32_t* ctx, uint64_t n_events, uint8_t* body,
                       cudaStream_t s) {
  if (n_events == 0) return;
  uint64_t groups = (n_events + 3) / 4;
  unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((groups + 255) / 256, 148ull * 16));
  k_soa_to_aos<<<blocks, 256, 0, s>>>(ts, ctx, n_events, reinterpret_cast<uint4*>(body));
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// K1v: one warp per trace checks the invariants validate_database reports.
__global__ void k_validate(trace_view tr, uint32_t n_ctx, unsigned long long* bad,
                           unsigned long long* first_bad) {
  uint32_t t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (t >= tr.n) return;
  uint64_t b = tr.off[t], e = tr.off[t + 1];
  bool ok = true;
  for (uint64_t i = b + lane; i < e; i += 32) {
    u64 x = ldg_u64(tr.ts + i);
    if (__ldg(tr.ctx + i) >= n_ctx) ok = false;
    if (i + 1 < e && ldg_u64(tr.ts + i + 1) < x) ok = false;
    if (i + 1 == e && tr.t_end[t] < x) ok = false;
  }
  if (!__all_sync(FULL, ok) && lane == 0) {
    atomicAdd(bad, 1ull);
    atomicMin(first_bad, static_cast<unsigned long long>(t));
  }
}

void launch_validate(const trace_view& tr, uint32_t n_ctx, unsigned long long* bad,
                     unsigned long long* first_bad, cudaStream_t s) {
  if (tr.n == 0) return;
  k_validate<<<(tr.n + 7) / 8, 256, 0, s>>>(tr, n_ctx, bad, first_bad);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K0: device replay of synthgen::generate_iterative_scenario.  The reference
// draws one xorshift64* value per (rank, iteration, kernel) from a single
// stream in rank-major order (synthgen.cpp:184-209).  xorshift64*'s state
// transition is linear over GF(2)^64, so the state before draw D is
// M^D * (seed | 1); jump_mats holds M^(2^b) as 64 column vectors each.
namespace {

__device__ __forceinline__ u64 gf2_apply(const uint64_t* __restrict__ m, u64 x) {
  u64 r = 0;
#pragma unroll 8
  for (int i = 0; i < 64; ++i)
    if ((x >> i) & 1ull) r ^= ldg_u64(m + i);
  return r;
}

__device__ u64 xs_jump(const uint64_t* __restrict__ mats, u64 state, u64 n) {
  for (int b = 0; n; ++b, n >>= 1)
    if (n & 1ull) state = gf2_apply(mats + 64 * b, state);
  return state;
}

struct xs64 {
  u64 s;
  __device__ __forceinline__ u64 next() {
    u64 x = s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    s = x;
    return x * 0x2545F4914F6CDD1DULL;
  }
  // next_signed_unit (util.hpp:35-38); every op is exact or explicitly rounded
  // (no FMA contraction) to match the host build bit for bit.
  __device__ __forceinline__ double signed_unit() {
    double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
    return __dsub_rn(__dmul_rn(2.0, u), 1.0);
  }
};

// to_ns(mean * factor * (1 + jitter * u)) (synthgen.cpp:22-24, 208-211)
__device__ __forceinline__ u64 kernel_ns(double mean, double factor, double jitter, double u) {
  double s = __dmul_rn(__dmul_rn(mean, factor), __dadd_rn(1.0, __dmul_rn(jitter, u)));
  return static_cast<u64>(llround(__dmul_rn(s, 1e9)));
}

constexpr uint32_t kGenItersPerThread = 16;

struct gen_args {
  const uint64_t* mats;
  u64 seed;
  uint32_t n_ranks, n_it, n_k;
  const double *mean, *jitter, *spread;
  u64 spread_kstride;
  u64 copy_ns;
  uint32_t rank_lo, n_local;
  u64 ept;  // events per trace
  u64* chunk;
  uint64_t* ts;
  uint32_t* ctx;
  uint64_t* t_end;
};

__device__ __forceinline__ double factor_of(const gen_args& a, uint32_t k, uint32_t r) {
  if (!a.spread) return 1.0;
  return __ldg(a.spread + static_cast<u64>(k) * a.spread_kstride + r);
}

}  // namespace

__global__ void k_gen_chunks(gen_args a) {
  uint32_t chunks = (a.n_it + kGenItersPerThread - 1) / kGenItersPerThread;
  u64 gid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  if (gid >= static_cast<u64>(a.n_local) * chunks) return;
  uint32_t rl = static_cast<uint32_t>(gid / chunks), j = static_cast<uint32_t>(gid % chunks);
  uint32_t r = a.rank_lo + rl;
  uint32_t it0 = j * kGenItersPerThread, it1 = min(a.n_it, it0 + kGenItersPerThread);
  xs64 g{xs_jump(a.mats, a.seed | 1ull,
                 (static_cast<u64>(r) * a.n_it + it0) * static_cast<u64>(a.n_k))};
  u64 total = 0;
  for (uint32_t it = it0; it < it1; ++it) {
    for (uint32_t k = 0; k < a.n_k; ++k)
      total += kernel_ns(__ldg(a.mean + k), factor_of(a, k, r), __ldg(a.jitter + k), g.signed_unit());
    total += a.copy_ns;
  }
  a.chunk[gid] = total;
}

__global__ void k_gen_write(gen_args a) {
  uint32_t chunks = (a.n_it + kGenItersPerThread - 1) / kGenItersPerThread;
  u64 gid = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  if (gid >= static_cast<u64>(a.n_local) * chunks) return;
  uint32_t rl = static_cast<uint32_t>(gid / chunks), j = static_cast<uint32_t>(gid % chunks);
  uint32_t r = a.rank_lo + rl;
  u64 t = 0;
  for (uint32_t jj = 0; jj < j; ++jj) t += a.chunk[static_cast<u64>(rl) * chunks + jj];
  uint32_t it0 = j * kGenItersPerThread, it1 = min(a.n_it, it0 + kGenItersPerThread);
  xs64 g{xs_jump(a.mats, a.seed | 1ull,
                 (static_cast<u64>(r) * a.n_it + it0) * static_cast<u64>(a.n_k))};
  const bool has_copy = a.copy_ns > 0;
  const uint32_t epi = a.n_k + 2 + (has_copy ? 1 : 0);
  u64 e = static_cast<u64>(rl) * a.ept + static_cast<u64>(it0) * epi;
  for (uint32_t it = it0; it < it1; ++it) {
    a.ts[e] = t;
    a.ctx[e++] = 1;  // anchor
    for (uint32_t k = 0; k < a.n_k; ++k) {
      u64 d = kernel_ns(__ldg(a.mean + k), factor_of(a, k, r), __ldg(a.jitter + k), g.signed_unit());
      a.ts[e] = t;
      a.ctx[e++] = 2 + k;
      t += d;
    }
    if (has_copy) {
      a.ts[e] = t;
      a.ctx[e++] = 2 + a.n_k;
      t += a.copy_ns;
    }
    a.ts[e] = t;
    a.ctx[e++] = 0;  // leave the anchor subtree
  }
  if (j == chunks - 1) a.t_end[rl] = t;
}

void launch_gen_iterative(const uint64_t* jump_mats, uint64_t seed, uint32_t n_ranks,
                          uint32_t n_it, uint32_t n_k, const double* mean, const double* jitter,
                          const double* spread, uint64_t spread_kstride, uint64_t copy_ns,
                          uint32_t rank_lo, uint32_t n_local, uint64_t events_per_trace,
                          uint64_t* chunk_scratch, uint64_t* ts, uint32_t* ctx, uint64_t* t_end,
                          cudaStream_t s) {
  gen_args a{jump_mats, seed, n_ranks, n_it, n_k, mean, jitter, spread, spread_kstride, copy_ns,
             rank_lo, n_local, events_per_trace, reinterpret_cast<u64*>(chunk_scratch), ts, ctx,
             t_end};
  uint32_t chunks = (n_it + kGenItersPerThread - 1) / kGenItersPerThread;
  u64 threads = static_cast<u64>(n_local) * chunks;
  if (threads == 0) return;
  unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
  k_gen_chunks<<<blocks, 128, 0, s>>>(a);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  k_gen_write<<<blocks, 128, 0, s>>>(a);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K4a: iterations per trace.  One warp per trace streams ctx only; ts is read
// just for candidate lanes (one per iteration), so the pass costs ~4 B/event.
__global__ void __launch_bounds__(256) k_iter_count(trace_view tr, const int32_t* __restrict__ sub_pre,
                                                    uint32_t* __restrict__ iter_count) {
  uint32_t t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (t >= tr.n) return;
  const u64 b = tr.off[t], e = tr.off[t + 1];
  bstate st{-1, 0, 0, 0};
  int nb = 0;
  u64 b_last = 0;
  for (u64 base = b; base < e; base += 128) {
    uint32_t cx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u64 i = base + j * 32 + lane;
      cx[j] = i < e ? __ldg(tr.ctx + i) : 0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u64 i0 = base + j * 32;
      if (i0 >= e) break;
      u64 i = i0 + lane;
      bool valid = i < e;
      bool in_sub = valid && __ldg(sub_pre + cx[j]) >= 0;
      int prev_in = __shfl_up_sync(FULL, (int)in_sub, 1);
      if (lane == 0) prev_in = st.inside;
      bool cand = valid && in_sub && !prev_in;
      u64 ts = cand ? ldg_u64(tr.ts + i) : 0;
      unsigned cmask, bmask;
      int ki = boundary_step(st, valid, in_sub, ts, lane, cmask, bmask);
      if (bmask) {
        int lb = 31 - __clz(bmask);
        b_last = __shfl_sync(FULL, ts, lb);
        nb += __popc(bmask);
      }
      int nvalid = static_cast<int>((e - i0) < 32ull ? (e - i0) : 32ull);
      boundary_advance(st, nvalid, in_sub, cmask, ts, ki);
    }
  }
  if (lane == 0) {
    uint32_t it = static_cast<uint32_t>(nb);
    if (nb > 0 && b_last >= tr.t_end[t]) it -= 1;  // empty last interval dropped
    iter_count[t] = it;
  }
}

void launch_iter_count(const trace_view& tr, const int32_t* sub_pre, uint32_t n_ctx,
                       uint32_t* iter_count, cudaStream_t s) {
  (void)n_ctx;
  if (tr.n == 0) return;
  k_iter_count<<<(tr.n + 7) / 8, 256, 0, s>>>(tr, sub_pre, iter_count);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// Cube layout: kept flags, cell counts, then exclusive scans (CUB).
__global__ void k_layout_prep(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint64_t* kept,
                              uint64_t* cells, unsigned long long* summary) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint32_t it = iter_count[t];
  kept[t] = it > 0 ? 1 : 0;
  cells[t] = static_cast<uint64_t>(it) * nn;
  if (it > 0) {
    atomicAdd(summary + 0, 1ull);
    atomicMin(summary + 1, static_cast<unsigned long long>(it));
    atomicAdd(summary + 2, static_cast<unsigned long long>(it) * nn);
  }
}

__global__ void k_u64_to_u32(const uint64_t* in, uint32_t* out, uint32_t n) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = static_cast<uint32_t>(in[t]);
}

size_t exclusive_scan_u64_scratch(uint32_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint64_t*>(nullptr),
                                static_cast<uint64_t*>(nullptr), static_cast<int>(n));
  return bytes;
}

void launch_exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint32_t n, void* scratch,
                               size_t scratch_bytes, cudaStream_t s) {
  if (n == 0) return;
  PSG_CUDA(cub::DeviceScan::ExclusiveSum(scratch, scratch_bytes, in, out, static_cast<int>(n), s));
}

size_t cube_layout_scratch_bytes(uint32_t n) {
  // kept (n u64) + cells (n u64) + tpos64 (n u64) + scan temp
  return 3ull * (n + 1) * sizeof(uint64_t) + exclusive_scan_u64_scratch(n) + 256;
}

void launch_cube_layout(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint32_t* tpos,
                        uint64_t* block_off, unsigned long long* summary, void* scratch,
                        size_t scratch_bytes, cudaStream_t s) {
  if (n == 0) return;
  uint64_t* kept = static_cast<uint64_t*>(scratch);
  uint64_t* cells = kept + (n + 1);
  uint64_t* tpos64 = cells + (n + 1);
  void* temp = tpos64 + (n + 1);
  size_t temp_bytes = scratch_bytes - 3ull * (n + 1) * sizeof(uint64_t);
  unsigned long long init[3] = {0ull, 0xFFFFFFFFull, 0ull};
  PSG_CUDA(cudaMemcpyAsync(summary, init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_layout_prep<<<(n + 255) / 256, 256, 0, s>>>(iter_count, n, nn, kept, cells, summary);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  launch_exclusive_scan_u64(kept, tpos64, n, temp, temp_bytes, s);
  launch_exclusive_scan_u64(cells, block_off, n, temp, temp_bytes, s);
  k_u64_to_u32<<<(n + 255) / 256, 256, 0, s>>>(tpos64, tpos, n);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K3+K4+K5+K6a: the fused trace pass.
//
// A CTA owns `warps` consecutive traces, one warp per trace.  Each warp walks
// its trace in 32-event steps (lane l <-> event pos+l, 4 steps of ts/ctx in
// registers per batch) and keeps, in its private shared-memory carve-out:
//   * the window table cnt/sum/min/max per ctx (non-atomic; conflict-free
//     fast path, __match_any_sync fold on duplicate keys);
//   * G+1 cube rows of exclusive ns in anchor-subtree preorder (G iterations
//     of the current chunk plus the gap row);
//   * within-trace sums over the first K iterations.
// The CTA advances in chunks of G iterations: every warp stops at its trace's
// boundary G*(c+1); rows are then rolled up to inclusive time with one warp
// prefix scan (preorder makes every subtree a contiguous range), stored to
// the dense cube, and reduced across the CTA's traces into the cross-rank
// (iteration, node) statistics with 64-bit global reductions.
__global__ void __launch_bounds__(512, 1) k_trace_query(query_params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t W = p.warps, n_ctx = p.n_ctx, nn = p.nn, G = p.G;

  int32_t* s_sub_pre = reinterpret_cast<int32_t*>(smem);
  int32_t* s_cct_pre = s_sub_pre + n_ctx;
  int32_t* s_cct_size = s_cct_pre + n_ctx;
  int32_t* s_node_pre = s_cct_size + n_ctx;
  int32_t* s_node_size = s_node_pre + nn;
  uint32_t* s_wkept = reinterpret_cast<uint32_t*>(s_node_size + nn);

  warp_smem_layout L;
  L.init(n_ctx, nn, G);
  uint8_t* wb = smem + cta_table_bytes(n_ctx, nn, W) + static_cast<size_t>(warp) * L.bytes;
  u64* wcnt = reinterpret_cast<u64*>(wb + L.off_wcnt);
  u64* wsum = reinterpret_cast<u64*>(wb + L.off_wsum);
  u64* wmin = reinterpret_cast<u64*>(wb + L.off_wmin);
  u64* wmax = reinterpret_cast<u64*>(wb + L.off_wmax);
  uint8_t* wtag = wb + L.off_wtag;
  u64* rows = reinterpret_cast<u64*>(wb + L.off_rows);
  uint8_t* rtag = wb + L.off_rtag;
  u64* scan = reinterpret_cast<u64*>(wb + L.off_scan);
  u64* wsx = reinterpret_cast<u64*>(wb + L.off_wsx);
  u64* wsqlo = reinterpret_cast<u64*>(wb + L.off_wsqlo);
  u64* wsqhi = reinterpret_cast<u64*>(wb + L.off_wsqhi);

  for (uint32_t i = threadIdx.x; i < n_ctx; i += blockDim.x) {
    s_sub_pre[i] = p.do_cube ? p.sub_pre[i] : -1;
    s_cct_pre[i] = p.do_window ? p.cct_pre[i] : 0;
    s_cct_size[i] = p.do_window ? p.cct_size[i] : 0;
  }
  for (uint32_t i = threadIdx.x; i < nn; i += blockDim.x) {
    s_node_pre[i] = p.node_pre[i];
    s_node_size[i] = p.node_size[i];
  }
  for (uint32_t c = lane; c < n_ctx; c += 32) {
    wcnt[c] = 0;
    wsum[c] = 0;
    wmin[c] = ~0ull;
    wmax[c] = 0;
  }
  for (uint32_t j = lane; j < (G + 1) * nn; j += 32) rows[j] = 0;
  for (uint32_t j = lane; j < nn; j += 32) {
    wsx[j] = 0;
    wsqlo[j] = 0;
    wsqhi[j] = 0;
  }

  const uint32_t t = blockIdx.x * W + warp;
  const bool active = t < p.tr.n;
  u64 pos = active ? p.tr.off[t] : 0, end = active ? p.tr.off[t + 1] : 0;
  const u64 tend = active ? p.tr.t_end[t] : 0;
  const uint32_t iters = (active && p.do_cube) ? p.iter_count[t] : 0;
  const bool kept = iters > 0;
  const uint32_t tp = kept ? p.tpos[t] : 0;
  const u64 bo = kept ? p.block_off[t] : 0;
  if (lane == 0) s_wkept[warp] = (active && kept) ? 1u : 0u;
  const u64 t0 = p.t0, t1 = (p.clamp_tend && tend < p.t1) ? tend : p.t1;

  bstate st{-1, 0, 0, 0};
  bool c_has = false;
  u64 c_ts = 0, c_d = 0;
  uint32_t c_ctx = 0;
  bool wdone = !active || pos >= end;
  __syncthreads();

  for (uint32_t chunk = 0;; ++chunk) {
    const int kbase = static_cast<int>(chunk * G);
    const int k_stop = p.do_cube ? static_cast<int>((chunk + 1) * G) : INT_MAX;
    if (!wdone) {
      bool stopped = false;
      while (!stopped && pos < end) {
        u64 bts[4];
        uint32_t bcx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          u64 i = pos + j * 32 + lane;
          bool v = i < end;
          bts[j] = v ? ldg_u64(p.tr.ts + i) : ~0ull;
          bcx[j] = v ? __ldg(p.tr.ctx + i) : 0u;
        }
        u64 tail = (lane == 0 && pos + 128 < end) ? ldg_u64(p.tr.ts + pos + 128) : ~0ull;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const u64 base = pos + j * 32;
          if (base >= end) break;
          const u64 i = base + lane;
          const bool valid = i < end;
          const u64 tsi = bts[j];
          const uint32_t ci = bcx[j];
          u64 nfirst = __shfl_sync(FULL, j + 1 < 4 ? bts[(j + 1) & 3] : tail, 0);
          u64 nxt = __shfl_down_sync(FULL, tsi, 1);
          if (lane == 31) nxt = nfirst;
          const bool is_last = valid && (i + 1 == end);
          const int nvalid = static_cast<int>((end - base) < 32ull ? (end - base) : 32ull);
          int nproc = nvalid;
          int ki = st.k;
          unsigned cmask = 0, bmask = 0;
          bool in_sub = false;
          int pp = -1;
          if (p.do_cube) {
            pp = valid ? s_sub_pre[ci] : -1;
            in_sub = pp >= 0;
            ki = boundary_step(st, valid, in_sub, tsi, lane, cmask, bmask);
            unsigned stopm = __ballot_sync(FULL, valid && ki >= k_stop);
            if (stopm) nproc = __ffs(stopm) - 1;
            const bool cu = lane < nproc && in_sub && ki < static_cast<int>(iters);
            const u64 cd = (is_last ? tend : nxt) - tsi;
            const int slot = ki < 0 ? static_cast<int>(G) : ki - kbase;
            const unsigned key = cu ? static_cast<unsigned>(slot) * nn + static_cast<unsigned>(pp) : 0u;
            warp_keyed_update<1>(rtag, key, cu, lane, cd, rows, nullptr, nullptr, nullptr);
          }
          const bool act = lane < nproc;
          if (p.do_window) {
            const bool carry_here = act && tsi < t0 && (is_last || nxt >= t0);
            unsigned cm = __ballot_sync(FULL, carry_here);
            if (cm) {
              int src = __ffs(cm) - 1;
              c_has = true;
              c_ts = __shfl_sync(FULL, tsi, src);
              c_ctx = __shfl_sync(FULL, ci, src);
              u64 e2 = __shfl_sync(FULL, is_last ? t1 : min(nxt, t1), src);
              c_d = e2 > t0 ? e2 - t0 : 0;
            }
            const bool in_w = act && tsi >= t0 && tsi < t1;
            const u64 wd = (is_last ? t1 : min(nxt, t1)) - tsi;
            warp_keyed_update<4>(wtag, in_w ? ci : 0u, in_w, lane, wd, wsum, wcnt, wmin, wmax);
          }
          if (p.do_cube) boundary_advance(st, nproc, in_sub, cmask, tsi, ki);
          if (nproc < nvalid) {
            pos = base + nproc;
            stopped = true;
            break;
          }
        }
        if (!stopped) pos = min(pos + 128, end);
      }
      if (pos >= end) wdone = true;
    }

    if (p.do_cube) {
      __syncwarp();
      if (active && kept) {
        const int k_hi = min(kbase + static_cast<int>(G), static_cast<int>(iters));
        for (int k = (chunk == 0 ? -1 : kbase); k < k_hi; ++k) {
          const int slot = k < 0 ? static_cast<int>(G) : k - kbase;
          u64* row = rows + static_cast<size_t>(slot) * nn;
          warp_prefix(row, scan, nn, lane);
          for (uint32_t n = lane; n < nn; n += 32) {
            const int pr = s_node_pre[n], sz = s_node_size[n];
            const u64 ex = scan[pr + 1] - scan[pr], in = scan[pr + sz] - scan[pr];
            if (k < 0) {
              p.gap_excl[static_cast<size_t>(tp) * nn + n] = ex;
              p.gap_incl[static_cast<size_t>(tp) * nn + n] = in;
            } else {
              if (p.store_cube) {
                p.cube_excl[bo + static_cast<u64>(k) * nn + n] = ex;
                p.cube_incl[bo + static_cast<u64>(k) * nn + n] = in;
              }
              if (p.do_stats && static_cast<uint32_t>(k) < p.K) {
                wsx[n] += in;
                u128 sq = static_cast<u128>(in) * in;
                u64 lo = wsqlo[n] + static_cast<u64>(sq);
                wsqhi[n] += static_cast<u64>(sq >> 64) + (lo < wsqlo[n] ? 1ull : 0ull);
                wsqlo[n] = lo;
              }
            }
          }
          __syncwarp();
          // keep inclusive values in node order for the CTA cross-rank reduction
          for (uint32_t n = lane; n < nn; n += 32) {
            const int pr = s_node_pre[n], sz = s_node_size[n];
            row[n] = scan[pr + sz] - scan[pr];
          }
          __syncwarp();
        }
      }
      __syncthreads();
      if (p.do_stats) {
        for (uint32_t idx = threadIdx.x; idx < G * nn; idx += blockDim.x) {
          const uint32_t s = idx / nn, n = idx - s * nn;
          const uint32_t k = static_cast<uint32_t>(kbase) + s;
          if (k >= p.K) continue;
          u64 sum = 0, mx = 0;
          u128 sq = 0;
          bool any = false;
          for (uint32_t w = 0; w < W; ++w) {
            if (!s_wkept[w]) continue;
            const u64 v = reinterpret_cast<const u64*>(smem + cta_table_bytes(n_ctx, nn, W) +
                                                       static_cast<size_t>(w) * L.bytes +
                                                       L.off_rows)[idx];
            sum += v;
            mx = max(mx, v);
            sq += static_cast<u128>(v) * v;
            any = true;
          }
          if (any) {
            const size_t cell = static_cast<size_t>(k) * nn + n;
            const size_t plane = static_cast<size_t>(p.K) * nn;
            atomicAdd(p.x_sum + cell, sum);
            atomicMax(p.x_max + cell, mx);
            const u64 mask43 = (1ull << 43) - 1;
            atomicAdd(p.x_sq + cell, static_cast<u64>(sq) & mask43);
            atomicAdd(p.x_sq + plane + cell, static_cast<u64>(sq >> 43) & mask43);
            atomicAdd(p.x_sq + 2 * plane + cell, static_cast<u64>(sq >> 86));
          }
        }
      }
      __syncthreads();
      for (uint32_t j = lane; j < (G + 1) * nn; j += 32) rows[j] = 0;
      __syncwarp();
    }
    if (__syncthreads_and(wdone ? 1 : 0)) break;
  }

  if (!active) return;
  if (p.do_window) {
    // excl incl. the carry-in segment, in CCT preorder, then inclusive roll-up
    u64* tmp = reinterpret_cast<u64*>(wb + L.off_tmp);
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      u64 ex = wsum[c] + ((c_has && c == c_ctx) ? c_d : 0ull);
      tmp[s_cct_pre[c]] = ex;
    }
    __syncwarp();
    warp_prefix(tmp, scan, n_ctx, lane);
    const size_t base = static_cast<size_t>(t) * n_ctx;
    for (uint32_t c = lane; c < n_ctx; c += 32) {
      const int pr = s_cct_pre[c], sz = s_cct_size[c];
      const u64 cnt = wcnt[c], sum = wsum[c];
      p.w_cnt[base + c] = cnt;
      p.w_sum[base + c] = sum;
      p.w_min[base + c] = cnt ? wmin[c] : 0ull;
      p.w_max[base + c] = wmax[c];
      p.w_mean[base + c] = cnt ? static_cast<double>(sum) / static_cast<double>(cnt) : 0.0;
      p.w_excl[base + c] = scan[pr + 1] - scan[pr];
      p.w_incl[base + c] = scan[pr + sz] - scan[pr];
    }
    if (lane == 0) {
      p.c_has[t] = c_has ? 1 : 0;
      p.c_ts[t] = c_has ? c_ts : 0;
      p.c_ctx[t] = c_has ? c_ctx : 0;
    }
  }
  if (p.do_stats && kept && p.K > 0) {
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

void launch_trace_query(const query_params& p, uint32_t smem_bytes, cudaStream_t s) {
  if (p.tr.n == 0) return;
  unsigned blocks = (p.tr.n + p.warps - 1) / p.warps;
  static int configured_bytes = 0;
  if (static_cast<int>(smem_bytes) > configured_bytes) {
    PSG_CUDA(cudaFuncSetAttribute(k_trace_query, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_bytes)));
    configured_bytes = static_cast<int>(smem_bytes);
  }
  k_trace_query<<<blocks, p.warps * 32, smem_bytes, s>>>(p);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K6b: within-rank CV mean over kept traces (fixed-order tree per node), then
// the per-node savings / across-rank CV rows.
__global__ void k_within_reduce(const double* within_cv, const uint8_t* within_ok, uint32_t n_kept,
                                uint32_t nn, double* out_sum, double* out_bad) {
  const uint32_t n = blockIdx.x;
  double s = 0.0, bad = 0.0;
  for (uint32_t t = threadIdx.x; t < n_kept; t += blockDim.x) {
    s += within_cv[static_cast<size_t>(t) * nn + n];
    bad += within_ok[static_cast<size_t>(t) * nn + n] ? 0.0 : 1.0;
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double ts = BR(tmp).Sum(s);
  __syncthreads();
  double tb = BR(tmp).Sum(bad);
  if (threadIdx.x == 0) {
    out_sum[n] = ts;
    out_bad[n] = tb;
  }
}

__global__ void k_stats_finalize(const unsigned long long* x_sum, const unsigned long long* x_max,
                                 const unsigned long long* x_sq, uint32_t K, uint32_t nn,
                                 uint32_t n_kept, const double* within_sum, const double* within_bad,
                                 double* out) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const size_t plane = static_cast<size_t>(K) * nn;
  double avg_mean = 0.0, avg_max = 0.0, across = 0.0;
  bool across_ok = true;
  for (uint32_t k = 0; k < K; ++k) {
    const size_t cell = static_cast<size_t>(k) * nn + n;
    const u64 s = x_sum[cell], mx = x_max[cell];
    const u128 sq = static_cast<u128>(x_sq[cell]) + (static_cast<u128>(x_sq[plane + cell]) << 43) +
                    (static_cast<u128>(x_sq[2 * plane + cell]) << 86);
    avg_mean += (static_cast<double>(s) / 1e9) / static_cast<double>(n_kept);
    avg_max += static_cast<double>(mx) / 1e9;
    if (s == 0) {
      across_ok = false;
    } else {
      const u128 num = static_cast<u128>(n_kept) * sq - static_cast<u128>(s) * s;
      across += 100.0 * sqrt(u128_to_double(num)) / static_cast<double>(s);
    }
  }
  avg_mean /= static_cast<double>(K);
  avg_max /= static_cast<double>(K);
  across /= static_cast<double>(K);
  double* o = out + static_cast<size_t>(n) * 8;
  o[0] = avg_mean;
  o[1] = avg_max;
  o[2] = avg_max - avg_mean;
  o[3] = (avg_max - avg_mean) * K;
  o[4] = across;
  o[5] = within_sum[n] / static_cast<double>(n_kept);
  o[6] = (across_ok && n_kept >= 2 && K >= 2) ? 1.0 : 0.0;
  o[7] = (within_bad[n] == 0.0 && n_kept >= 2 && K >= 2) ? 1.0 : 0.0;
}

void launch_stats_finalize(const unsigned long long* x_sum, const unsigned long long* x_max,
                           const unsigned long long* x_sq, uint32_t K, uint32_t nn,
                           uint32_t n_kept, const double* within_cv, const uint8_t* within_ok,
                           uint32_t n_kept_local, double* node_out, cudaStream_t s) {
  // node_out layout: [nn][8] result rows, then [nn] within sums, [nn] bad counts
  double* wsum = node_out + static_cast<size_t>(nn) * 8;
  double* wbad = wsum + nn;
  if (within_cv) {
    k_within_reduce<<<nn, 256, 0, s>>>(within_cv, within_ok, n_kept_local, nn, wsum, wbad);
    count_launch();
    PSG_CUDA(cudaGetLastError());
  }
  if (x_sum) {
    k_stats_finalize<<<(nn + 127) / 128, 128, 0, s>>>(x_sum, x_max, x_sq, K, nn, n_kept, wsum, wbad,
                                                      node_out);
    count_launch();
    PSG_CUDA(cudaGetLastError());
  }
}

// ===========================================================================
// K2: ingest_traces rows.  Per trace two lower_bounds (store.cpp:644-656),
// the carry-in event[i0-1] (store.cpp:667-670), then a warp copy of [i0,i1).
__device__ __forceinline__ u64 lower_bound_ts(const uint64_t* ts, u64 lo, u64 hi, u64 x) {
  while (lo < hi) {
    u64 mid = lo + (hi - lo) / 2;
    if (ldg_u64(ts + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void k_window_bounds(trace_view tr, u64 t0, u64 t1, uint64_t* cnt, uint8_t* c_has,
                                uint64_t* c_ts, uint32_t* c_ctx) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tr.n) return;
  u64 b = tr.off[t], e = tr.off[t + 1];
  u64 i0 = lower_bound_ts(tr.ts, b, e, t0);
  u64 i1 = lower_bound_ts(tr.ts, i0, e, t1);
  cnt[t] = i1 - i0;
  c_has[t] = i0 > b ? 1 : 0;
  c_ts[t] = i0 > b ? ldg_u64(tr.ts + i0 - 1) : 0;
  c_ctx[t] = i0 > b ? __ldg(tr.ctx + i0 - 1) : 0;
}

void launch_window_bounds(const trace_view& tr, uint64_t t0, uint64_t t1, uint64_t* cnt,
                          uint8_t* c_has, uint64_t* c_ts, uint32_t* c_ctx, cudaStream_t s) {
  if (tr.n == 0) return;
  k_window_bounds<<<(tr.n + 255) / 256, 256, 0, s>>>(tr, t0, t1, cnt, c_has, c_ts, c_ctx);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

__global__ void k_window_copy(trace_view tr, const uint32_t* pid, u64 t0, const uint64_t* row_off,
                              uint32_t* out_pid, uint64_t* out_ts, uint32_t* out_ctx) {
  uint32_t t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (t >= tr.n) return;
  u64 b = tr.off[t], e = tr.off[t + 1];
  u64 i0 = lower_bound_ts(tr.ts, b, e, t0);
  u64 n = row_off[t + 1] - row_off[t], o = row_off[t];
  uint32_t id = pid[t];
  for (u64 j = lane; j < n; j += 32) {
    out_pid[o + j] = id;
    out_ts[o + j] = ldg_u64(tr.ts + i0 + j);
    out_ctx[o + j] = __ldg(tr.ctx + i0 + j);
  }
}

void launch_window_copy(const trace_view& tr, const uint32_t* pid, uint64_t t0,
                        const uint64_t* row_off, uint32_t* out_pid, uint64_t* out_ts,
                        uint32_t* out_ctx, cudaStream_t s) {
  if (tr.n == 0) return;
  k_window_copy<<<(tr.n + 7) / 8, 256, 0, s>>>(tr, pid, t0, row_off, out_pid, out_ts, out_ctx);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K7: outliers.  phase 0: per-site cross-rank sum/max of the window-inclusive
// ns (rank_vector + balance_ratio, workflows.cpp:442-453); phase 1: pick the
// worst site (strict <, first wins, workflows.cpp:455-457); phase 2: per-node
// sums/counts of the worst site's values (node_correlate, diagnostics.cpp:378-403).
__global__ void k_site_acc(const uint64_t* w_incl, uint32_t n, uint32_t n_ctx, const uint32_t* site,
                           uint32_t n_sites, unsigned long long* acc) {
  u64 g = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
  if (g >= static_cast<u64>(n) * n_sites) return;
  uint32_t t = static_cast<uint32_t>(g / n_sites), s = static_cast<uint32_t>(g % n_sites);
  u64 v = w_incl[static_cast<size_t>(t) * n_ctx + site[s]];
  atomicAdd(acc + s, v);
  atomicMax(acc + n_sites + s, v);
}

__global__ void k_pick_worst(const unsigned long long* acc, uint32_t n_sites, uint32_t n_ranks,
                             uint32_t* worst, double* ratio) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t w = 0;
  for (uint32_t s = 0; s < n_sites; ++s) {
    double mx = static_cast<double>(acc[n_sites + s]) / 1e9;
    double sum = static_cast<double>(acc[s]) / 1e9;
    ratio[s] = mx == 0.0 ? 1.0 : sum / static_cast<double>(n_ranks) / mx;
    if (ratio[s] < ratio[w]) w = s;
  }
  *worst = w;
}

__global__ void k_node_acc(const uint64_t* w_incl, uint32_t n, uint32_t n_ctx, const uint32_t* site,
                           const uint32_t* worst, const uint32_t* node_of_trace,
                           unsigned long long* node_acc) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  u64 v = w_incl[static_cast<size_t>(t) * n_ctx + site[*worst]];
  uint32_t nd = node_of_trace[t];
  atomicAdd(node_acc + 2 * nd, v);
  atomicAdd(node_acc + 2 * nd + 1, 1ull);
}

void launch_outliers(const uint64_t* w_incl, uint32_t n_traces, uint32_t n_ctx,
                     const uint32_t* site_ctx, uint32_t n_sites, const uint32_t* node_of_trace,
                     uint32_t n_nodes, unsigned long long* site_acc,
                     unsigned long long* node_acc, uint32_t* worst, double* site_ratio,
                     uint32_t phase, cudaStream_t s) {
  (void)n_nodes;
  if (phase == 0) {
    u64 th = static_cast<u64>(n_traces) * n_sites;
    if (th) k_site_acc<<<static_cast<unsigned>((th + 255) / 256), 256, 0, s>>>(w_incl, n_traces, n_ctx,
                                                                              site_ctx, n_sites, site_acc);
  } else if (phase == 1) {
    k_pick_worst<<<1, 32, 0, s>>>(site_acc, n_sites, n_traces /* global rank count */, worst,
                                  site_ratio);
  } else {
    if (n_traces)
      k_node_acc<<<(n_traces + 255) / 256, 256, 0, s>>>(w_incl, n_traces, n_ctx, site_ctx, worst,
                                                        node_of_trace, node_acc);
  }
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// Node means, population z-scores, then the ranking: CUB radix sort of the
// means descending (stable, node ids ascending on ties), selection of the
// prefix with z >= z_min capped at top_k.
__global__ void k_node_stats(const unsigned long long* node_acc, uint32_t n_nodes, double* mean,
                             double* z, uint64_t* key, uint32_t* ids) {
  __shared__ double red[1024];
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < n_nodes; i += blockDim.x) {
    u64 c = node_acc[2 * i + 1];
    double m = c ? (static_cast<double>(node_acc[2 * i]) / 1e9) / static_cast<double>(c) : 0.0;
    mean[i] = m;
    s += m;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double mu = red[0] / static_cast<double>(n_nodes);
  __syncthreads();
  double v = 0.0;
  for (uint32_t i = threadIdx.x; i < n_nodes; i += blockDim.x) v += (mean[i] - mu) * (mean[i] - mu);
  red[threadIdx.x] = v;
  __syncthreads();
  for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double sd = sqrt(red[0] / static_cast<double>(n_nodes));
  for (uint32_t i = threadIdx.x; i < n_nodes; i += blockDim.x) {
    z[i] = sd > 0.0 ? (mean[i] - mu) / sd : 0.0;
    key[i] = __double_as_longlong(mean[i]);  // means are >= 0: bit order == value order
    ids[i] = i;
  }
}

__global__ void k_node_cut(const uint32_t* sorted_ids, const double* z, uint32_t n_nodes,
                           uint32_t top_k, double z_min, uint32_t* n_sel) {
  __shared__ uint32_t first_bad;
  if (threadIdx.x == 0) first_bad = n_nodes;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_nodes; i += blockDim.x)
    if (z[sorted_ids[i]] < z_min) atomicMin(&first_bad, i);
  __syncthreads();
  if (threadIdx.x == 0) *n_sel = top_k ? min(first_bad, top_k) : first_bad;
}

void launch_node_select(const unsigned long long* node_acc, uint32_t n_nodes, uint32_t top_k,
                        double z_min, double* node_mean, double* node_z, uint32_t* order,
                        uint32_t* n_sel, cudaStream_t s) {
  // scratch: keys/ids (in + out) allocated per call (small: n_nodes entries)
  uint64_t *k_in = nullptr, *k_out = nullptr;
  uint32_t* ids_in = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  PSG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, temp_bytes, k_in, k_out, ids_in, order,
                                                     static_cast<int>(n_nodes), 0, 64, s));
  PSG_CUDA(cudaMallocAsync(&k_in, sizeof(uint64_t) * n_nodes * 2 + sizeof(uint32_t) * n_nodes + temp_bytes + 64, s));
  k_out = k_in + n_nodes;
  ids_in = reinterpret_cast<uint32_t*>(k_out + n_nodes);
  temp = reinterpret_cast<uint8_t*>(ids_in + n_nodes + 8);
  k_node_stats<<<1, 1024, 0, s>>>(node_acc, n_nodes, node_mean, node_z, k_in, ids_in);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, k_in, k_out, ids_in, order,
                                                     static_cast<int>(n_nodes), 0, 64, s));
  k_node_cut<<<1, 1024, 0, s>>>(order, node_z, n_nodes, top_k, z_min, n_sel);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cudaFreeAsync(k_in, s));
}

// K8: topology.  Outlier nodes -> (rack index, chassis) histogram; a chassis
// is fully affected when its outlier count equals its universe node count.
__global__ void k_topology(const uint32_t* selected, const uint32_t* n_sel, const uint32_t* rack_idx,
                           const uint32_t* chassis, const uint32_t* uni_cnt, uint32_t n_racks,
                           uint32_t* rack_nodes, unsigned long long* rack_mask,
                           unsigned long long* rack_full) {
  extern __shared__ uint32_t cnt[];  // [n_racks][64]
  for (uint32_t i = threadIdx.x; i < n_racks * 64; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint32_t ns = *n_sel;
  for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
    uint32_t nd = selected[i];
    atomicAdd(&cnt[rack_idx[nd] * 64 + min(chassis[nd], 63u)], 1u);
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < n_racks; r += blockDim.x) {
    uint32_t nodes = 0;
    u64 m = 0, f = 0;
    for (uint32_t c = 0; c < 64; ++c) {
      uint32_t x = cnt[r * 64 + c];
      nodes += x;
      if (x) {
        m |= 1ull << c;
        if (x == uni_cnt[r * 64 + c]) f |= 1ull << c;
      }
    }
    rack_nodes[r] = nodes;
    rack_mask[r] = m;
    rack_full[r] = f;
  }
}

void launch_topology(const uint32_t* selected, const uint32_t* n_sel, const uint32_t* node_rack_idx,
                     const uint32_t* node_chassis, const uint32_t* uni_cnt, uint32_t n_racks,
                     uint32_t* rack_nodes, unsigned long long* rack_mask,
                     unsigned long long* rack_full, cudaStream_t s) {
  if (n_racks == 0) return;
  size_t sm = sizeof(uint32_t) * n_racks * 64;
  if (sm > 200 * 1024) fail(PS_E_INVALID_ARGUMENT, "too many racks for the topology kernel");
  if (sm > 48 * 1024)
    PSG_CUDA(cudaFuncSetAttribute(k_topology, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
  k_topology<<<1, 512, sm, s>>>(selected, n_sel, node_rack_idx, node_chassis, uni_cnt, n_racks,
                                rack_nodes, rack_mask, rack_full);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
