// Hand-written sm_100a kernels of the perfslice trace query path.
//
//   K1 k_aos_to_soa      trace.db 12-byte AoS -> SoA ts/ctx      (store.cpp:573-580, 678-692)
//   K1v k_validate       format invariants of the loaded events   (store.cpp:743-761)
//   K0 k_gen_*           device replay of synthgen's iterative scenario (synthgen.cpp:146-246)
//   (the two passes of the fused query, k_bounds and k_trace_query, are in psg_query.cu)
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

#include <algorithm>
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

__device__ __forceinline__ u64 ldg_u64(const uint64_t* p) {
  return static_cast<u64>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}
__device__ __forceinline__ double u128_to_double(u128 v) {
  return static_cast<double>(static_cast<u64>(v >> 64)) * 18446744073709551616.0 +
         static_cast<double>(static_cast<u64>(v));
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

// Dense int64 copy-out of the stored cube (itermodel.hpp:97-101): one CTA per
// loaded trace of [t_lo, t_lo + gridDim.x); a kept trace's iterations x nodes
// go to dense cell (iter_off[t] - dense_row0) * nn + k * nn + n, widened from
// the 32- or 64-bit storage cells (rows of stride nnp); excl is the leaf's
// incl, or the internal node's entry of the compact [row][m] excl table.
__global__ void k_cube_dense(const void* __restrict__ incl, uint32_t cube32,
                             const uint64_t* __restrict__ xint, const uint32_t* __restrict__ iter_count,
                             const uint64_t* __restrict__ block_off, const uint64_t* __restrict__ iter_off,
                             const int4* __restrict__ node_tab, uint32_t nn, uint32_t nnp, uint32_t m,
                             uint32_t t_lo, uint64_t dense_row0, int64_t* __restrict__ out_incl,
                             int64_t* __restrict__ out_excl) {
  const uint32_t t = t_lo + blockIdx.x;
  const uint32_t it = iter_count[t];
  if (it == 0) return;
  const uint64_t bo = block_off[t], row0 = iter_off[t];
  const uint64_t cells = static_cast<uint64_t>(it) * nn;
  int64_t* oi = out_incl ? out_incl + (row0 - dense_row0) * nn : nullptr;
  int64_t* oe = out_excl ? out_excl + (row0 - dense_row0) * nn : nullptr;
  for (uint64_t i = threadIdx.x; i < cells; i += blockDim.x) {
    const uint64_t k = i / nn;
    const uint32_t n = static_cast<uint32_t>(i - k * nn);
    const uint64_t src = bo + k * nnp + n;
    const int64_t v = cube32 ? static_cast<int64_t>(__ldg(static_cast<const uint32_t*>(incl) + src))
                             : static_cast<int64_t>(ldg_u64(static_cast<const uint64_t*>(incl) + src));
    if (oi) oi[i] = v;
    if (oe) {
      const int z = node_tab[n].z;
      oe[i] = z ? static_cast<int64_t>(ldg_u64(xint + (row0 + k) * m + (z - 1))) : v;
    }
  }
}

void launch_cube_dense(const void* incl, bool cube32, const uint64_t* xint, const uint32_t* iter_count,
                       const uint64_t* block_off, const uint64_t* iter_off, const int4* node_tab,
                       uint32_t nn, uint32_t nnp, uint32_t m, uint32_t t_lo, uint32_t t_hi,
                       uint64_t dense_row0, int64_t* out_incl, int64_t* out_excl, cudaStream_t s) {
  if (t_hi <= t_lo || nn == 0) return;
  k_cube_dense<<<t_hi - t_lo, 256, 0, s>>>(incl, cube32 ? 1u : 0u, xint, iter_count, block_off, iter_off,
                                           node_tab, nn, nnp, m, t_lo, dense_row0, out_incl, out_excl);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// K1v: one warp per trace checks the invariants validate_database reports.
__global__ void k_validate(trace_view tr, uint32_t n_ctx, const uint64_t* t_begin,
                           unsigned long long* bad, unsigned long long* first_bad) {
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
    if (i == b && t_begin && t_begin[t] != x) ok = false;  // store.cpp:750-751
  }
  if (!__all_sync(FULL, ok) && lane == 0) {
    atomicAdd(bad, 1ull);
    atomicMin(first_bad, static_cast<unsigned long long>(t));
  }
}

void launch_validate(const trace_view& tr, uint32_t n_ctx, const uint64_t* t_begin,
                     unsigned long long* bad, unsigned long long* first_bad, cudaStream_t s) {
  if (tr.n == 0) return;
  k_validate<<<(tr.n + 7) / 8, 256, 0, s>>>(tr, n_ctx, t_begin, bad, first_bad);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// K1n: the narrow ctx mirror pass 1 reads (1 B/event instead of 4): 16 ctx
// words (four 16-byte loads) -> 16 bytes (one 16-byte store) per thread, each
// ctx replaced by its preorder position in the CCT (any subtree is then one
// contiguous byte range).
__global__ void __launch_bounds__(256) k_ctx8(const uint32_t* __restrict__ ctx, uint64_t n,
                                              const int32_t* __restrict__ pre, uint32_t n_ctx,
                                              uint8_t* __restrict__ out) {
  __shared__ uint32_t s_pre[256];
  s_pre[threadIdx.x] = threadIdx.x < n_ctx ? static_cast<uint32_t>(pre[threadIdx.x]) : 0u;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 16;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; i < n;
       i += stride) {
    if (i + 16 <= n) {
      const uint4* src = reinterpret_cast<const uint4*>(ctx + i);
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(src + q);
        w[q] = s_pre[v.x & 255u] | (s_pre[v.y & 255u] << 8) | (s_pre[v.z & 255u] << 16) |
               (s_pre[v.w & 255u] << 24);
      }
      *reinterpret_cast<uint4*>(out + i) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (uint64_t j = i; j < n; ++j) out[j] = static_cast<uint8_t>(s_pre[ctx[j] & 255u]);
    }
  }
}

void launch_ctx8(const uint32_t* ctx, uint64_t n, const int32_t* pre, uint32_t n_ctx, uint8_t* out,
                 cudaStream_t s) {
  if (n == 0) return;
  if (n_ctx > 256) fail(PS_E_INTERNAL, "ctx8 mirror needs n_ctx <= 256");
  int dev = 0, sms = 148;
  PSG_CUDA(cudaGetDevice(&dev));
  PSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t need = (n + 16 * 256 - 1) / (16 * 256);
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(need, static_cast<uint64_t>(sms) * 8));
  k_ctx8<<<g, 256, 0, s>>>(ctx, n, pre, n_ctx, out);
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

// Cube layout: kept flags, storage cell counts (rows of stride nnp, each
// trace block padded to a multiple of 4 cells = 16 bytes of 32-bit cells),
// iteration counts, then exclusive scans (CUB).
__global__ void k_layout_prep(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint32_t nnp,
                              uint64_t* kept, uint64_t* cells, uint64_t* iters,
                              unsigned long long* summary) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // the grid covers whole warps
  const uint32_t it = t < n ? iter_count[t] : 0;
  if (t < n) {
    kept[t] = it > 0 ? 1 : 0;
    cells[t] = (static_cast<uint64_t>(it) * nnp + 3) & ~3ull;
    iters[t] = it;
  }
  // warp-aggregated summary atomics: kept count, min iterations, cells, storage cells
  unsigned long long k1 = it > 0 ? 1ull : 0ull, m1 = it > 0 ? it : 0xFFFFFFFFull;
  unsigned long long c2 = static_cast<unsigned long long>(it) * nn;
  unsigned long long c4 = (static_cast<unsigned long long>(it) * nnp + 3) & ~3ull;
  for (int d = 16; d > 0; d >>= 1) {
    k1 += __shfl_xor_sync(FULL, k1, d);
    m1 = min(m1, __shfl_xor_sync(FULL, m1, d));
    c2 += __shfl_xor_sync(FULL, c2, d);
    c4 += __shfl_xor_sync(FULL, c4, d);
  }
  if ((threadIdx.x & 31) == 0 && k1) {
    atomicAdd(summary + 0, k1);
    atomicMin(summary + 1, m1);
    atomicAdd(summary + 2, c2);
    atomicAdd(summary + 4, c4);
  }
}

// Kept-trace positions (u32) and the compact list of kept block offsets.
__global__ void k_finish_layout(const uint64_t* tpos64, const uint32_t* iter_count,
                                const uint64_t* block_off, uint32_t n, uint32_t* tpos,
                                uint64_t* kept_bo) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t tp = static_cast<uint32_t>(tpos64[t]);
  tpos[t] = tp;
  if (iter_count[t] > 0) kept_bo[tp] = block_off[t];
}

// One warp per trace: the longest stored iteration (itermodel.cpp:294-301:
// iteration k = [b_k, b_{k+1}), the last one ends at t_end).
__global__ void k_iter_spans(const uint64_t* cap_off, const uint64_t* bts, const uint32_t* iter_count,
                             const uint64_t* t_end, uint32_t n, unsigned long long* max_span) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n) return;
  const uint32_t it = iter_count[t];
  const uint64_t* b = bts + cap_off[t];
  unsigned long long m = 0;
  for (uint32_t j = lane; j < it; j += 32) {
    const uint64_t b0 = b[j], b1 = j + 1 < it ? b[j + 1] : t_end[t];
    m = max(m, static_cast<unsigned long long>(b1 - b0));
  }
  for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
  if (lane == 0 && it > 0) atomicMax(max_span, m);
}

void launch_iter_spans(const uint64_t* cap_off, const uint64_t* bts, const uint32_t* iter_count,
                       const uint64_t* t_end, uint32_t n, unsigned long long* max_span,
                       cudaStream_t s) {
  if (n == 0) return;
  k_iter_spans<<<(n + 7) / 8, 256, 0, s>>>(cap_off, bts, iter_count, t_end, n, max_span);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

size_t exclusive_scan_u64_scratch(uint32_t n) { return exclusive_sum_scratch_bytes(n); }

void launch_exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint32_t n, void* scratch,
                               size_t scratch_bytes, cudaStream_t s) {
  exclusive_sum_u64(in, out, n, scratch, scratch_bytes, s);
}

size_t cube_layout_scratch_bytes(uint32_t n) {
  // kept, cells, tpos64, iters (n u64 each) + scan temp
  return 4ull * (n + 1) * sizeof(uint64_t) + exclusive_scan_u64_scratch(n) + 256;
}

void launch_cube_layout(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint32_t nnp,
                        uint32_t* tpos, uint64_t* block_off, uint64_t* iter_off, uint64_t* kept_bo,
                        unsigned long long* summary, void* scratch, size_t scratch_bytes,
                        cudaStream_t s) {
  unsigned long long init[5] = {0ull, 0xFFFFFFFFull, 0ull, 0ull, 0ull};
  // an empty shard still reports its (empty) summary: no kept traces, the
  // "no minimum" sentinel, no cells (a rank may hold no traces)
  PSG_CUDA(cudaMemcpyAsync(summary, init, 3 * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  PSG_CUDA(cudaMemcpyAsync(summary + 4, init + 4, sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  if (n == 0) return;
  uint64_t* kept = static_cast<uint64_t*>(scratch);
  uint64_t* cells = kept + (n + 1);
  uint64_t* tpos64 = cells + (n + 1);
  uint64_t* iters = tpos64 + (n + 1);
  void* temp = iters + (n + 1);
  size_t temp_bytes = scratch_bytes - 4ull * (n + 1) * sizeof(uint64_t);
  k_layout_prep<<<(n + 255) / 256, 256, 0, s>>>(iter_count, n, nn, nnp, kept, cells, iters, summary);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  launch_exclusive_scan_u64(kept, tpos64, n, temp, temp_bytes, s);
  launch_exclusive_scan_u64(cells, block_off, n, temp, temp_bytes, s);
  launch_exclusive_scan_u64(iters, iter_off, n, temp, temp_bytes, s);
  k_finish_layout<<<(n + 255) / 256, 256, 0, s>>>(tpos64, iter_count, block_off, n, tpos, kept_bo);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// ===========================================================================
// K6b: within-rank CV mean over kept traces (fixed-order tree per node), then
// the per-node savings / across-rank CV rows.
// Stage 1: one CTA per tile of kept traces.  Threads cover (sub-row j, node
// n) so that consecutive threads read consecutive cells of a trace's row
// (coalesced); each thread sums its node over the tile's traces j, j + S, ...
// eight at a time (eight independent loads in flight, then added in trace
// order), and sub-row partials are added in fixed order: deterministic.
__global__ void __launch_bounds__(256) k_within_partial(const double* within_cv,
                                                        const uint8_t* within_ok, uint32_t n_kept,
                                                        uint32_t nn, uint32_t per_tile,
                                                        double* part /*[tiles][2][nn]*/,
                                                        const unsigned long long* qs) {
  __shared__ double s_sum[256], s_bad[256];
  if (qs) n_kept = min(n_kept, static_cast<uint32_t>(qs[QS_KEPT]));
  const uint32_t ne = min(nn, blockDim.x), S = blockDim.x / ne;
  const uint32_t j = threadIdx.x / ne, nl = threadIdx.x % ne;
  const uint32_t t0 = blockIdx.x * per_tile, t1 = min(n_kept, t0 + per_tile);
  for (uint32_t nb = 0; nb < nn; nb += ne) {
    const uint32_t n = nb + nl;
    double sm = 0.0, bad = 0.0;
    if (j < S && n < nn) {
      uint32_t t = t0 + j;
      for (; t + 7 * S < t1; t += 8 * S) {
        double v[8];
        uint8_t ok[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = __ldg(within_cv + static_cast<size_t>(t + u * S) * nn + n);
          ok[u] = __ldg(within_ok + static_cast<size_t>(t + u * S) * nn + n);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          sm += v[u];
          bad += ok[u] ? 0.0 : 1.0;
        }
      }
      for (; t < t1; t += S) {
        sm += within_cv[static_cast<size_t>(t) * nn + n];
        bad += within_ok[static_cast<size_t>(t) * nn + n] ? 0.0 : 1.0;
      }
    }
    s_sum[threadIdx.x] = sm;
    s_bad[threadIdx.x] = bad;
    __syncthreads();
    if (j == 0 && n < nn) {
      for (uint32_t q = 1; q < S; ++q) {
        sm += s_sum[q * ne + nl];
        bad += s_bad[q * ne + nl];
      }
      part[(static_cast<size_t>(blockIdx.x) * 2) * nn + n] = sm;
      part[(static_cast<size_t>(blockIdx.x) * 2 + 1) * nn + n] = bad;
    }
    __syncthreads();
  }
}

// Stage 2: per node (one warp), the tile partials in a fixed order: lane l
// sums tiles l, l + 32, ... in order, then a fixed butterfly.
__global__ void k_within_finish(const double* part, uint32_t tiles, uint32_t nn, double* out_sum,
                                double* out_bad) {
  const uint32_t n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= nn) return;
  double sm = 0.0, bad = 0.0;
  for (uint32_t b = lane; b < tiles; b += 32) {
    sm += part[(static_cast<size_t>(b) * 2) * nn + n];
    bad += part[(static_cast<size_t>(b) * 2 + 1) * nn + n];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    sm += __shfl_xor_sync(0xFFFFFFFFu, sm, d);
    bad += __shfl_xor_sync(0xFFFFFFFFu, bad, d);
  }
  if (lane == 0) {
    out_sum[n] = sm;
    out_bad[n] = bad;
  }
}

// One CTA per node: the per-iteration terms are summed with a fixed-order
// block reduction (deterministic; the fp64 association differs from the
// reference's sequential fold by ~1e-16 relative).
__global__ void __launch_bounds__(256) k_stats_finalize(const unsigned long long* x_sum,
                                                        const unsigned long long* x_max,
                                                        const unsigned long long* x_sq, uint32_t K,
                                                        uint32_t plane_k, uint32_t nn, uint32_t n_kept,
                                                        const double* within_sum,
                                                        const double* within_bad, double* out,
                                                        const unsigned long long* qs) {
  const uint32_t n = blockIdx.x;
  const size_t plane = static_cast<size_t>(plane_k) * nn;
  if (qs) {
    if (qs[QS_CAP_MISS]) return;  // the query re-runs
    K = qs_K(qs);
    n_kept = static_cast<uint32_t>(qs[QS_KEPT_G]);
  }
  if (K == 0) return;
  double m = 0.0, mx_s = 0.0, across = 0.0, bad = 0.0;
  for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) {
    const size_t cell = static_cast<size_t>(k) * nn + n;
    const u64 s = x_sum[cell], mx = x_max[cell];
    const u128 sq = static_cast<u128>(x_sq[cell]) + (static_cast<u128>(x_sq[plane + cell]) << 43) +
                    (static_cast<u128>(x_sq[2 * plane + cell]) << 86);
    m += (static_cast<double>(s) / 1e9) / static_cast<double>(n_kept);
    mx_s += static_cast<double>(mx) / 1e9;
    if (s == 0) {
      bad += 1.0;
    } else {
      const u128 num = static_cast<u128>(n_kept) * sq - static_cast<u128>(s) * s;
      across += 100.0 * sqrt(u128_to_double(num)) / static_cast<double>(s);
    }
  }
  __shared__ double s_warp[32];
  const double avg_mean = block_reduce(m, op_add(), s_warp) / static_cast<double>(K);
  const double avg_max = block_reduce(mx_s, op_add(), s_warp) / static_cast<double>(K);
  const double acr = block_reduce(across, op_add(), s_warp) / static_cast<double>(K);
  const double nbad = block_reduce(bad, op_add(), s_warp);
  if (threadIdx.x != 0) return;
  double* o = out + static_cast<size_t>(n) * 8;
  o[0] = avg_mean;
  o[1] = avg_max;
  o[2] = avg_max - avg_mean;
  o[3] = (avg_max - avg_mean) * K;
  o[4] = acr;
  o[5] = within_sum[n] / static_cast<double>(n_kept);
  o[6] = (nbad == 0.0 && n_kept >= 2 && K >= 2) ? 1.0 : 0.0;
  o[7] = (within_bad[n] == 0.0 && n_kept >= 2 && K >= 2) ? 1.0 : 0.0;
}

void launch_stats_finalize(const unsigned long long* x_sum, const unsigned long long* x_max,
                           const unsigned long long* x_sq, uint32_t K, uint32_t plane_k, uint32_t nn,
                           uint32_t n_kept, const double* within_cv, const uint8_t* within_ok,
                           uint32_t n_kept_local, double* node_out, const unsigned long long* qs,
                           cudaStream_t s) {
  // node_out layout: [nn][8] result rows, then [nn] within sums, [nn] bad counts
  double* wsum = node_out + static_cast<size_t>(nn) * 8;
  double* wbad = wsum + nn;
  if (within_cv) {
    // tile partials live after the bad counts in node_out (sized by the caller)
    const uint32_t tiles = std::max(1u, std::min(kWithinTiles, (n_kept_local + 31) / 32));
    const uint32_t per_tile = (std::max(1u, n_kept_local) + tiles - 1) / tiles;
    double* part = wbad + nn;
    k_within_partial<<<tiles, 256, 0, s>>>(within_cv, within_ok, n_kept_local, nn, per_tile, part, qs);
    k_within_finish<<<(nn + 7) / 8, 256, 0, s>>>(part, tiles, nn, wsum, wbad);
    count_launch(2);
    PSG_CUDA(cudaGetLastError());
  }
  if (x_sum) {
    k_stats_finalize<<<nn, 256, 0, s>>>(x_sum, x_max, x_sq, K, plane_k, nn, n_kept, wsum, wbad, node_out, qs);
    count_launch();
    PSG_CUDA(cudaGetLastError());
  }
}

__global__ void k_qs_check_k(unsigned long long* qs, uint32_t k_cap) {
  if (qs_K(qs) > k_cap) qs[QS_CAP_MISS] |= 4ull;
}

void launch_qs_check_k(unsigned long long* qs, uint32_t k_cap, cudaStream_t s) {
  k_qs_check_k<<<1, 1, 0, s>>>(qs, k_cap);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

__global__ void k_outlier_summary(const uint32_t* worst, const uint32_t* n_sel, const double* site_ratio,
                                  const uint32_t* rack_nodes, uint32_t n_racks, unsigned long long* qs) {
  uint32_t racks = 0;
  for (uint32_t r = threadIdx.x; r < n_racks; r += blockDim.x) racks += rack_nodes[r] > 0 ? 1u : 0u;
  for (int d = 16; d > 0; d >>= 1) racks += __shfl_xor_sync(FULL, racks, d);
  if (threadIdx.x == 0) {
    const uint32_t w = worst[0];
    qs[QS_WORST] = w;
    qs[QS_NSEL] = n_sel[0];
    qs[QS_WORST_RATIO] = static_cast<unsigned long long>(__double_as_longlong(site_ratio[w]));
    qs[QS_RACKS] = racks;
  }
}

void launch_outlier_summary(const uint32_t* worst, const uint32_t* n_sel, const double* site_ratio,
                            const uint32_t* rack_nodes, uint32_t n_racks, unsigned long long* qs,
                            cudaStream_t s) {
  k_outlier_summary<<<1, 32, 0, s>>>(worst, n_sel, site_ratio, rack_nodes, n_racks, qs);
  count_launch();
  PSG_CUDA(cudaGetLastError());
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
__global__ void __launch_bounds__(256) k_site_acc(const uint64_t* w_incl, uint32_t n, uint32_t n_ctx,
                                                  const uint32_t* site, uint32_t n_sites,
                                                  unsigned long long* acc) {
  const uint32_t s = blockIdx.y;
  const uint32_t c = site[s];
  u64 sum = 0, mx = 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const u64 v = w_incl[static_cast<size_t>(t) * n_ctx + c];
    sum += v;
    mx = max(mx, v);
  }
  __shared__ u64 s_warp[32];
  sum = block_reduce(sum, op_add(), s_warp);
  mx = block_reduce(mx, op_max(), s_warp);
  if (threadIdx.x == 0) {
    atomicAdd(acc + s, sum);
    atomicMax(acc + n_sites + s, mx);
  }
}

// Balance ratio per site, then the worst (smallest ratio, first on ties:
// workflows.cpp:478-495): one thread per site, a fixed-order argmin.
__global__ void k_pick_worst(const unsigned long long* acc, uint32_t n_sites, uint32_t n_ranks,
                             uint32_t* worst, double* ratio) {
  __shared__ double s_r[1024];
  for (uint32_t s = threadIdx.x; s < n_sites; s += blockDim.x) {
    const double mx = static_cast<double>(acc[n_sites + s]) / 1e9;
    const double sum = static_cast<double>(acc[s]) / 1e9;
    const double r = mx == 0.0 ? 1.0 : sum / static_cast<double>(n_ranks) / mx;
    ratio[s] = r;
    if (s < 1024) s_r[s] = r;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t w = 0;
  for (uint32_t s = 1; s < n_sites; ++s) {
    const double r = s < 1024 ? s_r[s] : ratio[s];
    if (r < (w < 1024 ? s_r[w] : ratio[w])) w = s;
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
    if (n_traces && n_sites) {
      const unsigned gx = std::max(1u, std::min(64u, (n_traces + 1023) / 1024));
      k_site_acc<<<dim3(gx, n_sites), 256, 0, s>>>(w_incl, n_traces, n_ctx, site_ctx, n_sites, site_acc);
    }
  } else if (phase == 1) {
    k_pick_worst<<<1, 256, 0, s>>>(site_acc, n_sites, n_traces /* global rank count */, worst,
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
    double m;
    if (node_acc) {
      u64 c = node_acc[2 * i + 1];
      m = c ? (static_cast<double>(node_acc[2 * i]) / 1e9) / static_cast<double>(c) : 0.0;
      mean[i] = m;
    } else {
      m = mean[i];  // given (profile-record path)
    }
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
    // order-preserving map of doubles to unsigned keys (negative: all bits flipped)
    const u64 bits = static_cast<u64>(__double_as_longlong(mean[i]));
    key[i] = (bits >> 63) ? ~bits : (bits | (1ull << 63));
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

size_t node_select_scratch_bytes(uint32_t n_nodes) {
  const size_t temp_bytes = sort_pairs_scratch_bytes<uint64_t, uint32_t>(n_nodes);
  return sizeof(uint64_t) * n_nodes * 2 + sizeof(uint32_t) * (n_nodes + 8) + temp_bytes + 64;
}

void launch_node_select(const unsigned long long* node_acc, uint32_t n_nodes, uint32_t top_k,
                        double z_min, double* node_mean, double* node_z, uint32_t* order,
                        uint32_t* n_sel, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  // scratch (owned by the context, reused across queries): keys/ids in + out, sort temp
  uint64_t* k_in = static_cast<uint64_t*>(scratch);
  uint64_t* k_out = k_in + n_nodes;
  uint32_t* ids_in = reinterpret_cast<uint32_t*>(k_out + n_nodes);
  void* temp = reinterpret_cast<uint8_t*>(ids_in + n_nodes + 8);
  size_t temp_bytes = scratch_bytes - (sizeof(uint64_t) * n_nodes * 2 + sizeof(uint32_t) * (n_nodes + 8));
  k_node_stats<<<1, 1024, 0, s>>>(node_acc, n_nodes, node_mean, node_z, k_in, ids_in);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  sort_pairs<uint64_t, uint32_t>(k_in, k_out, ids_in, order, n_nodes, 0, 64, true, temp, temp_bytes, s);
  k_node_cut<<<1, 1024, 0, s>>>(order, node_z, n_nodes, top_k, z_min, n_sel);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// K8: topology.  Outlier nodes -> (rack index, chassis) histogram; a chassis
// is fully affected when its outlier count equals its universe node count.
__global__ void k_topology(const uint32_t* selected, const uint32_t* n_sel, const uint32_t* rack_idx,
                           const uint32_t* chassis, const uint32_t* uni_cnt, uint32_t n_racks,
                           uint32_t* rack_nodes, unsigned long long* rack_mask,
                           unsigned long long* rack_full, uint32_t* rack_cnt) {
  extern __shared__ uint32_t cnt[];  // [n_racks][64]
  for (uint32_t i = threadIdx.x; i < n_racks * 64; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint32_t ns = *n_sel;
  for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
    uint32_t nd = selected[i];
    atomicAdd(&cnt[rack_idx[nd] * 64 + min(chassis[nd], 63u)], 1u);  // chassis slot < 64
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_racks * 64; i += blockDim.x) rack_cnt[i] = cnt[i];
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
                     unsigned long long* rack_full, uint32_t* rack_cnt, cudaStream_t s) {
  if (n_racks == 0) return;
  size_t sm = sizeof(uint32_t) * n_racks * 64;
  if (sm > 200 * 1024) fail(PS_E_INVALID_ARGUMENT, "too many racks for the topology kernel");
  if (sm > 48 * 1024)
    PSG_CUDA(cudaFuncSetAttribute(k_topology, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
  k_topology<<<1, 512, sm, s>>>(selected, n_sel, node_rack_idx, node_chassis, uni_cnt, n_racks,
                                rack_nodes, rack_mask, rack_full, rack_cnt);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
