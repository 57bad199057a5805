// The sparse window path: large calling-context trees.
//
// The fused query keeps one window record per ctx in each warp's shared
// memory and writes a dense [trace][ctx] result; past a few thousand
// contexts (the paper's AMG run has 97,833) neither fits.  This
// path computes the same two reference results as sparse, sorted rows:
//
//   groups  frame::group_aggregate over the window rows keyed by (pid, ctx)
//           (ingest.cpp:178-208 + frame.cpp:290-408): one row per (trace,
//           ctx) with count > 0 — count, sum / min / max of the clipped row
//           durations, mean = sum / count;
//   remat   itermodel::rematerialize over [t0, t1) per trace
//           (itermodel.cpp:145-183): one row per (trace, ctx) with incl or
//           excl nonzero, ascending ctx — excl = the window rows' durations
//           plus the carry-in segment, incl = excl summed over the subtree.
//
// Steps (trace-major throughout, so both outputs come out sorted by (trace,
// ctx)): per trace the window's event range by binary search (K2), one
// (key, duration) pair per row with key = trace << ctx_bits | ctx, a radix
// sort of the pairs (CUB), run starts, one thread folding each run (integer
// sums: exact and order-free).  For remat every nonzero exclusive
// contribution (a group's sum, a trace's carry segment) is emitted once per
// ancestor-or-self with a self flag, sorted by (trace, ancestor) and folded.
//
// Traces are processed in batches that bound the scratch; each batch appends
// to the outputs.

#include <algorithm>
#include <cstdint>

#include "psg_internal.h"

namespace psg {

namespace {

typedef unsigned long long u64;

__device__ __forceinline__ u64 ldg_u64s(const uint64_t* p) {
  return static_cast<u64>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}

__device__ __forceinline__ u64 lower_bound_s(const uint64_t* ts, u64 lo, u64 hi, u64 x) {
  while (lo < hi) {
    const u64 mid = lo + (hi - lo) / 2;
    if (ldg_u64s(ts + mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Per trace of the batch: window rows [i0, i1) (t0 <= ts < t1w) and the carry-in.
__global__ void k_sp_bounds(trace_view tr, uint32_t t_lo, uint32_t nb, u64 t0, u64 t1, uint32_t clamp,
                            uint64_t* rows, uint64_t* i0s, uint8_t* c_has, uint64_t* c_ts, uint32_t* c_ctx,
                            uint64_t* c_dur) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const uint32_t t = t_lo + i;
  const u64 b = tr.off[t], e = tr.off[t + 1];
  const u64 t1w = (clamp && tr.t_end[t] < t1) ? tr.t_end[t] : t1;
  const u64 a = lower_bound_s(tr.ts, b, e, t0);
  const u64 z = t1w > t0 ? lower_bound_s(tr.ts, a, e, t1w) : a;
  rows[i] = z - a;
  i0s[i] = a;
  const bool has = a > b;
  c_has[t] = has ? 1 : 0;
  c_ts[t] = has ? ldg_u64s(tr.ts + a - 1) : 0;
  c_ctx[t] = has ? __ldg(tr.ctx + a - 1) : 0;
  // the carry segment [t0, min(next ts, t1w)): the next event is a (or the
  // interval end when the carry is the trace's last event)
  u64 dur = 0;
  if (has) {
    const u64 nx = a < e ? min(ldg_u64s(tr.ts + a), t1w) : t1w;
    dur = nx > t0 ? nx - t0 : 0;
  }
  c_dur[i] = dur;
}

// One warp per trace: the (trace << cbits | ctx, duration) pair of each row.
__global__ void k_sp_pairs(trace_view tr, uint32_t t_lo, uint32_t nb, u64 t1, uint32_t clamp, uint32_t cbits,
                           const uint64_t* i0s, const uint64_t* row_off, uint64_t* key, uint64_t* dur) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= nb) return;
  const uint32_t t = t_lo + i;
  const u64 e = tr.off[t + 1];
  const u64 t1w = (clamp && tr.t_end[t] < t1) ? tr.t_end[t] : t1;
  const u64 a = i0s[i], o = row_off[i], n = row_off[i + 1] - o;
  for (u64 j = lane; j < n; j += 32) {
    const u64 x = a + j;
    const u64 ts = ldg_u64s(tr.ts + x);
    const u64 nx = x + 1 < e ? min(ldg_u64s(tr.ts + x + 1), t1w) : t1w;  // the last row runs to t1w
    key[o + j] = (static_cast<u64>(i) << cbits) | __ldg(tr.ctx + x);
    dur[o + j] = nx - ts;
  }
}

// flag[r] = 1 where a run of equal keys starts
__global__ void k_sp_flags(const uint64_t* key, uint64_t n, uint64_t* flag) {
  const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r < n) flag[r] = (r == 0 || key[r] != key[r - 1]) ? 1 : 0;
}

__global__ void k_sp_starts(const uint64_t* flag, const uint64_t* pos, uint64_t n, uint64_t* starts) {
  const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r < n && flag[r]) starts[pos[r]] = r;
  if (r == 0) starts[pos[n - 1] + flag[n - 1]] = n;
}

// One thread per run of the sorted window rows: the group's aggregates,
// appended at out + g.
__global__ void k_sp_groups(const uint64_t* key, const uint64_t* dur, const uint64_t* starts, uint64_t n_groups,
                            uint32_t cbits, uint32_t t_lo, uint64_t out, uint32_t* g_trace, uint32_t* g_ctx,
                            uint64_t* g_cnt, int64_t* g_sum, int64_t* g_min, int64_t* g_max, double* g_mean) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (g >= n_groups) return;
  const uint64_t a = starts[g], z = starts[g + 1];
  u64 s = 0, mn = ~0ull, mx = 0;
  for (uint64_t r = a; r < z; ++r) {
    const u64 d = dur[r];
    s += d;
    mn = min(mn, d);
    mx = max(mx, d);
  }
  const u64 k = key[a];
  g_trace[out + g] = t_lo + static_cast<uint32_t>(k >> cbits);
  g_ctx[out + g] = static_cast<uint32_t>(k & ((1ull << cbits) - 1));
  g_cnt[out + g] = z - a;
  g_sum[out + g] = static_cast<int64_t>(s);
  g_min[out + g] = static_cast<int64_t>(mn);
  g_max[out + g] = static_cast<int64_t>(mx);
  g_mean[out + g] = static_cast<double>(s) / static_cast<double>(z - a);
}

// Exclusive contributions: each group's sum (groups [0, n_groups) of this
// batch, read back from the outputs) and each trace's carry segment; one
// count per contribution = its ctx's depth + 1 (self and every ancestor).
__global__ void k_sp_contrib_count(const uint32_t* g_ctx, const int64_t* g_sum, uint64_t g0, uint64_t n_groups,
                                   const uint8_t* c_has, const uint32_t* c_ctx, const uint64_t* c_dur,
                                   uint32_t t_lo, uint32_t nb, const uint32_t* depth, uint64_t* cnt) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n_groups) {
    cnt[i] = g_sum[g0 + i] > 0 ? depth[g_ctx[g0 + i]] + 1ull : 0ull;
  } else if (i < n_groups + nb) {
    const uint32_t t = t_lo + static_cast<uint32_t>(i - n_groups);
    cnt[i] = (c_has[t] && c_dur[i - n_groups] > 0) ? depth[c_ctx[t]] + 1ull : 0ull;
  }
}

// The ancestor-or-self emissions: key = trace << cbits | ancestor, value =
// contribution << 1 | self (contributions are < 2^63: durations inside one
// trace's window).
__global__ void k_sp_contrib_emit(const uint32_t* g_trace, const uint32_t* g_ctx, const int64_t* g_sum,
                                  uint64_t g0, uint64_t n_groups, const uint8_t* c_has, const uint32_t* c_ctx,
                                  const uint64_t* c_dur, uint32_t t_lo, uint32_t nb, const uint32_t* parent,
                                  const uint64_t* off, uint32_t cbits, uint64_t* key, uint64_t* val) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_groups + nb) return;
  uint64_t o = off[i];
  const uint64_t n = off[i + 1] - o;
  if (n == 0) return;
  uint32_t tl, c;
  u64 v;
  if (i < n_groups) {
    tl = g_trace[g0 + i] - t_lo;
    c = g_ctx[g0 + i];
    v = static_cast<u64>(g_sum[g0 + i]);
  } else {
    tl = static_cast<uint32_t>(i - n_groups);
    c = c_ctx[t_lo + tl];
    v = c_dur[tl];
  }
  const u64 hi = static_cast<u64>(tl) << cbits;
  key[o] = hi | c;
  val[o] = (v << 1) | 1ull;
  for (uint32_t a = parent[c]; a != 0xFFFFFFFFu; a = parent[a]) {
    ++o;
    key[o] = hi | a;
    val[o] = v << 1;
  }
}

// One thread per run of the sorted emissions: incl = every value, excl = the self ones.
__global__ void k_sp_remat(const uint64_t* key, const uint64_t* val, const uint64_t* starts, uint64_t n_rows,
                           uint32_t cbits, uint32_t t_lo, uint64_t out, uint32_t* r_trace, uint32_t* r_ctx,
                           int64_t* r_incl, int64_t* r_excl) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (g >= n_rows) return;
  const uint64_t a = starts[g], z = starts[g + 1];
  u64 inc = 0, exc = 0;
  for (uint64_t r = a; r < z; ++r) {
    const u64 v = val[r];
    inc += v >> 1;
    if (v & 1) exc += v >> 1;
  }
  const u64 k = key[a];
  r_trace[out + g] = t_lo + static_cast<uint32_t>(k >> cbits);
  r_ctx[out + g] = static_cast<uint32_t>(k & ((1ull << cbits) - 1));
  r_incl[out + g] = static_cast<int64_t>(inc);
  r_excl[out + g] = static_cast<int64_t>(exc);
}

// Per trace, the incl of each site ctx from its remat rows (0 when absent):
// the dense [trace][site] values the outlier step reads.
__global__ void k_sp_site_values(const uint32_t* r_trace, const uint32_t* r_ctx, const int64_t* r_incl,
                                 uint64_t n_rows, const uint32_t* site, uint32_t n_sites, uint32_t n_traces,
                                 uint64_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<uint64_t>(n_traces) * n_sites) return;
  const uint32_t t = static_cast<uint32_t>(i / n_sites), s = static_cast<uint32_t>(i % n_sites);
  // lower bound of (t, site[s]) in the (trace, ctx)-sorted rows
  uint64_t lo = 0, hi = n_rows;
  const uint32_t c = site[s];
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    const bool less = r_trace[mid] < t || (r_trace[mid] == t && r_ctx[mid] < c);
    if (less)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[i] = (lo < n_rows && r_trace[lo] == t && r_ctx[lo] == c) ? static_cast<uint64_t>(r_incl[lo]) : 0ull;
}

template <typename T>
void grow_keep(dbuf<T>& b, size_t used, size_t need, cudaStream_t s) {
  if (b.n >= need && b.p) return;
  size_t cap = std::max<size_t>(need, b.n + b.n / 2 + 1024);
  T* p = nullptr;
  PSG_CUDA(cudaMalloc(&p, cap * sizeof(T)));
  if (used && b.p) PSG_CUDA(cudaMemcpyAsync(p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  b.release();
  b.p = p;
  b.n = cap;
}

unsigned blocks_for(uint64_t n, unsigned th) { return static_cast<unsigned>((n + th - 1) / th); }

// run starts of sorted keys[0, n) into starts[0 .. runs] (starts[runs] = n)
uint64_t run_starts(const uint64_t* keys, uint64_t n, dbuf<uint64_t>& flag, dbuf<uint64_t>& pos,
                    dbuf<uint64_t>& starts, dbuf<uint8_t>& scratch, cudaStream_t s) {
  if (n == 0) return 0;
  flag.ensure(n);
  pos.ensure(n);
  k_sp_flags<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, flag.p);
  const size_t sb = exclusive_sum_scratch_bytes(n);
  exclusive_sum_u64(flag.p, pos.p, n, scratch.ensure(sb), sb, s);
  uint64_t last[2];
  PSG_CUDA(cudaMemcpyAsync(&last[0], pos.p + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&last[1], flag.p + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  const uint64_t runs = last[0] + last[1];
  starts.ensure(runs + 1);
  k_sp_starts<<<blocks_for(n, 256), 256, 0, s>>>(flag.p, pos.p, n, starts.p);
  count_launch(2);
  PSG_CUDA(cudaGetLastError());
  return runs;
}

void sort_kv(dbuf<uint64_t>& k, dbuf<uint64_t>& v, dbuf<uint64_t>& k2, dbuf<uint64_t>& v2, uint64_t n,
                int end_bit, dbuf<uint8_t>& scratch, cudaStream_t s) {
  if (n == 0) return;
  k2.ensure(n);
  v2.ensure(n);
  const size_t sb = sort_pairs_scratch_bytes<uint64_t, uint64_t>(n);
  sort_pairs<uint64_t, uint64_t>(k.p, k2.p, v.p, v2.p, n, 0, end_bit, false, scratch.ensure(sb), sb, s);
  std::swap(k.p, k2.p);
  std::swap(k.n, k2.n);
  std::swap(v.p, v2.p);
  std::swap(v.n, v2.n);
}

int bits_for(uint64_t x) {  // bits to hold values < x
  int b = 1;
  while (b < 64 && (1ull << b) < x) ++b;
  return b;
}

}  // namespace

void sparse_window(const sparse_args& a, sparse_result& r, cudaStream_t s) {
  const trace_view& tr = a.tr;
  const uint32_t n = tr.n;
  const int cbits = bits_for(a.n_ctx);
  r.n_groups = r.n_remat = 0;
  dbuf<uint64_t>&rows = r.w_rows, &i0s = r.w_i0s, &roff = r.w_roff, &cdur = r.w_cdur, &key = r.w_key,
                &val = r.w_val, &key2 = r.w_key2, &val2 = r.w_val2, &flag = r.w_flag, &pos = r.w_pos,
                &starts = r.w_starts, &ccnt = r.w_ccnt, &coff = r.w_coff;
  dbuf<uint8_t>& scratch = r.w_scratch;
  rows.ensure(n + 1);
  i0s.ensure(n + 1);
  cdur.ensure(n + 1);
  std::vector<uint64_t> h_rows(n + 1, 0);
  // all traces' row counts first (one pass of binary searches), then batches
  // of whole traces whose rows fit the budget
  k_sp_bounds<<<blocks_for(n, 256), 256, 0, s>>>(tr, 0, n, a.t0, a.t1, a.clamp_tend, rows.p, i0s.p, a.c_has,
                                                 a.c_ts, a.c_ctx, cdur.p);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  if (n) PSG_CUDA(cudaMemcpyAsync(h_rows.data(), rows.p, 8ull * n, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  uint64_t total_rows = 0;
  for (uint32_t t = 0; t < n; ++t) total_rows += h_rows[t];
  r.n_rows = total_rows;
  const uint64_t budget = std::max<uint64_t>(a.row_budget, 1);
  uint32_t t_lo = 0;
  while (t_lo < n) {
    uint32_t t_hi = t_lo;
    uint64_t nr = 0;
    while (t_hi < n && (t_hi == t_lo || nr + h_rows[t_hi] <= budget)) nr += h_rows[t_hi++];
    const uint32_t nb = t_hi - t_lo;
    const int tbits = bits_for(nb);
    if (tbits + cbits > 64) fail(PS_E_INVALID_ARGUMENT, "sparse window: trace batch x ctx keys exceed 64 bits");
    // batch-local bounds and row offsets
    k_sp_bounds<<<blocks_for(nb, 256), 256, 0, s>>>(tr, t_lo, nb, a.t0, a.t1, a.clamp_tend, rows.p, i0s.p,
                                                    a.c_has, a.c_ts, a.c_ctx, cdur.p);
    std::vector<uint64_t> ho(nb + 1, 0);
    for (uint32_t i = 0; i < nb; ++i) ho[i + 1] = ho[i] + h_rows[t_lo + i];
    roff.ensure(nb + 1);
    PSG_CUDA(cudaMemcpyAsync(roff.p, ho.data(), 8ull * (nb + 1), cudaMemcpyHostToDevice, s));
    // ---- groups: (trace, ctx) runs of the window rows
    uint64_t ng = 0;
    if (nr) {
      key.ensure(nr);
      val.ensure(nr);
      k_sp_pairs<<<blocks_for(32ull * nb, 256), 256, 0, s>>>(tr, t_lo, nb, a.t1, a.clamp_tend, cbits, i0s.p,
                                                              roff.p, key.p, val.p);
      count_launch(2);
      PSG_CUDA(cudaGetLastError());
      sort_kv(key, val, key2, val2, nr, tbits + cbits, scratch, s);
      ng = run_starts(key.p, nr, flag, pos, starts, scratch, s);
      grow_keep(r.g_trace, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_ctx, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_cnt, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_sum, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_min, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_max, r.n_groups, r.n_groups + ng, s);
      grow_keep(r.g_mean, r.n_groups, r.n_groups + ng, s);
      k_sp_groups<<<blocks_for(ng, 256), 256, 0, s>>>(key.p, val.p, starts.p, ng, cbits, t_lo, r.n_groups,
                                                      r.g_trace.p, r.g_ctx.p, r.g_cnt.p, r.g_sum.p, r.g_min.p,
                                                      r.g_max.p, r.g_mean.p);
      count_launch();
      PSG_CUDA(cudaGetLastError());
    }
    // ---- remat: every nonzero exclusive contribution up its ancestor chain
    const uint64_t nc = ng + nb;
    ccnt.ensure(nc + 1);
    coff.ensure(nc + 1);
    k_sp_contrib_count<<<blocks_for(nc, 256), 256, 0, s>>>(r.g_ctx.p, r.g_sum.p, r.n_groups, ng, a.c_has, a.c_ctx,
                                                           cdur.p, t_lo, nb, a.depth, ccnt.p);
    PSG_CUDA(cudaMemsetAsync(ccnt.p + nc, 0, 8, s));
    const size_t sb = exclusive_sum_scratch_bytes(nc + 1);
    exclusive_sum_u64(ccnt.p, coff.p, nc + 1, scratch.ensure(sb), sb, s);
    uint64_t ne = 0;
    PSG_CUDA(cudaMemcpyAsync(&ne, coff.p + nc, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    count_launch();
    if (ne) {
      key.ensure(ne);
      val.ensure(ne);
      k_sp_contrib_emit<<<blocks_for(nc, 256), 256, 0, s>>>(r.g_trace.p, r.g_ctx.p, r.g_sum.p, r.n_groups, ng,
                                                           a.c_has, a.c_ctx, cdur.p, t_lo, nb, a.parent, coff.p,
                                                           cbits, key.p, val.p);
      count_launch();
      PSG_CUDA(cudaGetLastError());
      sort_kv(key, val, key2, val2, ne, tbits + cbits, scratch, s);
      const uint64_t nrm = run_starts(key.p, ne, flag, pos, starts, scratch, s);
      grow_keep(r.r_trace, r.n_remat, r.n_remat + nrm, s);
      grow_keep(r.r_ctx, r.n_remat, r.n_remat + nrm, s);
      grow_keep(r.r_incl, r.n_remat, r.n_remat + nrm, s);
      grow_keep(r.r_excl, r.n_remat, r.n_remat + nrm, s);
      k_sp_remat<<<blocks_for(nrm, 256), 256, 0, s>>>(key.p, val.p, starts.p, nrm, cbits, t_lo, r.n_remat,
                                                      r.r_trace.p, r.r_ctx.p, r.r_incl.p, r.r_excl.p);
      count_launch();
      PSG_CUDA(cudaGetLastError());
      r.n_remat += nrm;
    }
    r.n_groups += ng;
    t_lo = t_hi;
  }
  PSG_CUDA(cudaStreamSynchronize(s));
}

namespace {
// Dense [trace][ctx] results -> the same sparse rows (the copy-out of a dense
// query through the sparse accessors).
__global__ void k_dense_flags(const uint64_t* cnt, const uint64_t* incl, const uint64_t* excl, uint64_t cells,
                              uint64_t* fg, uint64_t* fr) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= cells) return;
  fg[i] = cnt[i] > 0 ? 1 : 0;
  fr[i] = (incl[i] | excl[i]) != 0 ? 1 : 0;
}

__global__ void k_dense_scatter(const uint64_t* fg, const uint64_t* pg, const uint64_t* fr, const uint64_t* pr,
                                uint64_t cells, uint32_t n_ctx, const uint64_t* cnt, const uint64_t* sum,
                                const uint64_t* mn, const uint64_t* mx, const double* mean, const uint64_t* incl,
                                const uint64_t* excl, sparse_result_view o) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= cells) return;
  const uint32_t t = static_cast<uint32_t>(i / n_ctx), c = static_cast<uint32_t>(i % n_ctx);
  if (fg[i]) {
    const uint64_t g = pg[i];
    o.g_trace[g] = t;
    o.g_ctx[g] = c;
    o.g_cnt[g] = cnt[i];
    o.g_sum[g] = static_cast<int64_t>(sum[i]);
    o.g_min[g] = static_cast<int64_t>(mn[i]);
    o.g_max[g] = static_cast<int64_t>(mx[i]);
    o.g_mean[g] = mean[i];
  }
  if (fr[i]) {
    const uint64_t r = pr[i];
    o.r_trace[r] = t;
    o.r_ctx[r] = c;
    o.r_incl[r] = static_cast<int64_t>(incl[i]);
    o.r_excl[r] = static_cast<int64_t>(excl[i]);
  }
}
}  // namespace

void dense_to_sparse(const dense_window& w, uint32_t n_traces, uint32_t n_ctx, sparse_result& r, cudaStream_t s) {
  const uint64_t cells = static_cast<uint64_t>(n_traces) * n_ctx;
  r.n_groups = r.n_remat = 0;
  if (cells == 0) return;
  // the workspace of the sparse path, reused (grow-only)
  dbuf<uint64_t>&fg = r.w_flag, &pg = r.w_pos, &fr = r.w_key, &pr = r.w_val;
  dbuf<uint8_t>& scratch = r.w_scratch;
  fg.ensure(cells + 1);
  pg.ensure(cells + 1);
  fr.ensure(cells + 1);
  pr.ensure(cells + 1);
  k_dense_flags<<<blocks_for(cells, 256), 256, 0, s>>>(w.cnt, w.incl, w.excl, cells, fg.p, fr.p);
  count_launch();
  PSG_CUDA(cudaMemsetAsync(fg.p + cells, 0, 8, s));
  PSG_CUDA(cudaMemsetAsync(fr.p + cells, 0, 8, s));
  const size_t sb = exclusive_sum_scratch_bytes(cells + 1);
  exclusive_sum_u64(fg.p, pg.p, cells + 1, scratch.ensure(sb), sb, s);
  exclusive_sum_u64(fr.p, pr.p, cells + 1, scratch.p, sb, s);
  uint64_t tot[2];
  PSG_CUDA(cudaMemcpyAsync(&tot[0], pg.p + cells, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&tot[1], pr.p + cells, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  r.n_groups = tot[0];
  r.n_remat = tot[1];
  sparse_result_view o{r.g_trace.ensure(tot[0] + 1), r.g_ctx.ensure(tot[0] + 1), r.g_cnt.ensure(tot[0] + 1),
                       r.g_sum.ensure(tot[0] + 1), r.g_min.ensure(tot[0] + 1), r.g_max.ensure(tot[0] + 1),
                       r.g_mean.ensure(tot[0] + 1), r.r_trace.ensure(tot[1] + 1), r.r_ctx.ensure(tot[1] + 1),
                       r.r_incl.ensure(tot[1] + 1), r.r_excl.ensure(tot[1] + 1)};
  k_dense_scatter<<<blocks_for(cells, 256), 256, 0, s>>>(fg.p, pg.p, fr.p, pr.p, cells, n_ctx, w.cnt, w.sum, w.mn,
                                                         w.mx, w.mean, w.incl, w.excl, o);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  PSG_CUDA(cudaStreamSynchronize(s));
}

void sparse_site_values(const sparse_result& r, const uint32_t* site, uint32_t n_sites, uint32_t n_traces,
                        uint64_t* out, cudaStream_t s) {
  const uint64_t n = static_cast<uint64_t>(n_traces) * n_sites;
  if (n == 0) return;
  k_sp_site_values<<<blocks_for(n, 256), 256, 0, s>>>(r.r_trace.p, r.r_ctx.p, r.r_incl.p, r.n_remat, site,
                                                      n_sites, n_traces, out);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
