// Profile-record path on sm_100a: profile.db bodies
// in HBM, the Query API's slice read (ingest::read_slices / ingest_profiles,
// ingest.cpp:122-176; store.cpp:582-631) and congestion_report's numeric core
// over profile records (workflows.cpp:42-62, 413-539; diagnostics.cpp:10-19,
// 378-403).
//
//   KP1 k_records_to_soa   packed 14-byte records {u32 ctx, u16 metric, f64}
//                          -> SoA ctx / metric / value (2-byte aligned loads)
//   KP2 k_slice            one warp per requested profile: ctx and metric
//                          filters as bit sets, ballot + popc placement; a
//                          counting pass, a scan, a writing pass (record order
//                          within a profile = the reference's per-ctx runs,
//                          because records are sorted by ctx)
//   KP3 k_site_values      rank_vector: per (rank profile, site) the record of
//                          (site ctx, metric) by binary search in the
//                          profile's ctx-sorted run, 0 when absent
//   KP4 k_site_ratio       balance_ratio per site: (Σ/n)/max (1 when max == 0)
//   KP5 k_node_mean        node_correlate: per node, the values of its ranks
//                          summed in rank order, / count
// The z-score / top-k selection and the topology are the trace path's kernels
// (psg_kernels.cu K7/K8) fed with these node means.

#include <cstdint>

#include "psg_internal.h"

namespace psg {

namespace {
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
}  // namespace

__global__ void k_records_to_soa(const uint16_t* body, uint64_t n, uint32_t* ctx, uint16_t* metric,
                                 double* value) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint16_t* r = body + 7 * i;  // 14 bytes = 7 halfwords, little endian
  ctx[i] = static_cast<uint32_t>(r[0]) | (static_cast<uint32_t>(r[1]) << 16);
  metric[i] = r[2];
  const unsigned long long v = static_cast<unsigned long long>(r[3]) |
                               (static_cast<unsigned long long>(r[4]) << 16) |
                               (static_cast<unsigned long long>(r[5]) << 32) |
                               (static_cast<unsigned long long>(r[6]) << 48);
  value[i] = __longlong_as_double(static_cast<long long>(v));
}

void launch_records_to_soa(const uint8_t* body, uint64_t n, uint32_t* ctx, uint16_t* metric,
                           double* value, cudaStream_t s) {
  if (n == 0) return;
  k_records_to_soa<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const uint16_t*>(body), n, ctx, metric, value);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// Records of a profile must be sorted by ctx (the reference binary-searches
// them, store.cpp:601-613): count the violations.
__global__ void k_records_check(const uint32_t* ctx, const uint64_t* off, uint32_t n_prof,
                                unsigned long long* bad) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n_prof) return;
  unsigned long long nb = 0;
  for (uint64_t i = off[p] + 1 + lane; i < off[p + 1]; i += 32) nb += ctx[i] < ctx[i - 1];
  for (int d = 16; d > 0; d >>= 1) nb += __shfl_xor_sync(FULL, nb, d);
  if (lane == 0 && nb) atomicAdd(bad, nb);
}

void launch_records_check(const uint32_t* ctx, const uint64_t* off, uint32_t n_prof,
                          unsigned long long* bad, cudaStream_t s) {
  if (n_prof == 0) return;
  k_records_check<<<(n_prof + 7) / 8, 256, 0, s>>>(ctx, off, n_prof, bad);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// KP2: WRITE = false counts the rows of each requested profile; WRITE = true
// writes them at row_off[i].  ctx_bits == nullptr: all contexts; metric_bits
// == nullptr: all metrics.
template <bool WRITE>
__global__ void k_slice(const profile_view pv, const uint32_t* slot, uint32_t n_req,
                        const uint32_t* ctx_bits, uint32_t ctx_words, const uint32_t* metric_bits,
                        unsigned long long* counts, const unsigned long long* row_off,
                        uint32_t* out_pid, uint32_t* out_ctx, uint16_t* out_metric, double* out_value) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_req) return;
  const uint32_t p = slot[i];
  const uint64_t b = pv.off[p], e = pv.off[p + 1];
  unsigned long long pos = WRITE ? row_off[i] : 0;
  for (uint64_t base = b; base < e; base += 32) {
    const uint64_t r = base + lane;
    bool keep = false;
    uint32_t c = 0;
    uint16_t m = 0;
    if (r < e) {
      c = pv.ctx[r];
      m = pv.metric[r];
      keep = (!ctx_bits || ((c >> 5) < ctx_words && ((ctx_bits[c >> 5] >> (c & 31)) & 1u))) &&
             (!metric_bits || ((metric_bits[m >> 5] >> (m & 31)) & 1u));
    }
    const uint32_t bal = __ballot_sync(FULL, keep);
    if (WRITE && keep) {
      const unsigned long long o = pos + __popc(bal & lanemask_lt());
      out_pid[o] = pv.pid[p];
      out_ctx[o] = c;
      out_metric[o] = m;
      out_value[o] = pv.value[r];
    }
    pos += __popc(bal);
  }
  if (!WRITE && lane == 0) counts[i] = pos;
}

void launch_slice(const profile_view& pv, const uint32_t* slot, uint32_t n_req,
                  const uint32_t* ctx_bits, uint32_t ctx_words, const uint32_t* metric_bits,
                  unsigned long long* counts, const unsigned long long* row_off, uint32_t* out_pid,
                  uint32_t* out_ctx, uint16_t* out_metric, double* out_value, cudaStream_t s) {
  if (n_req == 0) return;
  const unsigned g = (n_req + 7) / 8;
  if (row_off)
    k_slice<true><<<g, 256, 0, s>>>(pv, slot, n_req, ctx_bits, ctx_words, metric_bits, counts,
                                    row_off, out_pid, out_ctx, out_metric, out_value);
  else
    k_slice<false><<<g, 256, 0, s>>>(pv, slot, n_req, ctx_bits, ctx_words, metric_bits, counts,
                                     nullptr, nullptr, nullptr, nullptr, nullptr);
  count_launch();
  PSG_CUDA(cudaGetLastError());
}

// KP3: vals[r][s] for the rank profiles (rank_slot[r] = profile slot).
__global__ void k_site_values(const profile_view pv, const uint32_t* rank_slot, uint32_t n_ranks,
                              const uint32_t* site, uint32_t n_sites, uint16_t metric,
                              double* vals) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<uint64_t>(n_ranks) * n_sites) return;
  const uint32_t r = static_cast<uint32_t>(t / n_sites), s = static_cast<uint32_t>(t % n_sites);
  const uint32_t p = rank_slot[r], c = site[s];
  uint64_t lo = pv.off[p], hi = pv.off[p + 1];
  while (lo < hi) {  // lower_bound on ctx (store.cpp:601-613)
    const uint64_t mid = lo + (hi - lo) / 2;
    if (pv.ctx[mid] < c) lo = mid + 1; else hi = mid;
  }
  double v = 0.0;  // sparse zeros filled in (workflows.cpp:50-53)
  for (uint64_t i = lo; i < pv.off[p + 1] && pv.ctx[i] == c; ++i)
    if (pv.metric[i] == metric) v = pv.value[i];  // the last row wins (by_profile map)
  vals[t] = v;
}

// KP4: one block per site; ratio = (Σ/n)/max, 1 when max == 0 (diagnostics.cpp:10-19).
__global__ void __launch_bounds__(256) k_site_ratio(const double* vals, uint32_t n_ranks,
                                                    uint32_t n_sites, double* ratio) {
  const uint32_t s = blockIdx.x;
  double sum = 0.0, mx = 0.0;
  bool have = false;
  for (uint32_t r = threadIdx.x; r < n_ranks; r += blockDim.x) {
    const double v = vals[static_cast<size_t>(r) * n_sites + s];
    sum += v;
    mx = have ? fmax(mx, v) : v;
    have = true;
  }
  __shared__ double s_warp[32];
  const double s_sum = block_reduce(sum, op_add(), s_warp);
  // max over the ranks (ranks beyond n_ranks contribute nothing)
  const double m = block_reduce(have ? mx : -1.0e308, op_max(), s_warp);
  if (threadIdx.x == 0)
    ratio[s] = (n_ranks == 0 || m == 0.0) ? 1.0 : s_sum / static_cast<double>(n_ranks) / m;
}

__global__ void k_site_worst(const double* ratio, uint32_t n_sites, uint32_t* worst) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t w = 0;
  for (uint32_t s = 1; s < n_sites; ++s)
    if (ratio[s] < ratio[w]) w = s;  // the first minimal site (workflows.cpp:459-461)
  *worst = w;
}

// KP5: node means of the worst site's values; members of node i are
// node_rank[node_off[i] .. node_off[i+1]) in rank order.
__global__ void k_node_mean(const double* vals, uint32_t n_sites, const uint32_t* worst,
                            const uint32_t* node_off, const uint32_t* node_rank, uint32_t n_nodes,
                            double* mean) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  const uint32_t w = *worst;
  double sum = 0.0;
  for (uint32_t k = node_off[i]; k < node_off[i + 1]; ++k)
    sum += vals[static_cast<size_t>(node_rank[k]) * n_sites + w];
  const uint32_t cnt = node_off[i + 1] - node_off[i];
  mean[i] = cnt ? sum / static_cast<double>(cnt) : 0.0;
}

void launch_profile_outliers(const profile_view& pv, const uint32_t* rank_slot, uint32_t n_ranks,
                             const uint32_t* site, uint32_t n_sites, uint16_t metric, double* vals,
                             double* ratio, uint32_t* worst, const uint32_t* node_off,
                             const uint32_t* node_rank, uint32_t n_nodes, double* node_mean,
                             cudaStream_t s) {
  const uint64_t cells = static_cast<uint64_t>(n_ranks) * n_sites;
  if (cells) {
    k_site_values<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, s>>>(
        pv, rank_slot, n_ranks, site, n_sites, metric, vals);
    count_launch();
  }
  k_site_ratio<<<n_sites, 256, 0, s>>>(vals, n_ranks, n_sites, ratio);
  k_site_worst<<<1, 32, 0, s>>>(ratio, n_sites, worst);
  k_node_mean<<<(n_nodes + 255) / 256, 256, 0, s>>>(vals, n_sites, worst, node_off, node_rank,
                                                   n_nodes, node_mean);
  count_launch(3);
  PSG_CUDA(cudaGetLastError());
}

}  // namespace psg
