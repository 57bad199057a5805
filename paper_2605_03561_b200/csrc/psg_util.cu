// Device buffers for host-side callers, and the small diagnostics of the
// reference's hot-path signatures that are not part of the fused query
// (SURVEY.md §8(b) "Hot-path C++ signatures"): balance_ratio / cv_percent
// (diagnostics.cpp:10-31), node_correlate's per-host sums (diagnostics.cpp:
// 378-403) and localize_outliers' rack / chassis counts (topology.cpp:54-92).
// The drop-in binding (integration/perfslice_gpu.cpp) composes them with the
// host-side string bookkeeping (hostnames, parse errors) the reference does.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "psg_internal.h"

using namespace psg;

namespace {

typedef unsigned long long u64;

template <typename Fn>
ps_status uguard(Fn&& fn) {
  try {
    fn();
    return PS_OK;
  } catch (const failure& f) {
    set_last_error(f.what());
    return f.status;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PS_E_INTERNAL;
  }
}

cudaStream_t stream_of(psg_context* c) { return static_cast<cudaStream_t>(psg_stream(c)); }

constexpr unsigned kStatThreads = 1024;

// Σx and max x of values[0, n) by one CTA: each thread folds a strided
// subsequence, then a fixed-shape tree over the threads (deterministic).
__global__ void __launch_bounds__(kStatThreads) k_sum_max(const double* __restrict__ v, uint64_t n,
                                                          double* out /*[sum, max, sumsq-dev]*/) {
  __shared__ double s_sum[kStatThreads], s_max[kStatThreads];
  double sm = 0.0, mx = n ? v[0] : 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = v[i];
    sm += x;
    mx = fmax(mx, x);
  }
  s_sum[threadIdx.x] = sm;
  s_max[threadIdx.x] = mx;
  __syncthreads();
  for (unsigned w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      s_max[threadIdx.x] = fmax(s_max[threadIdx.x], s_max[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s_sum[0];
    out[1] = s_max[0];
  }
}

// Σ (x - mean)^2 with mean = sum / n (the second pass of cv_percent).
__global__ void __launch_bounds__(kStatThreads) k_sq_dev(const double* __restrict__ v, uint64_t n,
                                                         double* out) {
  __shared__ double s[kStatThreads];
  const double mean = out[0] / static_cast<double>(n);
  double acc = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = v[i] - mean;
    acc += d * d;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (unsigned w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[2] = s[0];
}

// node_correlate: one thread per node folds its values in input order
// (member lists are CSR in input order), so each Σ equals the reference's
// sequential `slot.first += value` bit for bit.
__global__ void k_node_sums(const double* __restrict__ v, const uint32_t* __restrict__ off,
                            const uint32_t* __restrict__ members, uint32_t n_nodes, double* mean,
                            uint32_t* count) {
  const uint32_t nd = blockIdx.x * blockDim.x + threadIdx.x;
  if (nd >= n_nodes) return;
  double s = 0.0;
  const uint32_t a = off[nd], b = off[nd + 1];
  for (uint32_t i = a; i < b; ++i) s += v[members[i]];
  count[nd] = b - a;
  mean[nd] = b > a ? s / static_cast<double>(b - a) : 0.0;
}

// localize_outliers: outlier count per (rack, chassis slot).
__global__ void k_localize(const uint32_t* __restrict__ out_node, uint32_t n_out,
                           const uint32_t* __restrict__ node_cell, uint32_t* cell_cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_out) atomicAdd(cell_cnt + node_cell[out_node[i]], 1u);
}

}  // namespace

extern "C" {

ps_status psg_dev_alloc(psg_context* c, uint64_t bytes, void** out) {
  if (!c || !out) return PS_E_INVALID_ARGUMENT;
  return uguard([&] {
    *out = nullptr;
    PSG_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  });
}

void psg_dev_free(psg_context* c, void* p) {
  if (c && p) {
    cudaStreamSynchronize(stream_of(c));
    cudaFree(p);
  }
}

ps_status psg_copy(psg_context* c, void* dst, const void* src, uint64_t bytes) {
  if (!c || (bytes && (!dst || !src))) return PS_E_INVALID_ARGUMENT;
  return uguard([&] {
    if (!bytes) return;
    PSG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream_of(c)));
    PSG_CUDA(cudaStreamSynchronize(stream_of(c)));
  });
}

ps_status psg_vector_stats(psg_context* c, const double* values, uint64_t n, uint32_t what,
                           double* result) {
  if (!c || !result || (n && !values) || what > 1) return PS_E_INVALID_ARGUMENT;
  return uguard([&] {
    if (n == 0)  // empty_input (diagnostics.cpp:11, 22)
      fail(PS_E_INVALID_ARGUMENT, what == 0 ? "balance_ratio of empty vector" : "cv of empty vector");
    cudaStream_t s = stream_of(c);
    double* d = nullptr;
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 3 * sizeof(double), s));
    const double* v = values;
    double* staged = nullptr;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, values) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&staged), 8 * n, s));
      PSG_CUDA(cudaMemcpyAsync(staged, values, 8 * n, cudaMemcpyHostToDevice, s));
      v = staged;
    }
    k_sum_max<<<1, kStatThreads, 0, s>>>(v, n, d);
    count_launch();
    if (what == 1) {
      k_sq_dev<<<1, kStatThreads, 0, s>>>(v, n, d);
      count_launch();
    }
    PSG_CUDA(cudaGetLastError());
    double h[3] = {0, 0, 0};
    PSG_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaFreeAsync(d, s));
    if (staged) PSG_CUDA(cudaFreeAsync(staged, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    const double nd = static_cast<double>(n);
    if (what == 0) {
      *result = h[1] == 0.0 ? 1.0 : h[0] / nd / h[1];
    } else {
      const double mean = h[0] / nd;
      if (mean == 0.0) fail(PS_E_INSUFFICIENT_DATA, "cv undefined for zero mean");  // undefined_cv
      *result = 100.0 * std::sqrt(h[2] / nd) / mean;
    }
  });
}

ps_status psg_node_means(psg_context* c, const double* values, const uint32_t* node_of, uint64_t n,
                         uint32_t n_nodes, double* mean, uint32_t* count) {
  if (!c || (n && (!values || !node_of)) || (n_nodes && (!mean || !count))) return PS_E_INVALID_ARGUMENT;
  return uguard([&] {
    std::vector<uint32_t> off(n_nodes + 1, 0), members(n);
    for (uint64_t i = 0; i < n; ++i) {
      if (node_of[i] >= n_nodes) fail(PS_E_INVALID_ARGUMENT, "node index out of range");
      ++off[node_of[i] + 1];
    }
    for (uint32_t i = 0; i < n_nodes; ++i) off[i + 1] += off[i];
    std::vector<uint32_t> fill(off.begin(), off.end() - 1);
    for (uint64_t i = 0; i < n; ++i) members[fill[node_of[i]]++] = static_cast<uint32_t>(i);
    cudaStream_t s = stream_of(c);
    double *dv = nullptr, *dm = nullptr;
    uint32_t *doff = nullptr, *dmem = nullptr, *dc = nullptr;
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dv), 8 * n + 8, s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dm), 8ull * n_nodes + 8, s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&doff), 4ull * (n_nodes + 1), s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dmem), 4 * n + 4, s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dc), 4ull * n_nodes + 4, s));
    if (n) {
      PSG_CUDA(cudaMemcpyAsync(dv, values, 8 * n, cudaMemcpyDefault, s));
      PSG_CUDA(cudaMemcpyAsync(dmem, members.data(), 4 * n, cudaMemcpyHostToDevice, s));
    }
    PSG_CUDA(cudaMemcpyAsync(doff, off.data(), 4ull * (n_nodes + 1), cudaMemcpyHostToDevice, s));
    if (n_nodes) {
      k_node_sums<<<(n_nodes + 127) / 128, 128, 0, s>>>(dv, doff, dmem, n_nodes, dm, dc);
      count_launch();
      PSG_CUDA(cudaGetLastError());
      PSG_CUDA(cudaMemcpyAsync(mean, dm, 8ull * n_nodes, cudaMemcpyDeviceToHost, s));
      PSG_CUDA(cudaMemcpyAsync(count, dc, 4ull * n_nodes, cudaMemcpyDeviceToHost, s));
    }
    for (void* p : {static_cast<void*>(dv), static_cast<void*>(dm), static_cast<void*>(doff),
                    static_cast<void*>(dmem), static_cast<void*>(dc)})
      PSG_CUDA(cudaFreeAsync(p, s));
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_localize(psg_context* c, const uint32_t* node_rack, const uint32_t* node_chassis,
                       uint32_t n_nodes, uint32_t n_universe, const uint32_t* outliers, uint32_t n_out,
                       uint32_t* n_rows, uint32_t* rows) {
  if (!c || !n_rows || (n_nodes && (!node_rack || !node_chassis)) || (n_out && !outliers) ||
      n_universe > n_nodes)
    return PS_E_INVALID_ARGUMENT;
  return uguard([&] {
    // (rack, chassis) cells of the universe, ascending; node -> cell
    std::vector<std::pair<uint32_t, uint32_t>> cells(n_nodes);
    for (uint32_t i = 0; i < n_nodes; ++i) cells[i] = {node_rack[i], node_chassis[i]};
    std::vector<std::pair<uint32_t, uint32_t>> uniq = cells;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    std::vector<uint32_t> node_cell(n_nodes), uni_cnt(uniq.size(), 0);
    for (uint32_t i = 0; i < n_nodes; ++i) {
      node_cell[i] = static_cast<uint32_t>(std::lower_bound(uniq.begin(), uniq.end(), cells[i]) - uniq.begin());
      if (i < n_universe) ++uni_cnt[node_cell[i]];
    }
    for (uint32_t i = 0; i < n_out; ++i)
      if (outliers[i] >= n_nodes) fail(PS_E_INVALID_ARGUMENT, "outlier node index out of range");
    cudaStream_t s = stream_of(c);
    uint32_t *dcell = nullptr, *dout = nullptr, *dcnt = nullptr;
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dcell), 4ull * n_nodes + 4, s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), 4ull * n_out + 4, s));
    PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dcnt), 4ull * uniq.size() + 4, s));
    PSG_CUDA(cudaMemsetAsync(dcnt, 0, 4ull * uniq.size() + 4, s));
    if (n_nodes) PSG_CUDA(cudaMemcpyAsync(dcell, node_cell.data(), 4ull * n_nodes, cudaMemcpyHostToDevice, s));
    if (n_out) PSG_CUDA(cudaMemcpyAsync(dout, outliers, 4ull * n_out, cudaMemcpyHostToDevice, s));
    if (n_out) {
      k_localize<<<(n_out + 255) / 256, 256, 0, s>>>(dout, n_out, dcell, dcnt);
      count_launch();
      PSG_CUDA(cudaGetLastError());
    }
    std::vector<uint32_t> cnt(uniq.size());
    if (!uniq.empty()) PSG_CUDA(cudaMemcpyAsync(cnt.data(), dcnt, 4ull * uniq.size(), cudaMemcpyDeviceToHost, s));
    for (void* p : {static_cast<void*>(dcell), static_cast<void*>(dout), static_cast<void*>(dcnt)})
      PSG_CUDA(cudaFreeAsync(p, s));
    PSG_CUDA(cudaStreamSynchronize(s));
    uint32_t j = 0;
    for (size_t k = 0; k < uniq.size(); ++k) {
      if (!cnt[k]) continue;
      if (rows) {
        rows[4ull * j] = uniq[k].first;
        rows[4ull * j + 1] = uniq[k].second;
        rows[4ull * j + 2] = cnt[k];
        rows[4ull * j + 3] = cnt[k] == uni_cnt[k] ? 1u : 0u;
      }
      ++j;
    }
    *n_rows = j;
  });
}

}  // extern "C"
