// GPU frame operators: the reference's columnar
// engine (frame.hpp / frame.cpp) for numeric columns, with its determinism
// contract kept bit for bit:
//   * sort / group keys: a stable multi-key argsort (original row index breaks
//     ties, frame.cpp:62-69) built from LSD passes of a stable radix sort over
//     order-preserving 64-bit keys (f64: NaN above every number and equal to
//     itself, -0 == +0, frame.cpp:19-25; descending keys inverted);
//   * group sums / min / max fold from the run's first row in ascending
//     original row index; mean = (0 + Σ cells as double) / n (frame.cpp:290-392);
//   * filter and merge keep the reference's output order (frame.cpp:424-572);
//   * reduce_sum / cumulative_sum fold left inside 4096-element blocks, then
//     fold the block sums left (frame.cpp:599-647): reduce_sum equals the last
//     element of cumulative_sum bit for bit.
// All column pointers are device pointers; results stay on the device.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "psg_internal.h"

using namespace psg;

namespace {

typedef unsigned long long u64;
constexpr uint64_t kBlock = 4096;  // frame::k_reduce_block

template <typename Fn>
ps_status fguard(Fn&& fn) {
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

// Stream-ordered scratch; the pool keeps its memory between operators.
struct scratch {
  cudaStream_t s;
  std::vector<void*> held;
  explicit scratch(cudaStream_t st) : s(st) {
    static bool once = false;
    if (!once) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      once = true;
    }
  }
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    PSG_CUDA(cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), s));
    held.push_back(p);
    return static_cast<T*>(p);
  }
  ~scratch() {
    for (void* p : held) cudaFreeAsync(p, s);
  }
};

// ---- order-preserving keys ----------------------------------------------------
__device__ __forceinline__ u64 key_of(const void* col, uint32_t dt, uint64_t i) {
  if (dt == PSG_I64) return static_cast<u64>(static_cast<const int64_t*>(col)[i]) ^ (1ull << 63);
  if (dt == PSG_U64) return static_cast<const uint64_t*>(col)[i];
  double v = static_cast<const double*>(col)[i];
  if (v != v) return ~0ull;  // every NaN: one key above all numbers
  if (v == 0.0) v = 0.0;     // -0 == +0
  const u64 b = static_cast<u64>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

__global__ void k_iota(uint64_t* p, uint64_t n) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = i;
}

// keys[i] = key of row perm[i] (inverted for a descending key)
__global__ void k_gather_key(const void* col, uint32_t dt, bool desc, const uint64_t* perm, uint64_t n,
                             u64* keys) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const u64 k = key_of(col, dt, perm[i]);
  keys[i] = desc ? ~k : k;
}

unsigned blocks(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

void check_dtype(uint32_t dt) {
  if (dt > PSG_F64) fail(PS_E_INVALID_ARGUMENT, "unsupported column dtype (i64, u64, f64 only)");
}

// Stable argsort over keys[0] (most significant) .. keys[k-1]: LSD radix passes.
void argsort(const psg_col* keys, uint32_t n_keys, const uint8_t* ascending, uint64_t n, uint64_t* perm,
             cudaStream_t s, scratch& sc) {
  if (n == 0) return;
  k_iota<<<blocks(n), 256, 0, s>>>(perm, n);
  count_launch();
  if (n_keys == 0) return;
  u64* kin = sc.get<u64>(n);
  u64* kout = sc.get<u64>(n);
  uint64_t* pout = sc.get<uint64_t>(n);
  const size_t tb = sort_pairs_scratch_bytes<uint64_t, uint64_t>(n);
  void* tmp = sc.get<uint8_t>(tb);
  for (uint32_t k = n_keys; k-- > 0;) {
    check_dtype(keys[k].dtype);
    k_gather_key<<<blocks(n), 256, 0, s>>>(keys[k].data, keys[k].dtype, ascending && !ascending[k], perm, n, kin);
    count_launch();
    sort_pairs<uint64_t, uint64_t>(reinterpret_cast<const uint64_t*>(kin), reinterpret_cast<uint64_t*>(kout),
                                   perm, pout, n, 0, 64, false, tmp, tb, s);
    PSG_CUDA(cudaMemcpyAsync(perm, pout, 8 * n, cudaMemcpyDeviceToDevice, s));
  }
  PSG_CUDA(cudaGetLastError());
}

// flag[i] = row perm[i] starts a new key tuple
__global__ void k_run_flags(const psg_col* keys, uint32_t n_keys, const uint64_t* perm, uint64_t n,
                            uint64_t* flag) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  bool nw = i == 0;
  for (uint32_t k = 0; k < n_keys && !nw; ++k)
    nw = key_of(keys[k].data, keys[k].dtype, perm[i - 1]) != key_of(keys[k].data, keys[k].dtype, perm[i]);
  flag[i] = nw ? 1 : 0;
}

__global__ void k_scatter_starts(const uint64_t* flag, const uint64_t* pos, uint64_t n, uint64_t* starts) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && flag[i]) starts[pos[i]] = i;
}

// exclusive scan of n u64 flags into pos; returns the total
uint64_t scan_count(const uint64_t* flag, uint64_t n, uint64_t* pos, cudaStream_t s, scratch& sc) {
  const size_t tb = exclusive_sum_scratch_bytes(n);
  exclusive_sum_u64(flag, pos, n, sc.get<uint8_t>(tb), tb, s);
  uint64_t last_pos = 0, last_flag = 0;
  PSG_CUDA(cudaMemcpyAsync(&last_pos, pos + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&last_flag, flag + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return last_pos + last_flag;
}

// ---- group aggregates -------------------------------------------------------------
template <typename T>
__global__ void k_group_fold(const T* src, const uint64_t* perm, const uint64_t* starts, uint64_t n_groups,
                             uint64_t n, uint32_t fn, T* out) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (g >= n_groups) return;
  const uint64_t lo = starts[g], hi = g + 1 < n_groups ? starts[g + 1] : n;
  T acc = src[perm[lo]];
  for (uint64_t i = lo + 1; i < hi; ++i) {
    const T x = src[perm[i]];
    if (fn == PSG_AGG_SUM)
      acc = static_cast<T>(acc + x);  // integers wrap (frame.cpp:346-348)
    else if (fn == PSG_AGG_MIN)
      acc = x < acc ? x : acc;  // std::min
    else
      acc = acc < x ? x : acc;  // std::max
  }
  out[g] = acc;
}

__global__ void k_group_mean(const void* src, uint32_t dt, const uint64_t* perm, const uint64_t* starts,
                             uint64_t n_groups, uint64_t n, double* out) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (g >= n_groups) return;
  const uint64_t lo = starts[g], hi = g + 1 < n_groups ? starts[g + 1] : n;
  double acc = 0.0;
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t r = perm[i];
    acc += dt == PSG_I64 ? static_cast<double>(static_cast<const int64_t*>(src)[r])
         : dt == PSG_U64 ? static_cast<double>(static_cast<const uint64_t*>(src)[r])
                         : static_cast<const double*>(src)[r];
  }
  out[g] = acc / static_cast<double>(hi - lo);
}

__global__ void k_group_count(const uint64_t* starts, uint64_t n_groups, uint64_t n, uint64_t* out) {
  const uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (g < n_groups) out[g] = (g + 1 < n_groups ? starts[g + 1] : n) - starts[g];
}

__global__ void k_has_nan(const double* v, uint64_t n, unsigned long long* flag) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && v[i] != v[i]) *flag = 1;
}

// ---- gather / filter ------------------------------------------------------------
__global__ void k_gather8(const uint64_t* src, const uint64_t* idx, uint64_t n, uint64_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = src[idx[i]];
}

__device__ __forceinline__ int cmp_cell(const void* col, uint32_t dt, uint64_t i, const void* lit) {
  if (dt == PSG_I64) {
    const int64_t a = static_cast<const int64_t*>(col)[i], b = *static_cast<const int64_t*>(lit);
    return a < b ? -1 : (b < a ? 1 : 0);
  }
  if (dt == PSG_U64) {
    const uint64_t a = static_cast<const uint64_t*>(col)[i], b = *static_cast<const uint64_t*>(lit);
    return a < b ? -1 : (b < a ? 1 : 0);
  }
  const double a = static_cast<const double*>(col)[i], b = *static_cast<const double*>(lit);
  const bool na = a != a, nb = b != b;  // cmp_f64 (frame.cpp:19-25)
  if (na || nb) return na == nb ? 0 : (na ? 1 : -1);
  return a < b ? -1 : (a > b ? 1 : 0);
}

__device__ __forceinline__ bool holds(int c, uint32_t op) {
  switch (op) {
    case PSG_LT: return c < 0;
    case PSG_LE: return c <= 0;
    case PSG_EQ: return c == 0;
    case PSG_GE: return c >= 0;
    case PSG_GT: return c > 0;
    default: return c != 0;
  }
}

__global__ void k_filter_flags(const void* col, uint32_t dt, uint32_t op, const void* lit, uint64_t n,
                               uint64_t* flag) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) flag[i] = holds(cmp_cell(col, dt, i, lit), op) ? 1 : 0;
}

__global__ void k_scatter_idx(const uint64_t* flag, const uint64_t* pos, uint64_t n, uint64_t* idx) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && flag[i]) idx[pos[i]] = i;
}

// ---- merge (inner join) ----------------------------------------------------------
struct key_tuple {
  const psg_col* keys;
  uint32_t n;
};

__device__ __forceinline__ int cmp_rows(const psg_col* lk, uint64_t li, const psg_col* rk, uint64_t ri,
                                        uint32_t n) {
  for (uint32_t k = 0; k < n; ++k) {
    const u64 a = key_of(lk[k].data, lk[k].dtype, li), b = key_of(rk[k].data, rk[k].dtype, ri);
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

// per left row: the matching right run (frame.cpp:503-520) -> its length
__global__ void k_merge_count(const psg_col* lk, const psg_col* rk, uint32_t nk, uint64_t nl,
                              const uint64_t* rperm, const uint64_t* rstarts, uint64_t n_runs, uint64_t nr,
                              uint64_t* run_of, uint64_t* cnt) {
  const uint64_t li = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (li >= nl) return;
  uint64_t lo = 0, hi = n_runs;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (cmp_rows(lk, li, rk, rperm[rstarts[mid]], nk) > 0) lo = mid + 1; else hi = mid;
  }
  uint64_t c = 0;
  if (lo < n_runs && cmp_rows(lk, li, rk, rperm[rstarts[lo]], nk) == 0)
    c = (lo + 1 < n_runs ? rstarts[lo + 1] : nr) - rstarts[lo];
  run_of[li] = lo;
  cnt[li] = c;
}

__global__ void k_merge_emit(const uint64_t* run_of, const uint64_t* cnt, const uint64_t* pos, uint64_t nl,
                             const uint64_t* rperm, const uint64_t* rstarts, uint64_t* lidx, uint64_t* ridx) {
  const uint64_t li = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (li >= nl || cnt[li] == 0) return;
  const uint64_t r0 = rstarts[run_of[li]];
  for (uint64_t j = 0; j < cnt[li]; ++j) {
    lidx[pos[li] + j] = li;
    ridx[pos[li] + j] = rperm[r0 + j];
  }
}

// ---- vector ops ------------------------------------------------------------------
__global__ void k_vadd(const double* a, const double* b, uint64_t n, double* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = a[i] + b[i];
}
__global__ void k_vmul(const double* a, double s, uint64_t n, double* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = a[i] * s;
}
__global__ void k_scmp(const double* a, uint32_t op, double s, uint64_t n, int64_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = holds(cmp_cell(a, PSG_F64, i, &s), op) ? 1 : 0;
}

// Block sums: one thread folds one 4096-element block left to right (the
// reference's association); the block is staged through shared memory by the
// CTA's warp with coalesced loads first.
__global__ void __launch_bounds__(32) k_block_sums(const double* v, uint64_t n, double* sums) {
  __shared__ double buf[kBlock];
  const uint64_t lo = blockIdx.x * kBlock, hi = min(lo + kBlock, n);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += 32) buf[i - lo] = v[i];
  __syncwarp();
  if (threadIdx.x == 0) {
    double acc = buf[0];
    for (uint64_t i = 1; i < hi - lo; ++i) acc += buf[i];
    sums[blockIdx.x] = acc;
  }
}

// carry[b] = fold of sums[0..b) (the reference's carry chain, frame.cpp:628-630)
__global__ void k_carry(const double* sums, uint64_t nb, double* carry, double* total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (uint64_t b = 0; b < nb; ++b) {
    carry[b] = acc;  // carry[0] unused
    acc = b == 0 ? sums[0] : acc + sums[b];
  }
  *total = acc;
}

__global__ void __launch_bounds__(32) k_block_scan(const double* v, uint64_t n, const double* carry, double* out) {
  __shared__ double buf[kBlock];
  const uint64_t lo = blockIdx.x * kBlock, hi = min(lo + kBlock, n);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += 32) buf[i - lo] = v[i];
  __syncwarp();
  if (threadIdx.x == 0) {
    const double c = carry[blockIdx.x];
    double running = buf[0];
    buf[0] = blockIdx.x == 0 ? running : c + running;
    for (uint64_t i = 1; i < hi - lo; ++i) {
      running += buf[i];
      buf[i] = blockIdx.x == 0 ? running : c + running;
    }
  }
  __syncwarp();
  for (uint64_t i = lo + threadIdx.x; i < hi; i += 32) out[i] = buf[i - lo];
}

psg_col* upload_cols(const psg_col* cols, uint32_t n, cudaStream_t s, scratch& sc) {
  psg_col* d = sc.get<psg_col>(n);
  if (n) PSG_CUDA(cudaMemcpyAsync(d, cols, sizeof(psg_col) * n, cudaMemcpyHostToDevice, s));
  return d;
}

}  // namespace

extern "C" {

ps_status psg_frame_argsort(psg_context* c, const psg_col* keys, uint32_t n_keys, const uint8_t* ascending,
                            uint64_t n, uint64_t* perm) {
  if (!c || (n_keys && !keys) || (n && !perm)) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    argsort(keys, n_keys, ascending, n, perm, s, sc);
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_group(psg_context* c, const psg_col* keys, uint32_t n_keys, uint64_t n, uint64_t* perm,
                          uint64_t* starts, uint64_t* n_groups) {
  if (!c || !keys || n_keys == 0 || !n_groups || (n && (!perm || !starts))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    *n_groups = 0;
    if (n == 0) return;
    argsort(keys, n_keys, nullptr, n, perm, s, sc);
    psg_col* dk = upload_cols(keys, n_keys, s, sc);
    uint64_t* flag = sc.get<uint64_t>(n);
    uint64_t* pos = sc.get<uint64_t>(n);
    k_run_flags<<<blocks(n), 256, 0, s>>>(dk, n_keys, perm, n, flag);
    const uint64_t g = scan_count(flag, n, pos, s, sc);
    k_scatter_starts<<<blocks(n), 256, 0, s>>>(flag, pos, n, starts);
    count_launch(2);
    PSG_CUDA(cudaStreamSynchronize(s));
    *n_groups = g;
  });
}

ps_status psg_frame_group_agg(psg_context* c, psg_col src, const uint64_t* perm, const uint64_t* starts,
                              uint64_t n_groups, uint64_t n, uint32_t fn, void* out) {
  if (!c || (n_groups && (!perm || !starts || !out))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    check_dtype(src.dtype);
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    if (src.dtype == PSG_F64 && n) {  // require_numeric: NaN in an aggregate column (frame.cpp:150-156)
      unsigned long long* f = sc.get<unsigned long long>(1);
      PSG_CUDA(cudaMemsetAsync(f, 0, 8, s));
      k_has_nan<<<blocks(n), 256, 0, s>>>(static_cast<const double*>(src.data), n, f);
      count_launch();
      unsigned long long hf = 0;
      PSG_CUDA(cudaMemcpyAsync(&hf, f, 8, cudaMemcpyDeviceToHost, s));
      PSG_CUDA(cudaStreamSynchronize(s));
      if (hf) fail(PS_E_INVALID_ARGUMENT, "NaN in aggregate column");
    }
    if (n_groups == 0) return;
    const unsigned g = blocks(n_groups, 128);
    if (fn == PSG_AGG_COUNT) {
      k_group_count<<<g, 128, 0, s>>>(starts, n_groups, n, static_cast<uint64_t*>(out));
    } else if (fn == PSG_AGG_MEAN) {
      k_group_mean<<<g, 128, 0, s>>>(src.data, src.dtype, perm, starts, n_groups, n, static_cast<double*>(out));
    } else if (fn <= PSG_AGG_MAX) {
      if (src.dtype == PSG_I64)
        k_group_fold<int64_t><<<g, 128, 0, s>>>(static_cast<const int64_t*>(src.data), perm, starts, n_groups, n,
                                                fn, static_cast<int64_t*>(out));
      else if (src.dtype == PSG_U64)
        k_group_fold<uint64_t><<<g, 128, 0, s>>>(static_cast<const uint64_t*>(src.data), perm, starts, n_groups,
                                                 n, fn, static_cast<uint64_t*>(out));
      else
        k_group_fold<double><<<g, 128, 0, s>>>(static_cast<const double*>(src.data), perm, starts, n_groups, n, fn,
                                               static_cast<double*>(out));
    } else {
      fail(PS_E_INVALID_ARGUMENT, "unknown aggregate function");
    }
    count_launch();
    PSG_CUDA(cudaGetLastError());
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_gather(psg_context* c, psg_col src, const uint64_t* idx, uint64_t n_idx, void* out) {
  if (!c || (n_idx && (!idx || !out || !src.data))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    check_dtype(src.dtype);
    cudaStream_t s = stream_of(c);
    if (n_idx) {
      k_gather8<<<blocks(n_idx), 256, 0, s>>>(static_cast<const uint64_t*>(src.data), idx, n_idx,
                                              static_cast<uint64_t*>(out));
      count_launch();
    }
    PSG_CUDA(cudaGetLastError());
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_filter(psg_context* c, psg_col col, uint32_t op, const void* literal, uint64_t n,
                           uint64_t* idx, uint64_t* n_out) {
  if (!c || !literal || !n_out || (n && (!idx || !col.data))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    check_dtype(col.dtype);
    if (op > PSG_NE) fail(PS_E_INVALID_ARGUMENT, "unknown comparison");
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    *n_out = 0;
    if (n == 0) return;
    uint64_t* lit = sc.get<uint64_t>(1);
    PSG_CUDA(cudaMemcpyAsync(lit, literal, 8, cudaMemcpyHostToDevice, s));
    uint64_t* flag = sc.get<uint64_t>(n);
    uint64_t* pos = sc.get<uint64_t>(n);
    k_filter_flags<<<blocks(n), 256, 0, s>>>(col.data, col.dtype, op, lit, n, flag);
    const uint64_t m = scan_count(flag, n, pos, s, sc);
    k_scatter_idx<<<blocks(n), 256, 0, s>>>(flag, pos, n, idx);
    count_launch(2);
    PSG_CUDA(cudaStreamSynchronize(s));
    *n_out = m;
  });
}

ps_status psg_frame_merge(psg_context* c, const psg_col* lkeys, const psg_col* rkeys, uint32_t n_keys,
                          uint64_t nl, uint64_t nr, uint64_t capacity, uint64_t* lidx, uint64_t* ridx,
                          uint64_t* n_out) {
  if (!c || !lkeys || !rkeys || n_keys == 0 || !n_out) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    for (uint32_t k = 0; k < n_keys; ++k) {
      check_dtype(lkeys[k].dtype);
      if (lkeys[k].dtype != rkeys[k].dtype) fail(PS_E_INVALID_ARGUMENT, "key dtype mismatch");
    }
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    *n_out = 0;
    if (nl == 0 || nr == 0) return;
    uint64_t* rperm = sc.get<uint64_t>(nr);
    argsort(rkeys, n_keys, nullptr, nr, rperm, s, sc);
    psg_col* dl = upload_cols(lkeys, n_keys, s, sc);
    psg_col* dr = upload_cols(rkeys, n_keys, s, sc);
    uint64_t* flag = sc.get<uint64_t>(nr);
    uint64_t* rpos = sc.get<uint64_t>(nr);
    k_run_flags<<<blocks(nr), 256, 0, s>>>(dr, n_keys, rperm, nr, flag);
    const uint64_t runs = scan_count(flag, nr, rpos, s, sc);
    uint64_t* rstarts = sc.get<uint64_t>(runs);
    k_scatter_starts<<<blocks(nr), 256, 0, s>>>(flag, rpos, nr, rstarts);
    uint64_t* run_of = sc.get<uint64_t>(nl);
    uint64_t* cnt = sc.get<uint64_t>(nl);
    uint64_t* pos = sc.get<uint64_t>(nl);
    k_merge_count<<<blocks(nl), 256, 0, s>>>(dl, dr, n_keys, nl, rperm, rstarts, runs, nr, run_of, cnt);
    count_launch(3);
    const uint64_t m = scan_count(cnt, nl, pos, s, sc);
    *n_out = m;
    if (m > capacity || !lidx || !ridx) return;  // size query (two-call pattern)
    k_merge_emit<<<blocks(nl), 256, 0, s>>>(run_of, cnt, pos, nl, rperm, rstarts, lidx, ridx);
    count_launch();
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_vector_add(psg_context* c, const double* a, const double* b, uint64_t n, double* out) {
  if (!c || (n && (!a || !b || !out))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    cudaStream_t s = stream_of(c);
    if (n) k_vadd<<<blocks(n), 256, 0, s>>>(a, b, n, out), count_launch();
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_multiply(psg_context* c, const double* a, double scalar, uint64_t n, double* out) {
  if (!c || (n && (!a || !out))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    cudaStream_t s = stream_of(c);
    if (n) k_vmul<<<blocks(n), 256, 0, s>>>(a, scalar, n, out), count_launch();
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_scalar_compare(psg_context* c, const double* a, uint32_t op, double scalar, uint64_t n,
                                   int64_t* out) {
  if (!c || (n && (!a || !out))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    if (op > PSG_NE) fail(PS_E_INVALID_ARGUMENT, "unknown comparison");
    cudaStream_t s = stream_of(c);
    if (n) k_scmp<<<blocks(n), 256, 0, s>>>(a, op, scalar, n, out), count_launch();
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_reduce_sum(psg_context* c, const double* a, uint64_t n, double* result) {
  if (!c || !result || (n && !a)) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    *result = 0.0;
    if (n == 0) return;
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    const uint64_t nb = (n + kBlock - 1) / kBlock;
    double* sums = sc.get<double>(nb);
    double* carry = sc.get<double>(nb);
    double* total = sc.get<double>(1);
    k_block_sums<<<static_cast<unsigned>(nb), 32, 0, s>>>(a, n, sums);
    k_carry<<<1, 32, 0, s>>>(sums, nb, carry, total);
    count_launch(2);
    PSG_CUDA(cudaMemcpyAsync(result, total, 8, cudaMemcpyDeviceToHost, s));
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

ps_status psg_frame_cumsum(psg_context* c, const double* a, uint64_t n, double* out) {
  if (!c || (n && (!a || !out))) return PS_E_INVALID_ARGUMENT;
  return fguard([&] {
    if (n == 0) return;
    cudaStream_t s = stream_of(c);
    scratch sc(s);
    const uint64_t nb = (n + kBlock - 1) / kBlock;
    double* sums = sc.get<double>(nb);
    double* carry = sc.get<double>(nb);
    double* total = sc.get<double>(1);
    k_block_sums<<<static_cast<unsigned>(nb), 32, 0, s>>>(a, n, sums);
    k_carry<<<1, 32, 0, s>>>(sums, nb, carry, total);
    k_block_scan<<<static_cast<unsigned>(nb), 32, 0, s>>>(a, n, carry, out);
    count_launch(3);
    PSG_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
