// Automatic anchor on the device: itermodel::suggest_anchor (itermodel.cpp:
// 45-109) over one trace (the reference uses the first requested trace only,
// itermodel.cpp:253-255).
//
//   k_anchor_walk   one thread per event: the contexts ENTERED at the event
//                   (its ancestor chain minus the previous event's; chains are
//                   compared with CCT preorder ranges), and the segment's
//                   duration added to the context's exclusive time
//   (CUB scan)      entry offsets per event; per-context entry counts
//   k_anchor_emit   (context, timestamp) entry pairs
//   (CUB sort)      stable radix sort by context: each context's entries in
//                   event (= time) order
//   k_anchor_pick   one thread: inclusive (covered) time by reverse-id
//                   roll-up (parent < id), then per context with >= min_iters
//                   entries the population CV of the entry gaps with the
//                   reference's own fp64 arithmetic and order (gap_cv,
//                   itermodel.cpp:27-41), and the candidate with the most
//                   covered time (ties: the smallest id)

#include <cstdint>
#include <vector>

#include "psg_internal.h"

namespace psg {

namespace {

typedef unsigned long long u64;
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ bool is_anc(const int32_t* pre, const int32_t* size, uint32_t x,
                                       uint32_t y) {
  return pre[x] <= pre[y] && pre[y] < pre[x] + size[x];
}

__global__ void k_anchor_walk(const uint64_t* ts, const uint32_t* ctx, uint64_t n, uint64_t t_end,
                              const uint32_t* parent, const int32_t* pre, const int32_t* size,
                              uint64_t* ent_cnt, unsigned long long* ctx_cnt,
                              unsigned long long* excl) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = ctx[i];
  const bool has_prev = i > 0;
  const uint32_t prev = has_prev ? ctx[i - 1] : 0u;
  uint32_t cnt = 0;
  for (uint32_t x = c; x != kNone; x = parent[x]) {
    if (has_prev && is_anc(pre, size, x, prev)) break;  // shared with the previous chain
    ++cnt;
    atomicAdd(ctx_cnt + x, 1ull);
  }
  ent_cnt[i] = cnt;
  const uint64_t end = i + 1 < n ? ts[i + 1] : (t_end > ts[i] ? t_end : ts[i]);
  const uint64_t dur = end - ts[i];
  if (dur) atomicAdd(excl + c, static_cast<unsigned long long>(dur));
}

__global__ void k_anchor_emit(const uint64_t* ts, const uint32_t* ctx, uint64_t n,
                              const uint32_t* parent, const int32_t* pre, const int32_t* size,
                              const uint64_t* ent_off, uint32_t* keys, uint64_t* vals) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const bool has_prev = i > 0;
  const uint32_t prev = has_prev ? ctx[i - 1] : 0u;
  uint64_t o = ent_off[i];
  for (uint32_t x = ctx[i]; x != kNone; x = parent[x]) {
    if (has_prev && is_anc(pre, size, x, prev)) break;
    keys[o] = x;
    vals[o] = ts[i];
    ++o;
  }
}

// gap_cv (itermodel.cpp:27-41), same operations in the same order.
__device__ double gap_cv(const uint64_t* e, uint64_t n) {
  double mean = 0.0;
  for (uint64_t i = 1; i < n; ++i) mean += static_cast<double>(e[i] - e[i - 1]);
  mean /= static_cast<double>(n - 1);
  if (mean <= 0.0) return __longlong_as_double(0x7FF0000000000000ll);  // +inf
  double var = 0.0;
  for (uint64_t i = 1; i < n; ++i) {
    const double g = static_cast<double>(e[i] - e[i - 1]);
    var += (g - mean) * (g - mean);
  }
  var /= static_cast<double>(n - 1);
  return sqrt(var) / mean;
}

__global__ void k_anchor_pick(const uint32_t* parent, uint32_t n_ctx,
                              const unsigned long long* ctx_cnt, unsigned long long* incl,
                              const uint64_t* vals, uint32_t min_iters, double cv_max,
                              uint32_t* best_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (uint32_t c = n_ctx; c-- > 1;) incl[parent[c]] += incl[c];  // covered = inclusive time
  uint32_t best = kNone;
  u64 best_cov = 0, off = 0;
  for (uint32_t c = 0; c < n_ctx; ++c) {
    const u64 n = ctx_cnt[c];
    const u64 o = off;
    off += n;
    if (n < min_iters) continue;
    if (gap_cv(vals + o, n) > cv_max) continue;
    if (best == kNone || incl[c] > best_cov) {
      best = c;
      best_cov = incl[c];
    }
  }
  *best_out = best;
}

}  // namespace

namespace {

// Stream-ordered device scratch, freed with the call.
struct scratch {
  cudaStream_t s;
  std::vector<void*> held;
  explicit scratch(cudaStream_t st) : s(st) {}
  ~scratch() {
    for (void* p : held) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* get(size_t count) {
    void* p = nullptr;
    PSG_CUDA(cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), s));
    held.push_back(p);
    return static_cast<T*>(p);
  }
};

}  // namespace

uint32_t launch_suggest_anchor(const uint64_t* ts, const uint32_t* ctx, uint64_t n, uint64_t t_end,
                               const uint32_t* parent, const int32_t* pre, const int32_t* size,
                               uint32_t n_ctx, uint32_t min_iters, double cv_max, cudaStream_t s) {
  if (n == 0) fail(PS_E_INVALID_ARGUMENT, "trace has no events");  // empty_input
  if (n >= (1ull << 31)) fail(PS_E_INVALID_ARGUMENT, "trace too long for the anchor pass");
  scratch sc(s);
  uint64_t* ent_cnt = sc.get<uint64_t>(n);
  uint64_t* ent_off = sc.get<uint64_t>(n);
  unsigned long long* ctx_cnt = sc.get<unsigned long long>(n_ctx);
  unsigned long long* excl = sc.get<unsigned long long>(n_ctx);
  uint32_t* best = sc.get<uint32_t>(1);
  PSG_CUDA(cudaMemsetAsync(ctx_cnt, 0, 8ull * n_ctx, s));
  PSG_CUDA(cudaMemsetAsync(excl, 0, 8ull * n_ctx, s));
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  k_anchor_walk<<<blocks, 256, 0, s>>>(ts, ctx, n, t_end, parent, pre, size, ent_cnt, ctx_cnt, excl);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  {  // entry offsets: exclusive scan of the per-event counts
    const size_t tb = exclusive_sum_scratch_bytes(n);
    exclusive_sum_u64(ent_cnt, ent_off, n, sc.get<uint8_t>(tb), tb, s);
  }
  uint64_t last_off = 0, last_cnt = 0;
  PSG_CUDA(cudaMemcpyAsync(&last_off, ent_off + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaMemcpyAsync(&last_cnt, ent_cnt + n - 1, 8, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  const uint64_t total = last_off + last_cnt;
  uint32_t* keys = sc.get<uint32_t>(total);
  uint32_t* keys2 = sc.get<uint32_t>(total);
  uint64_t* vals = sc.get<uint64_t>(total);
  uint64_t* vals2 = sc.get<uint64_t>(total);
  k_anchor_emit<<<blocks, 256, 0, s>>>(ts, ctx, n, parent, pre, size, ent_off, keys, vals);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  int bits = 1;
  while ((1ull << bits) < n_ctx && bits < 32) ++bits;
  // stable: each ctx's entries keep their event order
  const size_t sb = sort_pairs_scratch_bytes<uint32_t, uint64_t>(total);
  sort_pairs<uint32_t, uint64_t>(keys, keys2, vals, vals2, total, 0, bits, false, sc.get<uint8_t>(sb), sb, s);
  k_anchor_pick<<<1, 32, 0, s>>>(parent, n_ctx, ctx_cnt, excl, vals2, min_iters, cv_max, best);
  count_launch();
  PSG_CUDA(cudaGetLastError());
  uint32_t h = kNone;
  PSG_CUDA(cudaMemcpyAsync(&h, best, 4, cudaMemcpyDeviceToHost, s));
  PSG_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace psg
