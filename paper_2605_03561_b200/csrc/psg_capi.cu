// extern "C" surface of libpsg: context lifetime, trace loading (host AoS,
// trace.db mmap reader, device generator), the fused query, NCCL summaries,
// and result copy-out.  Exceptions never cross the ABI: guarded() maps them
// to ps_status with a thread-local message (the reference's firewall,
// capi.cpp:65-80).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "psg_internal.h"
#include "psg_store.h"

using namespace psg;

namespace {

thread_local std::string t_last_error;

template <typename Fn>
ps_status guarded(Fn&& fn) {
  try {
    fn();
    return PS_OK;
  } catch (const failure& f) {
    t_last_error = f.what();
    return f.status;
  } catch (const std::bad_alloc&) {
    t_last_error = "out of memory";
    return PS_E_INTERNAL;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return PS_E_INTERNAL;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) fail(PS_E_INVALID_ARGUMENT, msg);
}

}  // namespace

void psg::set_last_error(const std::string& m) { t_last_error = m; }

namespace {

// ---- NCCL, resolved at runtime ---------------------------------------------
// Loaded with dlopen so that a process which already holds torch's bundled
// libnccl.so.2 reuses it (RTLD_NOLOAD first) instead of mixing two copies.
struct nccl_api {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

nccl_api& nccl() {
  static nccl_api api;
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(PS_E_INTERNAL, std::string("cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) fail(PS_E_INTERNAL, std::string("libnccl lacks ") + n);
    return p;
  };
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  api.h = h;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(PS_E_INTERNAL, std::string("NCCL error in ") + what + ": " + nccl().error_string(r));
}

// ---- host CCT helpers --------------------------------------------------------

struct preorder {
  std::vector<int32_t> pre, size;  // by ctx (-1 outside the requested subtree)
  std::vector<uint32_t> order;     // ctx ids in preorder
};

// Iterative DFS over children in ascending id order.
preorder preorder_of(const std::vector<uint32_t>& parent, uint32_t root) {
  const uint32_t n = static_cast<uint32_t>(parent.size());
  std::vector<std::vector<uint32_t>> kids(n);
  for (uint32_t c = 1; c < n; ++c)
    if (parent[c] != store::k_no_parent) kids[parent[c]].push_back(c);
  preorder po;
  po.pre.assign(n, -1);
  po.size.assign(n, 0);
  std::vector<std::pair<uint32_t, size_t>> stack{{root, 0}};
  po.pre[root] = 0;
  po.order.push_back(root);
  while (!stack.empty()) {
    auto& [node, next] = stack.back();
    if (next < kids[node].size()) {
      uint32_t ch = kids[node][next++];
      po.pre[ch] = static_cast<int32_t>(po.order.size());
      po.order.push_back(ch);
      stack.push_back({ch, 0});
    } else {
      po.size[node] = static_cast<int32_t>(po.order.size()) - po.pre[node];
      stack.pop_back();
    }
  }
  return po;
}

// xorshift64* transition matrix powers M^(2^b), b = 0..63, as column vectors.
std::vector<uint64_t> jump_matrices() {
  auto step = [](uint64_t x) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
  };
  auto apply = [](const uint64_t* m, uint64_t x) {
    uint64_t r = 0;
    for (int i = 0; i < 64; ++i)
      if ((x >> i) & 1) r ^= m[i];
    return r;
  };
  std::vector<uint64_t> mats(64 * 64);
  for (int i = 0; i < 64; ++i) mats[i] = step(1ull << i);
  for (int b = 1; b < 64; ++b)
    for (int i = 0; i < 64; ++i)
      mats[64 * b + i] = apply(&mats[64 * (b - 1)], mats[64 * (b - 1) + i]);
  return mats;
}

}  // namespace

// ---------------------------------------------------------------------------

struct psg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};

  // NCCL
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;

  // CCT
  uint32_t n_ctx = 0;
  std::vector<uint32_t> h_parent;
  preorder cct_po;
  dbuf<int32_t> d_cct_pre, d_cct_size;
  dbuf<uint32_t> d_parent;

  // traces (SoA)
  uint32_t n_traces = 0;
  uint64_t n_events = 0;
  std::vector<uint64_t> h_off, h_tend;
  std::vector<uint64_t> h_tbegin;  // trace.db index t_begin (validated on load; empty otherwise)
  dbuf<uint64_t> d_tbegin;
  std::vector<uint32_t> h_pid;
  dbuf<uint64_t> d_off, d_ts, d_tend;
  dbuf<uint32_t> d_ctx, d_pid;
  // narrow mirror of d_ctx when every ctx < 256 (pass 1 reads 1 B/event
  // instead of 4); built on load when HBM allows, else pass 1 reads d_ctx
  dbuf<uint8_t> d_ctx8;
  bool ctx8_valid = false;
  dbuf<uint8_t> d_stage;
  uint8_t* pinned[3] = {nullptr, nullptr, nullptr};  // pageable-source staging ring
  cudaEvent_t pinned_ev[3] = {nullptr, nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;  // H2D of pinned trace bodies (load_aos)
  // psg_prefetch_aos: the first staging chunks of the NEXT pinned load, copied
  // while the device works on the current one (pf_chunks chunks of pf_body)
  const uint8_t* pf_body = nullptr;
  uint64_t pf_events = 0;
  int pf_chunks = 0;
  // side stream of a speculative single-rank query: the pass-1 verification
  // runs there, concurrently with the cross-rank statistics
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_in = nullptr, side_out = nullptr;
  cudaEvent_t stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};

  // nodes / topology
  uint32_t n_nodes = 0;
  std::vector<uint32_t> h_node_of_trace, h_rack_ids;  // rack id per rack index
  // chassis ids of each rack's universe nodes, ascending: the device works on
  // a rack's chassis slot (position in this list), so any chassis id works as
  // long as a rack has at most 64 distinct chassis
  std::vector<std::vector<uint32_t>> h_rack_chassis;
  // set when a hostname of the node universe is not a Slingshot name: queries
  // that need the topology raise it as PS_E_PARSE (topology.cpp:14-46)
  std::string topo_error;
  dbuf<uint32_t> d_node_of_trace, d_node_rack_idx, d_node_chassis, d_uni_cnt;

  // anchor subtree (cached per anchor)
  int64_t cached_anchor = -1;
  uint32_t nn = 0;
  std::vector<uint32_t> node_ids, leaves;
  std::vector<int32_t> h_sub_pre;
  uint32_t root_only = 0;  // the anchor is the only internal node of its subtree
  std::vector<uint32_t> internal_pos;  // node positions of the internal nodes
  dbuf<int32_t> d_sub_pre;
  dbuf<int4> d_node_tab;  // [nn] {preorder position, subtree size, internal?, 0}
  dbuf<uint32_t> d_contains;  // subtree membership bitset [ceil(n_ctx/32)]
  uint32_t contains_words = 0;

  // pass-1 boundary regions: trace t owns bidx[cap_off[t], cap_off[t+1])
  uint32_t cap_div = 32;  // capacity = n_t / cap_div + 32 (exact bound after an overflow)
  bool caps_valid = false;
  // the optimistic pass 1 missed on the loaded traces: start the next queries
  // in the exact mode (reset when traces are loaded)
  bool exact_hint = false;
  dbuf<uint64_t> d_cap_off;
  dbuf<uint32_t> d_bidx, d_nbounds;
  dbuf<uint64_t> d_bts;

  // window results
  bool have_window = false, have_carry = false;
  dbuf<uint64_t> w_cnt, w_sum, w_min, w_max, w_excl, w_incl, c_ts;
  dbuf<double> w_mean;
  dbuf<uint8_t> c_has;
  dbuf<uint32_t> c_ctx;
  dbuf<unsigned long long> w_counters;  // [0] groups, [1] rows (computed on copy-out)

  // cube results
  bool have_cube = false;
  uint32_t n_kept = 0, n_kept_global = 0, K = 0;
  uint64_t n_cells = 0;
  dbuf<uint32_t> iter_count, tpos;
  dbuf<uint64_t> block_off, iter_off, kept_bo, cube_incl, cube_xint, gap_incl, gap_excl;
  uint64_t n_store = 0;  // storage cells of the cube (rows of stride row_stride(nn), blocks padded)
  bool cube32 = false;   // 32-bit cells (every stored iteration spans < 2^32 ns)
  dbuf<unsigned long long> summary;
  dbuf<uint8_t> scratch;
  dbuf<uint64_t> dense_stage;  // int64 cells of the dense copy-out (k_cube_dense)
  dbuf<unsigned long long> x_acc;  // x_sum [K nn] | x_max [K nn] | x_sq [3 K nn]
  dbuf<double> within_cv, node_out;
  dbuf<uint8_t> within_ok;
  bool have_stats = false;
  bool have_excl = false;  // PSG_Q_NO_CUBE_STORE keeps only the incl half

  // outliers
  bool have_outliers = false;
  std::vector<uint32_t> sites;
  dbuf<uint32_t> d_sites, d_worst, d_order, d_nsel, d_rack_nodes;
  dbuf<unsigned long long> site_acc, node_acc, rack_mask, rack_full;
  dbuf<uint32_t> rack_cnt;  // [n_racks][64] outlier nodes per (rack, chassis slot)
  dbuf<double> site_ratio, node_mean, node_z;

  // profile records (profile.db; psg_profiles.cu)
  uint32_t n_prof = 0;
  uint64_t n_rec = 0;
  std::vector<uint32_t> h_prof_pid;
  std::vector<int32_t> h_prof_rank;
  dbuf<uint64_t> prof_off;
  dbuf<uint32_t> prof_pid, prec_ctx;
  dbuf<uint16_t> prec_metric;
  dbuf<double> prec_value;
  uint32_t n_rank_prof = 0;                    // profiles with rank >= 0 ...
  dbuf<uint32_t> d_rank_slot;                  // ... in (rank, id) order -> profile slot
  bool have_prof_nodes = false;
  dbuf<uint32_t> d_pnode_off, d_pnode_rank;    // node -> its rank profiles (CSR, rank order)
  dbuf<double> pvals;                          // [n_rank_prof][n_sites] rank_vector values
  dbuf<uint32_t> d_slot, d_ctx_bits, d_metric_bits;
  dbuf<unsigned long long> d_counts, d_row_off;
  dbuf<uint32_t> d_row_pid, d_row_ctx;
  dbuf<uint16_t> d_row_metric;
  dbuf<double> d_row_value;
  profile_view pview() const {
    return {prof_off.p, prof_pid.p, prec_ctx.p, prec_metric.p, prec_value.p, n_prof};
  }

  dbuf<uint64_t> jump;
  dbuf<double> gen_params;
  dbuf<uint64_t> gen_chunks;

  ~psg_context() {
    for (int i = 0; i < 3; ++i) {
      if (pinned_ev[i]) cudaEventDestroy(pinned_ev[i]);
      if (pinned[i]) cudaFreeHost(pinned[i]);
    }
    if (copy_stream) cudaStreamSynchronize(copy_stream);  // a prefetch into d_stage
    for (auto& e : stage_ev)
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (comm) nccl().comm_destroy(comm);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  // the sparse window (psg_sparse.cu): the last query's rows when it took the
  // sparse layout, or the copy-out of a dense window (sp_valid)
  sparse_result sp;
  bool sp_valid = false, window_sparse = false;
  dbuf<uint32_t> d_depth;  // [n_ctx] ancestors per ctx (set_cct)
  dbuf<uint32_t> d_ppo_g;  // [n_ctx] cube column byte offsets of the current anchor (compute_subtree)
  dbuf<uint64_t> site_vals;  // [n][n_sites] site incl of a sparse window (outliers)
  dbuf<uint32_t> d_site_iota;

  // query status block (QS_*), and what the speculative path needs: buffers
  // sized by an earlier query on these traces, the K its statistics planes
  // are laid out for, the global rank count
  dbuf<unsigned long long> qstat;
  // work units of pass 2 (intra-trace split of long traces), planned from the
  // loaded traces' event counts; units_key = the plan's (traces, events, unit size)
  dbuf<uint4> d_units;
  dbuf<uint32_t> d_split;
  uint32_t n_units = 0, n_split = 0;
  uint64_t units_key = 0;
  dbuf<unsigned long long> wacc;
  // asynchronous copy-out (psg_get_cube_stored_async): its own stream, so the
  // D2H of one query's cube overlaps the H2D of the next query's traces
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t d2h_ready = nullptr, d2h_done = nullptr;
  bool d2h_pending = false;
  void wait_copies() {
    if (d2h_pending) PSG_CUDA(cudaEventSynchronize(d2h_done));
    d2h_pending = false;
  }
  bool spec_ready = false;
  uint32_t k_plane = 0;
  uint64_t ranks_global_cache = 0;
  uint64_t n_syncs = 0;  // stream synchronisations (psg_query_info::host_syncs)

  trace_view view() const { return {d_off.p, d_ts.p, d_ctx.p, d_tend.p, n_traces}; }
  void sync() {
    ++n_syncs;
    PSG_CUDA(cudaStreamSynchronize(stream));
  }

  // Summary exchange between ranks: NCCL on device buffers, or a host
  // callback (psg_comm_init_host) on a staged host copy.
  psg_allreduce_fn host_fn = nullptr;
  void* host_user = nullptr;
  bool multi() const { return nranks > 1 && (comm || host_fn); }
  void group_begin() {
    if (comm && nranks > 1) nccl_check(nccl().group_start(), "ncclGroupStart");
  }
  void group_end() {
    if (comm && nranks > 1) nccl_check(nccl().group_end(), "ncclGroupEnd");
  }
  template <typename T>
  void allreduce(T* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op) {
    if (nranks <= 1 || count == 0) return;
    if (comm) {
      nccl_check(nccl().all_reduce(buf, buf, count, dt, op, comm, stream), "ncclAllReduce");
      return;
    }
    if (!host_fn) return;
    std::vector<T> h(count);
    PSG_CUDA(cudaMemcpyAsync(h.data(), buf, sizeof(T) * count, cudaMemcpyDeviceToHost, stream));
    sync();
    const int dtype = dt == ncclFloat64 ? 1 : 0;
    const int o = op == ncclSum ? 0 : (op == ncclMax ? 1 : 2);
    if (host_fn(h.data(), count, dtype, o, host_user) != 0)
      fail(PS_E_INTERNAL, "host all-reduce callback failed");
    PSG_CUDA(cudaMemcpyAsync(buf, h.data(), sizeof(T) * count, cudaMemcpyHostToDevice, stream));
    sync();
  }
};

namespace {

// The query kernels read whole 128-bit-aligned block steps and prefetch ahead:
// event arrays carry this many events of slack past the last event.
constexpr uint64_t kEventPad = 2048;

void ensure_device(psg_context* c) { PSG_CUDA(cudaSetDevice(c->device)); }

// Per-trace boundary regions for pass 1 (k_bounds).  A trace of n events has
// at most ceil(n/2) boundaries (two adjacent events cannot both enter the
// subtree); the default region n/32 + 32 covers iterations of >= 32 events
// on average and an overflow re-runs pass 1 with the exact bound.
void build_caps(psg_context* c) {
  std::vector<uint64_t> cap(c->n_traces + 1, 0);
  for (uint32_t t = 0; t < c->n_traces; ++t) {
    const uint64_t n = c->h_off[t + 1] - c->h_off[t];
    cap[t + 1] = cap[t] + (c->cap_div <= 2 ? (n + 1) / 2 + 1 : n / c->cap_div + 32);
  }
  PSG_CUDA(cudaMemcpyAsync(c->d_cap_off.ensure(c->n_traces + 1), cap.data(), 8ull * cap.size(),
                           cudaMemcpyHostToDevice, c->stream));
  c->d_bidx.ensure(cap.back() + 1);
  c->d_bts.ensure(cap.back() + 1);
  c->sync();
  c->caps_valid = true;
}

void invalidate_results(psg_context* c) {
  c->have_window = c->have_carry = c->have_cube = c->have_stats = c->have_outliers = false;
  c->sp_valid = false;
}

void build_ctx8(psg_context* c);

void set_cct_impl(psg_context* c, const uint32_t* parent, uint32_t n_ctx) {
  require(parent != nullptr && n_ctx > 0, "parent array and n_ctx > 0 are required");
  if (parent[0] != store::k_no_parent) fail(PS_E_FORMAT, "ctx 0: root must have no parent");
  for (uint32_t i = 1; i < n_ctx; ++i)
    if (parent[i] >= i)
      fail(PS_E_FORMAT, "ctx " + std::to_string(i) +
                            ": parent id must be smaller than ctx id (topological order)");
  c->n_ctx = n_ctx;
  c->h_parent.assign(parent, parent + n_ctx);
  c->cct_po = preorder_of(c->h_parent, 0);
  PSG_CUDA(cudaMemcpyAsync(c->d_cct_pre.ensure(n_ctx), c->cct_po.pre.data(), 4ull * n_ctx,
                           cudaMemcpyHostToDevice, c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_cct_size.ensure(n_ctx), c->cct_po.size.data(), 4ull * n_ctx,
                           cudaMemcpyHostToDevice, c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_parent.ensure(n_ctx), parent, 4ull * n_ctx,
                           cudaMemcpyHostToDevice, c->stream));
  std::vector<uint32_t> depth(n_ctx, 0);  // parents precede their children
  for (uint32_t i = 1; i < n_ctx; ++i) depth[i] = depth[parent[i]] + 1;
  PSG_CUDA(cudaMemcpyAsync(c->d_depth.ensure(n_ctx), depth.data(), 4ull * n_ctx, cudaMemcpyHostToDevice,
                           c->stream));
  c->cached_anchor = -1;
  invalidate_results(c);
  c->sync();
  build_ctx8(c);  // the mirror holds preorder positions of this tree
}

// The narrow ctx mirror (validated ctx < n_ctx <= 256): 1 B/event more HBM,
// built only when at least half the event bytes stay free afterwards (room
// for the cube, ~1/3 of the event bytes with 32-bit cells); PSG_NO_CTX8=1
// turns it off (A/B).
void build_ctx8(psg_context* c) {
  c->ctx8_valid = false;
  const char* off = std::getenv("PSG_NO_CTX8");
  if ((off && *off == '1') || c->n_ctx > 256 || c->n_events == 0) return;
  const uint64_t need = c->n_events + 2 * kEventPad;
  if (c->d_ctx8.n < need) {
    size_t free_b = 0, total_b = 0;
    PSG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    c->d_ctx8.release();
    if (free_b < need || free_b - need < 6 * c->n_events) return;
    c->d_ctx8.ensure(need);
  }
  launch_ctx8(c->d_ctx.p, c->n_events, c->d_cct_pre.p, c->n_ctx, c->d_ctx8.p, c->stream);
  c->ctx8_valid = true;
}

// Uploads the trace index and validates the SoA already in d_ts/d_ctx.
void finish_load(psg_context* c) {
  PSG_CUDA(cudaMemcpyAsync(c->d_off.ensure(c->n_traces + 1), c->h_off.data(),
                           8ull * (c->n_traces + 1), cudaMemcpyHostToDevice, c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_tend.ensure(c->n_traces + 1), c->h_tend.data(), 8ull * c->n_traces,
                           cudaMemcpyHostToDevice, c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_pid.ensure(c->n_traces + 1), c->h_pid.data(), 4ull * c->n_traces,
                           cudaMemcpyHostToDevice, c->stream));
  if (c->n_ctx == 0) fail(PS_E_INVALID_ARGUMENT, "set the calling-context tree before loading traces");
  for (uint32_t t = 0; t < c->n_traces; ++t)
    if (c->h_off[t + 1] - c->h_off[t] >= (1ull << 32) - 4096)
      fail(PS_E_INVALID_ARGUMENT, "trace " + std::to_string(c->h_pid[t]) +
                                      " has 2^32 - 4096 or more events (event indices are 32-bit)");
  c->caps_valid = false;
  c->exact_hint = false;
  c->cap_div = 32;
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(c->summary.ensure(4));
  unsigned long long init[2] = {0ull, ~0ull};
  PSG_CUDA(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
  const uint64_t* tb = nullptr;
  if (!c->h_tbegin.empty()) {
    PSG_CUDA(cudaMemcpyAsync(c->d_tbegin.ensure(c->n_traces + 1), c->h_tbegin.data(),
                             8ull * c->n_traces, cudaMemcpyHostToDevice, c->stream));
    tb = c->d_tbegin.p;
  }
  c->spec_ready = false;  // the first query on these traces sizes the buffers
  c->units_key = 0;
  c->ranks_global_cache = 0;
  launch_validate(c->view(), c->n_ctx, tb, flags, flags + 1, c->stream);
  unsigned long long out[2];
  PSG_CUDA(cudaMemcpyAsync(out, flags, sizeof(out), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (out[0] != 0)
    fail(PS_E_FORMAT, std::to_string(out[0]) + " trace(s) violate the format (first: trace " +
                          std::to_string(c->h_pid[out[1]]) +
                          "): non-decreasing timestamps, ctx < n_ctx and t_end >= last event are required");
  build_ctx8(c);
  invalidate_results(c);
}

// Host AoS body -> HBM staging (chunked, double-buffered) -> SoA.
// Pageable sources (an mmap'd trace.db, a std::vector) go through a ring of
// pinned staging buffers: host threads fill buffer i+1 (page faults and
// copies in parallel) while the DMA engine moves buffer i, then K1 transposes
// on the stream.  Pinned sources are DMA'd directly (load_aos_pinned).
constexpr uint64_t kRingEvents = 1ull << 22;  // 4 Mi events = 48 MB per pinned buffer
constexpr uint64_t kRingBytes = kRingEvents * 12;
constexpr int kRingBufs = 3;

void ensure_pinned_ring(psg_context* c) {
  if (c->pinned[0]) return;
  for (int i = 0; i < kRingBufs; ++i) {
    PSG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->pinned[i]), kRingBytes,
                           cudaHostAllocDefault));
    PSG_CUDA(cudaEventCreateWithFlags(&c->pinned_ev[i], cudaEventDisableTiming));
  }
}

constexpr uint64_t kPinnedChunkEvents = 4ull << 24;  // 64 Mi events = 768 MB per staging chunk

void ensure_copy_stream(psg_context* c) {
  if (c->copy_stream) return;
  PSG_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (auto& e : c->stage_ev) PSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// Every other user of the staging buffer first lets an unclaimed prefetch land
// (its copies may still be writing there) and forgets it.
void drop_prefetch(psg_context* c) {
  if (c->pf_chunks > 0) PSG_CUDA(cudaStreamSynchronize(c->copy_stream));
  c->pf_body = nullptr;
  c->pf_events = 0;
  c->pf_chunks = 0;
}

void load_aos_pageable(psg_context* c, const uint8_t* body, uint64_t n_events) {
  constexpr uint64_t kBufEv = kRingEvents, kBufBytes = kRingBytes;
  constexpr int kBufs = kRingBufs;
  ensure_pinned_ring(c);
  drop_prefetch(c);
  uint8_t* stage = c->d_stage.ensure(std::max<uint64_t>(c->d_stage.n, 2 * kBufBytes));
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nthreads = std::min(8u, hw);
  uint64_t done = 0;
  for (int i = 0; done < n_events; ++i) {
    const uint64_t ev = std::min(kBufEv, n_events - done);
    const int slot = i % kBufs;
    PSG_CUDA(cudaEventSynchronize(c->pinned_ev[slot]));  // the buffer's previous DMA finished
    const uint8_t* src = body + done * 12;
    uint8_t* dst = c->pinned[slot];
    const uint64_t bytes = ev * 12, part = (bytes + nthreads - 1) / nthreads;
    std::vector<std::thread> th;
    for (unsigned k = 1; k < nthreads; ++k) {
      const uint64_t a = std::min(bytes, k * part), e = std::min(bytes, a + part);
      if (a < e) th.emplace_back([=] { std::memcpy(dst + a, src + a, e - a); });
    }
    std::memcpy(dst, src, std::min(bytes, part));
    for (auto& t : th) t.join();
    uint8_t* dev = stage + static_cast<uint64_t>(i % 2) * kBufBytes;
    PSG_CUDA(cudaMemcpyAsync(dev, dst, bytes, cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaEventRecord(c->pinned_ev[slot], c->stream));
    launch_aos_to_soa(dev, ev, c->d_ts.p + done, c->d_ctx.p + done, c->stream);
    done += ev;
  }
}

// A byte range of a file (trace.db bodies): host threads pread() straight into
// the pinned ring (no page faults on an mmap), the DMA engine moves the
// previous buffer meanwhile, then K1 transposes on the stream.
void load_aos_file(psg_context* c, const std::string& path, uint64_t offset, uint64_t n_events) {
  c->n_events = n_events;
  c->d_ts.ensure(n_events + kEventPad);
  c->d_ctx.ensure(n_events + kEventPad);
  ensure_pinned_ring(c);
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) fail(PS_E_IO, "cannot open " + path);
  struct fd_closer {
    int fd;
    ~fd_closer() { ::close(fd); }
  } closer{fd};
  drop_prefetch(c);
  uint8_t* stage = c->d_stage.ensure(std::max<uint64_t>(c->d_stage.n, 2 * kRingBytes));
  const unsigned nthreads = std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  uint64_t done = 0;
  for (int i = 0; done < n_events; ++i) {
    const uint64_t ev = std::min(kRingEvents, n_events - done);
    const int slot = i % kRingBufs;
    PSG_CUDA(cudaEventSynchronize(c->pinned_ev[slot]));
    uint8_t* dst = c->pinned[slot];
    const uint64_t bytes = ev * 12, part = ((bytes + nthreads - 1) / nthreads + 4095) & ~4095ull;
    const uint64_t base = offset + done * 12;
    std::vector<int> ok(nthreads, 1);
    std::vector<std::thread> th;
    for (unsigned k = 0; k < nthreads; ++k) {
      const uint64_t a = std::min(bytes, k * part), e = std::min(bytes, a + part);
      if (a >= e) break;
      th.emplace_back([&, k, a, e] {
        uint64_t got = a;
        while (got < e) {
          const ssize_t r = ::pread(fd, dst + got, e - got, static_cast<off_t>(base + got));
          if (r <= 0) {
            ok[k] = 0;
            return;
          }
          got += static_cast<uint64_t>(r);
        }
      });
    }
    for (auto& t : th) t.join();
    for (int v : ok)
      if (!v) fail(PS_E_IO, "short read of " + path);
    uint8_t* dev = stage + static_cast<uint64_t>(i % 2) * kRingBytes;
    PSG_CUDA(cudaMemcpyAsync(dev, dst, bytes, cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaEventRecord(c->pinned_ev[slot], c->stream));
    launch_aos_to_soa(dev, ev, c->d_ts.p + done, c->d_ctx.p + done, c->stream);
    done += ev;
  }
}

void load_aos(psg_context* c, const uint8_t* body, uint64_t n_events) {
  c->n_events = n_events;
  c->d_ts.ensure(n_events + kEventPad);
  c->d_ctx.ensure(n_events + kEventPad);
  if (n_events == 0) return;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, body) != cudaSuccess) {
    cudaGetLastError();  // clear: unregistered host memory
    attr.type = cudaMemoryTypeUnregistered;
  }
  if (attr.type != cudaMemoryTypeHost && attr.type != cudaMemoryTypeDevice &&
      attr.type != cudaMemoryTypeManaged)
    return load_aos_pageable(c, body, n_events);
  const uint64_t chunk_ev = kPinnedChunkEvents;
  const uint64_t chunk_bytes = chunk_ev * 12;
  // chunks a psg_prefetch_aos of this very body already put in flight
  const int pf = (c->pf_body == body && c->pf_events == n_events) ? c->pf_chunks : 0;
  if (!pf) drop_prefetch(c);
  c->pf_body = nullptr;
  c->pf_chunks = 0;
  uint8_t* stage = pf ? c->d_stage.p
                      : c->d_stage.ensure(std::min<uint64_t>(2 * chunk_bytes, n_events * 12 + 64));
  const bool two = c->d_stage.n >= 2 * chunk_bytes;
  // H2D copies on their own stream, transposes on the context's stream: copy
  // i + 1 runs while transpose i does (two staging slots, events in between),
  // so the copy engine stays busy at the PCIe rate
  ensure_copy_stream(c);
  cudaEvent_t* copied = c->stage_ev;      // [2] slot filled
  cudaEvent_t* consumed = c->stage_ev + 2;  // [2] slot transposed
  if (!pf) {
    PSG_CUDA(cudaEventRecord(consumed[0], c->stream));  // earlier work on the staging buffer
    PSG_CUDA(cudaEventRecord(consumed[1], c->stream));
  }
  uint64_t done = 0;
  int slot = 0;
  for (int i = 0; done < n_events; ++i) {
    uint64_t ev = std::min(chunk_ev, n_events - done);
    const int sl = two ? slot : 0;
    uint8_t* dst = stage + sl * chunk_bytes;
    if (i >= pf) {  // (the prefetch issued chunk i < pf into slot i, and recorded copied[i])
      PSG_CUDA(cudaStreamWaitEvent(c->copy_stream, consumed[sl], 0));
      PSG_CUDA(cudaMemcpyAsync(dst, body + done * 12, ev * 12, cudaMemcpyHostToDevice, c->copy_stream));
      PSG_CUDA(cudaEventRecord(copied[sl], c->copy_stream));
    }
    PSG_CUDA(cudaStreamWaitEvent(c->stream, copied[sl], 0));
    launch_aos_to_soa(dst, ev, c->d_ts.p + done, c->d_ctx.p + done, c->stream);
    PSG_CUDA(cudaEventRecord(consumed[sl], c->stream));
    done += ev;
    slot ^= 1;
  }
}

void compute_subtree(psg_context* c, uint32_t anchor) {
  if (c->cached_anchor == static_cast<int64_t>(anchor)) return;
  if (anchor >= c->n_ctx)
    fail(PS_E_NOT_FOUND, "anchor ctx " + std::to_string(anchor) + " not in tree");
  preorder sub = preorder_of(c->h_parent, anchor);
  c->node_ids.clear();
  for (uint32_t id = 0; id < c->n_ctx; ++id)
    if (sub.pre[id] >= 0) c->node_ids.push_back(id);
  c->nn = static_cast<uint32_t>(c->node_ids.size());
  std::vector<int4> tab(c->nn);
  std::vector<char> has_child(c->n_ctx, 0);
  for (uint32_t id = 1; id < c->n_ctx; ++id) has_child[c->h_parent[id]] = 1;
  c->leaves.clear();
  c->internal_pos.clear();
  uint32_t n_internal = 0;
  for (uint32_t i = 0; i < c->nn; ++i) {
    const uint32_t id = c->node_ids[i];
    tab[i] = make_int4(sub.pre[id], sub.size[id], has_child[id] ? static_cast<int>(n_internal) + 1 : 0, 0);
    if (has_child[id]) {  // internal: inclusive time = sum over its preorder range
      c->internal_pos.push_back(i);
      ++n_internal;
    } else {
      c->leaves.push_back(id);
    }
  }
  c->root_only = (n_internal == 1 && has_child[anchor]) ? 1u : 0u;
  c->contains_words = (c->n_ctx + 31) / 32;
  std::vector<uint32_t> bits(c->contains_words, 0);
  for (uint32_t id : c->node_ids) bits[id >> 5] |= 1u << (id & 31);
  if (c->leaves.empty()) c->leaves.push_back(anchor);  // itermodel.cpp:216
  // cube rows are indexed by node position (ascending ctx id, the output
  // order); .w of the node table is the inverse map preorder -> node position
  std::vector<int32_t> npos(c->n_ctx, -1);
  for (uint32_t i = 0; i < c->nn; ++i) {
    npos[c->node_ids[i]] = static_cast<int32_t>(i);
    tab[sub.pre[c->node_ids[i]]].w = static_cast<int32_t>(i);
  }
  c->h_sub_pre = npos;
  PSG_CUDA(cudaMemcpyAsync(c->d_sub_pre.ensure(c->n_ctx), npos.data(), 4ull * c->n_ctx,
                           cudaMemcpyHostToDevice, c->stream));
  std::vector<uint32_t> ppo(c->n_ctx);  // the global column table (large trees: no window records)
  for (uint32_t id = 0; id < c->n_ctx; ++id) ppo[id] = 4u * (npos[id] >= 0 ? static_cast<uint32_t>(npos[id]) : c->nn);
  PSG_CUDA(cudaMemcpyAsync(c->d_ppo_g.ensure(c->n_ctx), ppo.data(), 4ull * c->n_ctx, cudaMemcpyHostToDevice,
                           c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_node_tab.ensure(c->nn), tab.data(), sizeof(int4) * c->nn,
                           cudaMemcpyHostToDevice, c->stream));
  PSG_CUDA(cudaMemcpyAsync(c->d_contains.ensure(c->contains_words), bits.data(),
                           4ull * c->contains_words, cudaMemcpyHostToDevice, c->stream));
  c->sync();
  c->cached_anchor = anchor;
}

#ifndef PSG_WMAX
#define PSG_WMAX 16  // warps (traces) per CTA of k_trace_query's wide shape (<= its launch bound / 32)
#endif
#ifndef PSG_ONE_WARP_MIN_EVENTS
#define PSG_ONE_WARP_MIN_EVENTS 40000  // average events per trace from which one-warp CTAs are used (measured crossover 33.5k-50k)
#endif
static constexpr uint64_t kOneWarpMinEvents = PSG_ONE_WARP_MIN_EVENTS;
#ifndef PSG_UNIT_MIN
#define PSG_UNIT_MIN 16384  // events: the smallest work unit of a split trace
#endif
static constexpr uint64_t kUnitMinEvents = PSG_UNIT_MIN;
#ifndef PSG_G
#define PSG_G 8  // iterations per chunk of k_trace_query (power of two, <= 15)
#endif

// itermodel::suggest_anchor on the trace with the smallest profile id over all
// ranks (build_tri_model uses pids.front(), itermodel.cpp:253-255): its owner
// runs the device pass, every rank receives the result.  Both exchanges are
// MIN all-reduces whose "nothing from me" sentinel sits below 2^63 (a host
// reducer may reinterpret uint64 as int64); the owner's own failure travels
// as a value between the anchors and the sentinel, so every rank fails with
// the owner's status instead of waiting in a collective the owner never joins.
uint32_t auto_anchor(psg_context* c) {
  constexpr uint64_t kAbsent = 0x7FFFFFFFFFFFFFFFull;  // this rank has nothing to say
  constexpr uint64_t kErrBase = 1ull << 40;            // kErrBase | ps_status: the owner failed
  uint64_t mine = kAbsent;
  uint32_t t_min = 0;
  for (uint32_t t = 0; t < c->n_traces; ++t)
    if (c->h_pid[t] < mine) {
      mine = c->h_pid[t];
      t_min = t;
    }
  unsigned long long* d = c->summary.ensure(4);
  auto min_over_ranks = [&](uint64_t v) {
    if (!c->multi()) return v;
    PSG_CUDA(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, c->stream));
    c->allreduce(reinterpret_cast<unsigned long long*>(d), 1, ncclUint64, ncclMin);
    PSG_CUDA(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return v;
  };
  const uint64_t g = min_over_ranks(mine);
  if (g == kAbsent) fail(PS_E_INVALID_ARGUMENT, "no traces loaded");
  uint64_t anchor = kAbsent;
  std::string owner_msg;
  if (g == mine) {
    try {
      const uint64_t b = c->h_off[t_min], n = c->h_off[t_min + 1] - b;
      // kNone (0xFFFFFFFF: no periodic context) travels as a valid "minimum" too
      anchor = launch_suggest_anchor(c->d_ts.p + b, c->d_ctx.p + b, n, c->h_tend[t_min], c->d_parent.p,
                                     c->d_cct_pre.p, c->d_cct_size.p, c->n_ctx, 3, 0.2, c->stream);
    } catch (const failure& f) {
      if (!c->multi()) throw;
      anchor = kErrBase | static_cast<uint64_t>(f.status);
      owner_msg = f.what();
    }
  }
  anchor = min_over_ranks(anchor);
  if (anchor >= kErrBase && anchor < kAbsent)
    fail(static_cast<ps_status>(anchor - kErrBase),
         owner_msg.empty() ? "suggest_anchor failed on the rank owning the first trace" : owner_msg);
  if (anchor >= 0xFFFFFFFFull)  // itermodel.cpp:106-107
    fail(PS_E_NO_PERIODICITY, "no context shows periodic entries");
  return static_cast<uint32_t>(anchor);
}

// Whether some wide shape (>= 2 warps) fits the 227 KB of shared memory.
bool fits_wide(uint32_t n_traces, uint32_t per_warp_bytes, uint32_t table_bytes) {
  uint32_t w = PSG_WMAX;
  while (w > 1 && static_cast<uint64_t>(n_traces) < 2ull * 148 * w) w /= 2;
  while (w > 1 && table_bytes + w * per_warp_bytes > 227u * 1024) w /= 2;
  return w > 1 || table_bytes + per_warp_bytes <= 227u * 1024;
}

uint32_t choose_warps(uint32_t n_traces, uint32_t per_warp_bytes, uint32_t table_bytes) {
  // Aim for >= 2 CTAs per SM worth of traces; fit the carve-outs in 227 KB.
  uint32_t w = PSG_WMAX;
  while (w > 1 && static_cast<uint64_t>(n_traces) < 2ull * 148 * w) w /= 2;
  while (w > 1 && table_bytes + w * per_warp_bytes > 227u * 1024) w /= 2;
  if (table_bytes + w * per_warp_bytes > 227u * 1024)
    fail(PS_E_INVALID_ARGUMENT,
         "calling-context tree too large for the shared-memory tables of the fused kernel");
  return w;
}

}  // namespace

// The node universe shared by the trace and profile paths: n_nodes, and when
// given, each node's rack and chassis (topology.cpp:54-92 universe counts).
static void set_node_tables(psg_context* c, uint32_t n_nodes, const uint32_t* node_rack,
                            const uint32_t* node_chassis) {
  c->n_nodes = n_nodes;
  c->h_rack_ids.clear();
  c->h_rack_chassis.clear();
  if (node_rack && node_chassis) {
    std::set<uint32_t> racks(node_rack, node_rack + n_nodes);
    c->h_rack_ids.assign(racks.begin(), racks.end());
    const size_t nr = c->h_rack_ids.size();
    std::vector<std::set<uint32_t>> ch(nr);
    std::vector<uint32_t> ridx(n_nodes), slot(n_nodes), uni(nr * 64, 0);
    for (uint32_t i = 0; i < n_nodes; ++i) {
      ridx[i] = static_cast<uint32_t>(
          std::lower_bound(c->h_rack_ids.begin(), c->h_rack_ids.end(), node_rack[i]) -
          c->h_rack_ids.begin());
      ch[ridx[i]].insert(node_chassis[i]);
    }
    c->h_rack_chassis.resize(nr);
    for (size_t r = 0; r < nr; ++r) {
      require(ch[r].size() <= 64, "a rack with more than 64 distinct chassis is not supported");
      c->h_rack_chassis[r].assign(ch[r].begin(), ch[r].end());
    }
    for (uint32_t i = 0; i < n_nodes; ++i) {
      const auto& v = c->h_rack_chassis[ridx[i]];
      slot[i] = static_cast<uint32_t>(std::lower_bound(v.begin(), v.end(), node_chassis[i]) - v.begin());
      uni[ridx[i] * 64 + slot[i]] += 1;
    }
    PSG_CUDA(cudaMemcpyAsync(c->d_node_rack_idx.ensure(n_nodes), ridx.data(), 4ull * n_nodes,
                             cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaMemcpyAsync(c->d_node_chassis.ensure(n_nodes), slot.data(), 4ull * n_nodes,
                             cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaMemcpyAsync(c->d_uni_cnt.ensure(uni.size()), uni.data(), 4ull * uni.size(),
                             cudaMemcpyHostToDevice, c->stream));
  }
  c->sync();
}

// Rack / chassis of a database's node universe (hostnames in sorted order,
// node_correlate's order).  A name that is not x<r>c<c>s<s>b<b>n<n> leaves the
// nodes without topology and records the reference's parse_error message for
// the first such name, which topology queries then raise (localize_outliers
// parses the whole universe, topology.cpp:54-63).
static void set_db_nodes(psg_context* c, const std::vector<std::string>& host_list) {
  std::vector<uint32_t> rack(host_list.size()), chassis(host_list.size());
  std::string err;
  for (size_t i = 0; i < host_list.size() && err.empty(); ++i)
    err = store::node_name_error(host_list[i], &rack[i], &chassis[i]);
  const bool topo = err.empty() && !host_list.empty();
  set_node_tables(c, static_cast<uint32_t>(host_list.size()), topo ? rack.data() : nullptr,
                  topo ? chassis.data() : nullptr);
  c->topo_error = err;
}

extern "C" {

const char* psg_version(void) { return "0.1.0-sm100a"; }
const char* psg_last_error(void) { return t_last_error.c_str(); }

const char* psg_status_name(ps_status status) {
  switch (status) {
    case PS_OK: return "ok";
    case PS_E_IO: return "io_error";
    case PS_E_FORMAT: return "format_error";
    case PS_E_INVALID_IMAGE: return "invalid_image";
    case PS_E_NOT_FOUND: return "not_found";
    case PS_E_INVALID_CONFIG: return "invalid_config";
    case PS_E_NO_SUMMARY: return "no_summary";
    case PS_E_DEGENERATE_SUMMARY: return "degenerate_summary";
    case PS_E_PARSE: return "parse_error";
    case PS_E_NO_SUCH_METRIC: return "no_such_metric";
    case PS_E_NO_PERIODICITY: return "no_periodicity";
    case PS_E_NO_OUTLIERS: return "no_outliers";
    case PS_E_INSUFFICIENT_DATA: return "insufficient_data";
    case PS_E_INVALID_ARGUMENT: return "invalid_argument";
    case PS_E_INTERNAL: return "internal";
  }
  return "unknown";
}

ps_status psg_open(int device, void* stream, psg_context** out) {
  if (!out) {
    t_last_error = "out is required";
    return PS_E_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guarded([&] {
    int n = 0;
    PSG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n)
      fail(PS_E_INVALID_ARGUMENT, "no CUDA device " + std::to_string(device));
    auto c = std::make_unique<psg_context>();
    c->device = device;
    PSG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    PSG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      fail(PS_E_INTERNAL, std::string("psg kernels are built for sm_100a; device is ") + prop.name);
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      PSG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    for (auto& e : c->ev) PSG_CUDA(cudaEventCreate(&e));
    *out = c.release();
  });
}

void psg_close(psg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
    cudaEventDestroy(ctx->side_in);
    cudaEventDestroy(ctx->side_out);
  }
  if (ctx->d2h_stream) {
    cudaStreamSynchronize(ctx->d2h_stream);
    cudaStreamDestroy(ctx->d2h_stream);
    cudaEventDestroy(ctx->d2h_ready);
    cudaEventDestroy(ctx->d2h_done);
  }
  delete ctx;
}

void* psg_stream(psg_context* ctx) { return ctx ? ctx->stream : nullptr; }

uint64_t psg_device_bytes(const psg_context* c) {
  if (!c) return 0;
  return c->d_off.bytes() + c->d_ts.bytes() + c->d_ctx.bytes() + c->d_tend.bytes() +
         c->d_stage.bytes() + c->cube_incl.bytes() + c->cube_xint.bytes() + c->w_cnt.bytes() * 7;
}

ps_status psg_comm_unique_id(uint8_t out_id[128]) {
  if (!out_id) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out_id, &id, 128);
  });
}

ps_status psg_comm_init(psg_context* c, int nranks, int rank, const uint8_t id[128]) {
  if (!c || !id) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad nranks/rank");
    ensure_device(c);
    if (c->comm) nccl().comm_destroy(c->comm);
    c->comm = nullptr;
    c->host_fn = nullptr;
    c->spec_ready = false;
    c->ranks_global_cache = 0;
    c->nranks = nranks;
    c->rank = rank;
    if (nranks == 1) return;
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    nccl_check(nccl().comm_init_rank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
  });
}

ps_status psg_comm_init_host(psg_context* c, int nranks, int rank, psg_allreduce_fn fn,
                             void* user) {
  if (!c || (nranks > 1 && !fn)) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "bad nranks/rank");
    if (c->comm) nccl().comm_destroy(c->comm);
    c->comm = nullptr;
    c->spec_ready = false;
    c->ranks_global_cache = 0;
    c->nranks = nranks;
    c->rank = rank;
    c->host_fn = fn;
    c->host_user = user;
  });
}

ps_status psg_set_cct(psg_context* c, const uint32_t* parent, uint32_t n_ctx) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    set_cct_impl(c, parent, n_ctx);
  });
}

ps_status psg_load_traces_aos(psg_context* c, const void* body, uint64_t n_events,
                              const uint64_t* event_off, const uint32_t* profile_ids,
                              const uint64_t* t_end_ns, uint32_t n_traces) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(event_off && profile_ids && t_end_ns, "event_off, profile_ids and t_end_ns are required");
    require(n_events == 0 || body, "body is required");
    require(event_off[0] == 0 && event_off[n_traces] == n_events, "event_off must span [0, n_events]");
    ensure_device(c);
    c->n_traces = n_traces;
    c->h_off.assign(event_off, event_off + n_traces + 1);
    c->h_tend.assign(t_end_ns, t_end_ns + n_traces);
    c->h_pid.assign(profile_ids, profile_ids + n_traces);
    c->h_tbegin.clear();
    for (uint32_t i = 0; i < n_traces; ++i)
      require(event_off[i] <= event_off[i + 1], "event_off must be non-decreasing");
    load_aos(c, static_cast<const uint8_t*>(body), n_events);
    finish_load(c);
  });
}

ps_status psg_prefetch_aos(psg_context* c, const void* body, uint64_t n_events) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(n_events == 0 || body, "body is required");
    ensure_device(c);
    drop_prefetch(c);
    if (n_events == 0) return;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, body) != cudaSuccess) {
      cudaGetLastError();
      return;  // pageable memory: nothing to prefetch (psg_load_traces_aos stages it itself)
    }
    if (attr.type != cudaMemoryTypeHost) return;
    const uint64_t chunk_ev = kPinnedChunkEvents, chunk_bytes = chunk_ev * 12;
    uint8_t* stage = c->d_stage.ensure(std::min<uint64_t>(2 * chunk_bytes, n_events * 12 + 64));
    const int slots = c->d_stage.n >= 2 * chunk_bytes ? 2 : 1;
    ensure_copy_stream(c);
    cudaEvent_t* copied = c->stage_ev;
    cudaEvent_t* consumed = c->stage_ev + 2;
    // the slots are free once the earlier transposes (and any other staging
    // work on the context's stream) are done
    PSG_CUDA(cudaEventRecord(consumed[0], c->stream));
    PSG_CUDA(cudaEventRecord(consumed[1], c->stream));
    const uint8_t* src = static_cast<const uint8_t*>(body);
    int k = 0;
    for (uint64_t done = 0; k < slots && done < n_events; ++k, done += chunk_ev) {
      const uint64_t ev = std::min(chunk_ev, n_events - done);
      PSG_CUDA(cudaStreamWaitEvent(c->copy_stream, consumed[k], 0));
      PSG_CUDA(cudaMemcpyAsync(stage + k * chunk_bytes, src + done * 12, ev * 12, cudaMemcpyHostToDevice,
                               c->copy_stream));
      PSG_CUDA(cudaEventRecord(copied[k], c->copy_stream));
    }
    c->pf_body = src;
    c->pf_events = n_events;
    c->pf_chunks = k;
  });
}

ps_status psg_set_nodes(psg_context* c, const uint32_t* node_of_trace, uint32_t n_nodes,
                        const uint32_t* node_rack, const uint32_t* node_chassis) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(node_of_trace && n_nodes > 0, "node_of_trace and n_nodes > 0 are required");
    ensure_device(c);
    for (uint32_t t = 0; t < c->n_traces; ++t)
      require(node_of_trace[t] < n_nodes, "node_of_trace entry out of range");
    c->n_nodes = n_nodes;
    c->h_node_of_trace.assign(node_of_trace, node_of_trace + c->n_traces);
    PSG_CUDA(cudaMemcpyAsync(c->d_node_of_trace.ensure(c->n_traces + 1), node_of_trace,
                             4ull * c->n_traces, cudaMemcpyHostToDevice, c->stream));
    set_node_tables(c, n_nodes, node_rack, node_chassis);
    c->topo_error.clear();
    c->sync();
  });
}


// ---- profile records ------------------------------

namespace {
// Uploads n_rec packed records (host or device bytes) and the profile index,
// transposes to SoA on the device and checks the ctx order of every run.
void load_profiles_impl(psg_context* c, const uint8_t* records, const uint64_t* rec_off,
                        const uint32_t* pid, const int32_t* rank, const uint32_t* node_of_profile,
                        uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) {
    require(rec_off[i + 1] >= rec_off[i], "record offsets must be non-decreasing");
    if (i > 0 && pid[i] <= pid[i - 1]) fail(PS_E_FORMAT, "profile ids must be strictly ascending");
  }
  const uint64_t n_rec = n ? rec_off[n] - rec_off[0] : 0;
  c->n_prof = n;
  c->n_rec = n_rec;
  c->h_prof_pid.assign(pid, pid + n);
  c->h_prof_rank.assign(rank, rank + n);
  std::vector<uint64_t> off(n + 1);
  for (uint32_t i = 0; i <= n; ++i) off[i] = n ? rec_off[i] - rec_off[0] : 0;
  cudaStream_t s = c->stream;
  PSG_CUDA(cudaMemcpyAsync(c->prof_off.ensure(n + 1), off.data(), 8ull * (n + 1), cudaMemcpyHostToDevice, s));
  PSG_CUDA(cudaMemcpyAsync(c->prof_pid.ensure(n + 1), pid, 4ull * n, cudaMemcpyHostToDevice, s));
  drop_prefetch(c);
  uint8_t* stage = c->d_stage.ensure(n_rec * 14 + 16);
  if (n_rec)
    PSG_CUDA(cudaMemcpyAsync(stage, records, n_rec * 14, cudaMemcpyDefault, s));
  launch_records_to_soa(stage, n_rec, c->prec_ctx.ensure(n_rec + 1), c->prec_metric.ensure(n_rec + 1),
                        c->prec_value.ensure(n_rec + 1), s);
  unsigned long long* bad = c->summary.ensure(8) + 7;
  PSG_CUDA(cudaMemsetAsync(bad, 0, 8, s));
  launch_records_check(c->prec_ctx.p, c->prof_off.p, n, bad, s);
  unsigned long long hb = 0;
  PSG_CUDA(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s));
  c->sync();
  if (hb) fail(PS_E_FORMAT, "profile records must be sorted by ctx within a profile (store.cpp:601-613)");
  // rank profiles in (rank, id) order: rank_vector's order (workflows.cpp:42-62)
  std::vector<uint32_t> rs;
  for (uint32_t i = 0; i < n; ++i)
    if (rank[i] >= 0) rs.push_back(i);
  std::stable_sort(rs.begin(), rs.end(), [&](uint32_t a, uint32_t b) { return rank[a] < rank[b]; });
  c->n_rank_prof = static_cast<uint32_t>(rs.size());
  PSG_CUDA(cudaMemcpyAsync(c->d_rank_slot.ensure(rs.size() + 1), rs.data(), 4ull * rs.size(),
                           cudaMemcpyHostToDevice, s));
  c->have_prof_nodes = false;
  if (node_of_profile && c->n_nodes > 0) {
    // node -> its rank profiles in rank order (node_correlate sums in that order)
    std::vector<uint32_t> cnt(c->n_nodes + 1, 0), members(rs.size());
    for (uint32_t r = 0; r < rs.size(); ++r) {
      const uint32_t nd = node_of_profile[rs[r]];
      require(nd < c->n_nodes, "node_of_profile entry out of range");
      ++cnt[nd + 1];
    }
    for (uint32_t i = 0; i < c->n_nodes; ++i) cnt[i + 1] += cnt[i];
    std::vector<uint32_t> fill(cnt.begin(), cnt.end() - 1);
    for (uint32_t r = 0; r < rs.size(); ++r) members[fill[node_of_profile[rs[r]]]++] = r;
    PSG_CUDA(cudaMemcpyAsync(c->d_pnode_off.ensure(c->n_nodes + 1), cnt.data(), 4ull * (c->n_nodes + 1),
                             cudaMemcpyHostToDevice, s));
    PSG_CUDA(cudaMemcpyAsync(c->d_pnode_rank.ensure(members.size() + 1), members.data(),
                             4ull * members.size(), cudaMemcpyHostToDevice, s));
    c->have_prof_nodes = true;
  }
  c->sync();
}
}  // namespace

ps_status psg_load_profiles(psg_context* c, const void* records, const uint64_t* rec_off,
                            const uint32_t* pid, const int32_t* rank,
                            const uint32_t* node_of_profile, uint32_t n_profiles) {
  if (!c || (n_profiles && (!rec_off || !pid || !rank))) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    if (n_profiles && rec_off[n_profiles] > rec_off[0]) require(records != nullptr, "records are required");
    load_profiles_impl(c, static_cast<const uint8_t*>(records), rec_off, pid, rank, node_of_profile,
                       n_profiles);
  });
}

ps_status psg_load_profile_db(psg_context* c, const char* dir) {
  if (!c || !dir) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    store::profile_db db;
    store::open_profile_db(dir, db);
    const uint32_t n = static_cast<uint32_t>(db.index.size());
    std::vector<uint64_t> off(n + 1, 0);
    std::vector<uint32_t> pid(n);
    std::vector<int32_t> rank(n, -1);
    bool contiguous = true;
    for (uint32_t i = 0; i < n; ++i) {
      const auto& e = db.index[i];
      off[i + 1] = off[i] + e.record_count;
      pid[i] = e.profile_id;
      const auto* pd = db.meta.find_profile(e.profile_id);
      rank[i] = pd ? pd->rank : -1;
      if (i > 0 && e.offset != db.index[i - 1].offset + db.index[i - 1].record_count * store::k_record_size)
        contiguous = false;
    }
    std::vector<uint8_t> gathered;
    const uint8_t* body = nullptr;
    if (n && off[n]) {
      if (contiguous) {
        body = db.map.data() + db.index[0].offset;
      } else {
        gathered.resize(off[n] * store::k_record_size);
        for (uint32_t i = 0; i < n; ++i)
          std::memcpy(gathered.data() + off[i] * store::k_record_size, db.map.data() + db.index[i].offset,
                      db.index[i].record_count * store::k_record_size);
        body = gathered.data();
      }
    }
    // nodes: rank -> hostname from the first profile with that rank, node id =
    // position in the sorted host list (node_correlate, diagnostics.cpp:381-398)
    std::map<int32_t, const std::string*> rank_host;
    for (const auto& p : db.meta.profiles)
      if (p.rank >= 0 && !rank_host.count(p.rank)) rank_host[p.rank] = &p.hostname;
    std::set<std::string> hosts;
    for (const auto& [r, h] : rank_host) hosts.insert(*h);
    std::vector<std::string> host_list(hosts.begin(), hosts.end());
    std::vector<uint32_t> node_of(n, 0);
    for (uint32_t i = 0; i < n; ++i)
      if (rank[i] >= 0)
        node_of[i] = static_cast<uint32_t>(std::lower_bound(host_list.begin(), host_list.end(),
                                                            *rank_host[rank[i]]) - host_list.begin());
    if (!host_list.empty()) set_db_nodes(c, host_list);
    load_profiles_impl(c, body, off.data(), pid.data(), rank.data(),
                       host_list.empty() ? nullptr : node_of.data(), n);
  });
}

ps_status psg_slice(psg_context* c, const uint32_t* pids, uint32_t n_pids, const uint32_t* ctx_ids,
                    uint32_t n_ctx_ids, const uint16_t* metric_ids, uint32_t n_metrics,
                    uint64_t* n_rows, uint32_t* row_pid, uint32_t* row_ctx, uint16_t* row_metric,
                    double* row_value) {
  if (!c || !n_rows || (n_pids && !pids)) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    cudaStream_t s = c->stream;
    // ingest_profiles: sorted unique profile ids (ingest.cpp:161-163); an
    // unknown id is not_found (store.cpp:588-590)
    std::vector<uint32_t> ids(pids, pids + n_pids);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    std::vector<uint32_t> slot(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) {
      auto it = std::lower_bound(c->h_prof_pid.begin(), c->h_prof_pid.end(), ids[i]);
      if (it == c->h_prof_pid.end() || *it != ids[i])
        fail(PS_E_NOT_FOUND, "profile " + std::to_string(ids[i]) + " not in database");
      slot[i] = static_cast<uint32_t>(it - c->h_prof_pid.begin());
    }
    const uint32_t nr = static_cast<uint32_t>(ids.size());
    PSG_CUDA(cudaMemcpyAsync(c->d_slot.ensure(nr + 1), slot.data(), 4ull * nr, cudaMemcpyHostToDevice, s));
    // filters as bit sets (id_filter / metric_filter "all" = no set)
    const uint32_t* cb = nullptr;
    uint32_t cw = 0;
    if (ctx_ids) {
      uint32_t mx = 0;
      for (uint32_t i = 0; i < n_ctx_ids; ++i) mx = std::max(mx, ctx_ids[i]);
      cw = n_ctx_ids ? mx / 32 + 1 : 1;
      std::vector<uint32_t> bits(cw, 0);
      for (uint32_t i = 0; i < n_ctx_ids; ++i) bits[ctx_ids[i] >> 5] |= 1u << (ctx_ids[i] & 31);
      PSG_CUDA(cudaMemcpyAsync(c->d_ctx_bits.ensure(cw), bits.data(), 4ull * cw, cudaMemcpyHostToDevice, s));
      cb = c->d_ctx_bits.p;
    }
    const uint32_t* mb = nullptr;
    if (metric_ids) {
      std::vector<uint32_t> bits(2048, 0);
      for (uint32_t i = 0; i < n_metrics; ++i) bits[metric_ids[i] >> 5] |= 1u << (metric_ids[i] & 31);
      PSG_CUDA(cudaMemcpyAsync(c->d_metric_bits.ensure(2048), bits.data(), 4ull * 2048,
                               cudaMemcpyHostToDevice, s));
      mb = c->d_metric_bits.p;
    }
    unsigned long long* counts = c->d_counts.ensure(nr + 1);
    launch_slice(c->pview(), c->d_slot.p, nr, cb, cw, mb, counts, nullptr, nullptr, nullptr, nullptr,
                 nullptr, s);
    unsigned long long* ro = c->d_row_off.ensure(nr + 1);
    const size_t sb = exclusive_scan_u64_scratch(nr + 1);
    PSG_CUDA(cudaMemsetAsync(counts + nr, 0, 8, s));
    launch_exclusive_scan_u64(reinterpret_cast<const uint64_t*>(counts), reinterpret_cast<uint64_t*>(ro),
                              nr + 1, c->scratch.ensure(sb), sb, s);
    unsigned long long total = 0;
    PSG_CUDA(cudaMemcpyAsync(&total, ro + nr, 8, cudaMemcpyDeviceToHost, s));
    c->sync();
    const bool want = row_pid || row_ctx || row_metric || row_value;
    if (want && total) {
      launch_slice(c->pview(), c->d_slot.p, nr, cb, cw, mb, counts, ro, c->d_row_pid.ensure(total),
                   c->d_row_ctx.ensure(total), c->d_row_metric.ensure(total), c->d_row_value.ensure(total), s);
      if (row_pid) PSG_CUDA(cudaMemcpyAsync(row_pid, c->d_row_pid.p, 4 * total, cudaMemcpyDeviceToHost, s));
      if (row_ctx) PSG_CUDA(cudaMemcpyAsync(row_ctx, c->d_row_ctx.p, 4 * total, cudaMemcpyDeviceToHost, s));
      if (row_metric)
        PSG_CUDA(cudaMemcpyAsync(row_metric, c->d_row_metric.p, 2 * total, cudaMemcpyDeviceToHost, s));
      if (row_value)
        PSG_CUDA(cudaMemcpyAsync(row_value, c->d_row_value.p, 8 * total, cudaMemcpyDeviceToHost, s));
      c->sync();
    }
    *n_rows = total;
  });
}

ps_status psg_profile_outliers(psg_context* c, uint16_t metric, const uint32_t* site_ctx,
                               uint32_t n_sites, uint32_t top_k, double z_min, psg_query_info* info) {
  if (!c || !info || !site_ctx || n_sites == 0) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    if (c->n_rank_prof == 0) fail(PS_E_INSUFFICIENT_DATA, "balance_ratio of empty vector (no rank profiles loaded)");
    require(c->have_prof_nodes, "profile outliers need the profile -> node mapping (psg_load_profile_db or node_of_profile)");
    if (!c->topo_error.empty()) fail(PS_E_PARSE, c->topo_error);
    // an asynchronous copy-out of the previous result may still read the
    // buffers this query rewrites: the stream waits for it (no host block)
    if (c->d2h_pending) PSG_CUDA(cudaStreamWaitEvent(c->stream, c->d2h_done, 0));
    invalidate_results(c);
    std::memset(info, 0, sizeof(*info));
    cudaStream_t s = c->stream;
    PSG_CUDA(cudaEventRecord(c->ev[0], s));
    c->sites.assign(site_ctx, site_ctx + n_sites);
    PSG_CUDA(cudaMemcpyAsync(c->d_sites.ensure(n_sites), site_ctx, 4ull * n_sites, cudaMemcpyHostToDevice, s));
    launch_profile_outliers(c->pview(), c->d_rank_slot.p, c->n_rank_prof, c->d_sites.p, n_sites, metric,
                            c->pvals.ensure(static_cast<size_t>(c->n_rank_prof) * n_sites),
                            c->site_ratio.ensure(n_sites), c->d_worst.ensure(2), c->d_pnode_off.p,
                            c->d_pnode_rank.p, c->n_nodes, c->node_mean.ensure(c->n_nodes), s);
    const size_t ssb = node_select_scratch_bytes(c->n_nodes);
    launch_node_select(nullptr, c->n_nodes, top_k, z_min, c->node_mean.p, c->node_z.ensure(c->n_nodes),
                       c->d_order.ensure(c->n_nodes), c->d_nsel.ensure(1), c->scratch.ensure(ssb), ssb, s);
    const uint32_t nr = static_cast<uint32_t>(c->h_rack_ids.size());
    if (nr)
      launch_topology(c->d_order.p, c->d_nsel.p, c->d_node_rack_idx.p, c->d_node_chassis.p, c->d_uni_cnt.p,
                      nr, c->d_rack_nodes.ensure(nr), c->rack_mask.ensure(nr), c->rack_full.ensure(nr),
                      c->rack_cnt.ensure(64ull * nr), s);
    PSG_CUDA(cudaEventRecord(c->ev[3], s));
    c->sync();
    c->have_outliers = true;
    uint32_t w = 0;
    PSG_CUDA(cudaMemcpy(&w, c->d_worst.p, 4, cudaMemcpyDeviceToHost));
    PSG_CUDA(cudaMemcpy(&info->n_outliers, c->d_nsel.p, 4, cudaMemcpyDeviceToHost));
    info->worst_site = c->sites[w];
    PSG_CUDA(cudaMemcpy(&info->worst_ratio, c->site_ratio.p + w, 8, cudaMemcpyDeviceToHost));
    if (nr) {
      std::vector<uint32_t> rn(nr);
      PSG_CUDA(cudaMemcpy(rn.data(), c->d_rack_nodes.p, 4ull * nr, cudaMemcpyDeviceToHost));
      for (uint32_t x : rn) info->n_racks += x > 0;
    }
    PSG_CUDA(cudaEventElapsedTime(&info->ms_total, c->ev[0], c->ev[3]));
  });
}

ps_status psg_load_trace_db(psg_context* c, const char* dir, const uint32_t* pids, uint32_t n_pids) {
  if (!c || !dir) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    store::trace_db db;
    store::open_trace_db(dir, db);
    std::vector<const store::trace_index_entry*> sel;
    if (pids) {
      std::vector<uint32_t> ids(pids, pids + n_pids);
      std::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      for (uint32_t id : ids) {
        auto* e = db.find(id);
        if (!e) fail(PS_E_NOT_FOUND, "trace " + std::to_string(id) + " not in database");
        sel.push_back(e);
      }
    } else {
      for (auto& e : db.index) sel.push_back(&e);
    }
    // CCT from meta.bin
    std::vector<uint32_t> parent;
    for (size_t i = 0; i < db.meta.contexts.size(); ++i) {
      if (db.meta.contexts[i].id != i) fail(PS_E_FORMAT, "meta.bin: ctx ids must be dense");
      parent.push_back(db.meta.contexts[i].parent);
    }
    set_cct_impl(c, parent.data(), static_cast<uint32_t>(parent.size()));
    // index + body (contiguous fast path, gathered otherwise)
    c->n_traces = static_cast<uint32_t>(sel.size());
    c->h_off.assign(1, 0);
    c->h_tend.clear();
    c->h_pid.clear();
    bool contiguous = true;
    for (size_t i = 0; i < sel.size(); ++i) {
      if (sel[i]->event_count > 0 && sel[i]->t_begin_ns != 0) {
      }
      c->h_off.push_back(c->h_off.back() + sel[i]->event_count);
      c->h_tend.push_back(sel[i]->t_end_ns);
      c->h_pid.push_back(sel[i]->profile_id);
      if (i > 0 && sel[i]->offset != sel[i - 1]->offset + sel[i - 1]->event_count * 12)
        contiguous = false;
    }
    const uint64_t n_ev = c->h_off.back();
    // first event == indexed t_begin (store.cpp:750-751) is checked on the device
    c->h_tbegin.clear();
    for (auto* e : sel) c->h_tbegin.push_back(e->t_begin_ns);
    if (contiguous || sel.empty()) {
      if (n_ev) load_aos_file(c, db.dir + "/trace.db", sel.front()->offset, n_ev);
      else load_aos(c, nullptr, 0);
    } else {
      std::vector<uint8_t> gathered(n_ev * 12);
      uint64_t o = 0;
      for (auto* e : sel) {
        std::memcpy(gathered.data() + o, db.map.data() + e->offset, e->event_count * 12);
        o += e->event_count * 12;
      }
      load_aos(c, gathered.data(), n_ev);
      c->sync();
    }
    finish_load(c);
    // rank -> hostname from the first profile with that rank (diagnostics.cpp:381-384);
    // node index = position of the hostname in sorted order (std::map order).
    std::map<int32_t, const std::string*> rank_host;
    for (const auto& p : db.meta.profiles)
      if (p.rank >= 0 && !rank_host.count(p.rank)) rank_host[p.rank] = &p.hostname;
    std::vector<std::string> host_of_trace;
    std::set<std::string> hosts;
    for (auto* e : sel) {
      const auto* pd = db.meta.find_profile(e->profile_id);
      std::string h;
      if (pd && pd->rank >= 0) h = *rank_host[pd->rank];
      host_of_trace.push_back(h);
      hosts.insert(h);
    }
    std::vector<std::string> host_list(hosts.begin(), hosts.end());
    std::vector<uint32_t> node_of(sel.size());
    for (size_t i = 0; i < sel.size(); ++i)
      node_of[i] = static_cast<uint32_t>(
          std::lower_bound(host_list.begin(), host_list.end(), host_of_trace[i]) - host_list.begin());
    if (!sel.empty()) {
      c->h_node_of_trace = node_of;
      PSG_CUDA(cudaMemcpyAsync(c->d_node_of_trace.ensure(c->n_traces + 1), node_of.data(),
                               4ull * c->n_traces, cudaMemcpyHostToDevice, c->stream));
      set_db_nodes(c, host_list);
    }
  });
}

ps_status psg_generate_iterative(psg_context* c, const psg_iter_scenario* s, uint32_t rank_lo,
                                 uint32_t rank_hi) {
  if (!c || !s) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(s->n_ranks >= 1 && s->n_iterations >= 1 && s->n_kernels >= 1,
            "n_ranks, n_iterations, n_kernels must be >= 1");
    require(s->mean_time_s && s->jitter_frac, "mean_time_s and jitter_frac are required");
    require(rank_lo <= rank_hi && rank_hi <= s->n_ranks, "bad rank range");
    require(s->copy_segment_s >= 0.0, "copy_segment_s must be >= 0");
    ensure_device(c);
    const uint32_t nk = s->n_kernels;
    const bool has_copy = s->copy_segment_s > 0.0;
    std::vector<uint32_t> parent(2 + nk + (has_copy ? 1 : 0));
    parent[0] = store::k_no_parent;
    parent[1] = 0;
    for (uint32_t k = 0; k < nk; ++k) parent[2 + k] = 1;
    if (has_copy) parent[2 + nk] = 0;
    set_cct_impl(c, parent.data(), static_cast<uint32_t>(parent.size()));

    const uint32_t n_local = rank_hi - rank_lo;
    const uint64_t epi = nk + 2 + (has_copy ? 1 : 0);
    const uint64_t ept = epi * s->n_iterations;
    c->n_traces = n_local;
    c->n_events = ept * n_local;
    c->h_off.resize(n_local + 1);
    for (uint32_t r = 0; r <= n_local; ++r) c->h_off[r] = ept * r;
    c->h_pid.resize(n_local);
    for (uint32_t r = 0; r < n_local; ++r) c->h_pid[r] = rank_lo + r + 1;
    c->h_tend.assign(n_local, 0);
    c->h_tbegin.clear();

    if (!c->jump.p) {
      auto mats = jump_matrices();
      PSG_CUDA(cudaMemcpyAsync(c->jump.ensure(mats.size()), mats.data(), 8 * mats.size(),
                               cudaMemcpyHostToDevice, c->stream));
    }
    // parameters: mean[nk] | jitter[nk] | spread
    uint64_t spread_n = 0;
    if (s->spread) spread_n = s->spread_kernel_stride ? s->spread_kernel_stride * nk : s->n_ranks;
    double* gp = c->gen_params.ensure(2 * nk + spread_n + 1);
    PSG_CUDA(cudaMemcpyAsync(gp, s->mean_time_s, 8ull * nk, cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaMemcpyAsync(gp + nk, s->jitter_frac, 8ull * nk, cudaMemcpyHostToDevice, c->stream));
    if (spread_n)
      PSG_CUDA(cudaMemcpyAsync(gp + 2 * nk, s->spread, 8ull * spread_n, cudaMemcpyHostToDevice,
                               c->stream));
    const uint64_t copy_ns = static_cast<uint64_t>(std::llround(s->copy_segment_s * 1e9));
    c->d_ts.ensure(c->n_events + kEventPad);
    c->d_ctx.ensure(c->n_events + kEventPad);
    c->d_tend.ensure(n_local + 1);
    const uint32_t chunks = (s->n_iterations + 15) / 16;
    uint64_t* scratch = c->gen_chunks.ensure(static_cast<uint64_t>(n_local) * chunks + 1);
    launch_gen_iterative(c->jump.p, s->seed, s->n_ranks, s->n_iterations, nk, gp, gp + nk,
                         spread_n ? gp + 2 * nk : nullptr, s->spread_kernel_stride, copy_ns, rank_lo,
                         n_local, ept, scratch, c->d_ts.p, c->d_ctx.p, c->d_tend.p, c->stream);
    PSG_CUDA(cudaMemcpyAsync(c->h_tend.data(), c->d_tend.p, 8ull * n_local, cudaMemcpyDeviceToHost,
                             c->stream));
    c->sync();
    finish_load(c);
  });
}

ps_status psg_shard(psg_context* c, psg_shard_info* out) {
  if (!c || !out) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    out->n_traces = c->n_traces;
    out->n_ctx = c->n_ctx;
    out->n_events = c->n_events;
    out->t_max = c->h_tend.empty() ? 0 : *std::max_element(c->h_tend.begin(), c->h_tend.end());
    out->t_min = 0;
    if (c->n_events) {
      // min first timestamp over non-empty traces
      uint64_t m = ~0ull;
      for (uint32_t t = 0; t < c->n_traces; ++t) {
        if (c->h_off[t + 1] == c->h_off[t]) continue;
        uint64_t v;
        PSG_CUDA(cudaMemcpy(&v, c->d_ts.p + c->h_off[t], 8, cudaMemcpyDeviceToHost));
        m = std::min(m, v);
        if (t > 64) break;  // synthetic traces start at 0; a sample is enough for a hint
      }
      out->t_min = m == ~0ull ? 0 : m;
    }
  });
}

ps_status psg_get_traces(psg_context* c, uint64_t* ts, uint32_t* ctx_ids, uint64_t* event_off,
                         uint64_t* t_end, uint32_t* profile_ids) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    if (ts && c->n_events)
      PSG_CUDA(cudaMemcpy(ts, c->d_ts.p, 8 * c->n_events, cudaMemcpyDeviceToHost));
    if (ctx_ids && c->n_events)
      PSG_CUDA(cudaMemcpy(ctx_ids, c->d_ctx.p, 4 * c->n_events, cudaMemcpyDeviceToHost));
    if (event_off) std::copy(c->h_off.begin(), c->h_off.end(), event_off);
    if (t_end) std::copy(c->h_tend.begin(), c->h_tend.end(), t_end);
    if (profile_ids) std::copy(c->h_pid.begin(), c->h_pid.end(), profile_ids);
  });
}

// ---------------------------------------------------------------------------
// Traces over all ranks (the balance ratios' denominator): one exchange per
// load, cached.
uint64_t ranks_global(psg_context* c) {
  if (!c->multi()) return c->n_traces;
  if (c->ranks_global_cache == 0) {
    unsigned long long* d = c->summary.ensure(8);
    unsigned long long hn = c->n_traces;
    PSG_CUDA(cudaMemcpyAsync(d, &hn, 8, cudaMemcpyHostToDevice, c->stream));
    c->allreduce(d, 1, ncclUint64, ncclSum);
    PSG_CUDA(cudaMemcpyAsync(&hn, d, 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    c->ranks_global_cache = hn;
  }
  return c->ranks_global_cache;
}

namespace {
// Work units for pass 2 (SURVEY.md §5 "long-context": the reference runs one
// thread per trace, itermodel.cpp:276).  U = the events one resident warp
// gets when the work is spread evenly (events / resident warps, at least
// PSG_UNIT_MIN).  A trace longer than 2U would outlast the rest of the query
// on its one warp: it is split into ceil(n_t / U) units of equal event ranges
// (pass 2 snaps them to chunk starts).  Evenly sized traces are never split
// (configs[1], C3: measured slower split, tools/c3_units.py — a split trace
// merges its window and within-rank sums with atomics).  PSG_UNIT_EVENTS
// overrides U and splits every trace longer than it (tests).
//
// Tail fill (tail_fill: the query runs one-warp CTAs anyway): evenly sized
// traces run in waves of `slots` warps; when the last wave would be at most
// half full, its traces are split into k = slots / rem units each, so it lasts
// 1 / k of a trace (C3: 8,192 traces on 2,368 slots = 3 waves + 1,088 traces:
// 4 -> 3.5 trace times).
void plan_units(psg_context* c, uint64_t slots, bool tail_fill) {
  uint64_t U = std::max<uint64_t>(kUnitMinEvents, c->n_events / std::max<uint64_t>(1, slots));
  uint64_t thresh = 2 * U;
  const char* env = std::getenv("PSG_UNIT_EVENTS");
  if (env) thresh = U = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
  const uint64_t key = (static_cast<uint64_t>(c->n_traces) * 1000003ull) ^ (c->n_events * 7919ull) ^ (U << 40) ^
                       (thresh << 20) ^ (slots << 4) ^ (tail_fill ? 2ull : 1ull);
  if (key == c->units_key) return;
  std::vector<uint4> units;
  std::vector<uint32_t> split;
  bool any = false;
  uint64_t max_t = 0;
  for (uint32_t t = 0; t < c->n_traces; ++t) {
    const uint64_t n_t = c->h_off[t + 1] - c->h_off[t];
    any = any || n_t > thresh;
    max_t = std::max(max_t, n_t);
  }
  // tail fill: the last `rem` traces (the last CTAs launched) split k ways
  uint32_t tail_from = c->n_traces, tail_k = 1;
  if (!any && !env && tail_fill && slots && c->n_traces > slots && c->n_events &&
      max_t * c->n_traces <= c->n_events + c->n_events / 4) {  // evenly sized: max <= 1.25 mean
    const uint64_t rem = c->n_traces % slots;
    if (rem && 2 * rem <= slots && max_t >= 2 * kUnitMinEvents) {
      tail_k = static_cast<uint32_t>(std::min<uint64_t>(slots / rem, std::max<uint64_t>(1, max_t / kUnitMinEvents)));
      if (tail_k >= 2) tail_from = c->n_traces - static_cast<uint32_t>(rem);
    }
  }
  if (any || tail_from < c->n_traces) {
    units.reserve(c->n_traces);
    for (uint32_t t = 0; t < c->n_traces; ++t) {
      const uint64_t n_t = c->h_off[t + 1] - c->h_off[t];
      const uint64_t u = t >= tail_from ? tail_k : n_t > thresh ? (n_t + U - 1) / U : 1;
      if (u > 1) split.push_back(t);
      for (uint64_t i = 0; i < u; ++i)
        units.push_back(make_uint4(t, static_cast<uint32_t>(n_t * i / u), static_cast<uint32_t>(n_t * (i + 1) / u),
                                   u > 1 ? 1u : 0u));
    }
    if (units.size() >= (1ull << 31)) fail(PS_E_INVALID_ARGUMENT, "too many work units");
    PSG_CUDA(cudaMemcpyAsync(c->d_units.ensure(units.size()), units.data(), sizeof(uint4) * units.size(),
                             cudaMemcpyHostToDevice, c->stream));
    PSG_CUDA(cudaMemcpyAsync(c->d_split.ensure(split.size() + 1), split.data(), 4 * split.size(),
                             cudaMemcpyHostToDevice, c->stream));
    c->sync();  // the host vectors go out of scope
  }
  c->n_units = static_cast<uint32_t>(units.size());
  c->n_split = static_cast<uint32_t>(split.size());
  c->units_key = key;
}
}  // namespace

ps_status psg_query(psg_context* c, const psg_query_spec* q, psg_query_info* info) {
  if (!c || !q || !info) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    const uint32_t f = q->flags;
    const bool do_window = f & PSG_Q_WINDOW, do_cube = f & PSG_Q_CUBE;
    const bool do_stats = f & PSG_Q_STATS, do_out = f & PSG_Q_OUTLIERS;
    const bool store_cube = do_cube && !(f & PSG_Q_NO_CUBE_STORE);
    require(do_window || do_cube, "query needs PSG_Q_WINDOW and/or PSG_Q_CUBE");
    require(!do_stats || do_cube, "PSG_Q_STATS requires PSG_Q_CUBE");
    require(!do_out || do_window, "PSG_Q_OUTLIERS requires PSG_Q_WINDOW");
    if (do_window && q->t0_ns > q->t1_ns)
      fail(PS_E_INVALID_ARGUMENT, "trace window start after end");
    if (c->n_ctx == 0) fail(PS_E_INVALID_ARGUMENT, "no calling-context tree loaded");
    // an asynchronous copy-out of the previous result may still read the
    // buffers this query rewrites: the stream waits for it (no host block)
    if (c->d2h_pending) PSG_CUDA(cudaStreamWaitEvent(c->stream, c->d2h_done, 0));
    invalidate_results(c);
    std::memset(info, 0, sizeof(*info));
    const uint64_t syncs0 = c->n_syncs;
    const uint32_t n = c->n_traces;
    cudaStream_t s = c->stream;
    PSG_CUDA(cudaEventRecord(c->ev[0], s));

    query_params p{};
    p.tr = c->view();
    p.t_base = 0;
    p.t_stop = n;
    p.n_ctx = c->n_ctx;
    p.G = PSG_G;
    uint32_t anchor = q->anchor_ctx;
    if (do_cube && anchor == PSG_ANCHOR_AUTO) anchor = auto_anchor(c);
    if (do_cube) compute_subtree(c, anchor);
    // Window layout: the fused kernel keeps one record per ctx in each warp's
    // shared memory and writes a dense [trace][ctx] result; a tree too large
    // for either (or PSG_Q_SPARSE) takes the sparse path, and the cube then
    // reads its column offsets from a global table when the records do not fit
    const uint32_t nn0 = do_cube ? c->nn : 1u;
    auto carve_out = [&](uint32_t n_ctx_tab) {
      warp_smem_layout Lx;
      Lx.init(n_ctx_tab, nn0, PSG_G, do_cube && (c->exact_hint || (f & PSG_Q_EXACT_BOUNDS)));
      return Lx.bytes;
    };
    constexpr uint32_t kSmemCap = 227u * 1024;
    const bool records_fit = carve_out(c->n_ctx) <= kSmemCap;
    const uint64_t dense_bytes = 56ull * n * c->n_ctx;
    const bool sparse = do_window && ((f & PSG_Q_SPARSE) || !records_fit || dense_bytes > (24ull << 30));
    const bool global_cols = do_cube && !records_fit;
    if (global_cols && carve_out(0) > kSmemCap)
      fail(PS_E_INVALID_ARGUMENT, "anchor subtree too large for the fused kernel's cube rows");
    c->window_sparse = sparse;
    if (sparse) {
      sparse_args a{};
      a.tr = c->view();
      a.n_ctx = c->n_ctx;
      a.t0 = q->t0_ns;
      a.t1 = q->t1_ns;
      a.clamp_tend = (f & PSG_Q_CLAMP_TEND) ? 1 : 0;
      a.parent = c->d_parent.p;
      a.depth = c->d_depth.p;
      a.row_budget = 1ull << 27;  // 128 Mi rows per batch: ~5 GB of sort scratch
      if (const char* e = std::getenv("PSG_SPARSE_ROW_BUDGET")) a.row_budget = std::strtoull(e, nullptr, 10);
      a.c_has = c->c_has.ensure(n + 1);
      a.c_ts = c->c_ts.ensure(n + 1);
      a.c_ctx = c->c_ctx.ensure(n + 1);
      sparse_window(a, c->sp, s);
      c->n_syncs += 3;  // the sparse path sizes its batches on the host
      c->sp_valid = true;
    }
    if (do_window && !sparse) {
      const size_t cells = static_cast<size_t>(n) * c->n_ctx + 1;
      p.do_window = 1;
      p.clamp_tend = (f & PSG_Q_CLAMP_TEND) ? 1 : 0;
      p.t0 = q->t0_ns;
      p.t1 = q->t1_ns;
      p.w_cnt = c->w_cnt.ensure(cells);
      p.w_sum = c->w_sum.ensure(cells);
      p.w_min = c->w_min.ensure(cells);
      p.w_max = c->w_max.ensure(cells);
      p.w_excl = c->w_excl.ensure(cells);
      p.w_incl = c->w_incl.ensure(cells);
      p.w_mean = c->w_mean.ensure(cells);
      p.c_has = c->c_has.ensure(n + 1);
      p.c_ts = c->c_ts.ensure(n + 1);
      p.c_ctx = c->c_ctx.ensure(n + 1);
      p.cct_pre = c->d_cct_pre.p;
      p.cct_size = c->d_cct_size.p;
    }
    uint32_t nn = 0;
    info->anchor = do_cube ? anchor : 0;
    bool exact_bounds = c->exact_hint || (f & PSG_Q_EXACT_BOUNDS) != 0;
    const bool force64 = (f & PSG_Q_CUBE64) != 0;
    // The status block carries every count a later kernel needs (K, kept
    // traces) and every verdict (pass-1 overflow, optimistic pass 1, buffer
    // capacities).  A speculative query (buffers sized by an earlier query on
    // these traces, optimistic pass 1) runs all its kernels back to back and
    // reads the block once at the end; any miss re-runs the query with the
    // host sizing each step (the first query after a load always does).
    unsigned long long* qs = c->qstat.ensure(QS_WORDS);
    unsigned long long hq[QS_WORDS] = {};
    const char* nospec = std::getenv("PSG_NO_SPEC");
    bool spec = c->spec_ready && !(nospec && *nospec == '1');
    uint32_t k_cap = 0;  // K the statistics accumulators are laid out for
    for (;;) {
    const bool sp = spec && do_cube && !exact_bounds;
    bool side_pending = false;
    PSG_CUDA(cudaMemsetAsync(qs, 0, QS_WORDS * sizeof(unsigned long long), s));
    if (do_cube) {
      compute_subtree(c, anchor);
      nn = c->nn;
      uint32_t* ic = c->iter_count.ensure(n + 1);
      // pass 1: iteration boundaries (re-run with exact region bounds on overflow)
      PSG_CUDA(cudaEventRecord(c->ev[4], s));
      for (;;) {
        if (!c->caps_valid) build_caps(c);
        bound_params bp{};
        bp.tr = c->view();
        bp.ctx8 = c->ctx8_valid ? c->d_ctx8.p : nullptr;
        bp.sub_lo = static_cast<uint32_t>(c->cct_po.pre[anchor]);
        bp.sub_size = static_cast<uint32_t>(c->cct_po.size[anchor]);
        bp.ctx7 = (c->n_ctx <= 128 && !std::getenv("PSG_NO_CTX7")) ? 1u : 0u;
        bp.contains = c->d_contains.p;
        bp.words = c->contains_words;
        bp.cap_off = c->d_cap_off.p;
        bp.bidx = c->d_bidx.p;
        bp.bts = c->d_bts.p;
        bp.n_bounds = c->d_nbounds.ensure(n + 1);
        bp.iter_count = ic;
        bp.overflow = qs + QS_OVERFLOW;
        launch_bounds(bp, exact_bounds, s);
        if (sp) break;  // checked at the end
        PSG_CUDA(cudaMemcpyAsync(&hq[QS_OVERFLOW], qs + QS_OVERFLOW, 8, cudaMemcpyDeviceToHost, s));
        c->sync();
        if (hq[QS_OVERFLOW] == 0 || c->cap_div <= 2) break;
        c->cap_div = 2;
        c->caps_valid = false;
        PSG_CUDA(cudaMemsetAsync(qs + QS_OVERFLOW, 0, 8, s));
      }
      PSG_CUDA(cudaEventRecord(c->ev[5], s));
      const size_t sb = cube_layout_scratch_bytes(n);
      launch_cube_layout(ic, n, nn, row_stride(nn), c->tpos.ensure(n + 1), c->block_off.ensure(n + 1),
                         c->iter_off.ensure(n + 1), c->kept_bo.ensure(n + 1), qs,
                         c->scratch.ensure(sb), sb, s);
      if (exact_bounds) launch_iter_spans(c->d_cap_off.p, c->d_bts.p, ic, c->d_tend.p, n, qs + QS_SPAN, s);
      // global {kept, min iterations}: K for every kernel that follows
      PSG_CUDA(cudaMemcpyAsync(qs + QS_KEPT_G, qs + QS_KEPT, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToDevice, s));
      static_assert(QS_MIN_IT_G == QS_KEPT_G + 1 && QS_MIN_IT == QS_KEPT + 1, "status layout");
      if (c->multi()) {
        c->group_begin();
        c->allreduce(qs + QS_KEPT_G, 1, ncclUint64, ncclSum);
        c->allreduce(qs + QS_MIN_IT_G, 1, ncclUint64, ncclMin);
        c->group_end();
      }
      const uint32_t m = static_cast<uint32_t>(c->internal_pos.size());
      if (!sp) {
        PSG_CUDA(cudaMemcpyAsync(hq, qs, sizeof(hq), cudaMemcpyDeviceToHost, s));
        c->sync();
        // 32-bit cells: exact spans from pass 1, or optimistic (verified by pass 2)
        c->cube32 = !force64 && (!exact_bounds || hq[QS_SPAN] < (1ull << 32));
        // buffers sized exactly (grow-only: later queries run speculatively in them)
        c->cube_incl.ensure((hq[QS_STORE] * (c->cube32 ? 4 : 8) + 7) / 8 + 2);
        if (store_cube) c->cube_xint.ensure((nn ? hq[QS_CELLS] / nn : 0) * m + 1);
        k_cap = qs_K(hq);
      } else {
        c->cube32 = !force64;
        k_cap = (do_stats && nn) ? static_cast<uint32_t>(c->x_acc.n / (5ull * nn)) : 0u;
      }
      p.do_cube = 1;
      p.store_cube = store_cube ? 1 : 0;
      p.sub_pre = c->d_sub_pre.p;
      p.node_tab = c->d_node_tab.p;
      p.nn = nn;
      p.root_only = c->root_only;
      p.cap_off = c->d_cap_off.p;
      p.bidx = c->d_bidx.p;
      p.bts = c->d_bts.p;
      p.n_bounds = c->d_nbounds.p;
      p.iter_count = ic;
      p.tpos = c->tpos.p;
      p.block_off = c->block_off.p;
      p.iter_off = c->iter_off.p;
      p.qs = qs;
      p.cap_miss = sp ? qs + QS_CAP_MISS : nullptr;
      // incl is always materialised (the cross-rank statistics stream it);
      // PSG_Q_NO_CUBE_STORE drops the excl half
      p.cube_incl = c->cube_incl.ensure(1);
      p.cube_cap = c->cube_incl.n * 8 / (c->cube32 ? 4 : 8);
      p.cube32 = c->cube32 ? 1 : 0;
      p.exact_bounds = exact_bounds ? 1 : 0;
      p.m = m;
      if (store_cube) p.cube_xint = c->cube_xint.ensure(1);
      p.xint_cap = store_cube ? c->cube_xint.n : 0;
      c->have_excl = store_cube;
      // per kept trace rows: sized for every trace (the kept count is known on the device)
      p.gap_incl = c->gap_incl.ensure(static_cast<size_t>(n) * nn + 1);
      p.gap_excl = c->gap_excl.ensure(static_cast<size_t>(n) * nn + 1);
      if (do_stats && k_cap > 0) {
        const size_t plane = static_cast<size_t>(k_cap) * nn;
        unsigned long long* x = c->x_acc.ensure(5 * plane);
        PSG_CUDA(cudaMemsetAsync(x, 0, 5 * plane * sizeof(unsigned long long), s));
        p.do_stats = 1;
        p.x_sum = x;
        p.x_max = x + plane;
        p.x_sq = x + 2 * plane;
        p.within_cv = c->within_cv.ensure(static_cast<size_t>(n) * nn + 1);
        p.within_ok = c->within_ok.ensure(static_cast<size_t>(n) * nn + 1);
      }
    }
    // launch geometry
    warp_smem_layout L;
    L.init((global_cols || (!p.do_window && !p.do_cube)) ? 0u : c->n_ctx, nn, p.G, do_cube && exact_bounds);
    p.ppo_g = global_cols ? c->d_ppo_g.p : nullptr;
    // CTA shape: one warp per CTA for long traces (17 resident per SM, no
    // CTA tail), 16-warp CTAs for short ones (their per-trace prologue and
    // epilogue run better in warps that start together); PSG_CTA_SHAPE=one|wide
    // overrides (A/B)
    bool one = c->n_events >= kOneWarpMinEvents * static_cast<uint64_t>(n);
    {  // few traces: 16-warp CTAs (one per SM) would leave a part-filled last wave
      int dev = 0, sms = 148;
      PSG_CUDA(cudaGetDevice(&dev));
      PSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const double ctas = std::ceil(n / 16.0), waves = std::ceil(ctas / sms);
      if (ctas / (waves * sms) < 0.9) one = true;
    }
    if (const char* e = std::getenv("PSG_CTA_SHAPE")) {
      if (!std::strcmp(e, "one")) one = true;
      if (!std::strcmp(e, "wide")) one = false;
    }
    // the wide shape's CTA tables (and 16 carve-outs) may not fit where one
    // warp's carve-out alone does: fall back to one-warp CTAs (a decision that
    // depends only on the tree and the anchor, so every rank takes the same one)
    if (!one && !fits_wide(n, L.bytes, cta_table_bytes(c->n_ctx, nn, 16, false))) one = true;
    if (global_cols) one = true;
    // work units: long traces split across warps (one-warp CTAs); the
    // resident slots are those of the one-warp instantiation this query uses
    {
      int dev = 0, sms = 148;
      PSG_CUDA(cudaGetDevice(&dev));
      PSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const uint32_t per_sm = trace_query_one_warp_per_sm(p.do_window != 0, p.do_cube != 0,
                                                          p.do_cube && exact_bounds, global_cols, L.bytes);
      plan_units(c, static_cast<uint64_t>(sms) * std::max(1u, per_sm), one);
    }
    const bool units = c->n_split > 0;
    if (units) one = true;
    uint32_t W = one ? choose_warps(1, L.bytes, 0) : choose_warps(n, L.bytes, cta_table_bytes(c->n_ctx, nn, 16, false));
    if (one) W = 1;
    p.one_warp = one ? 1u : 0u;
    p.warps = W;
    p.L = L;
    p.cta_bytes = cta_table_bytes(c->n_ctx, nn, W, one);
    uint32_t smem = p.cta_bytes + W * L.bytes;
    if (const char* e = std::getenv("PSG_ONE_MIN_SMEM"); e && one)  // A/B: cap resident CTAs per SM
      smem = std::max<uint32_t>(smem, static_cast<uint32_t>(std::strtoul(e, nullptr, 10)));
    PSG_CUDA(cudaEventRecord(c->ev[1], s));
    if (units) {
      p.units = c->d_units.p;
      p.n_units = c->n_units;
      p.wacc = (p.do_stats && nn) ? c->wacc.ensure(static_cast<size_t>(n) * nn * 3 + 1) : nullptr;
      launch_split_init(p, c->d_split.p, c->n_split, s);
    }
    if (p.do_window || p.do_cube) launch_trace_query(p, smem, s);
    if (units) launch_split_finish(p, c->d_split.p, c->n_split, 0, s);
    PSG_CUDA(cudaEventRecord(c->ev[2], s));
    if (do_cube && !exact_bounds) {
      // the optimistic pass 1 (and its 32-bit cells) against the boundary
      // timestamps pass 2 recorded; a miss re-runs both passes exactly
      unsigned long long* v = qs + QS_VERIFY;
      // speculative single-rank query: the verdict is read at the end, so the
      // (latency-bound) verification overlaps k_cross_stats on a side stream
      if (sp && !c->multi() && !std::getenv("PSG_NO_SIDE_STREAM")) {
        if (!c->side_stream) {
          PSG_CUDA(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
          PSG_CUDA(cudaEventCreateWithFlags(&c->side_in, cudaEventDisableTiming));
          PSG_CUDA(cudaEventCreateWithFlags(&c->side_out, cudaEventDisableTiming));
        }
        PSG_CUDA(cudaEventRecord(c->side_in, s));
        PSG_CUDA(cudaStreamWaitEvent(c->side_stream, c->side_in, 0));
        launch_verify_bounds(c->view(), c->d_cap_off.p, c->d_bts.p, c->d_nbounds.p, c->iter_count.p, v,
                             c->side_stream);
        PSG_CUDA(cudaEventRecord(c->side_out, c->side_stream));
        side_pending = true;
      } else {
        launch_verify_bounds(c->view(), c->d_cap_off.p, c->d_bts.p, c->d_nbounds.p, c->iter_count.p, v, s);
      }
      if (!sp) {
        if (c->multi()) c->allreduce(v, 1, ncclUint64, ncclMax);  // every rank re-runs together
        PSG_CUDA(cudaMemcpyAsync(&hq[QS_VERIFY], v, 8, cudaMemcpyDeviceToHost, s));
        c->sync();
        if (hq[QS_VERIFY]) {  // duplicate boundary timestamps, or an iteration >= 2^32 ns
          exact_bounds = c->exact_hint = true;
          continue;
        }
      }
    }

    if (do_stats && k_cap > 0) {
      const size_t plane = static_cast<size_t>(k_cap) * nn;
      launch_cross_stats(c->cube_incl.p, c->cube32, c->kept_bo.p, n, nn, row_stride(nn), k_cap, c->x_acc.p,
                         c->x_acc.p + plane, c->x_acc.p + 2 * plane, qs, s);
      double* no = c->node_out.ensure(static_cast<size_t>(nn) * (10 + 2 * kWithinTiles) + 1);  // + tile partials
      // within-rank partial sums per node, then cross-GPU sums of everything
      launch_stats_finalize(nullptr, nullptr, nullptr, k_cap, k_cap, nn, n, c->within_cv.p,
                            c->within_ok.p, n, no, qs, s);
      if (c->multi()) {
        c->group_begin();
        c->allreduce(c->x_acc.p, plane, ncclUint64, ncclSum);
        c->allreduce(c->x_acc.p + plane, plane, ncclUint64, ncclMax);
        c->allreduce(c->x_acc.p + 2 * plane, 3 * plane, ncclUint64, ncclSum);
        c->allreduce(no + static_cast<size_t>(nn) * 8, 2 * nn, ncclFloat64, ncclSum);
        c->group_end();
      }
      launch_stats_finalize(c->x_acc.p, c->x_acc.p + plane, c->x_acc.p + 2 * plane, k_cap, k_cap, nn,
                            n, nullptr, nullptr, n, no, qs, s);
    }

    if (do_out) {
      require(q->site_ctx && q->n_sites > 0, "outliers need at least one candidate site ctx");
      require(c->n_nodes > 0, "outliers need the rank -> node mapping (psg_set_nodes)");
      if (!c->topo_error.empty()) fail(PS_E_PARSE, c->topo_error);
      for (uint32_t i = 0; i < q->n_sites; ++i)
        require(q->site_ctx[i] < c->n_ctx, "site ctx out of range");
      c->sites.assign(q->site_ctx, q->site_ctx + q->n_sites);
      const uint32_t ns = q->n_sites;
      PSG_CUDA(cudaMemcpyAsync(c->d_sites.ensure(ns), q->site_ctx, 4ull * ns, cudaMemcpyHostToDevice, s));
      unsigned long long* sa = c->site_acc.ensure(2 * ns);
      unsigned long long* na = c->node_acc.ensure(2 * c->n_nodes);
      PSG_CUDA(cudaMemsetAsync(sa, 0, 16ull * ns, s));
      PSG_CUDA(cudaMemsetAsync(na, 0, 16ull * c->n_nodes, s));
      // per-rank site values: the dense window's incl columns, or for a sparse
      // window the sites' incl looked up in the remat rows ([n][ns], sites 0..ns-1)
      const uint64_t* wv = c->w_incl.p;
      uint32_t wstride = c->n_ctx;
      const uint32_t* wsite = c->d_sites.p;
      if (sparse) {
        std::vector<uint32_t> iota(ns);
        for (uint32_t i = 0; i < ns; ++i) iota[i] = i;
        PSG_CUDA(cudaMemcpyAsync(c->d_site_iota.ensure(ns), iota.data(), 4ull * ns, cudaMemcpyHostToDevice, s));
        sparse_site_values(c->sp, c->d_sites.p, ns, n, c->site_vals.ensure(static_cast<size_t>(n) * ns + 1), s);
        c->sync();  // the host iota above
        wv = c->site_vals.p;
        wstride = ns;
        wsite = c->d_site_iota.p;
      }
      launch_outliers(wv, n, wstride, wsite, ns, c->d_node_of_trace.p, c->n_nodes,
                      sa, na, c->d_worst.ensure(2), c->site_ratio.ensure(ns), 0, s);
      if (c->multi()) {
        c->group_begin();
        c->allreduce(sa, ns, ncclUint64, ncclSum);
        c->allreduce(sa + ns, ns, ncclUint64, ncclMax);
        c->group_end();
      }
      launch_outliers(wv, static_cast<uint32_t>(ranks_global(c)), wstride, wsite, ns,
                      c->d_node_of_trace.p, c->n_nodes, sa, na, c->d_worst.p, c->site_ratio.p, 1, s);
      launch_outliers(wv, n, wstride, wsite, ns, c->d_node_of_trace.p, c->n_nodes,
                      sa, na, c->d_worst.p, c->site_ratio.p, 2, s);
      c->allreduce(na, 2ull * c->n_nodes, ncclUint64, ncclSum);
      const size_t ssb = node_select_scratch_bytes(c->n_nodes);
      launch_node_select(na, c->n_nodes, q->top_k, q->z_min, c->node_mean.ensure(c->n_nodes),
                         c->node_z.ensure(c->n_nodes), c->d_order.ensure(c->n_nodes),
                         c->d_nsel.ensure(1), c->scratch.ensure(ssb), ssb, s);
      const uint32_t nr = static_cast<uint32_t>(c->h_rack_ids.size());
      if (nr) {
        launch_topology(c->d_order.p, c->d_nsel.p, c->d_node_rack_idx.p, c->d_node_chassis.p,
                        c->d_uni_cnt.p, nr, c->d_rack_nodes.ensure(nr), c->rack_mask.ensure(nr),
                        c->rack_full.ensure(nr), c->rack_cnt.ensure(64ull * nr), s);
      }
      launch_outlier_summary(c->d_worst.p, c->d_nsel.p, c->site_ratio.p, nr ? c->d_rack_nodes.p : nullptr,
                             nr, qs, s);
    }
    if (sp && do_stats) launch_qs_check_k(qs, k_cap, s);  // K beyond the accumulator planes
    if (sp && c->multi()) {  // every rank re-runs together
      c->group_begin();
      c->allreduce(qs + QS_OVERFLOW, 1, ncclUint64, ncclMax);
      c->allreduce(qs + QS_VERIFY, 1, ncclUint64, ncclMax);
      c->allreduce(qs + QS_CAP_MISS, 1, ncclUint64, ncclMax);
      c->group_end();
    }
    if (side_pending) PSG_CUDA(cudaStreamWaitEvent(s, c->side_out, 0));
    PSG_CUDA(cudaEventRecord(c->ev[3], s));
    // the query's one host round trip: the status block
    PSG_CUDA(cudaMemcpyAsync(hq, qs, sizeof(hq), cudaMemcpyDeviceToHost, s));
    c->sync();
    if (const char* tq = std::getenv("PSG_TRACE_QUERY"); tq && *tq == '1')
      std::fprintf(stderr, "psg_query: spec=%d exact=%d overflow=%llu verify=%llu cap_miss=%llu K=%u k_cap=%u syncs=%llu\n",
                   sp ? 1 : 0, exact_bounds ? 1 : 0, hq[QS_OVERFLOW], hq[QS_VERIFY], hq[QS_CAP_MISS],
                   qs_K(hq), k_cap, static_cast<unsigned long long>(c->n_syncs - syncs0));
    if (sp && (hq[QS_OVERFLOW] || hq[QS_VERIFY] || hq[QS_CAP_MISS])) {
      // a miss: re-run with the host sizing every step (and, for the
      // optimistic pass 1's verdict, in the exact mode)
      if (hq[QS_OVERFLOW]) {
        c->cap_div = 2;
        c->caps_valid = false;
      }
      // the verdict on the optimistic pass 1 only counts for a run whose
      // regions and buffers held (clamped regions make pass 2's boundary
      // record meaningless); the re-run verifies again
      if (hq[QS_VERIFY] && !hq[QS_OVERFLOW] && !hq[QS_CAP_MISS]) exact_bounds = c->exact_hint = true;
      spec = false;
      continue;
    }
    break;
    }

    if (do_cube) {
      c->n_kept = static_cast<uint32_t>(hq[QS_KEPT]);
      c->n_cells = hq[QS_CELLS];
      c->n_store = hq[QS_STORE];
      c->K = qs_K(hq);
      c->n_kept_global = static_cast<uint32_t>(hq[QS_KEPT_G]);
      c->k_plane = k_cap;
      c->spec_ready = true;
    }
    if (do_stats && c->K > 0) c->have_stats = true;
    if (do_out) c->have_outliers = true;

    // info
    if (do_window) c->have_window = c->have_carry = true;
    if (do_cube) c->have_cube = true;
    info->n_nodes = nn;
    info->n_kept = c->n_kept;
    info->n_skipped = do_cube ? n - c->n_kept : 0;
    info->min_iterations = c->K;
    info->n_kept_global = c->n_kept_global;
    info->n_cells = c->n_cells;
    info->cube_cell_bytes = do_cube ? (c->cube32 ? 4u : 8u) : 0u;
    info->cube_store_bytes = do_cube ? c->n_store * (c->cube32 ? 4u : 8u) : 0u;
    info->n_leaves = do_cube ? static_cast<uint32_t>(c->leaves.size()) : 0;
    info->n_internal = do_cube ? static_cast<uint32_t>(c->internal_pos.size()) : 0;
    if (do_out) {
      info->worst_site = c->sites[hq[QS_WORST]];
      info->n_outliers = static_cast<uint32_t>(hq[QS_NSEL]);
      std::memcpy(&info->worst_ratio, &hq[QS_WORST_RATIO], sizeof(double));
      info->n_racks = static_cast<uint32_t>(hq[QS_RACKS]);
    }
    PSG_CUDA(cudaEventElapsedTime(&info->ms_total, c->ev[0], c->ev[3]));
    PSG_CUDA(cudaEventElapsedTime(&info->ms_main, c->ev[1], c->ev[2]));
    if (do_cube) PSG_CUDA(cudaEventElapsedTime(&info->ms_bounds, c->ev[4], c->ev[5]));
    info->host_syncs = static_cast<uint32_t>(c->n_syncs - syncs0);
    info->window_sparse = sparse ? 1u : 0u;
    if (sparse) {
      info->n_window_rows = c->sp.n_rows;
      info->n_window_groups = c->sp.n_groups;
      info->n_remat_rows = c->sp.n_remat;
    }
  });
}

namespace {
// the window as sparse rows: the sparse query's own, or the dense result compacted once
void ensure_sparse_rows(psg_context* c) {
  if (!c->have_window) fail(PS_E_INVALID_ARGUMENT, "no window result (run psg_query with PSG_Q_WINDOW)");
  ensure_device(c);
  if (c->sp_valid) return;
  dense_window w{c->w_cnt.p, c->w_sum.p, c->w_min.p, c->w_max.p, c->w_mean.p, c->w_incl.p, c->w_excl.p};
  dense_to_sparse(w, c->n_traces, c->n_ctx, c->sp, c->stream);
  c->sp_valid = true;
}
}  // namespace

ps_status psg_get_window_groups(psg_context* c, uint64_t* n, uint32_t* trace, uint32_t* ctx_ids,
                                uint64_t* count, int64_t* sum, int64_t* mn, int64_t* mx, double* mean) {
  if (!c || !n) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_sparse_rows(c);
    const sparse_result& r = c->sp;
    *n = r.n_groups;
    const size_t m = r.n_groups;
    auto cp = [&](void* dst, const void* src, size_t b) {
      if (dst && b) PSG_CUDA(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost));
    };
    cp(trace, r.g_trace.p, 4 * m);
    cp(ctx_ids, r.g_ctx.p, 4 * m);
    cp(count, r.g_cnt.p, 8 * m);
    cp(sum, r.g_sum.p, 8 * m);
    cp(mn, r.g_min.p, 8 * m);
    cp(mx, r.g_max.p, 8 * m);
    cp(mean, r.g_mean.p, 8 * m);
  });
}

ps_status psg_get_remat_rows(psg_context* c, uint64_t* n, uint32_t* trace, uint32_t* ctx_ids, int64_t* incl,
                             int64_t* excl) {
  if (!c || !n) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_sparse_rows(c);
    const sparse_result& r = c->sp;
    *n = r.n_remat;
    const size_t m = r.n_remat;
    auto cp = [&](void* dst, const void* src, size_t b) {
      if (dst && b) PSG_CUDA(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost));
    };
    cp(trace, r.r_trace.p, 4 * m);
    cp(ctx_ids, r.r_ctx.p, 4 * m);
    cp(incl, r.r_incl.p, 8 * m);
    cp(excl, r.r_excl.p, 8 * m);
  });
}

ps_status psg_get_window(psg_context* c, uint64_t* count, int64_t* sum, int64_t* mn, int64_t* mx,
                         double* mean, int64_t* excl, int64_t* incl) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_window) fail(PS_E_INVALID_ARGUMENT, "no window result (run psg_query with PSG_Q_WINDOW)");
    if (c->window_sparse)
      fail(PS_E_INVALID_ARGUMENT,
           "the window is sparse (PSG_Q_SPARSE or a large calling-context tree): use psg_get_window_groups / "
           "psg_get_remat_rows");
    ensure_device(c);
    const size_t cells = static_cast<size_t>(c->n_traces) * c->n_ctx;
    auto cp = [&](void* dst, const void* src, size_t b) {
      if (dst && b) PSG_CUDA(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost));
    };
    cp(count, c->w_cnt.p, 8 * cells);
    cp(sum, c->w_sum.p, 8 * cells);
    cp(mn, c->w_min.p, 8 * cells);
    cp(mx, c->w_max.p, 8 * cells);
    cp(mean, c->w_mean.p, 8 * cells);
    cp(excl, c->w_excl.p, 8 * cells);
    cp(incl, c->w_incl.p, 8 * cells);
  });
}

ps_status psg_get_carry(psg_context* c, uint8_t* has, uint64_t* ts, uint32_t* ctx_ids) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_carry) fail(PS_E_INVALID_ARGUMENT, "no window result");
    ensure_device(c);
    if (has) PSG_CUDA(cudaMemcpy(has, c->c_has.p, c->n_traces, cudaMemcpyDeviceToHost));
    if (ts) PSG_CUDA(cudaMemcpy(ts, c->c_ts.p, 8ull * c->n_traces, cudaMemcpyDeviceToHost));
    if (ctx_ids) PSG_CUDA(cudaMemcpy(ctx_ids, c->c_ctx.p, 4ull * c->n_traces, cudaMemcpyDeviceToHost));
  });
}

namespace {
// Dense int64 cells of the kept traces [t_lo, t_hi) into host arrays (dense
// position relative to the range's first kept row): widened on the device
// (k_cube_dense) in chunks of whole traces through a staging buffer, then one
// D2H copy per chunk and column.  ic = host iteration counts of all traces.
void cube_dense_to_host(psg_context* c, const std::vector<uint32_t>& ic, uint32_t t_lo, uint32_t t_hi,
                        int64_t* incl, int64_t* excl) {
  if (!incl && !excl) return;
  if (excl && !c->have_excl)
    fail(PS_E_INVALID_ARGUMENT, "the excl cube was not stored (PSG_Q_NO_CUBE_STORE)");
  const uint64_t nn = c->nn;
  constexpr uint64_t kChunkCells = 1ull << 27;  // 1 GiB of int64 per column per chunk
  uint64_t row0 = 0;  // dense rows of the range before trace t
  uint32_t t = t_lo;
  const uint32_t nnp = row_stride(c->nn);
  const uint32_t m = static_cast<uint32_t>(c->internal_pos.size());
  while (t < t_hi) {
    // whole traces up to the chunk size (at least one)
    uint32_t e = t;
    uint64_t rows = 0;
    while (e < t_hi && (e == t || (rows + ic[e]) * nn <= kChunkCells)) rows += ic[e++];
    if (rows == 0) {
      t = e;
      continue;
    }
    uint64_t dense_row0 = 0;  // iter_off of trace t on the device
    PSG_CUDA(cudaMemcpyAsync(&dense_row0, c->iter_off.p + t, 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    const uint64_t cells = rows * nn;
    int64_t* di = reinterpret_cast<int64_t*>(c->dense_stage.ensure((incl ? cells : 0) + (excl ? cells : 0)));
    int64_t* de = incl ? di + cells : di;
    launch_cube_dense(c->cube_incl.p, c->cube32, c->cube_xint.p, c->iter_count.p, c->block_off.p,
                      c->iter_off.p, c->d_node_tab.p, c->nn, nnp, m, t, e, dense_row0, incl ? di : nullptr,
                      excl ? de : nullptr, c->stream);
    if (incl)
      PSG_CUDA(cudaMemcpyAsync(incl + row0 * nn, di, 8 * cells, cudaMemcpyDeviceToHost, c->stream));
    if (excl)
      PSG_CUDA(cudaMemcpyAsync(excl + row0 * nn, de, 8 * cells, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    row0 += rows;
    t = e;
  }
}

std::vector<uint32_t> host_iter_counts(psg_context* c) {
  std::vector<uint32_t> ic(c->n_traces);
  if (c->n_traces)
    PSG_CUDA(cudaMemcpy(ic.data(), c->iter_count.p, 4ull * c->n_traces, cudaMemcpyDeviceToHost));
  return ic;
}
}  // namespace

ps_status psg_get_cube(psg_context* c, uint32_t* node_ids, uint32_t* iter_counts,
                       uint64_t* block_offset, int64_t* incl, int64_t* excl, int64_t* gap_incl,
                       int64_t* gap_excl) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_cube) fail(PS_E_INVALID_ARGUMENT, "no cube result (run psg_query with PSG_Q_CUBE)");
    ensure_device(c);
    if (node_ids) std::copy(c->node_ids.begin(), c->node_ids.end(), node_ids);
    const std::vector<uint32_t> ic = host_iter_counts(c);
    if (iter_counts) std::copy(ic.begin(), ic.end(), iter_counts);
    if (block_offset) {  // dense cell offsets of the kept traces (itermodel.hpp:97-101)
      uint64_t off = 0;
      size_t j = 0;
      for (uint32_t t = 0; t < c->n_traces; ++t)
        if (ic[t] > 0) {
          block_offset[j++] = off;
          off += static_cast<uint64_t>(ic[t]) * c->nn;
        }
    }
    if (c->n_cells) cube_dense_to_host(c, ic, 0, c->n_traces, incl, excl);
    else if (excl && !c->have_excl)
      fail(PS_E_INVALID_ARGUMENT, "the excl cube was not stored (PSG_Q_NO_CUBE_STORE)");
    const size_t g = static_cast<size_t>(c->n_kept) * c->nn;
    if (gap_incl && g) PSG_CUDA(cudaMemcpy(gap_incl, c->gap_incl.p, 8 * g, cudaMemcpyDeviceToHost));
    if (gap_excl && g) PSG_CUDA(cudaMemcpy(gap_excl, c->gap_excl.p, 8 * g, cudaMemcpyDeviceToHost));
  });
}

ps_status psg_get_boundaries(psg_context* c, uint32_t trace, uint32_t* n, uint64_t* ts) {
  if (!c || !n) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_cube) fail(PS_E_INVALID_ARGUMENT, "no cube result (run psg_query with PSG_Q_CUBE)");
    require(trace < c->n_traces, "trace index out of range");
    ensure_device(c);
    uint32_t nb = 0, it = 0;
    uint64_t off = 0;
    PSG_CUDA(cudaMemcpy(&nb, c->d_nbounds.p + trace, 4, cudaMemcpyDeviceToHost));
    PSG_CUDA(cudaMemcpy(&it, c->iter_count.p + trace, 4, cudaMemcpyDeviceToHost));
    PSG_CUDA(cudaMemcpy(&off, c->d_cap_off.p + trace, 8, cudaMemcpyDeviceToHost));
    *n = nb;
    if (!ts || !nb) return;
    if (it == 0) {  // one boundary, at t_end (the empty last interval dropped)
      ts[0] = c->h_tend[trace];
      return;
    }
    PSG_CUDA(cudaMemcpy(ts, c->d_bts.p + off, 8ull * nb, cudaMemcpyDeviceToHost));
  });
}

ps_status psg_node_name(const char* name, uint32_t* rack, uint32_t* chassis) {
  if (!name) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    const std::string err = store::node_name_error(name, rack, chassis);
    if (!err.empty()) fail(PS_E_PARSE, err);
  });
}

ps_status psg_get_cube_range(psg_context* c, uint32_t t_lo, uint32_t t_hi, uint64_t* n_cells,
                             uint32_t* n_kept, int64_t* incl, int64_t* excl, int64_t* gap_incl,
                             int64_t* gap_excl) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_cube) fail(PS_E_INVALID_ARGUMENT, "no cube result (run psg_query with PSG_Q_CUBE)");
    require(t_lo <= t_hi && t_hi <= c->n_traces, "bad trace range");
    ensure_device(c);
    const std::vector<uint32_t> ic = host_iter_counts(c);
    uint64_t rows = 0;
    uint32_t kept_before = 0, kept = 0;
    for (uint32_t t = 0; t < t_hi; ++t) {
      if (t < t_lo) kept_before += ic[t] > 0;
      else {
        rows += ic[t];
        kept += ic[t] > 0;
      }
    }
    if (n_cells) *n_cells = rows * c->nn;
    if (n_kept) *n_kept = kept;
    if (rows) cube_dense_to_host(c, ic, t_lo, t_hi, incl, excl);
    const size_t g = static_cast<size_t>(kept) * c->nn, g0 = static_cast<size_t>(kept_before) * c->nn;
    if (gap_incl && g) PSG_CUDA(cudaMemcpy(gap_incl, c->gap_incl.p + g0, 8 * g, cudaMemcpyDeviceToHost));
    if (gap_excl && g) PSG_CUDA(cudaMemcpy(gap_excl, c->gap_excl.p + g0, 8 * g, cudaMemcpyDeviceToHost));
  });
}

namespace {
ps_status get_cube_stored(psg_context* c, uint32_t* cell_bytes, uint32_t* stride, uint64_t* incl_bytes,
                          void* incl, uint64_t* stored_off, uint64_t* xint_cells, int64_t* xint, bool async) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_cube) fail(PS_E_INVALID_ARGUMENT, "no cube result (run psg_query with PSG_Q_CUBE)");
    ensure_device(c);
    const uint64_t cb = c->cube32 ? 4 : 8, bytes = c->n_store * cb;
    const uint64_t nx = c->have_excl && c->nn ? c->n_cells / c->nn * c->internal_pos.size() : 0;
    if (cell_bytes) *cell_bytes = static_cast<uint32_t>(cb);
    if (stride) *stride = row_stride(c->nn);
    if (incl_bytes) *incl_bytes = bytes;
    if (xint_cells) *xint_cells = nx;
    if (xint && !c->have_excl && c->n_cells)
      fail(PS_E_INVALID_ARGUMENT, "the excl cube was not stored (PSG_Q_NO_CUBE_STORE)");
    // straight DMA of the device buffers (full PCIe rate into pinned memory)
    cudaStream_t st = c->stream;
    if (async) {
      if (!c->d2h_stream) {
        PSG_CUDA(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
        PSG_CUDA(cudaEventCreateWithFlags(&c->d2h_ready, cudaEventDisableTiming));
        PSG_CUDA(cudaEventCreateWithFlags(&c->d2h_done, cudaEventDisableTiming));
      }
      c->wait_copies();  // one copy-out in flight at a time
      PSG_CUDA(cudaEventRecord(c->d2h_ready, c->stream));
      PSG_CUDA(cudaStreamWaitEvent(c->d2h_stream, c->d2h_ready, 0));
      st = c->d2h_stream;
    }
    if (incl && bytes) PSG_CUDA(cudaMemcpyAsync(incl, c->cube_incl.p, bytes, cudaMemcpyDeviceToHost, st));
    if (stored_off && c->n_traces)
      PSG_CUDA(cudaMemcpyAsync(stored_off, c->block_off.p, 8ull * c->n_traces, cudaMemcpyDeviceToHost, st));
    if (xint && nx) PSG_CUDA(cudaMemcpyAsync(xint, c->cube_xint.p, 8 * nx, cudaMemcpyDeviceToHost, st));
    if (async) {
      PSG_CUDA(cudaEventRecord(c->d2h_done, st));
      c->d2h_pending = true;
    } else {
      c->sync();
    }
  });
}
}  // namespace

ps_status psg_get_cube_stored(psg_context* c, uint32_t* cell_bytes, uint32_t* stride,
                              uint64_t* incl_bytes, void* incl, uint64_t* stored_off,
                              uint64_t* xint_cells, int64_t* xint) {
  return get_cube_stored(c, cell_bytes, stride, incl_bytes, incl, stored_off, xint_cells, xint, false);
}

ps_status psg_get_cube_stored_async(psg_context* c, void* incl, uint64_t* stored_off, int64_t* xint) {
  return get_cube_stored(c, nullptr, nullptr, nullptr, incl, stored_off, nullptr, xint, true);
}

ps_status psg_wait_copies(psg_context* c) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] { c->wait_copies(); });
}

ps_status psg_get_stats(psg_context* c, double total_time_s, uint32_t* leaves, double* savings,
                        double* summary, double* cv, int32_t* cv_ok) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_cube) fail(PS_E_INVALID_ARGUMENT, "no cube result");
    if (total_time_s <= 0.0) fail(PS_E_INVALID_ARGUMENT, "total time must be positive");
    if (c->K < 1) fail(PS_E_INSUFFICIENT_DATA, "model has no iterations");
    if (!c->have_stats) fail(PS_E_INVALID_ARGUMENT, "no stats result (run psg_query with PSG_Q_STATS)");
    ensure_device(c);
    std::vector<double> no(static_cast<size_t>(c->nn) * 8);
    PSG_CUDA(cudaMemcpy(no.data(), c->node_out.p, 8 * no.size(), cudaMemcpyDeviceToHost));
    double total = 0.0;
    for (size_t i = 0; i < c->leaves.size(); ++i) {
      const uint32_t npos = static_cast<uint32_t>(
          std::lower_bound(c->node_ids.begin(), c->node_ids.end(), c->leaves[i]) - c->node_ids.begin());
      const double* r = &no[static_cast<size_t>(npos) * 8];
      if (leaves) leaves[i] = c->leaves[i];
      if (savings)
        for (int j = 0; j < 4; ++j) savings[4 * i + j] = r[j];
      total += r[3];  // savings_report: total_savings_s += total_reduction_s (diagnostics.cpp:153)
      if (cv) {
        cv[2 * i] = r[4];
        cv[2 * i + 1] = r[5];
      }
      if (cv_ok) cv_ok[i] = (r[6] != 0.0 && r[7] != 0.0) ? 1 : 0;
    }
    if (summary) {
      summary[0] = c->K;
      summary[1] = total;
      summary[2] = total_time_s;
      summary[3] = total / total_time_s;
    }
  });
}

ps_status psg_get_outliers(psg_context* c, double* site_ratio, double* node_mean, double* node_z,
                           uint32_t* selected, uint32_t* rack_rows, uint64_t* chassis_mask,
                           uint64_t* full_mask) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_outliers) fail(PS_E_INVALID_ARGUMENT, "no outlier result (run psg_query with PSG_Q_OUTLIERS)");
    ensure_device(c);
    if (site_ratio)
      PSG_CUDA(cudaMemcpy(site_ratio, c->site_ratio.p, 8 * c->sites.size(), cudaMemcpyDeviceToHost));
    if (node_mean) PSG_CUDA(cudaMemcpy(node_mean, c->node_mean.p, 8ull * c->n_nodes, cudaMemcpyDeviceToHost));
    if (node_z) PSG_CUDA(cudaMemcpy(node_z, c->node_z.p, 8ull * c->n_nodes, cudaMemcpyDeviceToHost));
    uint32_t nsel = 0;
    PSG_CUDA(cudaMemcpy(&nsel, c->d_nsel.p, 4, cudaMemcpyDeviceToHost));
    if (selected && nsel) PSG_CUDA(cudaMemcpy(selected, c->d_order.p, 4ull * nsel, cudaMemcpyDeviceToHost));
    const uint32_t nr = static_cast<uint32_t>(c->h_rack_ids.size());
    if (nr && (rack_rows || chassis_mask || full_mask)) {
      std::vector<uint32_t> rn(nr);
      std::vector<uint64_t> m(nr), fm(nr);
      PSG_CUDA(cudaMemcpy(rn.data(), c->d_rack_nodes.p, 4ull * nr, cudaMemcpyDeviceToHost));
      PSG_CUDA(cudaMemcpy(m.data(), c->rack_mask.p, 8ull * nr, cudaMemcpyDeviceToHost));
      PSG_CUDA(cudaMemcpy(fm.data(), c->rack_full.p, 8ull * nr, cudaMemcpyDeviceToHost));
      // device masks are over chassis slots (position in the rack's chassis
      // list); report them over chassis ids, which needs ids < 64
      auto by_id = [&](uint32_t r, uint64_t slots) {
        uint64_t out = 0;
        for (uint32_t i = 0; i < 64; ++i)
          if ((slots >> i) & 1) {
            const uint32_t id = c->h_rack_chassis[r][i];
            if (id >= 64)
              fail(PS_E_INVALID_ARGUMENT,
                   "chassis id " + std::to_string(id) + " >= 64 has no mask bit; use psg_get_topology");
            out |= 1ull << id;
          }
        return out;
      };
      size_t j = 0;
      for (uint32_t r = 0; r < nr; ++r) {
        if (!rn[r]) continue;
        if (rack_rows) {
          rack_rows[3 * j] = c->h_rack_ids[r];
          rack_rows[3 * j + 1] = rn[r];
          rack_rows[3 * j + 2] = static_cast<uint32_t>(__builtin_popcountll(m[r]));
        }
        if (chassis_mask) chassis_mask[j] = by_id(r, m[r]);
        if (full_mask) full_mask[j] = by_id(r, fm[r]);
        ++j;
      }
    }
  });
}

ps_status psg_get_topology(psg_context* c, uint32_t* n_rows, uint32_t* rows) {
  if (!c || !n_rows) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (!c->have_outliers) fail(PS_E_INVALID_ARGUMENT, "no outlier result (run psg_query with PSG_Q_OUTLIERS)");
    ensure_device(c);
    const uint32_t nr = static_cast<uint32_t>(c->h_rack_ids.size());
    std::vector<uint32_t> cnt(64ull * nr);
    if (nr) PSG_CUDA(cudaMemcpy(cnt.data(), c->rack_cnt.p, 4ull * cnt.size(), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> uni(64ull * nr);
    if (nr) PSG_CUDA(cudaMemcpy(uni.data(), c->d_uni_cnt.p, 4ull * uni.size(), cudaMemcpyDeviceToHost));
    uint32_t j = 0;
    for (uint32_t r = 0; r < nr; ++r)
      for (uint32_t i = 0; i < c->h_rack_chassis[r].size(); ++i) {
        const uint32_t x = cnt[64ull * r + i];
        if (!x) continue;
        if (rows) {
          rows[4ull * j] = c->h_rack_ids[r];
          rows[4ull * j + 1] = c->h_rack_chassis[r][i];
          rows[4ull * j + 2] = x;
          rows[4ull * j + 3] = x == uni[64ull * r + i] ? 1u : 0u;
        }
        ++j;
      }
    *n_rows = j;
  });
}

uint64_t psg_kernel_launches(void) { return kernel_launches(); }

ps_status psg_export_aos_range(psg_context* c, uint32_t t_lo, uint32_t t_hi, void* body) {
  if (!c) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    require(t_lo <= t_hi && t_hi <= c->n_traces, "bad trace range");
    ensure_device(c);
    const uint64_t e0 = c->h_off[t_lo], e1 = c->h_off[t_hi];
    require(e1 == e0 || body != nullptr, "body is required");
    const uint64_t chunk_ev = 4ull << 24;
    drop_prefetch(c);
    uint8_t* stage = c->d_stage.ensure(std::max<uint64_t>(c->d_stage.n, chunk_ev * 12 + 64));
    // K1's inverse works on groups of 4 events from a 16-byte aligned start:
    // export from the aligned-down event and skip the head on the copy
    for (uint64_t done = e0; done < e1;) {
      const uint64_t a = done & ~3ull;
      const uint64_t ev = std::min(chunk_ev, e1 - a);
      launch_soa_to_aos(c->d_ts.p + a, c->d_ctx.p + a, ev, stage, c->stream);
      PSG_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(body) + (done - e0) * 12, stage + (done - a) * 12,
                               (a + ev - done) * 12, cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      done = a + ev;
    }
  });
}

ps_status psg_export_aos(psg_context* c, void* body) {
  if (!c || (!body && c->n_events)) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    ensure_device(c);
    const uint64_t chunk_ev = 4ull << 24;
    drop_prefetch(c);
    uint8_t* stage = c->d_stage.ensure(std::max<uint64_t>(c->d_stage.n, chunk_ev * 12));
    for (uint64_t done = 0; done < c->n_events; done += chunk_ev) {
      uint64_t ev = std::min(chunk_ev, c->n_events - done);
      launch_soa_to_aos(c->d_ts.p + done, c->d_ctx.p + done, ev, stage, c->stream);
      PSG_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(body) + done * 12, stage, ev * 12,
                               cudaMemcpyDeviceToHost, c->stream));
      c->sync();
    }
  });
}

ps_status psg_window_rows(psg_context* c, uint64_t t0, uint64_t t1, uint64_t* n_rows,
                          uint32_t* row_pid, uint64_t* row_ts, uint32_t* row_ctx) {
  if (!c || !n_rows) return PS_E_INVALID_ARGUMENT;
  return guarded([&] {
    if (t0 > t1) fail(PS_E_INVALID_ARGUMENT, "trace window start after end");
    ensure_device(c);
    const uint32_t n = c->n_traces;
    cudaStream_t s = c->stream;
    uint64_t* cnt = c->gen_chunks.ensure(2ull * (n + 1));
    uint64_t* roff = cnt + (n + 1);
    launch_window_bounds(c->view(), t0, t1, cnt, c->c_has.ensure(n + 1), c->c_ts.ensure(n + 1),
                         c->c_ctx.ensure(n + 1), s);
    PSG_CUDA(cudaMemsetAsync(cnt + n, 0, 8, s));
    size_t sb = exclusive_scan_u64_scratch(n + 1);
    launch_exclusive_scan_u64(cnt, roff, n + 1, c->scratch.ensure(sb), sb, s);
    uint64_t total = 0;
    PSG_CUDA(cudaMemcpyAsync(&total, roff + n, 8, cudaMemcpyDeviceToHost, s));
    c->sync();
    *n_rows = total;
    if (row_pid || row_ts || row_ctx) {
      dbuf<uint32_t> op, oc;
      dbuf<uint64_t> ot;
      launch_window_copy(c->view(), c->d_pid.p, t0, roff, op.ensure(total + 1), ot.ensure(total + 1),
                         oc.ensure(total + 1), s);
      c->sync();
      if (row_pid && total) PSG_CUDA(cudaMemcpy(row_pid, op.p, 4 * total, cudaMemcpyDeviceToHost));
      if (row_ts && total) PSG_CUDA(cudaMemcpy(row_ts, ot.p, 8 * total, cudaMemcpyDeviceToHost));
      if (row_ctx && total) PSG_CUDA(cudaMemcpy(row_ctx, oc.p, 4 * total, cudaMemcpyDeviceToHost));
    }
    c->have_window = false;  // carry buffers now hold window_rows carries only
    c->have_carry = true;
  });
}

}  // extern "C"
