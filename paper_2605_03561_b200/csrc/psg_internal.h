// Internal types of the psg runtime: device buffers, the context, error
// plumbing, and the launch wrappers shared by psg_capi.cu and psg_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "psg.h"

namespace psg {

// Typed failure that crosses C++ frames inside the library and is mapped to
// ps_status at the C ABI (the reference's errc -> ps_status map, capi.cpp:35-63).
struct failure : std::runtime_error {
  ps_status status;
  failure(ps_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(ps_status s, const std::string& m) { throw failure(s, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(PS_E_INTERNAL, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define PSG_CUDA(call) ::psg::cuda_check((call), #call)

// Owning device allocation; grow-only so repeated queries reuse HBM.
template <typename T>
struct dbuf {
  T* p = nullptr;
  size_t n = 0;     // elements allocated
  dbuf() = default;
  dbuf(const dbuf&) = delete;
  dbuf& operator=(const dbuf&) = delete;
  ~dbuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* ensure(size_t count) {
    if (count <= n && p) return p;
    release();
    size_t bytes = (count ? count : 1) * sizeof(T);
    PSG_CUDA(cudaMalloc(&p, bytes));
    n = count;
    return p;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// ---- device-side parameter blocks ----------------------------------------

struct trace_view {
  const uint64_t* off;    // [n+1] event offsets
  const uint64_t* ts;     // [E]
  const uint32_t* ctx;    // [E]
  const uint64_t* t_end;  // [n]
  uint32_t n;
};

struct query_params {
  trace_view tr;
  uint32_t n_ctx;
  // window part
  uint32_t do_window, clamp_tend;
  uint64_t t0, t1;
  uint64_t *w_cnt, *w_sum, *w_min, *w_max, *w_excl, *w_incl;  // [n][n_ctx]
  double* w_mean;
  uint8_t* c_has;
  uint64_t* c_ts;
  uint32_t* c_ctx;
  const int32_t* cct_pre;   // [n_ctx] preorder position in the whole CCT
  const int32_t* cct_size;  // [n_ctx] subtree size
  // cube part
  uint32_t do_cube, store_cube, do_stats;
  const int32_t* sub_pre;    // [n_ctx] preorder position inside the anchor subtree or -1
  const int32_t* node_pre;   // [nn] per node position (ascending ctx id)
  const int32_t* node_size;  // [nn]
  uint32_t nn;               // anchor subtree size (cube nodes)
  const uint32_t* iter_count;  // [n] 0 = skipped
  const uint32_t* tpos;        // [n] position among kept traces
  const uint64_t* block_off;   // [n] cell offset of the trace's first row (kept traces)
  uint32_t K;                  // global min iterations over kept traces (0: none)
  uint64_t *cube_incl, *cube_excl, *gap_incl, *gap_excl;
  // cross-rank stats accumulators (k < K) and within-trace CVs
  unsigned long long *x_sum, *x_max, *x_sq;  // [K][nn], x_sq = 3 limbs [3][K][nn]
  double* within_cv;   // [n_kept][nn]
  uint8_t* within_ok;  // [n_kept][nn]
  uint32_t G;          // iterations per CTA chunk
  uint32_t warps;      // traces per CTA
};

// Per-warp shared-memory carve-out sizes (bytes), shared by host and device.
struct warp_smem_layout {
  uint32_t n_ctx, nn, G;
  uint32_t off_wcnt, off_wsum, off_wmin, off_wmax, off_wtag;
  uint32_t off_rows, off_rtag, off_scan, off_tmp, off_wsx, off_wsqlo, off_wsqhi;
  uint32_t bytes;
  __host__ __device__ void init(uint32_t nctx, uint32_t nnodes, uint32_t g) {
    n_ctx = nctx;
    nn = nnodes;
    G = g;
    uint32_t o = 0;
    auto take = [&](uint32_t b) {
      uint32_t r = o;
      o += (b + 15u) & ~15u;
      return r;
    };
    off_wcnt = take(8u * nctx);
    off_wsum = take(8u * nctx);
    off_wmin = take(8u * nctx);
    off_wmax = take(8u * nctx);
    off_wtag = take(nctx);
    off_rows = take(8u * (g + 1) * nnodes);
    off_rtag = take((g + 1) * nnodes);
    uint32_t m = nctx > nnodes ? nctx : nnodes;
    off_scan = take(8u * (m + 1));
    off_tmp = take(8u * m);
    off_wsx = take(8u * nnodes);
    off_wsqlo = take(8u * nnodes);
    off_wsqhi = take(8u * nnodes);
    bytes = o;
  }
};

// CTA-shared tables placed before the per-warp carve-outs.
__host__ __device__ inline uint32_t cta_table_bytes(uint32_t n_ctx, uint32_t nn, uint32_t warps) {
  uint32_t b = 4u * n_ctx * 3 + 4u * nn * 2 + 4u * warps * 2;
  return (b + 15u) & ~15u;
}

// ---- launchers (psg_kernels.cu) ------------------------------------------

// Process-wide count of psg kernel launches (library kernels such as CUB's
// scans/sorts are not counted).
void count_launch(unsigned n = 1);
unsigned long long kernel_launches();
void launch_soa_to_aos(const uint64_t* ts, const uint32_t* ctx, uint64_t n_events, uint8_t* body,
                       cudaStream_t s);

void launch_aos_to_soa(const uint8_t* body, uint64_t n_events, uint64_t* ts, uint32_t* ctx,
                       cudaStream_t s);
void launch_validate(const trace_view& tr, uint32_t n_ctx, unsigned long long* bad,
                     unsigned long long* first_bad, cudaStream_t s);
void launch_gen_iterative(const uint64_t* jump_mats, uint64_t seed, uint32_t n_ranks,
                          uint32_t n_it, uint32_t n_k, const double* mean, const double* jitter,
                          const double* spread, uint64_t spread_kstride, uint64_t copy_ns,
                          uint32_t rank_lo, uint32_t n_local, uint64_t events_per_trace,
                          uint64_t* chunk_scratch, uint64_t* ts, uint32_t* ctx, uint64_t* t_end,
                          cudaStream_t s);
void launch_iter_count(const trace_view& tr, const int32_t* sub_pre, uint32_t n_ctx,
                       uint32_t* iter_count, cudaStream_t s);
void launch_cube_layout(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint32_t* tpos,
                        uint64_t* block_off,
                        unsigned long long* summary /*[0]=kept [1]=min_it [2]=cells*/,
                        void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t cube_layout_scratch_bytes(uint32_t n);
void launch_trace_query(const query_params& p, uint32_t smem_bytes, cudaStream_t s);
void launch_stats_finalize(const unsigned long long* x_sum, const unsigned long long* x_max,
                           const unsigned long long* x_sq, uint32_t K, uint32_t nn,
                           uint32_t n_kept, const double* within_cv, const uint8_t* within_ok,
                           uint32_t n_kept_local, double* node_out /*[nn][8]*/, cudaStream_t s);
void launch_window_bounds(const trace_view& tr, uint64_t t0, uint64_t t1, uint64_t* cnt,
                          uint8_t* c_has, uint64_t* c_ts, uint32_t* c_ctx, cudaStream_t s);
void launch_window_copy(const trace_view& tr, const uint32_t* pid, uint64_t t0,
                        const uint64_t* row_off, uint32_t* out_pid, uint64_t* out_ts,
                        uint32_t* out_ctx, cudaStream_t s);
void launch_exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint32_t n, void* scratch,
                               size_t scratch_bytes, cudaStream_t s);
size_t exclusive_scan_u64_scratch(uint32_t n);
void launch_outliers(const uint64_t* w_incl, uint32_t n_traces, uint32_t n_ctx,
                     const uint32_t* site_ctx, uint32_t n_sites, const uint32_t* node_of_trace,
                     uint32_t n_nodes, unsigned long long* site_acc /*[n_sites][2]*/,
                     unsigned long long* node_acc /*[n_nodes][2]*/, uint32_t* worst,
                     double* site_ratio, uint32_t phase, cudaStream_t s);
void launch_node_select(const unsigned long long* node_acc, uint32_t n_nodes, uint32_t top_k,
                        double z_min, double* node_mean, double* node_z, uint32_t* order,
                        uint32_t* n_sel, cudaStream_t s);
void launch_topology(const uint32_t* selected, const uint32_t* n_sel, const uint32_t* node_rack_idx,
                     const uint32_t* node_chassis, const uint32_t* uni_cnt, uint32_t n_racks,
                     uint32_t* rack_nodes, unsigned long long* rack_mask,
                     unsigned long long* rack_full, cudaStream_t s);

}  // namespace psg
