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

// The thread-local message behind psg_last_error (psg_capi.cu).
void set_last_error(const std::string& m);

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

// Profile records in HBM (profile.db bodies as SoA; store.cpp:563-571).
struct profile_view {
  const uint64_t* off;    // [n+1] record offsets per profile slot
  const uint32_t* pid;    // [n] ascending profile ids
  const uint32_t* ctx;    // [R] sorted by ctx within a profile
  const uint16_t* metric; // [R]
  const double* value;    // [R]
  uint32_t n;
};

// The query's device-side status block (u64 words).  The layout kernels,
// pass 1, pass 2 and the verification write it; the statistics kernels read
// K and the kept counts from it, so a query needs no host round trip between
// its kernels: the host reads the block once, at the end (psg_capi.cu).
enum : uint32_t {
  QS_KEPT = 0,       // kept traces (this rank)
  QS_MIN_IT = 1,     // min iterations over kept traces (this rank; ~0 when none)
  QS_CELLS = 2,      // logical cube cells (Σ iters * nn)
  QS_OVERFLOW = 3,   // pass-1 traces whose boundaries did not fit their region
  QS_STORE = 4,      // storage cells of the cube
  QS_SPAN = 5,       // longest stored iteration (exact pass 1)
  QS_VERIFY = 6,     // verdict on the optimistic pass 1 (bits; k_verify_bounds)
  QS_CAP_MISS = 7,   // the speculative capacities did not hold (bits: 1 cube, 2 excl, 4 K)
  QS_KEPT_G = 8,     // kept traces over all ranks
  QS_MIN_IT_G = 9,   // min iterations over all ranks' kept traces
  QS_WORST = 10,     // outliers: worst site index
  QS_NSEL = 11,      // outliers: selected nodes
  QS_WORST_RATIO = 12,  // outliers: the worst site's ratio (f64 bits)
  QS_RACKS = 13,     // outliers: racks holding a selected node
  QS_WORDS = 16
};
// K = the global min iterations over kept traces (0 when none: diagnostics.cpp:101)
__host__ __device__ inline uint32_t qs_K(const unsigned long long* qs) {
  return qs[QS_KEPT_G] ? static_cast<uint32_t>(qs[QS_MIN_IT_G]) : 0u;
}

// Pass 1 (k_bounds): iteration boundaries per trace (itermodel.cpp:111-143).
struct bound_params {
  trace_view tr;
  // narrow mirror of tr.ctx (every ctx < 256), or null: 1 B/event holding the
  // ctx's preorder position in the whole CCT, so the anchor subtree is the
  // byte range [sub_lo, sub_lo + sub_size) and membership is a SIMD compare
  const uint8_t* ctx8;
  uint32_t sub_lo, sub_size;
  uint32_t ctx7;             // every preorder byte < 128 (n_ctx <= 128): the 3-op SWAR test
  const uint32_t* contains;  // [ceil(n_ctx/32)] bit c set iff ctx c is in the anchor subtree
  uint32_t words;
  const uint64_t* cap_off;   // [n+1] offsets of the per-trace boundary regions in bidx
  uint32_t* bidx;            // boundary event index, relative to the trace's first event
  uint64_t* bts;             // boundary timestamp (same layout as bidx)
  uint32_t* n_bounds;        // [n] boundaries found (may exceed the region capacity)
  uint32_t* iter_count;      // [n] iterations (n_bounds minus a zero-length last interval)
  unsigned long long* overflow;  // traces whose boundaries did not fit their region
};

// Per-warp shared-memory carve-out (bytes), shared by host and device.
// Cube cells and window sums are split into 32-bit words so that the hot
// loop can use native 32-bit shared reductions (RED) without return values;
// the overflow guards are the time spans of iterations and block steps (see
// psg_query.cu).
//
// Cube rows are node-indexed with stride nnp = nn + 1 rounded up to even (the
// cube's storage stride): a chunk's G rows are byte for byte its block in the cube, and the pad
// column nn absorbs the events of contexts outside the anchor subtree, so the
// interior loop adds every event without a branch.  The ring holds 2G rows
// and the gap row (2G).
//
// The window table is one 36-byte record per ctx, so one address serves all
// of an event's reductions: {cnt, pending 32-bit sum, min, max, byte offset of
// the ctx's cube column in a row (the pad column outside the anchor subtree),
// count of durations >= 2^32, folded 64-bit
// sum (lo, hi words), -}.  The odd stride of 9 words puts the same field of 32
// consecutive contexts in 32 distinct banks.  The rare min/max of durations
// >= 2^32 accumulate in the trace's global output row (64-bit global atomics).
enum : uint32_t { WT_CNT = 0, WT_LO = 1, WT_MIN = 2, WT_MAX = 3, WT_PPO = 4, WT_NBIG = 5,
                  WT_ACC = 6 /* lo, hi words */, WT_STRIDE = 9 };
// First word of ctx c's record.  Lanes hold runs of 8 consecutive events, so
// in an iterative trace the lanes of one instruction touch contexts 8 apart
// (mod the iteration's length): with a stride of 9 words alone those share a
// bank every 4 lanes.  Skipping one record slot after every 8 contexts
// (PSG_WT_SWIZZLE 1) or every 32 (2) spreads them: a bank-conflict model of
// configs[1] (67 contexts per iteration) gives 2.97 / 2.21 / 2.00 shared
// wavefronts per record access for 0 / 1 / 2, and k_trace_query measured
// 18.36 / 17.60 / 17.40 ms (profiles/r2g_ab_wt_swizzle.txt).
// IL = the interleaved lane layout (one-warp CTAs: the lanes of an
// instruction hold consecutive events, so consecutive contexts, which the odd
// stride alone puts in distinct banks); the run layout (wide CTAs) skips one
// record slot every 32 contexts instead (model: 2.00 instead of 2.97
// wavefronts per access at configs[1]; measured 17.40 vs 18.36 ms, r2g).
template <bool IL>
__host__ __device__ inline uint32_t wt_word_l(uint32_t c) {
  return WT_STRIDE * (IL ? c : c + (c >> 5));
}
__host__ __device__ inline uint32_t wt_word(uint32_t c, bool il) {
  return il ? wt_word_l<true>(c) : wt_word_l<false>(c);
}

// Cube row stride in cells: nn + 1 rounded up to even (pad columns).
__host__ __device__ inline uint32_t row_stride(uint32_t nn) { return (nn + 2) & ~1u; }

struct warp_smem_layout {
  uint32_t nnp;               // cube row stride (nn + 1 rounded up to even)
  uint32_t off_rlo, off_rhi;  // (2G+1) x nnp u32: cube rows (ring of 2G, gap), high words
  uint32_t off_pref;   // nn+1 u64     prefix scratch for the generic inclusive roll-up
  uint32_t off_bwin;   // 2G+2 u32     boundary window (event indices relative to the trace)
  uint32_t off_bts;    // 2G+2 u64     timestamps of those boundaries
  uint32_t off_wtab;   // n_ctx x 36 B window records (WT_*)
  uint32_t off_wsx, off_wsqlo, off_wsqhi;  // nn u64: within-trace sums over k < K
  uint32_t off_carry;  // {u64 ts, u64 dur, u64 (has << 32 | ctx)}
  uint32_t off_scan;   // 2 x (n_ctx + 1) u64 at finalize (aliases the rows)
  uint32_t bytes;
  // wide_rows: 64-bit cells possible (exact pass 1), so the rows need their
  // high words; the optimistic mode runs 32-bit throughout and aliases them
  __host__ __device__ void init(uint32_t n_ctx, uint32_t nn, uint32_t G, bool wide_rows) {
    uint32_t o = 0;
    auto take = [&](uint32_t b) {
      uint32_t r = o;
      o += (b + 15u) & ~15u;
      return r;
    };
    nnp = row_stride(nn);
    const uint32_t rows = 4u * (2 * G + 1) * nnp, scan = 16u * (n_ctx + 1);
    off_rlo = take(rows > scan ? rows : scan);
    off_scan = off_rlo;
    off_rhi = wide_rows ? take(rows) : off_rlo;
    off_pref = take(8u * (nn + 1));  // generic rows and the gap row
    off_bwin = take(4u * (2 * G + 2));
    off_bts = take(8u * (2 * G + 2));
    off_wtab = take(4u * WT_STRIDE * (n_ctx + n_ctx / 32 + 1));
    off_wsx = take(8u * nn);
    off_wsqlo = take(8u * nn);
    off_wsqhi = take(8u * nn);
    off_carry = take(24);
    bytes = o;
  }
};

// Pass 2 (k_trace_query): window + cube + stats in one read of the events.
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
  const int32_t* sub_pre;    // [n_ctx] node position (ascending ctx id) in the anchor subtree or -1
  const int4* node_tab;      // [nn] {preorder position, subtree size, internal index + 1 (0: leaf),
                             //       node at preorder position n}, indexed by node position
  uint32_t nn;
  uint32_t root_only;        // the only internal node is the anchor: incl(anchor) = row total
  const uint64_t* cap_off;     // pass-1 boundary regions
  const uint32_t* bidx;
  uint64_t* bts;               // boundary timestamps (written by pass 2 after an optimistic pass 1)
  const uint32_t* n_bounds;
  const uint32_t* iter_count;  // [n] 0 = skipped
  const uint32_t* tpos;        // [n] position among kept traces
  const uint64_t* block_off;   // [n] storage cell offset of the trace's first row (kept traces)
  const uint64_t* iter_off;    // [n] iterations stored before the trace (kept traces)
  uint32_t K;                  // global min iterations over kept traces (0: none) ...
  const unsigned long long* qs;  // ... or, when set, qs_K(qs) of the device status block
  unsigned long long* cap_miss;  // speculative capacities: QS_CAP_MISS word (or null)
  uint64_t cube_cap;             // storage cells the cube buffer holds
  uint64_t xint_cap;             // entries the compact excl buffer holds
  // The cube is stored compactly: incl in rows of stride nnp (nn + 1 rounded
  // up to even: pad columns), each trace's block padded to 16 bytes, as 32-bit cells when every
  // stored iteration spans < 2^32 ns (cube32) else 64-bit; excl only for the m
  // internal nodes [Σ iters][m] (a leaf's exclusive time IS its inclusive
  // time).  Copy-out rebuilds the reference's dense int64 layout.
  uint64_t *cube_incl, *cube_xint, *gap_incl, *gap_excl;
  uint32_t cube32;
  uint32_t exact_bounds;        // pass 1 ran exact (boundary timestamps in bts)

  uint32_t m;  // internal nodes of the anchor subtree
  // cross-rank stats accumulators (k < K) and within-trace CVs
  unsigned long long *x_sum, *x_max, *x_sq;  // [K][nn], x_sq = 3 limbs [3][K][nn]
  double* within_cv;   // [n_kept][nn]
  uint8_t* within_ok;  // [n_kept][nn]
  uint32_t G;          // iterations per chunk (power of two); the row ring holds 2G + gap
  uint32_t warps;      // traces per CTA
  warp_smem_layout L;  // per-warp shared-memory carve-out (computed on the host)
  uint32_t cta_bytes;  // cta_table_bytes(n_ctx, nn, warps), computed on the host
  uint32_t one_warp;   // CTA shape: one warp per CTA (long traces) or up to 16
  uint32_t t_base, t_stop;  // this launch's traces [t_base, t_stop) (a part of tr.n)
  const uint32_t* ppo_g;    // [n_ctx] cube column byte offsets (4 * node position, pad 4 * nn),
                            // or null: they live in the per-warp window records
  // Work units (intra-trace split): when set, warp i of the grid runs unit i =
  // {trace, first event, end event, split} instead of trace t_base + i.  A
  // split trace's units snap their event ranges to chunk starts (G-iteration
  // boundaries) on the device, accumulate the window and the within-rank
  // sums into global rows with atomics (rows prepared by k_split_init), and
  // k_split_finish derives mean / min / within CV afterwards.
  const uint4* units;
  uint32_t n_units;
  unsigned long long* wacc;  // [n][nn][3] within-rank Σx, Σx² lo, hi of split traces (by tpos)
};

// CTA-shared tables placed before the per-warp carve-outs: node_tab [nn]
// (int4), then sub_pre, cct_pre, cct_size [n_ctx], then per-warp kept flags.
// One-warp CTAs read the tables from global memory instead (no CTA tables).
__host__ __device__ inline uint32_t cta_table_bytes(uint32_t n_ctx, uint32_t nn, uint32_t warps,
                                                   bool one_warp) {
  if (one_warp) return 0;
  uint32_t b = 16u * nn + 4u * n_ctx * 3 + 4u * warps;
  return (b + 15u) & ~15u;
}

// ---- the sparse window path (psg_sparse.cu): large calling-context trees --
struct sparse_args {
  trace_view tr;
  uint32_t n_ctx;
  uint64_t t0, t1;
  uint32_t clamp_tend;
  const uint32_t* parent;  // [n_ctx] (0xFFFFFFFF for the root)
  const uint32_t* depth;   // [n_ctx] ancestors of each ctx
  uint64_t row_budget;     // window rows per batch of traces (scratch bound)
  uint8_t* c_has;          // [n] carry-in outputs
  uint64_t* c_ts;
  uint32_t* c_ctx;
};
struct sparse_result {
  uint64_t n_rows = 0, n_groups = 0, n_remat = 0;
  // group_aggregate rows, sorted by (trace, ctx)
  dbuf<uint32_t> g_trace, g_ctx;
  dbuf<uint64_t> g_cnt;
  dbuf<int64_t> g_sum, g_min, g_max;
  dbuf<double> g_mean;
  // rematerialize rows (incl or excl nonzero), sorted by (trace, ctx)
  dbuf<uint32_t> r_trace, r_ctx;
  dbuf<int64_t> r_incl, r_excl;
  // the path's device workspace, kept across queries (grow-only): the sort
  // and scan scratch alone is GBs, and allocating it per query stalled the
  // stream for up to ~0.5 s (cudaMalloc / cudaFree of large buffers)
  dbuf<uint64_t> w_rows, w_i0s, w_roff, w_cdur, w_key, w_val, w_key2, w_val2, w_flag, w_pos, w_starts, w_ccnt,
      w_coff;
  dbuf<uint8_t> w_scratch;
};
void sparse_window(const sparse_args& a, sparse_result& r, cudaStream_t s);
struct sparse_result_view {
  uint32_t *g_trace, *g_ctx;
  uint64_t* g_cnt;
  int64_t *g_sum, *g_min, *g_max;
  double* g_mean;
  uint32_t *r_trace, *r_ctx;
  int64_t *r_incl, *r_excl;
};
struct dense_window {
  const uint64_t *cnt, *sum, *mn, *mx;
  const double* mean;
  const uint64_t *incl, *excl;
};
// the dense [trace][ctx] window result as sparse rows (count > 0 groups;
// incl or excl nonzero remat rows)
void dense_to_sparse(const dense_window& w, uint32_t n_traces, uint32_t n_ctx, sparse_result& r, cudaStream_t s);
// [n_traces][n_sites] incl of each site ctx (0 when the trace has no row for it)
void sparse_site_values(const sparse_result& r, const uint32_t* site, uint32_t n_sites, uint32_t n_traces,
                        uint64_t* out, cudaStream_t s);

// ---- launchers (psg_kernels.cu) ------------------------------------------

// Process-wide count of psg kernel launches (library kernels such as CUB's
// scans/sorts are not counted).
void count_launch(unsigned n = 1);
unsigned long long kernel_launches();
void launch_soa_to_aos(const uint64_t* ts, const uint32_t* ctx, uint64_t n_events, uint8_t* body,
                       cudaStream_t s);

void launch_aos_to_soa(const uint8_t* body, uint64_t n_events, uint64_t* ts, uint32_t* ctx,
                       cudaStream_t s);
// Narrow mirror of the ctx words (every ctx < 256): out[i] = pre[ctx[i]] (the
// ctx's preorder position in the CCT), n events.
void launch_ctx8(const uint32_t* ctx, uint64_t n, const int32_t* pre, uint32_t n_ctx, uint8_t* out,
                 cudaStream_t s);
void launch_validate(const trace_view& tr, uint32_t n_ctx, const uint64_t* t_begin,
                     unsigned long long* bad, unsigned long long* first_bad, cudaStream_t s);
void launch_gen_iterative(const uint64_t* jump_mats, uint64_t seed, uint32_t n_ranks,
                          uint32_t n_it, uint32_t n_k, const double* mean, const double* jitter,
                          const double* spread, uint64_t spread_kstride, uint64_t copy_ns,
                          uint32_t rank_lo, uint32_t n_local, uint64_t events_per_trace,
                          uint64_t* chunk_scratch, uint64_t* ts, uint32_t* ctx, uint64_t* t_end,
                          cudaStream_t s);
void launch_bounds(const bound_params& p, bool exact, cudaStream_t s);
// After pass 2 on an optimistic pass 1: duplicate boundary timestamps (bit 0)
// or a gap / iteration >= 2^32 ns (bit 1), OR-ed into *verify.
void launch_verify_bounds(const trace_view& tr, const uint64_t* cap_off, const uint64_t* bts,
                          const uint32_t* n_bounds, const uint32_t* iter_count,
                          unsigned long long* verify, cudaStream_t s);
// itermodel::suggest_anchor on one trace (psg_anchor.cu); returns the anchor
// ctx or 0xFFFFFFFF when no context shows periodic entries.
uint32_t launch_suggest_anchor(const uint64_t* ts, const uint32_t* ctx, uint64_t n, uint64_t t_end,
                               const uint32_t* parent, const int32_t* pre, const int32_t* size,
                               uint32_t n_ctx, uint32_t min_iters, double cv_max, cudaStream_t s);
// Cube layout from the iteration counts: kept positions, storage offsets of
// the trace blocks (rows of stride nnp, blocks padded to 4 cells), iteration
// offsets, the compact list of kept block offsets.  summary: [0] kept,
// [1] min iterations, [2] logical cells (Σ iters * nn), [4] storage cells.
void launch_cube_layout(const uint32_t* iter_count, uint32_t n, uint32_t nn, uint32_t nnp,
                        uint32_t* tpos, uint64_t* block_off, uint64_t* iter_off, uint64_t* kept_bo,
                        unsigned long long* summary, void* scratch, size_t scratch_bytes,
                        cudaStream_t s);
// Longest stored iteration of any trace (b_{k+1} - b_k, the last one ending at
// t_end) into *max_span (atomicMax): decides 32- vs 64-bit cube cells.
void launch_iter_spans(const uint64_t* cap_off, const uint64_t* bts, const uint32_t* iter_count,
                       const uint64_t* t_end, uint32_t n, unsigned long long* max_span,
                       cudaStream_t s);
size_t cube_layout_scratch_bytes(uint32_t n);
void launch_trace_query(const query_params& p, uint32_t smem_bytes, cudaStream_t s);
// resident one-warp CTAs per SM of the pass-2 instantiation a query would use
uint32_t trace_query_one_warp_per_sm(bool win, bool cube, bool exact, bool gt, uint32_t smem_bytes);
// split traces (list of loaded-trace indices): prepare their global window rows
// and within-rank accumulators before pass 2, finish them after
void launch_split_init(const query_params& p, const uint32_t* split_traces, uint32_t n_split, cudaStream_t s);
void launch_split_finish(const query_params& p, const uint32_t* split_traces, uint32_t n_split, uint32_t K,
                         cudaStream_t s);
// Dense int64 incl / excl cells (the reference layout) of the kept traces in
// [t_lo, t_hi), relative to dense row dense_row0 (= iter_off[t_lo]).
void launch_cube_dense(const void* incl, bool cube32, const uint64_t* xint, const uint32_t* iter_count,
                       const uint64_t* block_off, const uint64_t* iter_off, const int4* node_tab,
                       uint32_t nn, uint32_t nnp, uint32_t m, uint32_t t_lo, uint32_t t_hi,
                       uint64_t dense_row0, int64_t* out_incl, int64_t* out_excl, cudaStream_t s);
// Cross-rank sums over k < K, n_kept kept traces; with qs set, K and n_kept
// come from the status block and the arguments are capacities (K_cap sets the
// accumulator plane stride K_cap * nn); a set QS_CAP_MISS word skips the work.
// part: with tpos set, only the kept traces of loaded traces [ta, tb) (kept
// positions tpos[ta] .. tpos[tb], tpos[n] = QS_KEPT), in CTAs of `threads`.
struct cross_part {
  const uint32_t* tpos = nullptr;
  uint32_t ta = 0, tb = 0, n = 0;
  uint32_t threads = 512;
};
void launch_cross_stats(const void* incl, bool cube32, const uint64_t* kept_bo, uint32_t n_kept,
                        uint32_t nn, uint32_t nnp, uint32_t K, unsigned long long* x_sum,
                        unsigned long long* x_max, unsigned long long* x_sq,
                        const unsigned long long* qs, cudaStream_t s, const cross_part& part = {});
// plane_k: the K of the accumulator layout (x_sq limbs at plane_k * nn strides);
// with qs set, K / n_kept (global) / n_kept_local come from the status block.
#ifdef __CUDACC__
// Fixed-order CTA reduction (warp butterflies, then the warps' results in
// warp order; every thread receives the result): deterministic for a fixed
// block size.  s_warp holds 32 values; the block is a multiple of 32 threads.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* s_warp) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = op(v, __shfl_xor_sync(0xFFFFFFFFu, v, d));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) s_warp[w] = v;
  __syncthreads();
  T r = s_warp[0];
  for (int i = 1; i < nw; ++i) r = op(r, s_warp[i]);
  __syncthreads();  // s_warp is free for the next reduction
  return r;
}
struct op_add {
  template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct op_max {
  template <typename T> __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

#endif  // __CUDACC__

// ---- device-wide primitives (psg_sort.cu, hand-written) -------------------
size_t exclusive_sum_scratch_bytes(uint64_t n);
void exclusive_sum_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* scratch, size_t scratch_bytes,
                       cudaStream_t s);
template <typename K, typename V>
size_t sort_pairs_scratch_bytes(uint64_t n);
// stable LSD radix sort of (key, value) pairs over key bits [begin_bit, end_bit)
template <typename K, typename V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit, int end_bit, bool desc,
                void* scratch, size_t scratch_bytes, cudaStream_t s);

// tiles of the within-CV mean's first stage (node_out holds their partials)
constexpr uint32_t kWithinTiles = 592;
void launch_stats_finalize(const unsigned long long* x_sum, const unsigned long long* x_max,
                           const unsigned long long* x_sq, uint32_t K, uint32_t plane_k, uint32_t nn,
                           uint32_t n_kept, const double* within_cv, const uint8_t* within_ok,
                           uint32_t n_kept_local, double* node_out /*[nn][8]*/,
                           const unsigned long long* qs, cudaStream_t s);
// QS_CAP_MISS |= 4 when the query's K exceeds k_cap (the statistics planes).
void launch_qs_check_k(unsigned long long* qs, uint32_t k_cap, cudaStream_t s);
// The end-of-query summary of the outlier step into the status block
// (QS_WORST, QS_NSEL, QS_WORST_RATIO, QS_RACKS).
void launch_outlier_summary(const uint32_t* worst, const uint32_t* n_sel, const double* site_ratio,
                            const uint32_t* rack_nodes, uint32_t n_racks, unsigned long long* qs,
                            cudaStream_t s);
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
size_t node_select_scratch_bytes(uint32_t n_nodes);
// node means from node_acc ({Σ ns, count} per node), or given in node_mean
// when node_acc is null; then z-scores and the (mean desc, id asc) order, cut
// at top_k / z_min.
void launch_node_select(const unsigned long long* node_acc, uint32_t n_nodes, uint32_t top_k,
                        double z_min, double* node_mean, double* node_z, uint32_t* order,
                        uint32_t* n_sel, void* scratch, size_t scratch_bytes, cudaStream_t s);
// profile-record path (psg_profiles.cu)
void launch_records_to_soa(const uint8_t* body, uint64_t n, uint32_t* ctx, uint16_t* metric,
                           double* value, cudaStream_t s);
void launch_records_check(const uint32_t* ctx, const uint64_t* off, uint32_t n_prof,
                          unsigned long long* bad, cudaStream_t s);
void launch_slice(const profile_view& pv, const uint32_t* slot, uint32_t n_req,
                  const uint32_t* ctx_bits, uint32_t ctx_words, const uint32_t* metric_bits,
                  unsigned long long* counts, const unsigned long long* row_off, uint32_t* out_pid,
                  uint32_t* out_ctx, uint16_t* out_metric, double* out_value, cudaStream_t s);
void launch_profile_outliers(const profile_view& pv, const uint32_t* rank_slot, uint32_t n_ranks,
                             const uint32_t* site, uint32_t n_sites, uint16_t metric, double* vals,
                             double* ratio, uint32_t* worst, const uint32_t* node_off,
                             const uint32_t* node_rank, uint32_t n_nodes, double* node_mean,
                             cudaStream_t s);
void launch_topology(const uint32_t* selected, const uint32_t* n_sel, const uint32_t* node_rack_idx,
                     const uint32_t* node_chassis, const uint32_t* uni_cnt, uint32_t n_racks,
                     uint32_t* rack_nodes, unsigned long long* rack_mask,
                     unsigned long long* rack_full, uint32_t* rack_cnt, cudaStream_t s);

}  // namespace psg
