// Device-wide primitives of the query path, hand-written for sm_100a:
//
//   exclusive_sum_u64   exclusive prefix sums (cube layout, anchor entry
//                       offsets, run starts of the sparse window and the frame
//                       operators): per-tile reduction, one-CTA scan of the
//                       tile sums, per-tile scan with the tile's offset.
//   sort_pairs<K, V>    stable LSD radix sort of (key, value) pairs with 8-bit
//                       digits (frame argsort passes, sparse (trace, ctx) keys,
//                       the anchor's entry lists, the outlier order): per pass
//                       a per-tile digit histogram, an exclusive scan of the
//                       digit-major histogram (every tile's first slot per
//                       digit), and a stable in-tile ranking by warp
//                       (a ballot-based match per round of 32 keys, per-warp digit
//                       counters, a prefix over warps) that scatters each key
//                       to its digit's slot.  Descending order inverts the
//                       digits.  Stable: ties keep their input order, which
//                       the LSD multi-key frame sort relies on.
//
// Tiles are 2048 keys (256 threads x 8) for the sort and 4096 elements for
// the scan; both are HBM-bound streaming passes (the sort moves key + value
// twice per pass: the histogram read and the scatter's read + write).
#include "psg_internal.h"

namespace psg {
namespace {

constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
#ifndef PSG_SORT_ITEMS
#define PSG_SORT_ITEMS 8
#endif
constexpr int kSortThreads = 256, kSortItems = PSG_SORT_ITEMS, kSortTile = kSortThreads * kSortItems;
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ unsigned lanemask_lt_s() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of one value per thread across the CTA (warp shuffles, then
// the warp totals); *total receives the CTA's sum.
template <typename T, int THREADS>
__device__ __forceinline__ T block_exclusive(T v, T* s_warp, T* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    T t = lane < THREADS / 32 ? s_warp[lane] : T(0);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T y = __shfl_up_sync(0xFFFFFFFFu, t, d);
      if (lane >= d) t += y;
    }
    if (lane < THREADS / 32) s_warp[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const T before = w ? s_warp[w - 1] : T(0);
  *total = s_warp[THREADS / 32 - 1];
  __syncthreads();  // s_warp is reused by the caller's next round
  return before + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint64_t* in, uint64_t n, uint64_t* tile_sum) {
  __shared__ uint64_t s_warp[32];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t j = base + static_cast<uint64_t>(i) * kScanThreads + threadIdx.x;  // coalesced
    if (j < n) sum += in[j];
  }
  uint64_t total;
  block_exclusive<uint64_t, kScanThreads>(sum, s_warp, &total);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// One CTA: exclusive scan of the tile sums in place, in chunks of 1024.
__global__ void __launch_bounds__(1024) k_scan_tiles(uint64_t* tile_sum, uint64_t n_tiles) {
  __shared__ uint64_t s_warp[32];
  uint64_t carry = 0;
  for (uint64_t b = 0; b < n_tiles; b += 1024) {
    const uint64_t j = b + threadIdx.x;
    const uint64_t v = j < n_tiles ? tile_sum[j] : 0;
    uint64_t total;
    const uint64_t ex = block_exclusive<uint64_t, 1024>(v, s_warp, &total);
    if (j < n_tiles) tile_sum[j] = carry + ex;
    carry += total;
  }
}

// Per tile: each thread owns kScanItems consecutive elements (read through
// shared memory so the global accesses stay coalesced).
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const uint64_t* in, uint64_t* out, uint64_t n,
                                                             const uint64_t* tile_off) {
  __shared__ uint64_t s_tile[kScanTile + kScanTile / 32];  // padded: thread-consecutive reads
  __shared__ uint64_t s_warp[32];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  auto slot = [](uint32_t i) { return i + (i >> 5); };
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint32_t li = static_cast<uint32_t>(i) * kScanThreads + threadIdx.x;
    s_tile[slot(li)] = base + li < n ? in[base + li] : 0;
  }
  __syncthreads();
  uint64_t v[kScanItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = s_tile[slot(threadIdx.x * kScanItems + i)];
    sum += v[i];
  }
  uint64_t total;
  uint64_t run = tile_off[blockIdx.x] + block_exclusive<uint64_t, kScanThreads>(sum, s_warp, &total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    s_tile[slot(threadIdx.x * kScanItems + i)] = run;
    run += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint32_t li = static_cast<uint32_t>(i) * kScanThreads + threadIdx.x;
    if (base + li < n) out[base + li] = s_tile[slot(li)];
  }
}

// Lanes of the warp holding the same 9-bit value (digit, or 256 + lane for an
// empty slot): nine ballots, one per bit (a __match_any_sync equivalent that
// every execution model, including compute-sanitizer's, treats alike).
__device__ __forceinline__ unsigned match_digit(uint32_t v) {
  unsigned peers = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const bool bit = (v >> b) & 1u;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift, bool desc) {
  const uint32_t d = static_cast<uint32_t>(key >> shift) & 0xFFu;
  return desc ? 255u - d : d;
}

// Per tile: digit counts, digit-major into hist[d * n_tiles + tile].
template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_hist(const K* keys, uint64_t n, int shift, bool desc,
                                                             uint64_t* hist, uint32_t n_tiles) {
  __shared__ uint32_t s_cnt[kSortWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint64_t j = base + static_cast<uint64_t>(r) * kSortThreads + threadIdx.x;
    if (j < n) atomicAdd(&s_cnt[w][digit_of(keys[j], shift, desc)], 1u);
  }
  __syncthreads();
  (void)lane;
  for (int d = threadIdx.x; d < 256; d += kSortThreads) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kSortWarps; ++q) c += s_cnt[q][d];
    hist[static_cast<uint64_t>(d) * n_tiles + blockIdx.x] = c;
  }
}

// Per tile: stable ranks (warp w owns items [w * 32 * kSortItems, ...) of the
// tile, round r the 32 consecutive items r * 32 + lane of them: the order
// (w, r, lane) is the input order), then the scatter through shared memory:
// the tile is first placed in digit order locally, so that consecutive
// threads write consecutive addresses of each digit's run (coalesced).
template <typename K, typename V>
__global__ void __launch_bounds__(kSortThreads) k_radix_scatter(const K* kin, K* kout, const V* vin, V* vout,
                                                                uint64_t n, int shift, bool desc,
                                                                const uint64_t* off, uint32_t n_tiles) {
  __shared__ uint32_t s_cnt[kSortWarps][256];
  __shared__ uint32_t s_start[256];  // tile-local start of each digit
  __shared__ uint32_t s_gdelta[256];  // global start - local start, per digit
  __shared__ uint32_t s_warp[32];
  __shared__ uint64_t s_buf[kSortTile];  // keys, then values, in local digit order
  __shared__ uint8_t s_dig[kSortTile];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tbase = static_cast<uint64_t>(blockIdx.x) * kSortTile;
  const uint64_t wbase = tbase + static_cast<uint64_t>(w) * 32 * kSortItems;
  const uint32_t tn = static_cast<uint32_t>(min(static_cast<uint64_t>(kSortTile), n - tbase));
  K key[kSortItems];
  uint32_t dig[kSortItems], rank[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint64_t j = wbase + static_cast<uint64_t>(r) * 32 + lane;
    const bool ok = j < n;
    key[r] = ok ? kin[j] : K(0);
    dig[r] = ok ? digit_of(key[r], shift, desc) : 256u + static_cast<uint32_t>(lane);
  }
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const unsigned peers = match_digit(dig[r]);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && dig[r] < 256u) {
      old = s_cnt[w][dig[r]];
      s_cnt[w][dig[r]] = old + static_cast<uint32_t>(__popc(peers));
    }
    old = __shfl_sync(0xFFFFFFFFu, old, leader);
    rank[r] = old + static_cast<uint32_t>(__popc(peers & lanemask_lt_s()));
    __syncwarp();
  }
  __syncthreads();
  // per digit: the warps' exclusive prefix within the digit, the digit's total
  uint32_t tot = 0;
  {
    const int d = threadIdx.x;  // kSortThreads == 256 digits
#pragma unroll
    for (int q = 0; q < kSortWarps; ++q) {
      const uint32_t c = s_cnt[q][d];
      s_cnt[q][d] = tot;
      tot += c;
    }
  }
  uint32_t all;
  const uint32_t start = block_exclusive<uint32_t, kSortThreads>(tot, s_warp, &all);
  s_start[threadIdx.x] = start;
  s_gdelta[threadIdx.x] = static_cast<uint32_t>(off[static_cast<uint64_t>(threadIdx.x) * n_tiles + blockIdx.x]) - start;
  __syncthreads();
  uint32_t lpos[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    if (dig[r] < 256u) {
      lpos[r] = s_start[dig[r]] + s_cnt[w][dig[r]] + rank[r];
      s_buf[lpos[r]] = static_cast<uint64_t>(key[r]);
      s_dig[lpos[r]] = static_cast<uint8_t>(dig[r]);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads)
    kout[s_gdelta[s_dig[i]] + i] = static_cast<K>(s_buf[i]);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    const uint64_t j = wbase + static_cast<uint64_t>(r) * 32 + lane;
    if (dig[r] < 256u) s_buf[lpos[r]] = static_cast<uint64_t>(vin[j]);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads)
    vout[s_gdelta[s_dig[i]] + i] = static_cast<V>(s_buf[i]);
}

// Small inputs (n <= kSmallSort, e.g. the outlier order over nodes): every
// pair is ranked by counting (stable: equal keys keep their input order),
// instead of the 5 launches per digit pass of the general path.  One warp per
// pair, its lanes splitting the comparisons (n / 32 each), 32 pairs per CTA:
// ceil(n / 32) CTAs spread the n^2 compares over the SMs (one CTA doing all
// of them took ~0.1 ms at n = 1,000).
constexpr uint32_t kSmallSort = 2048;
template <typename K, typename V>
__global__ void __launch_bounds__(1024) k_sort_small(const K* kin, K* kout, const V* vin, V* vout, uint32_t n,
                                                     int begin_bit, int end_bit, bool desc) {
  __shared__ K s_key[kSmallSort];
  const int nb = end_bit - begin_bit;
  const K mask = nb >= static_cast<int>(8 * sizeof(K)) ? ~K(0) : ((K(1) << nb) - K(1));
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s_key[i] = (kin[i] >> begin_bit) & mask;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t i = blockIdx.x * 32u + (threadIdx.x >> 5);
  if (i >= n) return;
  const K ki = s_key[i];
  uint32_t rank = 0;
  for (uint32_t j = lane; j < n; j += 32) {
    const K kj = s_key[j];
    const bool before = desc ? (kj > ki) : (kj < ki);
    rank += (before || (kj == ki && j < i)) ? 1u : 0u;
  }
  rank = __reduce_add_sync(0xffffffffu, rank);
  if (lane == 0) {
    kout[rank] = kin[i];
    vout[rank] = vin[i];
  }
}

}  // namespace

size_t exclusive_sum_scratch_bytes(uint64_t n) {
  return 8 * ((n + kScanTile - 1) / kScanTile + 1) + 256;
}

void exclusive_sum_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* scratch, size_t scratch_bytes,
                       cudaStream_t s) {
  if (n == 0) return;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (scratch_bytes < 8 * tiles) fail(PS_E_INTERNAL, "exclusive_sum_u64: scratch too small");
  uint64_t* ts = static_cast<uint64_t*>(scratch);
  k_scan_reduce<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, ts);
  k_scan_tiles<<<1, 1024, 0, s>>>(ts, tiles);
  k_scan_apply<<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, ts);
  count_launch(3);
  PSG_CUDA(cudaGetLastError());
}

template <typename K, typename V>
size_t sort_pairs_scratch_bytes(uint64_t n) {
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
  const uint64_t cells = 256 * tiles;
  auto al = [](uint64_t b) { return (b + 255) & ~255ull; };
  return al(n * sizeof(K)) + al(n * sizeof(V)) + 2 * al(cells * 8) + al(exclusive_sum_scratch_bytes(cells)) + 256;
}

template <typename K, typename V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int begin_bit, int end_bit, bool desc,
                void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (n == 0) return;
  if (n >= (1ull << 32)) fail(PS_E_INTERNAL, "sort_pairs: more than 2^32 - 1 pairs");
  if (scratch_bytes < sort_pairs_scratch_bytes<K, V>(n)) fail(PS_E_INTERNAL, "sort_pairs: scratch too small");
  const uint32_t tiles = static_cast<uint32_t>((n + kSortTile - 1) / kSortTile);
  const uint64_t cells = 256ull * tiles;
  auto al = [](uint64_t b) { return (b + 255) & ~255ull; };
  uint8_t* p = static_cast<uint8_t*>(scratch);
  K* ktmp = reinterpret_cast<K*>(p);
  p += al(n * sizeof(K));
  V* vtmp = reinterpret_cast<V*>(p);
  p += al(n * sizeof(V));
  uint64_t* hist64 = reinterpret_cast<uint64_t*>(p);
  p += al(cells * 8);
  uint64_t* off64 = reinterpret_cast<uint64_t*>(p);
  p += al(cells * 8);
  void* sscr = p;
  const size_t sscr_bytes = exclusive_sum_scratch_bytes(cells);
  const int passes = (end_bit - begin_bit + 7) / 8;
  if (passes <= 0) {  // no key bits: the stable order is the input order
    PSG_CUDA(cudaMemcpyAsync(kout, kin, n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    PSG_CUDA(cudaMemcpyAsync(vout, vin, n * sizeof(V), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (n <= kSmallSort) {
    k_sort_small<K, V><<<static_cast<unsigned>((n + 31) / 32), 1024, 0, s>>>(kin, kout, vin, vout, static_cast<uint32_t>(n), begin_bit, end_bit, desc);
    count_launch();
    PSG_CUDA(cudaGetLastError());
    return;
  }
  const K* ks = kin;
  const V* vs = vin;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = begin_bit + 8 * pass;
    // the last pass writes the output; the others alternate so that it does
    const bool to_out = ((passes - 1 - pass) & 1) == 0;
    K* kd = to_out ? kout : ktmp;
    V* vd = to_out ? vout : vtmp;
    k_radix_hist<K><<<tiles, kSortThreads, 0, s>>>(ks, n, shift, desc, hist64, tiles);
    exclusive_sum_u64(hist64, off64, cells, sscr, sscr_bytes, s);
    k_radix_scatter<K, V><<<tiles, kSortThreads, 0, s>>>(ks, kd, vs, vd, n, shift, desc, off64, tiles);
    count_launch(2);
    PSG_CUDA(cudaGetLastError());
    ks = kd;
    vs = vd;
  }
}

template size_t sort_pairs_scratch_bytes<uint64_t, uint64_t>(uint64_t);
template size_t sort_pairs_scratch_bytes<uint32_t, uint64_t>(uint64_t);
template size_t sort_pairs_scratch_bytes<uint64_t, uint32_t>(uint64_t);
template void sort_pairs<uint64_t, uint64_t>(const uint64_t*, uint64_t*, const uint64_t*, uint64_t*, uint64_t, int,
                                             int, bool, void*, size_t, cudaStream_t);
template void sort_pairs<uint32_t, uint64_t>(const uint32_t*, uint32_t*, const uint64_t*, uint64_t*, uint64_t, int,
                                             int, bool, void*, size_t, cudaStream_t);
template void sort_pairs<uint64_t, uint32_t>(const uint64_t*, uint64_t*, const uint32_t*, uint32_t*, uint64_t, int,
                                             int, bool, void*, size_t, cudaStream_t);

}  // namespace psg
