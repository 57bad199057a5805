/*
 * TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the reference's
 * trace query path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.  The product
 * (paper_2605_03561_b200/libpsg.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * golden vectors written by the UNMODIFIED reference (oracle/_ref, built by
 * oracle/build_ref.sh; vectors in tests/golden/, script tests/golden/make_golden.py).
 *
 * Inputs are the SoA view of a trace set: off[n+1] event offsets, ts[E],
 * ctx[E], t_end[n]; the calling-context tree as parent[n_ctx]
 * (parent[0] = 0xFFFFFFFF, parent[c] < c).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NO_PARENT 0xFFFFFFFFu

/* itermodel.cpp:14-25 containment(): contains[c] = c == anchor || contains[parent[c]] */
static void containment(const uint32_t* parent, uint32_t n_ctx, uint32_t anchor, char* contains) {
  for (uint32_t c = 0; c < n_ctx; ++c) {
    if (c == anchor)
      contains[c] = 1;
    else if (c > 0 && parent[c] != NO_PARENT)
      contains[c] = contains[parent[c]];
    else
      contains[c] = 0;
  }
}

/* itermodel.cpp:145-183 rematerialize(): add every clipped segment to excl of
 * its leaf and incl of the leaf and each ancestor.  Dense outputs. */
static void rematerialize(const uint64_t* ts, const uint32_t* ctx, uint64_t n, int has_carry,
                          uint64_t carry_ts, uint32_t carry_ctx, uint64_t t0, uint64_t t1,
                          const uint32_t* parent, int64_t* incl, int64_t* excl) {
#define ADD_SEG(leaf, s0, s1)                                  \
  do {                                                         \
    uint64_t lo_ = (s0) > t0 ? (s0) : t0;                      \
    uint64_t hi_ = (s1) < t1 ? (s1) : t1;                      \
    if (lo_ < hi_) {                                           \
      int64_t d_ = (int64_t)(hi_ - lo_);                       \
      excl[leaf] += d_;                                        \
      for (uint32_t c_ = (leaf);; c_ = parent[c_]) {           \
        incl[c_] += d_;                                        \
        if (parent[c_] == NO_PARENT) break;                    \
      }                                                        \
    }                                                          \
  } while (0)
  if (has_carry) {
    uint64_t first = n == 0 ? t1 : ts[0];
    ADD_SEG(carry_ctx, carry_ts, first);
  }
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t s1 = i + 1 < n ? ts[i + 1] : t1;
    ADD_SEG(ctx[i], ts[i], s1);
  }
#undef ADD_SEG
}

static uint64_t lower_bound(const uint64_t* ts, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (ts[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* Window composition: ingest_traces rows t0 <= ts < t1
 * (store.cpp:633-676, ingest.cpp:178-208), row duration = next row of the
 * same trace or t1, group_aggregate by (trace, ctx) with sum/min/max/mean/
 * count (frame.cpp:290-408; mean = (0.0 + sum)/count in row order), and the
 * time-integrated excl/incl of rematerialize(window, carry, [t0,t1)).
 * Outputs are dense [n][n_ctx]; count == 0 marks an absent group.
 * clamp_tend (may be NULL): per-trace t_end; the window end becomes
 * min(t1, t_end[t]). */
void orc_window(const uint64_t* off, const uint64_t* ts, const uint32_t* ctx, uint32_t n,
                const uint32_t* parent, uint32_t n_ctx, uint64_t t0, uint64_t t1_all,
                const uint64_t* clamp_tend, uint64_t* count,
                int64_t* sum, int64_t* mn, int64_t* mx, double* mean, int64_t* excl, int64_t* incl,
                uint8_t* c_has, uint64_t* c_ts, uint32_t* c_ctx) {
  for (uint32_t t = 0; t < n; ++t) {
    const uint64_t b = off[t], e = off[t + 1];
    const size_t base = (size_t)t * n_ctx;
    /* clamp_tend (psg PSG_Q_CLAMP_TEND): the window ends at min(t1, t_end) per
     * trace, so [0, t_end) integrates the whole trace like its profile record */
    const uint64_t t1 = clamp_tend && clamp_tend[t] < t1_all ? clamp_tend[t] : t1_all;
    uint64_t i0 = lower_bound(ts, b, e, t0), i1 = lower_bound(ts, i0, e, t1);
    double* acc = (double*)calloc(n_ctx, sizeof(double));
    for (uint32_t c = 0; c < n_ctx; ++c) {
      count[base + c] = 0;
      sum[base + c] = mn[base + c] = mx[base + c] = 0;
      excl[base + c] = incl[base + c] = 0;
    }
    for (uint64_t i = i0; i < i1; ++i) {
      uint64_t next = i + 1 < i1 ? ts[i + 1] : t1;
      int64_t d = (int64_t)(next - ts[i]);
      size_t k = base + ctx[i];
      if (count[k] == 0) {
        sum[k] = mn[k] = mx[k] = d;
      } else {
        sum[k] = (int64_t)((uint64_t)sum[k] + (uint64_t)d);
        if (d < mn[k]) mn[k] = d;
        if (d > mx[k]) mx[k] = d;
      }
      acc[ctx[i]] += (double)d;
      count[k] += 1;
    }
    for (uint32_t c = 0; c < n_ctx; ++c)
      mean[base + c] = count[base + c] ? acc[c] / (double)count[base + c] : 0.0;
    free(acc);
    c_has[t] = i0 > b;
    c_ts[t] = i0 > b ? ts[i0 - 1] : 0;
    c_ctx[t] = i0 > b ? ctx[i0 - 1] : 0;
    if (t0 < t1)
      rematerialize(ts + i0, ctx + i0, i1 - i0, i0 > b, c_ts[t], c_ctx[t], t0, t1, parent,
                    incl + base, excl + base);
  }
}

/* itermodel.cpp:111-143 detect_iterations(): boundaries at transitions into
 * the anchor subtree, deduplicated by timestamp; iteration k = [b_k, b_k+1),
 * the last ends at t_end; empty intervals dropped.  Returns the interval
 * count (0: the trace is skipped, as build_tri_model does, :283-290) and
 * writes the interval starts/ends when the arrays are given. */
uint32_t orc_detect(const uint64_t* ts, const uint32_t* ctx, uint64_t n, uint64_t t_end,
                    const char* contains, uint64_t* starts, uint64_t* ends) {
  uint64_t nb = 0, last = 0;
  int inside = 0;
  uint64_t* bnd = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  for (uint64_t i = 0; i < n; ++i) {
    int now = contains[ctx[i]] != 0;
    if (now && !inside && (nb == 0 || last < ts[i])) {
      bnd[nb++] = ts[i];
      last = ts[i];
    }
    inside = now;
  }
  uint32_t out = 0;
  for (uint64_t k = 0; k < nb; ++k) {
    uint64_t t1 = k + 1 < nb ? bnd[k + 1] : t_end;
    if (bnd[k] < t1) {
      if (starts) starts[out] = bnd[k];
      if (ends) ends[out] = t1;
      ++out;
    }
  }
  free(bnd);
  return out;
}

/* Subtree node ids (ascending) of `anchor`; returns the count. */
uint32_t orc_subtree(const uint32_t* parent, uint32_t n_ctx, uint32_t anchor, uint32_t* node_ids) {
  char* contains = (char*)malloc(n_ctx);
  containment(parent, n_ctx, anchor, contains);
  uint32_t nn = 0;
  for (uint32_t c = 0; c < n_ctx; ++c)
    if (contains[c]) {
      if (node_ids) node_ids[nn] = c;
      ++nn;
    }
  free(contains);
  return nn;
}

/* Iteration counts per trace (0 = skipped). */
void orc_iter_counts(const uint64_t* off, const uint64_t* ts, const uint32_t* ctx,
                     const uint64_t* t_end, uint32_t n, const uint32_t* parent, uint32_t n_ctx,
                     uint32_t anchor, uint32_t* iter_counts) {
  char* contains = (char*)malloc(n_ctx);
  containment(parent, n_ctx, anchor, contains);
  for (uint32_t t = 0; t < n; ++t)
    iter_counts[t] = orc_detect(ts + off[t], ctx + off[t], off[t + 1] - off[t], t_end[t], contains,
                                NULL, NULL);
  free(contains);
}

/* itermodel.cpp:242-360 build_tri_model() with an explicit anchor: per kept
 * trace, per interval, rematerialize(window, carry, interval) projected onto
 * the anchor subtree; cells iteration-major, node-minor, kept traces in input
 * order; gap rows [first_ts, b_0).  Buffers sized from orc_iter_counts. */
void orc_cube(const uint64_t* off, const uint64_t* ts, const uint32_t* ctx, const uint64_t* t_end,
              uint32_t n, const uint32_t* parent, uint32_t n_ctx, uint32_t anchor, int64_t* incl,
              int64_t* excl, int64_t* gap_incl, int64_t* gap_excl) {
  char* contains = (char*)malloc(n_ctx);
  containment(parent, n_ctx, anchor, contains);
  int32_t* npos = (int32_t*)malloc(sizeof(int32_t) * n_ctx);
  uint32_t nn = 0;
  for (uint32_t c = 0; c < n_ctx; ++c) npos[c] = contains[c] ? (int32_t)nn++ : -1;
  int64_t* pi = (int64_t*)malloc(sizeof(int64_t) * n_ctx);
  int64_t* pe = (int64_t*)malloc(sizeof(int64_t) * n_ctx);
  size_t cell = 0, kept = 0;
  for (uint32_t t = 0; t < n; ++t) {
    const uint64_t* T = ts + off[t];
    const uint32_t* X = ctx + off[t];
    const uint64_t ne = off[t + 1] - off[t];
    uint64_t* st = (uint64_t*)malloc(sizeof(uint64_t) * (ne + 1));
    uint64_t* en = (uint64_t*)malloc(sizeof(uint64_t) * (ne + 1));
    uint32_t ni = orc_detect(T, X, ne, t_end[t], contains, st, en);
    if (ni == 0) {
      free(st);
      free(en);
      continue;
    }
    for (int part = -1; part < (int)ni; ++part) {
      uint64_t a, b;
      if (part < 0) {
        if (!(ne > 0 && T[0] < st[0])) continue;
        a = T[0];
        b = st[0];
      } else {
        a = st[part];
        b = en[part];
      }
      uint64_t lo = lower_bound(T, 0, ne, a), hi = lower_bound(T, lo, ne, b);
      memset(pi, 0, sizeof(int64_t) * n_ctx);
      memset(pe, 0, sizeof(int64_t) * n_ctx);
      rematerialize(T + lo, X + lo, hi - lo, lo > 0, lo > 0 ? T[lo - 1] : 0, lo > 0 ? X[lo - 1] : 0,
                    a, b, parent, pi, pe);
      int64_t* di = part < 0 ? gap_incl + kept * nn : incl + cell + (size_t)part * nn;
      int64_t* de = part < 0 ? gap_excl + kept * nn : excl + cell + (size_t)part * nn;
      for (uint32_t c = 0; c < n_ctx; ++c)
        if (npos[c] >= 0) {
          di[npos[c]] = pi[c];
          de[npos[c]] = pe[c];
        }
    }
    if (!(ne > 0 && T[0] < st[0]))
      for (uint32_t j = 0; j < nn; ++j) gap_incl[kept * nn + j] = gap_excl[kept * nn + j] = 0;
    cell += (size_t)ni * nn;
    ++kept;
    free(st);
    free(en);
  }
  free(contains);
  free(npos);
  free(pi);
  free(pe);
}

/* diagnostics.cpp:21-31 cv_percent (population, two-pass); returns 0 and sets
 * *ok = 0 where the reference raises undefined_cv. */
static double cv_percent(const double* v, size_t n, int* ok) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += v[i];
  double mean = s / (double)n;
  if (mean == 0.0) {
    *ok = 0;
    return 0.0;
  }
  double var = 0.0;
  for (size_t i = 0; i < n; ++i) var += (v[i] - mean) * (v[i] - mean);
  var /= (double)n;
  return 100.0 * sqrt(var) / mean;
}

/* diagnostics.cpp:83-158: node_matrix over the ordinal intersection
 * (min_iterations), savings_report and iteration_cv_report for one node
 * position.  out[0..5] = avg_mean, avg_max, savings, total, across, within;
 * *ok = 0 where iteration_cv_report would raise. */
void orc_node_stats(const int64_t* incl, const uint64_t* block_offset, const uint32_t* iter_counts,
                    uint32_t n_kept, uint32_t nn, uint32_t npos, double* out, int* ok) {
  uint32_t K = 0xFFFFFFFFu;
  for (uint32_t t = 0; t < n_kept; ++t)
    if (iter_counts[t] < K) K = iter_counts[t];
  if (n_kept == 0) K = 0;
  double* col = (double*)malloc(sizeof(double) * (n_kept + 1));
  double* row = (double*)malloc(sizeof(double) * (K + 1));
  double avg_mean = 0.0, avg_max = 0.0, across = 0.0, within = 0.0;
  *ok = (n_kept >= 2 && K >= 2);
  for (uint32_t k = 0; k < K; ++k) {
    double sum = 0.0, max = 0.0;
    for (uint32_t t = 0; t < n_kept; ++t) {
      double v = (double)incl[block_offset[t] + (size_t)k * nn + npos] / 1e9;
      col[t] = v;
      if (t == 0) max = v;
      sum += v;
      if (v > max) max = v;
    }
    avg_mean += sum / (double)n_kept;
    avg_max += max;
    if (*ok) across += cv_percent(col, n_kept, ok);
  }
  avg_mean /= (double)K;
  avg_max /= (double)K;
  if (*ok) {
    across /= (double)K;
    for (uint32_t t = 0; t < n_kept && *ok; ++t) {
      for (uint32_t k = 0; k < K; ++k)
        row[k] = (double)incl[block_offset[t] + (size_t)k * nn + npos] / 1e9;
      within += cv_percent(row, K, ok);
    }
    within /= (double)n_kept;
  }
  out[0] = avg_mean;
  out[1] = avg_max;
  out[2] = avg_max - avg_mean;
  out[3] = (avg_max - avg_mean) * K;
  out[4] = across;
  out[5] = within;
  free(col);
  free(row);
}

/* Outlier chain on per-rank values (workflows.cpp:442-476, diagnostics.cpp:
 * 10-19, 378-403): balance ratio per site over ranks (sum / n / max, 1.0 when
 * max == 0), worst = first minimum, node means as sequential sums of seconds
 * in rank order, then the z-score / top-k restatement: population z over node
 * means, order by (mean desc, node asc), keep z >= z_min, cap at top_k.
 * values[s * n_ranks + r] in ns; node_of_rank[r] in [0, n_nodes).
 * Returns the number of selected nodes. */
uint32_t orc_outliers(const int64_t* values, uint32_t n_sites, uint32_t n_ranks,
                      const uint32_t* node_of_rank, uint32_t n_nodes, uint32_t top_k, double z_min,
                      double* site_ratio, uint32_t* worst, double* node_mean, double* node_z,
                      uint32_t* selected) {
  uint32_t w = 0;
  for (uint32_t s = 0; s < n_sites; ++s) {
    double sum = 0.0, mx = (double)values[(size_t)s * n_ranks] / 1e9;
    for (uint32_t r = 0; r < n_ranks; ++r) {
      double v = (double)values[(size_t)s * n_ranks + r] / 1e9;
      if (v > mx) mx = v;
      sum += v;
    }
    site_ratio[s] = mx == 0.0 ? 1.0 : sum / (double)n_ranks / mx;
    if (site_ratio[s] < site_ratio[w]) w = s;
  }
  *worst = w;
  double* acc = (double*)calloc(n_nodes, sizeof(double));
  uint32_t* cnt = (uint32_t*)calloc(n_nodes, sizeof(uint32_t));
  for (uint32_t r = 0; r < n_ranks; ++r) {
    acc[node_of_rank[r]] += (double)values[(size_t)w * n_ranks + r] / 1e9;
    cnt[node_of_rank[r]] += 1;
  }
  double mu = 0.0;
  for (uint32_t i = 0; i < n_nodes; ++i) {
    node_mean[i] = cnt[i] ? acc[i] / cnt[i] : 0.0;
    mu += node_mean[i];
  }
  mu /= (double)n_nodes;
  double var = 0.0;
  for (uint32_t i = 0; i < n_nodes; ++i) var += (node_mean[i] - mu) * (node_mean[i] - mu);
  double sd = sqrt(var / (double)n_nodes);
  for (uint32_t i = 0; i < n_nodes; ++i) node_z[i] = sd > 0.0 ? (node_mean[i] - mu) / sd : 0.0;
  /* insertion order by (mean desc, id asc) — n_nodes is small in the tests */
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n_nodes);
  for (uint32_t i = 0; i < n_nodes; ++i) {
    uint32_t j = i;
    while (j > 0 && node_mean[order[j - 1]] < node_mean[i]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = i;
  }
  uint32_t ns = 0;
  for (uint32_t i = 0; i < n_nodes; ++i) {
    if (node_z[order[i]] < z_min) break;
    if (top_k && ns >= top_k) break;
    selected[ns++] = order[i];
  }
  free(order);
  free(acc);
  free(cnt);
  return ns;
}

/* itermodel.cpp:27-41 gap_cv(): population CV (fraction) of inter-entry gaps. */
static double gap_cv(const uint64_t* e, uint64_t n) {
  double mean = 0.0;
  for (uint64_t i = 1; i < n; ++i) mean += (double)(e[i] - e[i - 1]);
  mean /= (double)(n - 1);
  if (mean <= 0.0) return INFINITY;
  double var = 0.0;
  for (uint64_t i = 1; i < n; ++i) {
    double g = (double)(e[i] - e[i - 1]);
    var += (g - mean) * (g - mean);
  }
  var /= (double)(n - 1);
  return sqrt(var) / mean;
}

/* itermodel.cpp:45-109 suggest_anchor(): walk the step function once; a
 * context is ENTERED at event i when it is on the ancestor chain of ctx[i]
 * but not on the previous event's chain; covered time = inclusive time of the
 * segments (the last one ends at max(t_end, ts)).  Candidates have >=
 * min_iters entries and gap CV <= cv_max; the winner covers the most time
 * (ties: smallest id).  Returns 0xFFFFFFFF when there is no candidate (the
 * reference raises no_periodicity). */
uint32_t orc_suggest_anchor(const uint64_t* ts, const uint32_t* ctx, uint64_t n, uint64_t t_end,
                            const uint32_t* parent, uint32_t n_ctx, uint32_t min_iters,
                            double cv_max) {
  uint64_t* cnt = (uint64_t*)calloc(n_ctx, sizeof(uint64_t));
  uint64_t* covered = (uint64_t*)calloc(n_ctx, sizeof(uint64_t));
  char* on_prev = (char*)calloc(n_ctx, 1);
  char* on_cur = (char*)calloc(n_ctx, 1);
  /* pass 1: entry counts and covered time */
  for (uint64_t i = 0; i < n; ++i) {
    memset(on_cur, 0, n_ctx);
    for (uint32_t c = ctx[i];; c = parent[c]) {
      on_cur[c] = 1;
      if (!on_prev[c]) cnt[c] += 1;
      if (parent[c] == NO_PARENT) break;
    }
    uint64_t end = i + 1 < n ? ts[i + 1] : (t_end > ts[i] ? t_end : ts[i]);
    uint64_t dur = end - ts[i];
    if (dur)
      for (uint32_t c = ctx[i];; c = parent[c]) {
        covered[c] += dur;
        if (parent[c] == NO_PARENT) break;
      }
    char* tmp = on_prev;
    on_prev = on_cur;
    on_cur = tmp;
  }
  /* pass 2: entry timestamps per context, in order */
  uint64_t* off = (uint64_t*)calloc(n_ctx + 1, sizeof(uint64_t));
  for (uint32_t c = 0; c < n_ctx; ++c) off[c + 1] = off[c] + cnt[c];
  uint64_t* ent = (uint64_t*)malloc(sizeof(uint64_t) * (off[n_ctx] + 1));
  uint64_t* fill = (uint64_t*)calloc(n_ctx, sizeof(uint64_t));
  memset(on_prev, 0, n_ctx);
  for (uint64_t i = 0; i < n; ++i) {
    memset(on_cur, 0, n_ctx);
    for (uint32_t c = ctx[i];; c = parent[c]) {
      on_cur[c] = 1;
      if (!on_prev[c]) ent[off[c] + fill[c]++] = ts[i];
      if (parent[c] == NO_PARENT) break;
    }
    char* tmp = on_prev;
    on_prev = on_cur;
    on_cur = tmp;
  }
  uint32_t best = NO_PARENT;
  uint64_t best_cov = 0;
  for (uint32_t c = 0; c < n_ctx; ++c) {
    if (cnt[c] < min_iters) continue;
    if (gap_cv(ent + off[c], cnt[c]) > cv_max) continue;
    if (best == NO_PARENT || covered[c] > best_cov) {
      best = c;
      best_cov = covered[c];
    }
  }
  free(cnt);
  free(covered);
  free(on_prev);
  free(on_cur);
  free(off);
  free(ent);
  free(fill);
  return best;
}
