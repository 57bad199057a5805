// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Harness over the UNMODIFIED reference core (built by oracle/build_ref.sh
// from /root/reference/proj into oracle/_ref/).  It exposes extern "C" entry
// points so the Python tests and bench.py's CPU arms can drive the reference's
// own functions:
//   * golden-vector writers (raw little-endian arrays, one file per column);
//   * the reference's report renderers (iterations / congestion);
//   * timing of the reference CPU compositions named in SURVEY.md §8(d).
//
// The window composition is the one SURVEY.md §3(3) and §8(d) define:
//   ingest::ingest_traces (ingest.cpp:178-208)
//   -> dur_ns = (next row of the same profile ? next.ts : t1) - ts   [glue]
//   -> frame::group_aggregate({profile_id, ctx_id},
//                             {sum,min,max,mean,count}(dur_ns))   (frame.cpp:290-408)
// plus the per-trace time integration itermodel::rematerialize(window, carry,
// [t0,t1)) (itermodel.cpp:145-183).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "core/diagnostics.hpp"
#include "core/frame.hpp"
#include "core/ingest.hpp"
#include "core/itermodel.hpp"
#include "core/query.hpp"
#include "core/store.hpp"
#include "core/topology.hpp"
#include "core/util.hpp"
#include "core/workflows.hpp"

using namespace perfslice;

namespace {

thread_local std::string g_err;

template <typename T>
void dump(const std::string& dir, const std::string& name, const std::vector<T>& v) {
  std::ofstream f(dir + "/" + name + ".bin", std::ios::binary | std::ios::trunc);
  if (!v.empty()) f.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
  if (!f) throw std::runtime_error("cannot write " + dir + "/" + name);
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const perfslice::error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

char* copy_out(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::vector<uint32_t> all_trace_ids(const store::db_handle& h) {
  std::vector<uint32_t> ids;
  for (const auto& e : h.trace_index()) ids.push_back(e.profile_id);
  return ids;
}

struct window_out {
  frame::table agg;
  ingest::trace_ingest_result ing;
};

window_out window_composition(const store::db_handle& h, uint64_t t0, uint64_t t1,
                              unsigned jobs) {
  window_out w;
  w.ing = ingest::ingest_traces(h, all_trace_ids(h), t0, t1, jobs);
  const auto& ev = w.ing.events;
  const std::size_t n = ev.size();
  std::vector<uint64_t> pid(n), ctx(n);
  std::vector<int64_t> dur(n);
  for (std::size_t i = 0; i < n; ++i) {
    pid[i] = ev.profile_id[i];
    ctx[i] = ev.ctx_id[i];
    uint64_t next = (i + 1 < n && ev.profile_id[i + 1] == ev.profile_id[i])
                        ? ev.timestamp_ns[i + 1]
                        : t1;
    dur[i] = static_cast<int64_t>(next - ev.timestamp_ns[i]);
  }
  frame::table t;
  t.add(frame::column::of_u64("profile_id", std::move(pid)));
  t.add(frame::column::of_u64("ctx_id", std::move(ctx)));
  t.add(frame::column::of_i64("dur_ns", std::move(dur)));
  frame::backend be = jobs > 1 ? frame::backend::par(jobs) : frame::backend::seq();
  w.agg = frame::group_aggregate(t, {"profile_id", "ctx_id"},
                                 {{"dur_ns", frame::agg_fn::sum},
                                  {"dur_ns", frame::agg_fn::min},
                                  {"dur_ns", frame::agg_fn::max},
                                  {"dur_ns", frame::agg_fn::mean},
                                  {"dur_ns", frame::agg_fn::count}},
                                 be);
  return w;
}

itermodel::anchor_policy policy_of(int64_t anchor) {
  return anchor < 0 ? itermodel::anchor_policy::auto_detect()
                    : itermodel::anchor_policy::explicit_ctx(static_cast<uint32_t>(anchor));
}

template <typename Fn>
double time_mean(unsigned repeat, Fn&& fn) {
  if (repeat == 0) repeat = 1;
  double total = 0.0;
  for (unsigned r = 0; r < repeat; ++r) {
    auto a = std::chrono::steady_clock::now();
    fn();
    auto b = std::chrono::steady_clock::now();
    total += std::chrono::duration<double>(b - a).count();
  }
  return total / repeat;
}

}  // namespace

extern "C" {

const char* refh_last_error(void) { return g_err.c_str(); }
void refh_free(char* p) { std::free(p); }
unsigned refh_default_jobs(void) { return util::default_jobs(); }

// workflows::generate_database (workflows.cpp:64-81): scenario JSON -> DB dir.
int refh_generate(const char* config_json, const char* dir, char** truth_out) {
  return guarded([&] {
    std::string truth = workflows::generate_database(config_json, dir);
    if (truth_out) *truth_out = copy_out(truth);
  });
}

// Writes raw SoA traces as a reference database through the reference's own
// writer (store::write_database, store.cpp:313-392): contexts from parent[]
// (kind function), one profile per trace (rank = position, hostname given per
// trace or "x1000c0s0b0n0"), no profile records.  Lets the golden-vector
// script pin arbitrary (random, edge-case) trace sets on the reference.
int refh_write_traces(const char* dir, const uint32_t* parent, uint32_t n_ctx,
                      const uint32_t* pid, const uint64_t* off, const uint64_t* ts,
                      const uint32_t* ctx, const uint64_t* t_end, uint32_t n) {
  return guarded([&] {
    store::database_image img;
    img.meta.metrics.push_back({0, store::metric_scope::inclusive, "cputime", "s"});
    for (uint32_t c = 0; c < n_ctx; ++c)
      img.meta.contexts.push_back(
          {c, parent[c], store::ctx_kind::function, "c" + std::to_string(c)});
    for (uint32_t t = 0; t < n; ++t) {
      img.meta.profiles.push_back({pid[t], static_cast<int32_t>(t), 0, "x1000c0s0b0n0", 0});
      img.records.emplace_back();
      store::trace_data td;
      td.profile_id = pid[t];
      td.t_end_ns = t_end[t];
      for (uint64_t i = off[t]; i < off[t + 1]; ++i) td.events.push_back({ts[i], ctx[i]});
      img.traces.push_back(std::move(td));
    }
    store::write_database(img, dir);
  });
}

// Window composition goldens (see file header).
int refh_window(const char* dir, uint64_t t0, uint64_t t1, unsigned jobs,
                const char* outdir, int write_rows) {
  return guarded([&] {
    auto h = store::db_handle::open(dir);
    window_out w = window_composition(h, t0, t1, jobs);
    std::string o = outdir;
    std::filesystem::create_directories(o);
    dump(o, "wa_pid", w.agg.col("profile_id").u64s());
    dump(o, "wa_ctx", w.agg.col("ctx_id").u64s());
    dump(o, "wa_sum", w.agg.col("dur_ns_sum").i64s());
    dump(o, "wa_min", w.agg.col("dur_ns_min").i64s());
    dump(o, "wa_max", w.agg.col("dur_ns_max").i64s());
    dump(o, "wa_mean", w.agg.col("dur_ns_mean").f64s());
    dump(o, "wa_count", w.agg.col("dur_ns_count").u64s());
    std::vector<uint32_t> cpid, cctx;
    std::vector<uint8_t> chas;
    std::vector<uint64_t> cts;
    std::vector<uint32_t> rm_pid, rm_ctx;
    std::vector<int64_t> rm_incl, rm_excl;
    const auto& ev = w.ing.events;
    std::size_t row = 0;
    for (const auto& [pid, carry] : w.ing.carry_in) {
      cpid.push_back(pid);
      chas.push_back(carry ? 1 : 0);
      cts.push_back(carry ? carry->timestamp_ns : 0);
      cctx.push_back(carry ? carry->ctx_id : 0);
      if (t0 < t1) {
        std::vector<store::trace_event> win;
        while (row < ev.size() && ev.profile_id[row] == pid) {
          win.push_back({ev.timestamp_ns[row], ev.ctx_id[row]});
          ++row;
        }
        for (const auto& e : itermodel::rematerialize(win, carry, {t0, t1}, h.meta())) {
          rm_pid.push_back(pid);
          rm_ctx.push_back(e.ctx_id);
          rm_incl.push_back(e.incl_ns);
          rm_excl.push_back(e.excl_ns);
        }
      }
    }
    dump(o, "carry_pid", cpid);
    dump(o, "carry_has", chas);
    dump(o, "carry_ts", cts);
    dump(o, "carry_ctx", cctx);
    dump(o, "rm_pid", rm_pid);
    dump(o, "rm_ctx", rm_ctx);
    dump(o, "rm_incl", rm_incl);
    dump(o, "rm_excl", rm_excl);
    if (write_rows) {
      dump(o, "rows_pid", ev.profile_id);
      dump(o, "rows_ts", ev.timestamp_ns);
      dump(o, "rows_ctx", ev.ctx_id);
    }
  });
}

// ingest::ingest_profiles (ingest.cpp:155-176): the profile-record slice of
// the requested profiles; all_ctx = a keep set covering the whole tree.
int refh_slices(const char* dir, const uint32_t* pids, uint32_t n_pids, const uint32_t* ctxs,
                uint32_t n_ctx, int all_ctx, const uint16_t* metrics, uint32_t n_metrics,
                unsigned jobs, const char* outdir) {
  return guarded([&] {
    auto h = store::db_handle::open(dir);
    ingest::keep_set keep;
    if (all_ctx) {
      for (uint32_t i = 0; i < h.meta().contexts.size(); ++i) keep.ids.push_back(i);
    } else {
      keep.ids.assign(ctxs, ctxs + n_ctx);
    }
    std::vector<uint16_t> m(metrics, metrics + n_metrics);
    auto t = ingest::ingest_profiles(h, std::vector<uint32_t>(pids, pids + n_pids), keep, m, jobs);
    std::string o = outdir;
    std::filesystem::create_directories(o);
    dump(o, "pid", t.profile_id);
    dump(o, "ctx", t.ctx_id);
    dump(o, "metric", t.metric_id);
    dump(o, "value", t.value);
  });
}

// Mean wall time of ingest_profiles over all rank profiles for the given ctx
// set and metric (the CPU baseline of the profile slice path).
double refh_time_slices(const char* dir, const uint32_t* ctxs, uint32_t n_ctx, uint16_t metric,
                        unsigned jobs, unsigned repeat) {
  try {
    auto h = store::db_handle::open(dir);
    std::vector<uint32_t> pids;
    for (const auto& p : h.meta().profiles)
      if (p.rank >= 0) pids.push_back(p.id);
    ingest::keep_set keep;
    keep.ids.assign(ctxs, ctxs + n_ctx);
    return time_mean(repeat, [&] { ingest::ingest_profiles(h, pids, keep, {metric}, jobs); });
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// itermodel::build_tri_model (itermodel.cpp:242-360) + savings_report /
// iteration_cv_report on the subtree leaves (diagnostics.cpp:100-158).
int refh_trimodel(const char* dir, int64_t anchor, unsigned jobs, double total_time,
                  const char* outdir) {
  return guarded([&] {
    auto h = store::db_handle::open(dir);
    auto m = itermodel::build_tri_model(h, all_trace_ids(h), policy_of(anchor), jobs);
    std::string o = outdir;
    std::filesystem::create_directories(o);
    dump(o, "anchor", std::vector<uint32_t>{m.anchor_ctx});
    dump(o, "node_ids", m.node_ids);
    dump(o, "trace_ids", m.trace_ids);
    dump(o, "iter_counts", m.iter_counts);
    dump(o, "skipped", m.skipped_traces);
    std::vector<uint64_t> bo(m.block_offset.begin(), m.block_offset.end());
    dump(o, "block_offset", bo);
    dump(o, "incl", m.incl_ns);
    dump(o, "excl", m.excl_ns);
    dump(o, "gap_incl", m.gap_incl_ns);
    dump(o, "gap_excl", m.gap_excl_ns);
    auto leaves = m.subtree_leaves(h.meta());
    dump(o, "leaves", leaves);
    if (total_time <= 0.0)
      for (const auto& e : h.trace_index())
        total_time = std::max(total_time, static_cast<double>(e.t_end_ns - e.t_begin_ns) / 1e9);
    std::vector<double> sv;  // per leaf: avg_mean, avg_max, savings, total
    std::vector<double> summary(4, 0.0);
    int sav_ok = 1;
    try {
      auto s = diagnostics::savings_report(m, leaves, total_time);
      for (const auto& r : s.rows) {
        sv.push_back(r.avg_mean_s);
        sv.push_back(r.avg_max_s);
        sv.push_back(r.savings_per_iter_s);
        sv.push_back(r.total_reduction_s);
      }
      summary = {static_cast<double>(s.n_iterations), s.total_savings_s, total_time,
                 s.speedup_frac};
    } catch (const perfslice::error&) {
      sav_ok = 0;
    }
    dump(o, "savings", sv);
    dump(o, "savings_summary", summary);
    dump(o, "savings_ok", std::vector<int32_t>{sav_ok});
    std::vector<double> cv;
    std::vector<int32_t> cv_ok;
    for (uint32_t c : leaves) {
      try {
        auto r = diagnostics::iteration_cv_report(m, c);
        cv.push_back(r.across_rank_cv_pct);
        cv.push_back(r.within_rank_cv_pct);
        cv_ok.push_back(1);
      } catch (const perfslice::error&) {
        cv.push_back(0.0);
        cv.push_back(0.0);
        cv_ok.push_back(0);
      }
    }
    dump(o, "cv", cv);
    dump(o, "cv_ok", cv_ok);
  });
}

// workflows::iterations_report (workflows.cpp:281-411).
int refh_iterations_report(const char* dir, const char* anchor, double total_time,
                           int json, unsigned jobs, char** out) {
  return guarded([&] {
    auto h = store::db_handle::open(dir);
    workflows::session_options so;
    so.jobs = jobs;
    auto s = workflows::open_session(h, so);
    workflows::iterations_options io;
    io.anchor = anchor;
    io.total_time_s = total_time;
    *out = copy_out(workflows::iterations_report(
        *s, io, json ? workflows::output_format::json : workflows::output_format::csv));
  });
}

// workflows::congestion_report (workflows.cpp:413-599).
int refh_congestion_report(const char* dir, const char* glob, const char* method, unsigned k,
                           double eps, double min_share, int json, unsigned jobs, char** out) {
  return guarded([&] {
    auto h = store::db_handle::open(dir);
    workflows::session_options so;
    so.min_inclusive_share = min_share;
    so.jobs = jobs;
    auto s = workflows::open_session(h, so);
    workflows::congestion_options co;
    co.callsite_glob = glob;
    co.method = method;
    co.k = k;
    co.eps = eps;
    *out = copy_out(workflows::congestion_report(
        *s, co, json ? workflows::output_format::json : workflows::output_format::csv));
  });
}

// topology::localize_outliers (topology.cpp:54-92) rendered as JSON.
int refh_localize(const char* const* outliers, size_t n_out, const char* const* universe,
                  size_t n_uni, char** out) {
  return guarded([&] {
    std::vector<std::string> o(outliers, outliers + n_out), u(universe, universe + n_uni);
    auto r = topology::localize_outliers(o, u);
    *out = copy_out(topology::render_report(r, topology::report_format::json));
  });
}

// ---- CPU timing of the reference compositions (steady_clock mean) ----------

double refh_time_window(const char* dir, uint64_t t0, uint64_t t1, unsigned jobs,
                        unsigned repeat) {
  double t = -1.0;
  guarded([&] {
    auto h = store::db_handle::open(dir);
    t = time_mean(repeat, [&] { (void)window_composition(h, t0, t1, jobs); });
  });
  return t;
}

double refh_time_trimodel(const char* dir, int64_t anchor, unsigned jobs, unsigned repeat) {
  double t = -1.0;
  guarded([&] {
    auto h = store::db_handle::open(dir);
    auto ids = all_trace_ids(h);
    double total_time = 0.0;
    for (const auto& e : h.trace_index())
      total_time = std::max(total_time, static_cast<double>(e.t_end_ns - e.t_begin_ns) / 1e9);
    t = time_mean(repeat, [&] {
      auto m = itermodel::build_tri_model(h, ids, policy_of(anchor), jobs);
      auto leaves = m.subtree_leaves(h.meta());
      (void)diagnostics::savings_report(m, leaves, total_time);
      for (uint32_t c : leaves) {
        try {
          (void)diagnostics::iteration_cv_report(m, c);
        } catch (const perfslice::error&) {
        }
      }
    });
  });
  return t;
}

// The full trace query of BASELINE configs[1] on a sample: window composition
// + tri-model + savings + CV.
double refh_time_query(const char* dir, uint64_t t0, uint64_t t1, int64_t anchor,
                       unsigned jobs, unsigned repeat) {
  double t = -1.0;
  guarded([&] {
    auto h = store::db_handle::open(dir);
    auto ids = all_trace_ids(h);
    double total_time = 0.0;
    for (const auto& e : h.trace_index())
      total_time = std::max(total_time, static_cast<double>(e.t_end_ns - e.t_begin_ns) / 1e9);
    t = time_mean(repeat, [&] {
      (void)window_composition(h, t0, t1, jobs);
      auto m = itermodel::build_tri_model(h, ids, policy_of(anchor), jobs);
      auto leaves = m.subtree_leaves(h.meta());
      (void)diagnostics::savings_report(m, leaves, total_time);
      for (uint32_t c : leaves) {
        try {
          (void)diagnostics::iteration_cv_report(m, c);
        } catch (const perfslice::error&) {
        }
      }
    });
  });
  return t;
}

double refh_time_congestion(const char* dir, unsigned jobs, unsigned repeat) {
  double t = -1.0;
  guarded([&] {
    auto h = store::db_handle::open(dir);
    workflows::session_options so;
    so.min_inclusive_share = 0.01;
    so.jobs = jobs;
    t = time_mean(repeat, [&] {
      auto s = workflows::open_session(h, so);
      workflows::congestion_options co;
      (void)workflows::congestion_report(*s, co, workflows::output_format::json);
    });
  });
  return t;
}

// ---- frame operators (frame.cpp) on raw columns: dtype 0 i64, 1 u64, 2 f64 ----
namespace {
frame::column make_col(const std::string& name, int dt, const void* data, uint64_t n) {
  if (dt == 0) {
    const int64_t* p = static_cast<const int64_t*>(data);
    return frame::column::of_i64(name, std::vector<int64_t>(p, p + n));
  }
  if (dt == 1) {
    const uint64_t* p = static_cast<const uint64_t*>(data);
    return frame::column::of_u64(name, std::vector<uint64_t>(p, p + n));
  }
  const double* p = static_cast<const double*>(data);
  return frame::column::of_f64(name, std::vector<double>(p, p + n));
}
std::vector<uint64_t> iota_u64(uint64_t n) {
  std::vector<uint64_t> v(n);
  for (uint64_t i = 0; i < n; ++i) v[i] = i;
  return v;
}
void copy_col(const frame::column& c, void* out) {
  switch (c.type()) {
    case frame::dtype::i64: std::memcpy(out, c.i64s().data(), 8 * c.size()); break;
    case frame::dtype::u64: std::memcpy(out, c.u64s().data(), 8 * c.size()); break;
    case frame::dtype::f64: std::memcpy(out, c.f64s().data(), 8 * c.size()); break;
    default: throw std::runtime_error("string column");
  }
}
frame::backend be_of(unsigned jobs) { return jobs > 1 ? frame::backend::par(jobs) : frame::backend::seq(); }
}  // namespace

// frame::sort -> the permutation (gathered row ids)
int refh_frame_sort(uint64_t n, uint32_t nk, const int* dts, const void* const* keys, const uint8_t* asc,
                    unsigned jobs, uint64_t* perm) {
  return guarded([&] {
    frame::table t;
    std::vector<std::string> names;
    std::vector<bool> a;
    for (uint32_t k = 0; k < nk; ++k) {
      names.push_back("k" + std::to_string(k));
      t.add(make_col(names.back(), dts[k], keys[k], n));
      a.push_back(asc ? asc[k] != 0 : true);
    }
    t.add(frame::column::of_u64("_row", iota_u64(n)));
    frame::table o = frame::sort(t, names, asc ? a : std::vector<bool>{}, be_of(jobs));
    copy_col(o.col("_row"), perm);
  });
}

// frame::group_aggregate with one aggregate; outputs the group keys' first
// key column as row ids of the group heads is not available, so the keys are
// returned as columns (each 8 bytes) plus the aggregate column
int refh_frame_group(uint64_t n, uint32_t nk, const int* dts, const void* const* keys, int sdt,
                     const void* src, int fn, unsigned jobs, uint64_t* n_groups, void* const* key_out,
                     void* agg_out) {
  return guarded([&] {
    frame::table t;
    std::vector<std::string> names;
    for (uint32_t k = 0; k < nk; ++k) {
      names.push_back("k" + std::to_string(k));
      t.add(make_col(names.back(), dts[k], keys[k], n));
    }
    t.add(make_col("v", sdt, src, n));
    const frame::agg_fn fns[5] = {frame::agg_fn::sum, frame::agg_fn::min, frame::agg_fn::max,
                                  frame::agg_fn::mean, frame::agg_fn::count};
    frame::table o = frame::group_aggregate(t, names, {{"v", fns[fn]}}, be_of(jobs));
    *n_groups = o.n_rows();
    if (key_out)
      for (uint32_t k = 0; k < nk; ++k) copy_col(o.col(names[k]), key_out[k]);
    if (agg_out) copy_col(o.columns().back(), agg_out);
  });
}

int refh_frame_filter(uint64_t n, int dt, const void* col, int op, const void* lit, unsigned jobs,
                      uint64_t* n_out, uint64_t* idx) {
  return guarded([&] {
    frame::table t;
    t.add(make_col("c", dt, col, n));
    t.add(frame::column::of_u64("_row", iota_u64(n)));
    frame::literal l;
    if (dt == 0) l = *static_cast<const int64_t*>(lit);
    else if (dt == 1) l = *static_cast<const uint64_t*>(lit);
    else l = *static_cast<const double*>(lit);
    frame::table o = frame::filter(t, "c", static_cast<frame::cmp_op>(op), l, be_of(jobs));
    *n_out = o.n_rows();
    if (idx) copy_col(o.col("_row"), idx);
  });
}

int refh_frame_merge(uint64_t nl, uint64_t nr, uint32_t nk, const int* dts, const void* const* lkeys,
                     const void* const* rkeys, unsigned jobs, uint64_t* n_out, uint64_t* lidx, uint64_t* ridx) {
  return guarded([&] {
    frame::table l, r;
    std::vector<std::string> names;
    for (uint32_t k = 0; k < nk; ++k) {
      names.push_back("k" + std::to_string(k));
      l.add(make_col(names.back(), dts[k], lkeys[k], nl));
      r.add(make_col(names.back(), dts[k], rkeys[k], nr));
    }
    l.add(frame::column::of_u64("_l", iota_u64(nl)));
    r.add(frame::column::of_u64("_r", iota_u64(nr)));
    frame::table o = frame::merge(l, r, names, be_of(jobs));
    *n_out = o.n_rows();
    if (lidx) copy_col(o.col("_l"), lidx);
    if (ridx) copy_col(o.col("_r"), ridx);
  });
}

// op 0 vector_add, 1 in_place_multiply, 2 scalar_compare (cmp), 3 cumulative_sum, 4 reduce_sum
int refh_frame_vec(int op, uint64_t n, const double* a, const double* b, double scalar, int cmp, unsigned jobs,
                   void* out) {
  return guarded([&] {
    frame::column ca = frame::column::of_f64("a", std::vector<double>(a, a + n));
    frame::backend bk = be_of(jobs);
    if (op == 0) copy_col(frame::vector_add(ca, frame::column::of_f64("b", std::vector<double>(b, b + n)), bk), out);
    else if (op == 1) copy_col(frame::in_place_multiply(ca, scalar, bk), out);
    else if (op == 2) copy_col(frame::scalar_compare(ca, static_cast<frame::cmp_op>(cmp), scalar, bk), out);
    else if (op == 3) copy_col(frame::cumulative_sum(ca, bk), out);
    else *static_cast<double*>(out) = frame::reduce_sum(ca, bk);
  });
}

// Mean wall time of one frame operator on the reference engine (par backend
// with `jobs` workers): op 0 group_aggregate(keys k0,k1; v sum,min,max,mean,count),
// 1 sort(k0 asc, k2 desc), 2 filter(k2 >= lit), 3 merge(on k0 with a [m] table),
// 4 vector_add, 5 in_place_multiply, 6 scalar_compare, 7 reduce_sum, 8 cumulative_sum.
double refh_time_frame(int op, uint64_t n, const uint64_t* k0, const uint64_t* k1, const uint64_t* k2,
                       const double* v, uint64_t m, const uint64_t* mk, const double* mv, uint64_t lit,
                       unsigned jobs, unsigned repeat) {
  try {
    frame::table t;
    t.add(frame::column::of_u64("k0", std::vector<uint64_t>(k0, k0 + n)));
    t.add(frame::column::of_u64("k1", std::vector<uint64_t>(k1, k1 + n)));
    t.add(frame::column::of_u64("k2", std::vector<uint64_t>(k2, k2 + n)));
    t.add(frame::column::of_f64("v", std::vector<double>(v, v + n)));
    frame::table r;
    r.add(frame::column::of_u64("k0", std::vector<uint64_t>(mk, mk + m)));
    r.add(frame::column::of_f64("w", std::vector<double>(mv, mv + m)));
    const frame::column& cv = t.col("v");
    frame::backend bk = be_of(jobs);
    return time_mean(repeat, [&] {
      switch (op) {
        case 0: frame::group_aggregate(t, {"k0", "k1"}, {{"v", frame::agg_fn::sum}, {"v", frame::agg_fn::min},
                                                         {"v", frame::agg_fn::max}, {"v", frame::agg_fn::mean},
                                                         {"v", frame::agg_fn::count}}, bk); break;
        case 1: frame::sort(t, {"k0", "k2"}, {true, false}, bk); break;
        case 2: frame::filter(t, "k2", frame::cmp_op::ge, frame::literal{lit}, bk); break;
        case 3: frame::merge(t, r, {"k0"}, bk); break;
        case 4: frame::vector_add(cv, cv, bk); break;
        case 5: frame::in_place_multiply(cv, 1.5, bk); break;
        case 6: frame::scalar_compare(cv, frame::cmp_op::gt, 0.5, bk); break;
        case 7: frame::reduce_sum(cv, bk); break;
        default: frame::cumulative_sum(cv, bk); break;
      }
    });
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

}  // extern "C"
