// TEST INFRASTRUCTURE — drop-in parity of integration/perfslice_gpu.* against
// the UNMODIFIED reference, through the reference's own types.
//
// Linked with the reference core built by oracle/build_ref.sh (the checker)
// and with libpsg.so (the product under test).  Each case calls a reference
// function and its perfslice::gpu counterpart on the same database and
// compares the results with the reference's own operator== (bit-exact) or
// within 1e-9 relative for fp64 diagnostics — the style of the reference's
// acceptance suite (proj/tests/acceptance.cpp): PASS/FAIL lines, exit code =
// number of failures.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "core/diagnostics.hpp"
#include "core/frame.hpp"
#include "core/ingest.hpp"
#include "core/itermodel.hpp"
#include "core/store.hpp"
#include "core/synthgen.hpp"
#include "core/topology.hpp"
#include "core/util.hpp"
#include "helpers.hpp"
#include "perfslice_gpu.hpp"

using namespace perfslice;
using testutil::scratch_dir;

namespace {

int g_failures = 0;

struct check_failure {
  std::string message;
};

void expect(bool ok, const std::string& what) {
  if (!ok) throw check_failure{what};
}

// 1e-9 relative; `abs` is the floor for values that are zero up to rounding
// (a CV over identical values is exactly 0 in exact integers but may come out
// as ~1e-14 % from the reference's two-pass fp64 fold).
void expect_rel(double got, double want, const std::string& what, double rel = 1e-9,
                double abs = 0.0) {
  const double d = std::abs(got - want);
  if (!(got == want || d <= rel * std::abs(want) || d <= abs))
    throw check_failure{what + ": got " + std::to_string(got) + ", want " + std::to_string(want)};
}

void run(const std::string& name, const std::function<void()>& body) {
  std::string failure;
  try {
    body();
  } catch (const check_failure& f) {
    failure = f.message;
  } catch (const std::exception& e) {
    failure = std::string("exception: ") + e.what();
  }
  if (failure.empty()) {
    std::printf("PASS  %s\n", name.c_str());
  } else {
    std::printf("FAIL  %s: %s\n", name.c_str(), failure.c_str());
    ++g_failures;
  }
  std::fflush(stdout);
}

template <typename Fn>
errc raised(Fn&& fn) {
  try {
    fn();
  } catch (const error& e) {
    return e.code();
  }
  return errc::ok;
}

struct db {
  scratch_dir dir{"dropin"};
  std::unique_ptr<store::db_handle> h;
  explicit db(const store::database_image& image) {
    store::write_database(image, dir.path());
    h = std::make_unique<store::db_handle>(store::db_handle::open(dir.path()));
  }
  std::vector<uint32_t> ids() const {
    std::vector<uint32_t> v;
    for (const auto& e : h->trace_index()) v.push_back(e.profile_id);
    return v;
  }
  uint64_t t_max() const {
    uint64_t m = 0;
    for (const auto& e : h->trace_index()) m = std::max(m, e.t_end_ns);
    return m;
  }
};

// ingest_traces -> dur glue -> group_aggregate
frame::table ref_window_aggregate(const store::db_handle& h, const std::vector<uint32_t>& ids,
                                  uint64_t t0, uint64_t t1) {
  auto ing = ingest::ingest_traces(h, ids, t0, t1, 1);
  const auto& ev = ing.events;
  const size_t n = ev.size();
  std::vector<uint64_t> pid(n), ctx(n);
  std::vector<int64_t> dur(n);
  for (size_t i = 0; i < n; ++i) {
    pid[i] = ev.profile_id[i];
    ctx[i] = ev.ctx_id[i];
    const uint64_t next =
        (i + 1 < n && ev.profile_id[i + 1] == ev.profile_id[i]) ? ev.timestamp_ns[i + 1] : t1;
    dur[i] = static_cast<int64_t>(next - ev.timestamp_ns[i]);
  }
  frame::table t;
  t.add(frame::column::of_u64("profile_id", std::move(pid)));
  t.add(frame::column::of_u64("ctx_id", std::move(ctx)));
  t.add(frame::column::of_i64("dur_ns", std::move(dur)));
  return frame::group_aggregate(t, {"profile_id", "ctx_id"},
                                {{"dur_ns", frame::agg_fn::sum},
                                 {"dur_ns", frame::agg_fn::min},
                                 {"dur_ns", frame::agg_fn::max},
                                 {"dur_ns", frame::agg_fn::mean},
                                 {"dur_ns", frame::agg_fn::count}},
                                frame::backend::seq());
}

void same_model(const itermodel::tri_model& a, const itermodel::tri_model& b) {
  expect(a.anchor_ctx == b.anchor_ctx, "anchor");
  expect(a.node_ids == b.node_ids, "node_ids");
  expect(a.trace_ids == b.trace_ids, "trace_ids");
  expect(a.iter_counts == b.iter_counts, "iter_counts");
  expect(a.skipped_traces == b.skipped_traces, "skipped_traces");
  expect(a.block_offset == b.block_offset, "block_offset");
  expect(a.incl_ns == b.incl_ns, "incl_ns");
  expect(a.excl_ns == b.excl_ns, "excl_ns");
  expect(a.gap_incl_ns == b.gap_incl_ns, "gap_incl_ns");
  expect(a.gap_excl_ns == b.gap_excl_ns, "gap_excl_ns");
  expect(a.to_csv() == b.to_csv(), "to_csv");
}

// Random CCT + traces with repeated timestamps, empty traces and t_end == last ts.
store::database_image random_image(uint64_t seed) {
  util::xorshift64s rng(seed);
  store::database_image img;
  img.meta.metrics.push_back({0, store::metric_scope::inclusive, "cputime", "s"});
  const uint32_t n_ctx = 3 + static_cast<uint32_t>(rng.next_below(20));
  for (uint32_t c = 0; c < n_ctx; ++c)
    img.meta.contexts.push_back({c, c == 0 ? store::k_no_parent
                                           : static_cast<uint32_t>(rng.next_below(c)),
                                 store::ctx_kind::function, "c" + std::to_string(c)});
  const uint32_t n_tr = 1 + static_cast<uint32_t>(rng.next_below(12));
  for (uint32_t t = 0; t < n_tr; ++t) {
    const uint32_t pid = 1 + t * 2;
    img.meta.profiles.push_back({pid, static_cast<int32_t>(t), 0, "x1000c0s0b0n0", 0});
    img.records.emplace_back();
    store::trace_data td;
    td.profile_id = pid;
    const uint32_t n = t % 5 == 4 ? 0 : static_cast<uint32_t>(rng.next_below(600));
    uint64_t ts = rng.next_below(1000);
    for (uint32_t i = 0; i < n; ++i) {
      if (rng.next_below(3)) ts += rng.next_below(40);
      td.events.push_back({ts, static_cast<uint32_t>(rng.next_below(n_ctx))});
    }
    td.t_end_ns = ts + (rng.next_below(3) ? rng.next_below(300) : 0);
    img.traces.push_back(std::move(td));
  }
  return img;
}

void check_everything(const db& d, const std::string& tag, std::vector<uint32_t> anchors) {
  const auto ids = d.ids();
  const uint64_t T = d.t_max();
  const std::vector<std::pair<uint64_t, uint64_t>> windows = {
      {T / 4, 3 * T / 4}, {0, T + 1}, {T / 3, T / 3}, {T / 5, T / 5 + 7}, {T + 5, T + 9}};
  run(tag + ": ingest_traces == reference (5 windows)", [&] {
    for (auto [t0, t1] : windows) {
      auto a = ingest::ingest_traces(*d.h, ids, t0, t1, 2);
      auto b = gpu::ingest_traces(*d.h, ids, t0, t1, 2);
      expect(a.events == b.events, "events for window " + std::to_string(t0));
      expect(a.carry_in == b.carry_in, "carry_in for window " + std::to_string(t0));
    }
    // a subset, unsorted with duplicates (ingest.cpp:184-186)
    if (ids.size() >= 2) {
      std::vector<uint32_t> sub = {ids.back(), ids.front(), ids.back()};
      auto a = ingest::ingest_traces(*d.h, sub, T / 4, T / 2, 1);
      auto b = gpu::ingest_traces(*d.h, sub, T / 4, T / 2, 1);
      expect(a.events == b.events && a.carry_in == b.carry_in, "subset");
    }
  });
  run(tag + ": window aggregate == ingest_traces + group_aggregate", [&] {
    for (auto [t0, t1] : windows)
      expect(ref_window_aggregate(*d.h, ids, t0, t1) == gpu::window_aggregate(*d.h, ids, t0, t1),
             "table for window " + std::to_string(t0));
  });
  for (uint32_t a : anchors)
    run(tag + ": build_tri_model == reference (anchor " + std::to_string(a) + ")", [&] {
      auto pol = itermodel::anchor_policy::explicit_ctx(a);
      same_model(itermodel::build_tri_model(*d.h, ids, pol, 2),
                 gpu::build_tri_model(*d.h, ids, pol, 2));
    });
}

void check_profiles(const db& d, const std::string& tag) {
  run(tag + ": ingest_profiles == reference (keep sets x metric filters)", [&] {
    const auto& meta = d.h->meta();
    std::vector<uint32_t> all_pids;
    for (const auto& p : meta.profiles) all_pids.push_back(p.id);
    ingest::keep_set all_ctx, some, none;
    for (uint32_t c = 0; c < meta.contexts.size(); ++c) {
      all_ctx.ids.push_back(c);
      if (c % 3 != 1) some.ids.push_back(c);
    }
    std::vector<uint32_t> sub = {all_pids.back(), all_pids.front(), all_pids.back()};
    for (const auto* pids : {&all_pids, &sub})
      for (const auto* keep : {&all_ctx, &some, &none})
        for (const std::vector<uint16_t>& m : {std::vector<uint16_t>{}, std::vector<uint16_t>{0},
                                               std::vector<uint16_t>{1}, std::vector<uint16_t>{0, 1}}) {
          auto a = ingest::ingest_profiles(*d.h, *pids, *keep, m, 2);
          auto b = gpu::ingest_profiles(*d.h, *pids, *keep, m, 2);
          expect(a == b, "slice table");
        }
    expect(raised([&] { gpu::ingest_profiles(*d.h, {all_pids.back() + 1000}, all_ctx, {}, 1); }) ==
               errc::not_found,
           "missing profile");
  });
}

void check_diagnostics(const db& d, const std::string& tag, uint32_t anchor, double total) {
  run(tag + ": savings_report + iteration_cv_report == reference (1e-9)", [&] {
    const auto ids = d.ids();
    auto model = itermodel::build_tri_model(*d.h, ids, itermodel::anchor_policy::explicit_ctx(anchor), 1);
    auto leaves = model.subtree_leaves(d.h->meta());
    auto want = diagnostics::savings_report(model, leaves, total);
    auto got = gpu::iteration_report(*d.h, ids, anchor, total);
    expect(got.leaves == leaves, "leaves");
    expect(got.savings.n_iterations == want.n_iterations, "n_iterations");
    expect(got.savings.rows.size() == want.rows.size(), "rows");
    for (size_t i = 0; i < want.rows.size(); ++i) {
      const auto &g = got.savings.rows[i], &w = want.rows[i];
      expect(g.ctx_id == w.ctx_id, "row ctx");
      expect_rel(g.avg_mean_s, w.avg_mean_s, "avg_mean");
      expect_rel(g.avg_max_s, w.avg_max_s, "avg_max");
      expect_rel(g.savings_per_iter_s, w.savings_per_iter_s, "savings");
      expect_rel(g.total_reduction_s, w.total_reduction_s, "total_reduction");
      std::optional<diagnostics::cv_report> cv;
      try {
        cv = diagnostics::iteration_cv_report(model, w.ctx_id);
      } catch (const error&) {
      }
      expect(cv.has_value() == got.cv[i].has_value(), "cv availability");
      if (cv) {
        expect_rel(got.cv[i]->across_rank_cv_pct, cv->across_rank_cv_pct, "across cv", 1e-9, 1e-9);
        expect_rel(got.cv[i]->within_rank_cv_pct, cv->within_rank_cv_pct, "within cv", 1e-9, 1e-9);
      }
    }
    expect_rel(got.savings.total_savings_s, want.total_savings_s, "total savings");
    expect_rel(got.savings.speedup_frac, want.speedup_frac, "speedup");
  });
}

// The automatic anchor (itermodel.cpp:253-255): suggest_anchor on the first
// requested trace.  The drop-in picks it on the device; the reference's result
// (or the errc it raises) must come back.
void check_auto_anchor(const db& d, const std::string& tag, std::vector<uint32_t> ids = {}) {
  run(tag + ": auto anchor (device suggest_anchor) == reference", [&] {
    const auto pids = ids.empty() ? d.ids() : ids;
    auto pol = itermodel::anchor_policy::auto_detect();
    itermodel::tri_model want;
    const errc e = raised([&] { want = itermodel::build_tri_model(*d.h, pids, pol, 1); });
    if (e != errc::ok) {
      const errc g = raised([&] { gpu::build_tri_model(*d.h, pids, pol, 1); });
      expect(g == e, "errc " + std::string(errc_name(g)) + " != reference " + errc_name(e));
      return;
    }
    same_model(want, gpu::build_tri_model(*d.h, pids, pol, 1));
  });
}

// frame::group_aggregate / filter over a host table built from the window
// rows (the composition's own input) plus a string and an f64 column.
void check_frame(const db& d, const std::string& tag) {
  run(tag + ": frame group_aggregate / filter == reference (host table)", [&] {
    const auto ids = d.ids();
    const uint64_t T = d.t_max();
    auto ing = ingest::ingest_traces(*d.h, ids, T / 5, 4 * T / 5, 1);
    const auto& ev = ing.events;
    const size_t n = ev.size();
    std::vector<uint64_t> pid(n), ctx(n);
    std::vector<int64_t> dur(n);
    std::vector<double> durf(n);
    std::vector<std::string> tag_col(n);
    for (size_t i = 0; i < n; ++i) {
      pid[i] = ev.profile_id[i];
      ctx[i] = ev.ctx_id[i];
      const uint64_t next = (i + 1 < n && ev.profile_id[i + 1] == ev.profile_id[i]) ? ev.timestamp_ns[i + 1] : 4 * T / 5;
      dur[i] = static_cast<int64_t>(next - ev.timestamp_ns[i]);
      durf[i] = static_cast<double>(dur[i]) / 1e9;
      tag_col[i] = "r" + std::to_string(i % 7);
    }
    frame::table t;
    t.add(frame::column::of_u64("profile_id", pid));
    t.add(frame::column::of_u64("ctx_id", ctx));
    t.add(frame::column::of_i64("dur_ns", dur));
    t.add(frame::column::of_f64("dur_s", durf));
    t.add(frame::column::of_str("tag", tag_col));
    const std::vector<frame::agg_spec> aggs = {
        {"dur_ns", frame::agg_fn::sum}, {"dur_ns", frame::agg_fn::min},  {"dur_ns", frame::agg_fn::max},
        {"dur_ns", frame::agg_fn::mean}, {"dur_ns", frame::agg_fn::count}, {"dur_s", frame::agg_fn::sum},
        {"dur_s", frame::agg_fn::min},  {"dur_s", frame::agg_fn::max},   {"dur_s", frame::agg_fn::mean}};
    for (const std::vector<std::string>& keys :
         {std::vector<std::string>{"profile_id", "ctx_id"}, std::vector<std::string>{"ctx_id"},
          std::vector<std::string>{"dur_s", "profile_id"}})
      expect(frame::group_aggregate(t, keys, aggs, frame::backend::seq()) ==
                 gpu::group_aggregate(t, keys, aggs, frame::backend::seq()),
             "group_aggregate keys " + keys.front());
    for (auto op : {frame::cmp_op::lt, frame::cmp_op::le, frame::cmp_op::eq, frame::cmp_op::ge, frame::cmp_op::gt,
                    frame::cmp_op::ne}) {
      expect(frame::filter(t, "dur_ns", op, frame::literal{int64_t{1000}}, frame::backend::seq()) ==
                 gpu::filter(t, "dur_ns", op, frame::literal{int64_t{1000}}, frame::backend::seq()),
             "filter i64");
      expect(frame::filter(t, "ctx_id", op, frame::literal{uint64_t{3}}, frame::backend::seq()) ==
                 gpu::filter(t, "ctx_id", op, frame::literal{uint64_t{3}}, frame::backend::seq()),
             "filter u64");
      expect(frame::filter(t, "dur_s", op, frame::literal{1e-3}, frame::backend::seq()) ==
                 gpu::filter(t, "dur_s", op, frame::literal{1e-3}, frame::backend::seq()),
             "filter f64");
    }
    expect(raised([&] { gpu::filter(t, "dur_ns", frame::cmp_op::lt, frame::literal{1.0}, frame::backend::seq()); }) ==
               errc::type_mismatch,
           "literal type mismatch");
    expect(raised([&] { gpu::group_aggregate(t, {"tag"}, aggs, frame::backend::seq()); }) == errc::type_mismatch,
           "string key");
    expect(raised([&] { gpu::group_aggregate(t, {"nope"}, aggs, frame::backend::seq()); }) ==
               raised([&] { frame::group_aggregate(t, {"nope"}, aggs, frame::backend::seq()); }),
           "missing column");
  });
}

// detect_iterations / rematerialize on single traces given as events.
void check_span_itermodel(const db& d, const std::string& tag, std::vector<uint32_t> anchors) {
  run(tag + ": detect_iterations / rematerialize (span inputs) == reference", [&] {
    const auto& meta = d.h->meta();
    const uint64_t T = d.t_max();
    for (uint32_t pid : d.ids()) {
      auto [events, t_end] = d.h->read_trace_full(pid);
      for (uint32_t a : anchors) {
        std::vector<itermodel::interval> want;
        const errc e = raised([&] { want = itermodel::detect_iterations(events, t_end, meta, a); });
        std::vector<itermodel::interval> got;
        const errc g = raised([&] { got = gpu::detect_iterations(events, t_end, meta, a); });
        expect(e == g, "detect_iterations errc, trace " + std::to_string(pid));
        if (e == errc::ok) expect(want == got, "intervals, trace " + std::to_string(pid));
      }
      for (auto [t0, t1] : std::vector<std::pair<uint64_t, uint64_t>>{{T / 4, 3 * T / 4}, {0, T + 1}, {T / 3, T / 3 + 5}}) {
        auto w = d.h->read_trace_window(pid, t0, t1);
        const itermodel::interval iv{t0, t1};
        expect(itermodel::rematerialize(w.events, w.carry_in, iv, meta) ==
                   gpu::rematerialize(w.events, w.carry_in, iv, meta),
               "rematerialize, trace " + std::to_string(pid));
      }
    }
  });
}

void check_small_diagnostics() {
  run("balance_ratio / cv_percent / node_correlate / localize_outliers == reference", [&] {
    util::xorshift64s rng(99);
    for (size_t n : {1, 2, 7, 1000, 100000}) {
      std::vector<double> v(n);
      for (auto& x : v) x = rng.next_unit() * 3.0;
      expect_rel(gpu::balance_ratio(v), diagnostics::balance_ratio(v), "balance_ratio n=" + std::to_string(n));
      expect_rel(gpu::cv_percent(v), diagnostics::cv_percent(v), "cv n=" + std::to_string(n), 1e-9, 1e-12);
    }
    std::vector<double> zeros(5, 0.0), empty;
    expect(gpu::balance_ratio(zeros) == 1.0, "all-zero ratio");
    expect(raised([&] { gpu::cv_percent(zeros); }) == errc::undefined_cv, "zero-mean cv");
    expect(raised([&] { gpu::balance_ratio(empty); }) == errc::empty_input, "empty ratio");
    expect(raised([&] { gpu::cv_percent(empty); }) == errc::empty_input, "empty cv");
    // node_correlate on the aurora-like layout (10 ranks per node)
    auto [img, truth] = synthgen::generate_congestion_scenario(testutil::aurora_like_config(42));
    std::vector<std::pair<int32_t, double>> rv;
    for (const auto& p : img.meta.profiles)
      if (p.rank >= 0) rv.push_back({p.rank, rng.next_unit()});
    auto a = diagnostics::node_correlate(rv, img.meta), b = gpu::node_correlate(rv, img.meta);
    expect(a.size() == b.size(), "node count");
    for (size_t i = 0; i < a.size(); ++i)
      expect(a[i].hostname == b[i].hostname && a[i].mean_value == b[i].mean_value &&
                 a[i].rank_count == b[i].rank_count,
             "node " + a[i].hostname);
    rv.push_back({1 << 30, 1.0});
    expect(raised([&] { gpu::node_correlate(rv, img.meta); }) == errc::not_found, "unknown rank");
    // localize_outliers: the truth outliers, an outlier outside the universe,
    // duplicates, chassis ids >= 64, and parse errors
    std::vector<std::string> outl = truth.outlier_hostnames, uni = truth.node_hostnames;
    outl.push_back(outl.front());
    outl.push_back("x9000c70s0b0n0");
    uni.push_back("x9000c70s1b0n1");
    uni.push_back("x9001c4096s0b0n0");
    outl.push_back("x9001c4096s0b0n0");
    expect(topology::localize_outliers(outl, uni) == gpu::localize_outliers(outl, uni), "localize");
    for (const std::string bad : {"nid0001", "x1c2s3b4", "x1c2s3b4n5z", "x1cXs0b0n0"}) {
      auto u2 = uni;
      u2.push_back(bad);
      std::string want_msg, got_msg;
      try { topology::localize_outliers(outl, u2); } catch (const error& e) { want_msg = e.what(); }
      try { gpu::localize_outliers(outl, u2); } catch (const error& e) { got_msg = e.what(); }
      expect(!want_msg.empty() && want_msg == got_msg, "parse error message for " + bad + ": " + got_msg);
    }
  });
}

// No context enters periodically: suggest_anchor raises no_periodicity.
store::database_image aperiodic_image() {
  store::database_image img;
  img.meta.metrics.push_back({0, store::metric_scope::inclusive, "cputime", "s"});
  for (uint32_t c = 0; c < 4; ++c)
    img.meta.contexts.push_back({c, c == 0 ? store::k_no_parent : c - 1, store::ctx_kind::function,
                                 "c" + std::to_string(c)});
  for (uint32_t t = 0; t < 3; ++t) {
    img.meta.profiles.push_back({t + 1, static_cast<int32_t>(t), 0, "x1000c0s0b0n0", 0});
    img.records.emplace_back();
    store::trace_data td;
    td.profile_id = t + 1;
    // each context entered once, then the root: no context has 3 entries
    td.events = {{0, 0}, {10, 1}, {25, 2}, {70, 3}, {200, 0}};
    td.t_end_ns = 300;
    img.traces.push_back(std::move(td));
  }
  return img;
}

}  // namespace

int main() {
  {
    auto [image, truth] = synthgen::generate_iterative_scenario(testutil::small_iter_config(52, 5, 7, 0.1));
    db d(image);
    check_everything(d, "small_iter", {0, 1, 2});
    check_diagnostics(d, "small_iter", 1, 10.0);
    check_profiles(d, "small_iter");
    check_auto_anchor(d, "small_iter");
    check_frame(d, "small_iter");
    check_span_itermodel(d, "small_iter", {0, 1, 2, 3});
    check_auto_anchor(d, "small_iter (subset, first = last trace)", {d.ids().back()});
    run("small_iter: concurrent callers share one device (4 threads)", [&] {
      auto want = itermodel::build_tri_model(*d.h, d.ids(), itermodel::anchor_policy::explicit_ctx(1), 1);
      std::vector<std::thread> th;
      std::vector<int> ok(4, 0);
      for (int i = 0; i < 4; ++i)
        th.emplace_back([&, i] {
          try {
            auto got = gpu::build_tri_model(*d.h, d.ids(), itermodel::anchor_policy::explicit_ctx(1), 1);
            ok[i] = got.incl_ns == want.incl_ns && got.iter_counts == want.iter_counts;
          } catch (...) {
          }
        });
      for (auto& t : th) t.join();
      for (int v : ok) expect(v == 1, "thread result");
    });
    run("small_iter: boundaries == generator truth", [&] {
      auto m = gpu::build_tri_model(*d.h, d.ids(), itermodel::anchor_policy::explicit_ctx(truth.anchor_ctx), 1);
      for (size_t t = 0; t < m.trace_ids.size(); ++t)
        expect(m.iter_counts[t] == truth.boundaries_ns[t].size(), "iteration count");
    });
    run("errors map to the reference's errc", [&] {
      expect(raised([&] { gpu::ingest_traces(*d.h, d.ids(), 5, 4, 1); }) == errc::invalid_argument,
             "t0 > t1");
      expect(raised([&] { gpu::ingest_traces(*d.h, {999}, 0, 1, 1); }) == errc::not_found,
             "missing trace");
      expect(raised([&] { gpu::build_tri_model(*d.h, {}, itermodel::anchor_policy::explicit_ctx(1), 1); }) ==
                 errc::invalid_argument,
             "no traces");
      expect(raised([&] { gpu::build_tri_model(*d.h, d.ids(), itermodel::anchor_policy::explicit_ctx(10000), 1); }) ==
                 errc::not_found,
             "anchor out of range");
      expect(raised([&] { gpu::iteration_report(*d.h, d.ids(), 1, 0.0); }) == errc::invalid_total,
             "total time");
    });
  }
  {
    auto [image, truth] = synthgen::generate_iterative_scenario(testutil::gamess_like_config());
    db d(image);
    check_everything(d, "gamess_like", {1});
    check_auto_anchor(d, "gamess_like");
    check_diagnostics(d, "gamess_like", truth.anchor_ctx, 87.0);
  }
  for (uint64_t seed = 1; seed <= 6; ++seed) {
    db d(random_image(seed));
    check_everything(d, "random_" + std::to_string(seed), {0, 1, static_cast<uint32_t>(d.h->meta().contexts.size() - 1)});
    check_auto_anchor(d, "random_" + std::to_string(seed));
    check_frame(d, "random_" + std::to_string(seed));
    check_span_itermodel(d, "random_" + std::to_string(seed), {0, 1, static_cast<uint32_t>(d.h->meta().contexts.size() - 1)});
  }
  {
    db d(aperiodic_image());
    check_auto_anchor(d, "aperiodic");
    run("aperiodic: auto anchor raises no_periodicity", [&] {
      expect(raised([&] { gpu::build_tri_model(*d.h, d.ids(), itermodel::anchor_policy::auto_detect(), 1); }) ==
                 errc::no_periodicity,
             "errc");
    });
  }
  check_small_diagnostics();
  run("a database rewritten in place is reloaded (resident-trace cache keyed by file identity)", [&] {
    scratch_dir dir{"dropin_rewrite"};
    for (uint64_t seed : {11, 12, 13}) {
      store::write_database(random_image(seed), dir.path());
      auto h = store::db_handle::open(dir.path());
      std::vector<uint32_t> ids;
      for (const auto& e : h.trace_index()) ids.push_back(e.profile_id);
      uint64_t T = 0;
      for (const auto& e : h.trace_index()) T = std::max(T, e.t_end_ns);
      auto a = ingest::ingest_traces(h, ids, T / 4, 3 * T / 4, 1);
      auto b = gpu::ingest_traces(h, ids, T / 4, 3 * T / 4, 1);
      expect(a.events == b.events && a.carry_in == b.carry_in, "seed " + std::to_string(seed));
    }
  });
  std::printf("%s: %d failure(s)\n", g_failures ? "FAILED" : "OK", g_failures);
  return g_failures;
}
