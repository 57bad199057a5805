// perfslice_gpu.hpp — the drop-in C++ binding of the reference's trace query
// path onto libpsg (include/psg.h).
//
// Compiled against the reference's own headers (proj/src/core) and linked
// into the reference's build: every function here has
// the signature and result type of the reference function it replaces, so a
// caller switches by changing the namespace (perfslice::ingest::ingest_traces
// -> perfslice::gpu::ingest_traces, ...).  The trace bodies are read through
// the reference's reader: the db_handle's parsed index supplies the event
// offsets, counts and t_end of every trace, and the same trace.db bytes are
// handed to psg_load_traces_aos (K1 transposes them to SoA in HBM).  All
// compute runs on the GPU; there is no CPU fallback.  Errors come back as
// perfslice::error with the errc the reference would raise for the same
// condition (inverse of capi.cpp:35-63).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <optional>
#include <span>
#include <vector>

#include "core/diagnostics.hpp"
#include "core/frame.hpp"
#include "core/ingest.hpp"
#include "core/itermodel.hpp"
#include "core/store.hpp"
#include "core/topology.hpp"

struct psg_context;

namespace perfslice::gpu {

// One GPU context with a resident trace set.  Binding the same (database,
// profile ids) again reuses the traces already in HBM.
class device {
 public:
  explicit device(int cuda_device = 0);
  ~device();
  device(const device&) = delete;
  device& operator=(const device&) = delete;

  // Loads the traces of `profile_ids` (sorted, deduplicated; all traces when
  // empty) of `h` unless they are already resident.  Raises not_found for an
  // id without a trace (store.cpp:639-642).
  void bind(const store::db_handle& h, std::vector<uint32_t> profile_ids);
  // Loads every profile's records (profile.db of h) unless already resident.
  void bind_profiles(const store::db_handle& h);
  psg_context* ctx() const { return ctx_; }
  const std::vector<uint32_t>& profile_ids() const { return pids_; }

 private:
  psg_context* ctx_ = nullptr;
  // what is resident: database identity (path, size, mtime, inode of its
  // files) + profile ids; empty = nothing
  std::string bound_key_, bound_profiles_key_;
  std::vector<uint32_t> pids_;
};

// The process-wide device (CUDA device 0), created on first use and shared by
// every calling thread, so a trace set is resident once (the reference's
// db_handle is shared by concurrent readers).
device& default_device();
// The same device with its lock held: the drop-in functions below take it for
// the whole call, so concurrent callers serialise on the GPU context.
struct device_lease {
  std::unique_lock<std::mutex> lock;
  device& dev;
};
device_lease acquire_device();

// ingest::ingest_traces (ingest.hpp:105-108, ingest.cpp:178-208).  `jobs` is
// accepted for signature compatibility and ignored.
ingest::trace_ingest_result ingest_traces(const store::db_handle& h,
                                          std::vector<uint32_t> profile_ids,
                                          uint64_t t0_ns, uint64_t t1_ns, unsigned jobs);

// The window aggregate of SURVEY.md §3(3): ingest_traces rows with
// dur_ns = (next row of the same profile or t1) - ts, then
// frame::group_aggregate(table, {"profile_id", "ctx_id"},
// {sum, min, max, mean, count of "dur_ns"}) (frame.cpp:290-408) — the same
// frame::table, column for column.
frame::table window_aggregate(const store::db_handle& h, std::vector<uint32_t> profile_ids,
                              uint64_t t0_ns, uint64_t t1_ns);

// ingest::ingest_profiles (ingest.hpp:83-87, ingest.cpp:155-176): the
// profile-record slice of the requested profiles, filtered by the keep set and
// metric ids, on the device (psg_slice).  `jobs` is accepted and ignored.
ingest::slice_table ingest_profiles(const store::db_handle& h, std::vector<uint32_t> profile_ids,
                                    const ingest::keep_set& keep,
                                    const std::vector<uint16_t>& metric_ids, unsigned jobs);

// ingest::read_slices (ingest.hpp:77-80, ingest.cpp:122-153): the session's
// cache-miss reads (query.cpp:337-338) on the device; requests with the same
// (ctx, metric) filters share one psg_slice, and the rows come back in
// request order exactly as the reference assembles them.
ingest::slice_table read_slices(const store::db_handle& h,
                                const std::vector<ingest::slice_request>& requests, unsigned jobs);

// frame::group_aggregate / frame::filter (frame.hpp:100-113, frame.cpp:
// 290-470) over a host table: the key / predicate / aggregate columns go to
// the device (psg_frame_group, _group_agg, _filter: the reference's fold
// order and NaN rules, bit for bit); the rows are gathered back on the host.
// Numeric columns only on the device: a string key, predicate or aggregate
// column raises type_mismatch (string columns in other positions are
// gathered).  The backend argument is accepted and ignored.
frame::table group_aggregate(const frame::table& t, const std::vector<std::string>& keys,
                             const std::vector<frame::agg_spec>& aggs, frame::backend b);
frame::table filter(const frame::table& t, const std::string& column, frame::cmp_op op,
                    const frame::literal& lit, frame::backend b);

// itermodel::detect_iterations / rematerialize (itermodel.hpp:54-64,
// itermodel.cpp:111-183) on one trace given as events: the fused query's
// boundary pass and window integration on a second device context (the
// shared one keeps its resident traces).  Events must be timestamp-ordered
// (a trace.db invariant; PS_E_FORMAT -> format_error otherwise).
std::vector<itermodel::interval> detect_iterations(std::span<const store::trace_event> events,
                                                   uint64_t t_end_ns, const store::meta_data& cct,
                                                   uint32_t anchor);
itermodel::interval_profile rematerialize(std::span<const store::trace_event> events,
                                          std::optional<store::trace_event> carry_in,
                                          itermodel::interval iv, const store::meta_data& cct);

// diagnostics::balance_ratio / cv_percent (diagnostics.hpp:23-26): device
// tree sums (within 1e-9 of the reference's sequential fold).
double balance_ratio(std::span<const double> values);
double cv_percent(std::span<const double> values);
// diagnostics::node_correlate (diagnostics.hpp:128-130): hostname
// bookkeeping on the host, per-host sums on the device in input order (bit
// for bit the reference's fold).
std::vector<diagnostics::node_stat> node_correlate(
    const std::vector<std::pair<int32_t, double>>& rank_values, const store::meta_data& meta);
// topology::localize_outliers (topology.hpp:52-53): names parsed by
// psg_node_name (parse_error, the reference's message), counts on the device.
topology::congestion_report localize_outliers(const std::vector<std::string>& outliers,
                                              const std::vector<std::string>& universe);

// itermodel::build_tri_model (itermodel.hpp:118-120, itermodel.cpp:242-360).
// An automatic anchor is chosen on the device (psg_query with
// PSG_ANCHOR_AUTO: suggest_anchor's entry walk, gap CV and covered-time pick
// on the first requested trace, itermodel.cpp:45-109, 253-255).
itermodel::tri_model build_tri_model(const store::db_handle& h,
                                     const std::vector<uint32_t>& profile_ids,
                                     itermodel::anchor_policy policy, unsigned jobs);

// diagnostics::savings_report + iteration_cv_report over the subtree leaves
// (diagnostics.cpp:100-158, as workflows::iterations_report uses them),
// computed on the device in the same pass as the cube.  cv[i] is empty where
// the reference raises (insufficient data / undefined CV).
struct iteration_diagnostics {
  std::vector<uint32_t> leaves;
  diagnostics::savings_summary savings;
  std::vector<std::optional<diagnostics::cv_report>> cv;
};
iteration_diagnostics iteration_report(const store::db_handle& h,
                                       const std::vector<uint32_t>& profile_ids,
                                       uint32_t anchor_ctx, double total_time_s);

}  // namespace perfslice::gpu
