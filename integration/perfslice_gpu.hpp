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
#include <vector>

#include "core/diagnostics.hpp"
#include "core/frame.hpp"
#include "core/ingest.hpp"
#include "core/itermodel.hpp"
#include "core/store.hpp"

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
