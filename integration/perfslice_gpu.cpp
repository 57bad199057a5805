// perfslice_gpu.cpp — see perfslice_gpu.hpp.  Everything here is host glue:
// index bookkeeping, result marshalling into the reference's types, and error
// mapping.  The compute is libpsg's (include/psg.h).
#include "perfslice_gpu.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "core/common.hpp"
#include "psg.h"

namespace perfslice::gpu {

namespace {

// ps_status -> the errc the reference raises for the same condition (the
// inverse of capi.cpp:35-63, taking the first errc of each status).
errc errc_of(ps_status s) {
  switch (s) {
    case PS_OK: return errc::ok;
    case PS_E_IO: return errc::io_error;
    case PS_E_FORMAT: return errc::format_error;
    case PS_E_INVALID_IMAGE: return errc::invalid_image;
    case PS_E_NOT_FOUND: return errc::not_found;
    case PS_E_INVALID_CONFIG: return errc::invalid_config;
    case PS_E_NO_SUMMARY: return errc::no_summary;
    case PS_E_DEGENERATE_SUMMARY: return errc::degenerate_summary;
    case PS_E_PARSE: return errc::parse_error;
    case PS_E_NO_SUCH_METRIC: return errc::no_such_metric;
    case PS_E_NO_PERIODICITY: return errc::no_periodicity;
    case PS_E_NO_OUTLIERS: return errc::no_outliers;
    case PS_E_INSUFFICIENT_DATA: return errc::insufficient_data;
    case PS_E_INVALID_ARGUMENT: return errc::invalid_argument;
    case PS_E_INTERNAL: return errc::internal;
  }
  return errc::internal;
}

void check(ps_status s) {
  if (s == PS_OK) return;
  const std::string msg = psg_last_error();
  errc e = errc_of(s);
  // ps_status folds several errc into one; the library's message names the
  // reference condition where the C++ caller can tell them apart
  if (s == PS_E_INVALID_ARGUMENT && msg.find("trace has no events") != std::string::npos)
    e = errc::empty_input;  // suggest_anchor on an empty trace (itermodel.cpp:48)
  raise(e, "psg: " + msg);
}

// Identity of a database's on-disk files: a reopened or replaced database at
// the same path (or a new handle at a reused address) is a different key.
std::string db_key(const store::db_handle& h, const char* file) {
  struct stat st{};
  const std::filesystem::path p = h.path() / file;
  if (::stat(p.c_str(), &st) != 0) return p.string();
  return p.string() + "|" + std::to_string(st.st_size) + "|" + std::to_string(st.st_mtim.tv_sec) +
         "." + std::to_string(st.st_mtim.tv_nsec) + "|" + std::to_string(st.st_ino);
}

std::vector<uint32_t> sorted_unique(std::vector<uint32_t> v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

// Read-only mapping of <db>/trace.db: the bytes behind the reference
// reader's index entries (store.cpp:395-413 maps the same file).
struct trace_file {
  const uint8_t* data = nullptr;
  size_t size = 0;
  explicit trace_file(const std::filesystem::path& p) {
    const int fd = ::open(p.c_str(), O_RDONLY);
    if (fd < 0) raise(errc::io_error, "cannot open " + p.string());
    struct stat st{};
    if (::fstat(fd, &st) != 0) {
      ::close(fd);
      raise(errc::io_error, "cannot stat " + p.string());
    }
    size = static_cast<size_t>(st.st_size);
    if (size) {
      void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) {
        ::close(fd);
        raise(errc::io_error, "mmap failed: " + p.string());
      }
      data = static_cast<const uint8_t*>(m);
    }
    ::close(fd);
  }
  ~trace_file() {
    if (data) ::munmap(const_cast<uint8_t*>(data), size);
  }
};

}  // namespace

device::device(int cuda_device) { check(psg_open(cuda_device, nullptr, &ctx_)); }

device::~device() { psg_close(ctx_); }

void device::bind(const store::db_handle& h, std::vector<uint32_t> profile_ids) {
  profile_ids = sorted_unique(std::move(profile_ids));
  const std::string key = db_key(h, "trace.db") + "|" + db_key(h, "meta.bin");
  if (key == bound_key_ && profile_ids == pids_) return;
  bound_key_.clear();
  std::vector<const store::trace_index_entry*> sel;
  sel.reserve(profile_ids.size());
  for (uint32_t id : profile_ids) {
    const store::trace_index_entry* e = h.find_trace_entry(id);
    if (e == nullptr)  // store.cpp:639-642
      raise(errc::not_found, "trace " + std::to_string(id) + " not in database");
    sel.push_back(e);
  }
  // calling-context tree (meta.bin; parent < id is a format invariant)
  const auto& cct = h.meta().contexts;
  std::vector<uint32_t> parent(cct.size());
  for (size_t i = 0; i < cct.size(); ++i) parent[i] = cct[i].parent;
  check(psg_set_cct(ctx_, parent.data(), static_cast<uint32_t>(parent.size())));

  std::vector<uint64_t> off(1, 0), t_end;
  std::vector<uint32_t> pid;
  bool contiguous = true;
  for (size_t i = 0; i < sel.size(); ++i) {
    off.push_back(off.back() + sel[i]->event_count);
    t_end.push_back(sel[i]->t_end_ns);
    pid.push_back(sel[i]->profile_id);
    if (i > 0 && sel[i]->offset != sel[i - 1]->offset + sel[i - 1]->event_count * store::k_event_size)
      contiguous = false;
  }
  const uint64_t n_ev = off.back();
  trace_file f(h.path() / "trace.db");
  std::vector<uint8_t> gathered;
  const uint8_t* body = nullptr;
  if (n_ev) {
    if (contiguous) {
      body = f.data + sel.front()->offset;
    } else {
      gathered.resize(n_ev * store::k_event_size);
      size_t o = 0;
      for (auto* e : sel) {
        std::memcpy(gathered.data() + o, f.data + e->offset, e->event_count * store::k_event_size);
        o += e->event_count * store::k_event_size;
      }
      body = gathered.data();
    }
  }
  check(psg_load_traces_aos(ctx_, body, n_ev, off.data(), pid.data(), t_end.data(),
                            static_cast<uint32_t>(pid.size())));
  bound_key_ = key;
  pids_ = std::move(profile_ids);
}

void device::bind_profiles(const store::db_handle& h) {
  const std::string key = db_key(h, "profile.db") + "|" + db_key(h, "meta.bin");
  if (key == bound_profiles_key_) return;
  bound_profiles_key_.clear();
  check(psg_load_profile_db(ctx_, (h.path()).c_str()));
  bound_profiles_key_ = key;
}

ingest::slice_table ingest_profiles(const store::db_handle& h, std::vector<uint32_t> profile_ids,
                                    const ingest::keep_set& keep,
                                    const std::vector<uint16_t>& metric_ids, unsigned /*jobs*/) {
  device_lease lease = acquire_device();
  device& d = lease.dev;
  d.bind_profiles(h);
  const bool all_ctx = keep.size() == h.meta().contexts.size();
  uint64_t n = 0;
  const uint32_t* cx = all_ctx ? nullptr : keep.ids.data();
  const uint32_t ncx = all_ctx ? 0 : static_cast<uint32_t>(keep.ids.size());
  static const uint32_t k_none = 0;
  if (!all_ctx && keep.ids.empty()) cx = &k_none;  // an empty keep set keeps nothing
  const uint16_t* mt = metric_ids.empty() ? nullptr : metric_ids.data();
  const uint32_t nmt = static_cast<uint32_t>(metric_ids.size());
  const uint32_t np = static_cast<uint32_t>(profile_ids.size());
  check(psg_slice(d.ctx(), profile_ids.data(), np, cx, ncx, mt, nmt, &n, nullptr, nullptr, nullptr, nullptr));
  ingest::slice_table out;
  out.profile_id.resize(n);
  out.ctx_id.resize(n);
  out.metric_id.resize(n);
  out.value.resize(n);
  if (n)
    check(psg_slice(d.ctx(), profile_ids.data(), np, cx, ncx, mt, nmt, &n, out.profile_id.data(),
                    out.ctx_id.data(), out.metric_id.data(), out.value.data()));
  return out;
}

namespace {
std::mutex g_device_mu;
std::unique_ptr<device> g_device;
}  // namespace

device& default_device() {
  std::lock_guard<std::mutex> lk(g_device_mu);
  if (!g_device) g_device = std::make_unique<device>(0);
  return *g_device;
}

device_lease acquire_device() {
  std::unique_lock<std::mutex> lk(g_device_mu);
  if (!g_device) g_device = std::make_unique<device>(0);
  return device_lease{std::move(lk), *g_device};
}

ingest::trace_ingest_result ingest_traces(const store::db_handle& h,
                                          std::vector<uint32_t> profile_ids,
                                          uint64_t t0_ns, uint64_t t1_ns, unsigned /*jobs*/) {
  if (t0_ns > t1_ns) raise(errc::invalid_argument, "trace window start after end");
  ingest::trace_ingest_result out;
  profile_ids = sorted_unique(std::move(profile_ids));
  if (profile_ids.empty()) return out;
  device_lease lease = acquire_device();
  device& d = lease.dev;
  d.bind(h, profile_ids);
  uint64_t n = 0;
  check(psg_window_rows(d.ctx(), t0_ns, t1_ns, &n, nullptr, nullptr, nullptr));
  out.events.profile_id.resize(n);
  out.events.timestamp_ns.resize(n);
  out.events.ctx_id.resize(n);
  check(psg_window_rows(d.ctx(), t0_ns, t1_ns, &n, out.events.profile_id.data(),
                        out.events.timestamp_ns.data(), out.events.ctx_id.data()));
  const size_t nt = profile_ids.size();
  std::vector<uint8_t> has(nt);
  std::vector<uint64_t> ts(nt);
  std::vector<uint32_t> cx(nt);
  check(psg_get_carry(d.ctx(), has.data(), ts.data(), cx.data()));
  for (size_t i = 0; i < nt; ++i)
    out.carry_in[profile_ids[i]] =
        has[i] ? std::optional<store::trace_event>(store::trace_event{ts[i], cx[i]}) : std::nullopt;
  return out;
}

frame::table window_aggregate(const store::db_handle& h, std::vector<uint32_t> profile_ids,
                              uint64_t t0_ns, uint64_t t1_ns) {
  if (t0_ns > t1_ns) raise(errc::invalid_argument, "trace window start after end");
  profile_ids = sorted_unique(std::move(profile_ids));
  std::vector<uint64_t> kp, kc, cnt;
  std::vector<int64_t> sum, mn, mx;
  std::vector<double> mean;
  if (!profile_ids.empty()) {
    device_lease lease = acquire_device();
    device& d = lease.dev;
    d.bind(h, profile_ids);
    psg_query_spec q{};
    q.flags = PSG_Q_WINDOW;
    q.t0_ns = t0_ns;
    q.t1_ns = t1_ns;
    psg_query_info info{};
    check(psg_query(d.ctx(), &q, &info));
    psg_shard_info sh{};
    check(psg_shard(d.ctx(), &sh));
    const size_t cells = static_cast<size_t>(sh.n_traces) * sh.n_ctx;
    std::vector<uint64_t> c(cells);
    std::vector<int64_t> s(cells), lo(cells), hi(cells);
    std::vector<double> m(cells);
    check(psg_get_window(d.ctx(), c.data(), s.data(), lo.data(), hi.data(), m.data(), nullptr,
                         nullptr));
    // group_aggregate's output: one row per present (profile_id, ctx_id),
    // ascending (traces are loaded in ascending profile id)
    for (uint32_t t = 0; t < sh.n_traces; ++t)
      for (uint32_t x = 0; x < sh.n_ctx; ++x) {
        const size_t i = static_cast<size_t>(t) * sh.n_ctx + x;
        if (c[i] == 0) continue;
        kp.push_back(profile_ids[t]);
        kc.push_back(x);
        sum.push_back(s[i]);
        mn.push_back(lo[i]);
        mx.push_back(hi[i]);
        mean.push_back(m[i]);
        cnt.push_back(c[i]);
      }
  }
  frame::table out;
  out.add(frame::column::of_u64("profile_id", std::move(kp)));
  out.add(frame::column::of_u64("ctx_id", std::move(kc)));
  out.add(frame::column::of_i64("dur_ns_sum", std::move(sum)));
  out.add(frame::column::of_i64("dur_ns_min", std::move(mn)));
  out.add(frame::column::of_i64("dur_ns_max", std::move(mx)));
  out.add(frame::column::of_f64("dur_ns_mean", std::move(mean)));
  out.add(frame::column::of_u64("dur_ns_count", std::move(cnt)));
  return out;
}

namespace {

struct cube_run {
  psg_query_info info{};
  std::vector<uint32_t> pids;
};

// One cube query on the bound device (the caller holds the device lease).
// anchor = PSG_ANCHOR_AUTO runs suggest_anchor on the device on the first
// requested trace (itermodel.cpp:253-255); info.anchor is the one used.
cube_run run_cube(device& d, const store::db_handle& h, const std::vector<uint32_t>& profile_ids,
                  uint32_t anchor, bool stats) {
  cube_run r;
  r.pids = sorted_unique(profile_ids);
  if (anchor != PSG_ANCHOR_AUTO && anchor >= h.meta().contexts.size())  // itermodel.cpp:258-260
    raise(errc::not_found, "anchor ctx " + std::to_string(anchor) + " not in tree");
  d.bind(h, r.pids);
  psg_query_spec q{};
  q.flags = static_cast<uint32_t>(PSG_Q_CUBE) | (stats ? static_cast<uint32_t>(PSG_Q_STATS) : 0u);
  q.anchor_ctx = anchor;
  check(psg_query(d.ctx(), &q, &r.info));
  return r;
}

}  // namespace

itermodel::tri_model build_tri_model(const store::db_handle& h,
                                     const std::vector<uint32_t>& profile_ids,
                                     itermodel::anchor_policy policy, unsigned /*jobs*/) {
  if (profile_ids.empty()) raise(errc::invalid_argument, "no traces requested");
  const std::vector<uint32_t> pids = sorted_unique(profile_ids);
  itermodel::tri_model model;
  device_lease lease = acquire_device();
  device& d = lease.dev;
  cube_run r = run_cube(d, h, pids, policy.automatic ? PSG_ANCHOR_AUTO : policy.ctx, false);
  model.anchor_ctx = r.info.anchor;
  const psg_query_info& info = r.info;
  const size_t n = pids.size(), nn = info.n_nodes, kept = info.n_kept;
  model.node_ids.resize(nn);
  std::vector<uint32_t> ic(n);
  std::vector<uint64_t> bo(kept);
  model.incl_ns.resize(info.n_cells);
  model.excl_ns.resize(info.n_cells);
  model.gap_incl_ns.resize(kept * nn);
  model.gap_excl_ns.resize(kept * nn);
  check(psg_get_cube(d.ctx(), model.node_ids.data(), ic.data(), bo.data(), model.incl_ns.data(),
                     model.excl_ns.data(), model.gap_incl_ns.data(), model.gap_excl_ns.data()));
  for (size_t t = 0; t < n; ++t) {
    if (ic[t] == 0) {
      model.skipped_traces.push_back(pids[t]);
    } else {
      model.trace_ids.push_back(pids[t]);
      model.iter_counts.push_back(ic[t]);
    }
  }
  model.block_offset.assign(bo.begin(), bo.end());
  return model;
}

iteration_diagnostics iteration_report(const store::db_handle& h,
                                       const std::vector<uint32_t>& profile_ids,
                                       uint32_t anchor_ctx, double total_time_s) {
  if (profile_ids.empty()) raise(errc::invalid_argument, "no traces requested");
  if (!(total_time_s > 0.0))  // diagnostics.cpp:124-125
    raise(errc::invalid_total, "total time must be positive");
  device_lease lease = acquire_device();
  device& d = lease.dev;
  cube_run r = run_cube(d, h, profile_ids, anchor_ctx, true);
  if (r.info.n_kept_global == 0 || r.info.min_iterations == 0)
    raise(errc::insufficient_data, "model has no iterations");
  const uint32_t nl = r.info.n_leaves;
  iteration_diagnostics out;
  out.leaves.resize(nl);
  std::vector<double> sav(4ull * nl), summary(4), cv(2ull * nl);
  std::vector<int32_t> ok(nl);
  check(psg_get_stats(d.ctx(), total_time_s, out.leaves.data(), sav.data(), summary.data(),
                      cv.data(), ok.data()));
  for (uint32_t i = 0; i < nl; ++i) {
    diagnostics::savings_row row;
    row.ctx_id = out.leaves[i];
    row.avg_mean_s = sav[4 * i];
    row.avg_max_s = sav[4 * i + 1];
    row.savings_per_iter_s = sav[4 * i + 2];
    row.total_reduction_s = sav[4 * i + 3];
    out.savings.rows.push_back(row);
    if (ok[i])
      out.cv.push_back(diagnostics::cv_report{cv[2 * i], cv[2 * i + 1]});
    else
      out.cv.push_back(std::nullopt);
  }
  out.savings.n_iterations = static_cast<uint32_t>(summary[0]);
  out.savings.total_savings_s = summary[1];
  out.savings.speedup_frac = summary[3];
  return out;
}

}  // namespace perfslice::gpu
