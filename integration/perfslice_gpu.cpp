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
#include <map>
#include <mutex>
#include <set>
#include <span>
#include <tuple>
#include <type_traits>
#include <variant>
#include <string>

#include "core/common.hpp"
#include "core/topology.hpp"
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
  if (s == PS_E_PARSE) raise(e, msg);  // the reference's own parse message, verbatim
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

ingest::slice_table read_slices(const store::db_handle& h,
                                const std::vector<ingest::slice_request>& requests, unsigned /*jobs*/) {
  ingest::slice_table out;
  if (requests.empty()) return out;
  device_lease lease = acquire_device();
  device& d = lease.dev;
  d.bind_profiles(h);
  // requests with identical (ctx, metric) filters go to the device together;
  // each profile appears at most once per filter pair (query.cpp:322-334)
  using key = std::tuple<bool, std::vector<uint32_t>, bool, std::vector<uint16_t>>;
  std::map<key, std::vector<size_t>> groups;
  for (size_t i = 0; i < requests.size(); ++i) {
    const auto& r = requests[i];
    groups[key{r.ctxs.all, r.ctxs.ids, r.metrics.all, r.metrics.ids}].push_back(i);
  }
  struct part {
    size_t begin = 0, end = 0;  // rows of this request in its group's table
    const ingest::slice_table* rows = nullptr;
  };
  std::vector<part> parts(requests.size());
  std::vector<ingest::slice_table> tables;
  tables.reserve(groups.size());
  static const uint32_t k_no_ctx = 0;
  static const uint16_t k_no_metric = 0;
  for (const auto& [k, idx] : groups) {
    const auto& [ctx_all, ctx_ids, m_all, m_ids] = k;
    std::vector<uint32_t> pids;
    for (size_t i : idx) pids.push_back(requests[i].profile_id);
    // an explicit empty filter keeps nothing (non-null pointer, zero ids)
    const uint32_t* cx = ctx_all ? nullptr : (ctx_ids.empty() ? &k_no_ctx : ctx_ids.data());
    const uint16_t* mt = m_all ? nullptr : (m_ids.empty() ? &k_no_metric : m_ids.data());
    const uint32_t ncx = static_cast<uint32_t>(ctx_ids.size()), nmt = static_cast<uint32_t>(m_ids.size());
    const uint32_t np = static_cast<uint32_t>(pids.size());
    uint64_t n = 0;
    check(psg_slice(d.ctx(), pids.data(), np, cx, ncx, mt, nmt, &n, nullptr, nullptr, nullptr, nullptr));
    ingest::slice_table t;
    t.profile_id.resize(n);
    t.ctx_id.resize(n);
    t.metric_id.resize(n);
    t.value.resize(n);
    if (n)
      check(psg_slice(d.ctx(), pids.data(), np, cx, ncx, mt, nmt, &n, t.profile_id.data(), t.ctx_id.data(),
                      t.metric_id.data(), t.value.data()));
    tables.push_back(std::move(t));
    const ingest::slice_table& tb = tables.back();
    // the device returns profiles ascending, each one's records contiguous
    for (size_t i : idx) {
      const uint32_t pid = requests[i].profile_id;
      auto lo = std::lower_bound(tb.profile_id.begin(), tb.profile_id.end(), pid);
      auto hi = std::upper_bound(lo, tb.profile_id.end(), pid);
      parts[i] = part{static_cast<size_t>(lo - tb.profile_id.begin()),
                      static_cast<size_t>(hi - tb.profile_id.begin()), &tb};
    }
  }
  // ingest.cpp:122-153: request slots back to back in request order
  size_t total = 0;
  for (const auto& pt : parts) total += pt.end - pt.begin;
  out.profile_id.reserve(total);
  out.ctx_id.reserve(total);
  out.metric_id.reserve(total);
  out.value.reserve(total);
  for (const auto& pt : parts)
    for (size_t j = pt.begin; j < pt.end; ++j)
      out.append(pt.rows->profile_id[j], pt.rows->ctx_id[j], pt.rows->metric_id[j], pt.rows->value[j]);
  return out;
}

// ---- frame operators over a host frame::table --------------------------

namespace {

// Device allocation on the shared context, freed on scope exit.
struct dev_buf {
  psg_context* ctx = nullptr;
  void* p = nullptr;
  dev_buf(psg_context* c, uint64_t bytes) : ctx(c) { check(psg_dev_alloc(c, bytes, &p)); }
  ~dev_buf() { psg_dev_free(ctx, p); }
  dev_buf(const dev_buf&) = delete;
  dev_buf& operator=(const dev_buf&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

uint32_t psg_dtype(const frame::column& c) {
  switch (c.type()) {
    case frame::dtype::i64: return PSG_I64;
    case frame::dtype::u64: return PSG_U64;
    case frame::dtype::f64: return PSG_F64;
    case frame::dtype::str: break;
  }
  raise(errc::type_mismatch, "gpu frame: column " + c.name() + " is a string column (host only)");
}

const void* host_data(const frame::column& c) {
  switch (c.type()) {
    case frame::dtype::i64: return c.i64s().data();
    case frame::dtype::u64: return c.u64s().data();
    case frame::dtype::f64: return c.f64s().data();
    case frame::dtype::str: break;
  }
  return nullptr;
}

std::unique_ptr<dev_buf> upload(psg_context* ctx, const frame::column& c) {
  psg_dtype(c);
  auto b = std::make_unique<dev_buf>(ctx, 8ull * c.size() + 8);
  check(psg_copy(ctx, b->p, host_data(c), 8ull * c.size()));
  return b;
}

frame::column host_gather(const frame::column& c, const std::vector<uint64_t>& idx) {
  auto pick = [&](const auto& v) {
    std::remove_cvref_t<decltype(v)> out;
    out.reserve(idx.size());
    for (uint64_t i : idx) out.push_back(v[i]);
    return out;
  };
  switch (c.type()) {
    case frame::dtype::i64: return frame::column::of_i64(c.name(), pick(c.i64s()));
    case frame::dtype::u64: return frame::column::of_u64(c.name(), pick(c.u64s()));
    case frame::dtype::f64: return frame::column::of_f64(c.name(), pick(c.f64s()));
    case frame::dtype::str: return frame::column::of_str(c.name(), pick(c.strs()));
  }
  return c;
}

}  // namespace

frame::table group_aggregate(const frame::table& t, const std::vector<std::string>& keys,
                             const std::vector<frame::agg_spec>& aggs, frame::backend /*b*/) {
  std::vector<const frame::column*> kc;
  for (const auto& k : keys) kc.push_back(&t.col(k));  // no_such_column like the reference
  if (kc.empty()) raise(errc::invalid_argument, "at least one key column is required");
  for (const auto& a : aggs) {
    const frame::column& c = t.col(a.column);
    if (c.type() == frame::dtype::str)  // require_numeric (frame.cpp:295-297)
      raise(errc::type_mismatch, "column " + a.column + " is not numeric");
  }
  const uint64_t n = t.n_rows();
  device_lease lease = acquire_device();
  psg_context* ctx = lease.dev.ctx();
  std::vector<std::unique_ptr<dev_buf>> kd;
  std::vector<psg_col> cols;
  for (const auto* c : kc) {
    kd.push_back(upload(ctx, *c));
    cols.push_back(psg_col{psg_dtype(*c), kd.back()->p});
  }
  dev_buf perm(ctx, 8 * n + 8), starts(ctx, 8 * n + 8);
  uint64_t ng = 0;
  check(psg_frame_group(ctx, cols.data(), static_cast<uint32_t>(cols.size()), n, perm.as<uint64_t>(),
                        starts.as<uint64_t>(), &ng));
  std::vector<uint64_t> hp(n), hs(ng);
  check(psg_copy(ctx, hp.data(), perm.p, 8 * n));
  check(psg_copy(ctx, hs.data(), starts.p, 8 * ng));
  std::vector<uint64_t> heads(ng);
  for (uint64_t g = 0; g < ng; ++g) heads[g] = hp[hs[g]];
  frame::table out;
  for (const auto* c : kc) out.add(host_gather(*c, heads));
  for (const auto& a : aggs) {
    const frame::column& src = t.col(a.column);
    auto sd = upload(ctx, src);
    dev_buf res(ctx, 8 * ng + 8);
    check(psg_frame_group_agg(ctx, psg_col{psg_dtype(src), sd->p}, perm.as<uint64_t>(), starts.as<uint64_t>(),
                              ng, n, static_cast<uint32_t>(a.fn == frame::agg_fn::sum     ? PSG_AGG_SUM
                                                           : a.fn == frame::agg_fn::min   ? PSG_AGG_MIN
                                                           : a.fn == frame::agg_fn::max   ? PSG_AGG_MAX
                                                           : a.fn == frame::agg_fn::mean  ? PSG_AGG_MEAN
                                                                                          : PSG_AGG_COUNT),
                              res.p));
    const std::string name = a.column + "_" + frame::agg_fn_name(a.fn);
    if (a.fn == frame::agg_fn::count) {
      std::vector<uint64_t> v(ng);
      check(psg_copy(ctx, v.data(), res.p, 8 * ng));
      out.add(frame::column::of_u64(name, std::move(v)));
    } else if (a.fn == frame::agg_fn::mean || src.type() == frame::dtype::f64) {
      std::vector<double> v(ng);
      check(psg_copy(ctx, v.data(), res.p, 8 * ng));
      out.add(frame::column::of_f64(name, std::move(v)));
    } else if (src.type() == frame::dtype::i64) {
      std::vector<int64_t> v(ng);
      check(psg_copy(ctx, v.data(), res.p, 8 * ng));
      out.add(frame::column::of_i64(name, std::move(v)));
    } else {
      std::vector<uint64_t> v(ng);
      check(psg_copy(ctx, v.data(), res.p, 8 * ng));
      out.add(frame::column::of_u64(name, std::move(v)));
    }
  }
  return out;
}

frame::table filter(const frame::table& t, const std::string& column, frame::cmp_op op,
                    const frame::literal& lit, frame::backend /*b*/) {
  const frame::column& c = t.col(column);
  if (static_cast<size_t>(c.type()) != lit.index())  // frame.cpp:427-429
    raise(errc::type_mismatch, "literal type does not match column " + column);
  const uint64_t n = t.n_rows();
  device_lease lease = acquire_device();
  psg_context* ctx = lease.dev.ctx();
  auto cd = upload(ctx, c);
  dev_buf idx(ctx, 8 * n + 8);
  uint64_t m = 0;
  const void* litp = std::visit([](const auto& v) -> const void* { return &v; }, lit);
  check(psg_frame_filter(ctx, psg_col{psg_dtype(c), cd->p}, static_cast<uint32_t>(op), litp, n,
                         idx.as<uint64_t>(), &m));
  std::vector<uint64_t> sel(m);
  check(psg_copy(ctx, sel.data(), idx.p, 8 * m));
  frame::table out;
  for (const auto& col : t.columns()) out.add(host_gather(col, sel));
  return out;
}

// ---- single-trace iteration model (itermodel.cpp:111-183) ----------------

namespace {

// A second device context for span inputs (one trace given as events), so the
// shared device keeps its resident trace set.
struct span_device {
  std::mutex mu;
  std::unique_ptr<device> dev;
};
span_device& span_dev() {
  static span_device s;
  return s;
}

void load_span(psg_context* ctx, std::span<const store::trace_event> events, uint64_t t_end,
               const store::meta_data& cct) {
  std::vector<uint32_t> parent(cct.contexts.size());
  for (size_t i = 0; i < parent.size(); ++i) parent[i] = cct.contexts[i].parent;
  check(psg_set_cct(ctx, parent.data(), static_cast<uint32_t>(parent.size())));
  std::vector<uint8_t> body(events.size() * store::k_event_size);
  for (size_t i = 0; i < events.size(); ++i) {
    std::memcpy(body.data() + 12 * i, &events[i].timestamp_ns, 8);
    std::memcpy(body.data() + 12 * i + 8, &events[i].ctx_id, 4);
  }
  const uint64_t off[2] = {0, events.size()};
  const uint32_t pid = 0;
  check(psg_load_traces_aos(ctx, body.data(), events.size(), off, &pid, &t_end, 1));
}

}  // namespace

std::vector<itermodel::interval> detect_iterations(std::span<const store::trace_event> events,
                                                   uint64_t t_end_ns, const store::meta_data& cct,
                                                   uint32_t anchor) {
  if (anchor >= cct.contexts.size())  // itermodel.cpp:114-116
    raise(errc::not_found, "anchor ctx " + std::to_string(anchor) + " not in tree");
  for (const auto& e : events)
    if (e.ctx_id >= cct.contexts.size())
      raise(errc::dangling_context, "trace event ctx " + std::to_string(e.ctx_id) + " not in tree");
  span_device& sd = span_dev();
  std::lock_guard<std::mutex> lk(sd.mu);
  if (!sd.dev) sd.dev = std::make_unique<device>(0);
  psg_context* ctx = sd.dev->ctx();
  load_span(ctx, events, std::max(t_end_ns, events.empty() ? t_end_ns : events.back().timestamp_ns), cct);
  psg_query_spec q{};
  q.flags = PSG_Q_CUBE | PSG_Q_NO_CUBE_STORE;
  q.anchor_ctx = anchor;
  psg_query_info info{};
  check(psg_query(ctx, &q, &info));
  uint32_t nb = 0;
  check(psg_get_boundaries(ctx, 0, &nb, nullptr));
  if (nb == 0) raise(errc::no_iterations, "anchor never entered in trace");
  std::vector<uint64_t> b(nb);
  check(psg_get_boundaries(ctx, 0, &nb, b.data()));
  std::vector<itermodel::interval> out;
  for (uint32_t k = 0; k < nb; ++k) {
    const uint64_t t1 = k + 1 < nb ? b[k + 1] : t_end_ns;
    if (b[k] < t1) out.push_back({b[k], t1});
  }
  if (out.empty()) raise(errc::no_iterations, "all detected iterations are empty");
  return out;
}

itermodel::interval_profile rematerialize(std::span<const store::trace_event> events,
                                          std::optional<store::trace_event> carry_in,
                                          itermodel::interval iv, const store::meta_data& cct) {
  if (iv.t0_ns >= iv.t1_ns) raise(errc::invalid_argument, "interval must have positive length");
  // the carry-in event prepended to the span: the window query integrates
  // [carry.ts, first.ts) and every event to its successor or t1, clipped to
  // [t0, t1) -- rematerialize's segments (itermodel.cpp:168-176)
  std::vector<store::trace_event> ev;
  ev.reserve(events.size() + 1);
  if (carry_in) ev.push_back(*carry_in);
  ev.insert(ev.end(), events.begin(), events.end());
  for (const auto& e : ev)
    if (e.ctx_id >= cct.contexts.size())
      raise(errc::dangling_context, "trace event ctx " + std::to_string(e.ctx_id) + " not in tree");
  const size_t n_ctx = cct.contexts.size();
  itermodel::interval_profile out;
  if (ev.empty()) return out;
  span_device& sd = span_dev();
  std::lock_guard<std::mutex> lk(sd.mu);
  if (!sd.dev) sd.dev = std::make_unique<device>(0);
  psg_context* ctx = sd.dev->ctx();
  load_span(ctx, ev, std::max(ev.back().timestamp_ns, iv.t1_ns), cct);
  psg_query_spec q{};
  q.flags = PSG_Q_WINDOW;
  q.t0_ns = iv.t0_ns;
  q.t1_ns = iv.t1_ns;
  psg_query_info info{};
  check(psg_query(ctx, &q, &info));
  std::vector<int64_t> incl(n_ctx), excl(n_ctx);
  check(psg_get_window(ctx, nullptr, nullptr, nullptr, nullptr, nullptr, excl.data(), incl.data()));
  for (uint32_t c = 0; c < n_ctx; ++c)
    if (incl[c] != 0 || excl[c] != 0) out.push_back({c, incl[c], excl[c]});
  return out;
}

// ---- diagnostics and topology -------------------------------------------

double balance_ratio(std::span<const double> values) {
  if (values.empty()) raise(errc::empty_input, "balance_ratio of empty vector");
  device_lease lease = acquire_device();
  double r = 0.0;
  check(psg_vector_stats(lease.dev.ctx(), values.data(), values.size(), 0, &r));
  return r;
}

double cv_percent(std::span<const double> values) {
  if (values.empty()) raise(errc::empty_input, "cv of empty vector");
  device_lease lease = acquire_device();
  double r = 0.0;
  const ps_status st = psg_vector_stats(lease.dev.ctx(), values.data(), values.size(), 1, &r);
  if (st == PS_E_INSUFFICIENT_DATA) raise(errc::undefined_cv, "cv undefined for zero mean");
  check(st);
  return r;
}

std::vector<diagnostics::node_stat> node_correlate(
    const std::vector<std::pair<int32_t, double>>& rank_values, const store::meta_data& meta) {
  // rank -> hostname from the first profile with that rank; hosts in string
  // order (diagnostics.cpp:381-398): host bookkeeping stays on the host
  std::map<int32_t, const std::string*> rank_host;
  for (const auto& p : meta.profiles)
    if (p.rank >= 0 && rank_host.find(p.rank) == rank_host.end()) rank_host[p.rank] = &p.hostname;
  std::map<std::string, uint32_t> host_id;
  std::vector<const std::string*> host_of(rank_values.size());
  for (size_t i = 0; i < rank_values.size(); ++i) {
    auto it = rank_host.find(rank_values[i].first);
    if (it == rank_host.end())
      raise(errc::not_found, "rank " + std::to_string(rank_values[i].first) + " has no profile descriptor");
    host_of[i] = it->second;
    host_id.emplace(*it->second, 0);
  }
  uint32_t k = 0;
  for (auto& [h, id] : host_id) id = k++;
  std::vector<uint32_t> node(rank_values.size());
  std::vector<double> vals(rank_values.size());
  for (size_t i = 0; i < rank_values.size(); ++i) {
    node[i] = host_id[*host_of[i]];
    vals[i] = rank_values[i].second;
  }
  std::vector<double> mean(host_id.size());
  std::vector<uint32_t> count(host_id.size());
  device_lease lease = acquire_device();
  check(psg_node_means(lease.dev.ctx(), vals.data(), node.data(), vals.size(),
                       static_cast<uint32_t>(host_id.size()), mean.data(), count.data()));
  std::vector<diagnostics::node_stat> out;
  for (const auto& [h, id] : host_id) out.push_back({h, mean[id], count[id]});
  return out;
}

topology::congestion_report localize_outliers(const std::vector<std::string>& outliers,
                                              const std::vector<std::string>& universe) {
  // parse_error on the first bad name, universe first (topology.cpp:58-69)
  std::vector<std::string> names = universe;
  std::set<std::string> outlier_set(outliers.begin(), outliers.end());
  std::map<std::string, uint32_t> idx;
  for (size_t i = 0; i < universe.size(); ++i) idx.emplace(universe[i], static_cast<uint32_t>(i));
  for (const auto& o : outlier_set)
    if (!idx.count(o)) {
      idx.emplace(o, static_cast<uint32_t>(names.size()));
      names.push_back(o);
    }
  std::vector<uint32_t> rack(names.size()), chassis(names.size());
  for (size_t i = 0; i < universe.size(); ++i)  // raises parse_error
    check(psg_node_name(universe[i].c_str(), &rack[i], &chassis[i]));
  for (const auto& o : outlier_set) check(psg_node_name(o.c_str(), &rack[idx[o]], &chassis[idx[o]]));
  std::vector<uint32_t> sel;
  for (const auto& o : outlier_set) sel.push_back(idx[o]);
  device_lease lease = acquire_device();
  uint32_t nr = 0;
  check(psg_localize(lease.dev.ctx(), rack.data(), chassis.data(), static_cast<uint32_t>(names.size()),
                     static_cast<uint32_t>(universe.size()), sel.data(), static_cast<uint32_t>(sel.size()),
                     &nr, nullptr));
  std::vector<uint32_t> rows(4ull * nr + 4);
  check(psg_localize(lease.dev.ctx(), rack.data(), chassis.data(), static_cast<uint32_t>(names.size()),
                     static_cast<uint32_t>(universe.size()), sel.data(), static_cast<uint32_t>(sel.size()),
                     &nr, rows.data()));
  topology::congestion_report rep;
  rep.outlier_count = outlier_set.size();
  for (uint32_t j = 0; j < nr; ++j) {
    const uint32_t r = rows[4 * j], c = rows[4 * j + 1], cnt = rows[4 * j + 2], full = rows[4 * j + 3];
    if (rep.racks.empty() || rep.racks.back().rack != r) {
      rep.racks.emplace_back();
      rep.racks.back().rack = r;
    }
    auto& e = rep.racks.back();
    e.affected_nodes += cnt;
    e.affected_chassis.push_back(c);
    if (full) e.fully_affected_chassis.push_back(c);
  }
  return rep;
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
