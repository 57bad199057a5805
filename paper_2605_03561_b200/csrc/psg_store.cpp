// trace.db / meta.bin reader.  Format and validation rules follow the
// reference store (store.hpp:5-23; open: store.cpp:436-534).  Bodies are not
// decoded here: the GPU loader transposes them (psg_kernels.cu K1).
#include "psg_store.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstring>
#include <fstream>
#include <iterator>

#include "psg_internal.h"

namespace psg::store {

namespace {

constexpr char k_meta_magic[4] = {'H', 'P', 'A', 'N'};
constexpr char k_trace_magic[4] = {'H', 'P', 'T', 'R'};
constexpr char k_profile_magic[4] = {'H', 'P', 'P', 'R'};
constexpr uint32_t k_version = 1;
constexpr uint64_t k_event_size = 12;

// Bounds-checked little-endian cursor (the reference's `cursor`, store.cpp:44-110).
struct cursor {
  const uint8_t* p;
  uint64_t size, pos;
  const char* what;
  void need(uint64_t n) const {
    if (pos + n > size)
      fail(PS_E_FORMAT, std::string(what) + " truncated at byte " + std::to_string(pos));
  }
  template <typename T>
  T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  std::string str() {
    uint16_t n = get<uint16_t>();
    need(n);
    std::string s(reinterpret_cast<const char*>(p + pos), n);
    pos += n;
    return s;
  }
  void magic(const char m[4]) {
    need(4);
    if (std::memcmp(p + pos, m, 4) != 0) fail(PS_E_FORMAT, std::string(what) + ": bad magic");
    pos += 4;
  }
  void version() {
    uint32_t v = get<uint32_t>();
    if (v != k_version)
      fail(PS_E_FORMAT, std::string(what) + ": unsupported version " + std::to_string(v));
  }
};

}  // namespace

const profile_desc* meta_data::find_profile(uint32_t id) const {
  auto it = std::lower_bound(profiles.begin(), profiles.end(), id,
                             [](const profile_desc& p, uint32_t x) { return p.id < x; });
  return (it == profiles.end() || it->id != id) ? nullptr : &*it;
}

void mapped_file::open(const std::string& path) {
  if (data_) ::munmap(const_cast<uint8_t*>(data_), size_);
  data_ = nullptr;
  size_ = 0;
  int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) fail(PS_E_IO, "cannot open " + path);
  struct stat st {};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    fail(PS_E_IO, "cannot stat " + path);
  }
  size_ = static_cast<uint64_t>(st.st_size);
  if (size_ > 0) {
    void* m = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) {
      ::close(fd);
      fail(PS_E_IO, "mmap failed: " + path);
    }
    data_ = static_cast<const uint8_t*>(m);
  }
  ::close(fd);
}

mapped_file::~mapped_file() {
  if (data_) ::munmap(const_cast<uint8_t*>(data_), size_);
}

const trace_index_entry* trace_db::find(uint32_t pid) const {
  auto it = std::lower_bound(index.begin(), index.end(), pid,
                             [](const trace_index_entry& e, uint32_t x) { return e.profile_id < x; });
  return (it == index.end() || it->profile_id != pid) ? nullptr : &*it;
}

void read_meta(const std::string& dir, meta_data& meta) {
  meta = meta_data{};
  std::ifstream mf(dir + "/meta.bin", std::ios::binary);
  if (!mf) fail(PS_E_IO, "cannot open " + dir + "/meta.bin");
  std::string bytes((std::istreambuf_iterator<char>(mf)), std::istreambuf_iterator<char>());
  cursor mc{reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size(), 0, "meta.bin"};
  mc.magic(k_meta_magic);
  mc.version();
  uint32_t n_metrics = mc.get<uint32_t>();
  for (uint32_t i = 0; i < n_metrics; ++i) {
    metric_desc m;
    m.id = mc.get<uint32_t>();
    m.scope = mc.get<uint8_t>();
    if (m.scope > 1) fail(PS_E_FORMAT, "meta.bin: bad metric scope");
    m.name = mc.str();
    m.unit = mc.str();
    meta.metrics.push_back(std::move(m));
  }
  uint32_t n_profiles = mc.get<uint32_t>();
  for (uint32_t i = 0; i < n_profiles; ++i) {
    profile_desc p;
    p.id = mc.get<uint32_t>();
    p.rank = mc.get<int32_t>();
    p.thread = mc.get<int32_t>();
    p.hostname = mc.str();
    p.posix_node_id = mc.get<uint64_t>();
    meta.profiles.push_back(std::move(p));
  }
  uint32_t n_ctx = mc.get<uint32_t>();
  for (uint32_t i = 0; i < n_ctx; ++i) {
    cct_node n;
    n.id = mc.get<uint32_t>();
    n.parent = mc.get<uint32_t>();
    n.kind = mc.get<uint8_t>();
    n.name = mc.str();
    meta.contexts.push_back(std::move(n));
  }
}

void open_trace_db(const std::string& dir, trace_db& db) {
  db.dir = dir;
  read_meta(dir, db.meta);
  db.map.open(dir + "/trace.db");
  cursor tc{db.map.data(), db.map.size(), 0, "trace.db"};
  tc.magic(k_trace_magic);
  tc.version();
  uint32_t count = tc.get<uint32_t>();
  db.index.reserve(count);
  for (uint32_t i = 0; i < count; ++i) {
    trace_index_entry e;
    e.profile_id = tc.get<uint32_t>();
    e.offset = tc.get<uint64_t>();
    e.event_count = tc.get<uint64_t>();
    e.t_begin_ns = tc.get<uint64_t>();
    e.t_end_ns = tc.get<uint64_t>();
    if (e.offset + e.event_count * k_event_size > db.map.size())
      fail(PS_E_FORMAT, "trace.db: body out of bounds for trace " + std::to_string(e.profile_id));
    if (e.t_begin_ns > e.t_end_ns)
      fail(PS_E_FORMAT, "trace.db: t_begin after t_end for trace " + std::to_string(e.profile_id));
    if (i > 0 && e.profile_id <= db.index[i - 1].profile_id)
      fail(PS_E_FORMAT, "trace.db: index not sorted by profile id");
    db.index.push_back(e);
  }
}

const profile_index_entry* profile_db::find(uint32_t pid) const {
  auto it = std::lower_bound(index.begin(), index.end(), pid,
                             [](const profile_index_entry& e, uint32_t x) { return e.profile_id < x; });
  return (it == index.end() || it->profile_id != pid) ? nullptr : &*it;
}

// profile.db: magic "HPPR", u32 version, u32 count, 20-byte index entries
// {u32 profile_id, u64 offset, u64 record_count}, then packed 14-byte records
// (the reference's open, store.cpp:484-503, with its validation).
void open_profile_db(const std::string& dir, profile_db& db) {
  db.dir = dir;
  read_meta(dir, db.meta);
  db.map.open(dir + "/profile.db");
  cursor pc{db.map.data(), db.map.size(), 0, "profile.db"};
  pc.magic(k_profile_magic);
  pc.version();
  uint32_t count = pc.get<uint32_t>();
  db.index.reserve(count);
  for (uint32_t i = 0; i < count; ++i) {
    profile_index_entry e;
    e.profile_id = pc.get<uint32_t>();
    e.offset = pc.get<uint64_t>();
    e.record_count = pc.get<uint64_t>();
    if (e.offset + e.record_count * k_record_size > db.map.size())
      fail(PS_E_FORMAT, "profile.db: body out of bounds for profile " + std::to_string(e.profile_id));
    if (i > 0 && e.profile_id <= db.index[i - 1].profile_id)
      fail(PS_E_FORMAT, "profile.db: index not sorted by profile id");
    db.index.push_back(e);
  }
}

std::string node_name_error(const std::string& name, uint32_t* rack, uint32_t* chassis) {
  // topology.cpp:14-46: the same checks in the same order, the same messages
  const char tags[5] = {'x', 'c', 's', 'b', 'n'};
  uint32_t v[5];
  size_t pos = 0;
  for (int f = 0; f < 5; ++f) {
    if (pos >= name.size() || name[pos] != tags[f])
      return "node name parse error at byte " + std::to_string(pos) + ": expected '" +
             std::string(1, tags[f]) + "' in \"" + name + "\"";
    ++pos;
    auto [p, ec] = std::from_chars(name.data() + pos, name.data() + name.size(), v[f]);
    if (ec != std::errc() || p == name.data() + pos)
      return "node name parse error at byte " + std::to_string(pos) +
             ": expected decimal integer in \"" + name + "\"";
    pos = static_cast<size_t>(p - name.data());
  }
  if (pos != name.size())
    return "node name parse error at byte " + std::to_string(pos) + ": trailing characters in \"" +
           name + "\"";
  if (rack) *rack = v[0];
  if (chassis) *chassis = v[1];
  return std::string();
}

bool parse_node_name(const std::string& name, uint32_t* rack, uint32_t* chassis) {
  return node_name_error(name, rack, chassis).empty();
}

}  // namespace psg::store
